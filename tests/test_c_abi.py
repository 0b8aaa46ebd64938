"""The C ABI from plain C: tests/c/abi_host.c includes only include/la.h,
links libla.so and calls it with host buffers.  On CPU the program must
compile warning-free as C99, link, and report the missing GPU (exit 77); on a
B200 it must pass (exact integer product, error paths)."""
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


CUDA = "/usr/local/cuda"


def _build(tmp_path, name="abi_host"):
    import paper_1306_6192_b200 as la
    libdir = os.path.dirname(la.LIB_PATH)
    exe = str(tmp_path / name)
    cmd = ["gcc", "-std=c99", "-Wall", "-Wextra", "-Werror", "-pedantic", "-O2",
           "-I", os.path.join(ROOT, "include"), os.path.join(ROOT, "tests", "c", name + ".c"),
           "-o", exe, "-L", libdir, "-l:libla.so", f"-Wl,-rpath,{libdir}"]
    if name == "abi_device":  # the CUDA runtime's C API for device buffers and a stream
        cmd += ["-isystem", f"{CUDA}/include", "-L", f"{CUDA}/lib64", "-lcudart", f"-Wl,-rpath,{CUDA}/lib64"]
    subprocess.run(cmd, check=True)
    return exe


def _has_gpu():
    import torch
    return torch.cuda.is_available()


@pytest.mark.parametrize("name", ["abi_host", "abi_device"])
def test_c_consumer_builds_and_reports_no_gpu(tmp_path, name):
    if _has_gpu():
        pytest.skip("a GPU is present; see test_c_consumer_on_gpu")
    r = subprocess.run([_build(tmp_path, name)], capture_output=True, text=True, timeout=120)
    assert r.returncode == 77, r.stdout + r.stderr
    assert "la_init" in r.stderr


@pytest.mark.gpu
@pytest.mark.parametrize("name", ["abi_host", "abi_device"])
def test_c_consumer_on_gpu(tmp_path, name):
    r = subprocess.run([_build(tmp_path, name)], capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "exact" in r.stdout
