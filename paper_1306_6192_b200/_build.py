"""Build the C-ABI shared library libla.so in-tree with nvcc for sm_100a."""
from __future__ import annotations

import glob
import os
import subprocess
import sys

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
LIB = os.path.join(PKG, "libla.so")
SOURCES = [os.path.join(CSRC, "la.cu"), os.path.join(CSRC, "multi.cu")]


def _nccl_dirs():
    import nvidia.nccl  # the NCCL wheel torch uses (2.28.x)
    base = list(nvidia.nccl.__path__)[0]
    return os.path.join(base, "include"), os.path.join(base, "lib")


def nvcc_flags():
    inc, _ = _nccl_dirs()
    return [
        "-gencode", "arch=compute_100a,code=sm_100a",
        "-O3", "-lineinfo", "-std=c++17",
        "-Xcompiler", "-fPIC", "-Xcompiler", "-fvisibility=hidden",
        "-Xptxas", "-v" if os.environ.get("LA_PTXAS_VERBOSE") else "-O3",
        "-I", os.path.join(ROOT, "include"), "-I", CSRC, "-I", inc,
        "-DLA_BUILD",
    ] + (["-DLA_DIAGNOSTICS"] if os.environ.get("LA_BUILD_DIAGNOSTICS") else [])


def build(force: bool = False, verbose: bool = False) -> str:
    deps = SOURCES + glob.glob(os.path.join(CSRC, "*.cuh")) + glob.glob(os.path.join(CSRC, "*.h")) + \
        [os.path.join(ROOT, "include", "la.h"), __file__]
    stamp = LIB + ".flags"
    flags_now = " ".join(nvcc_flags())
    same_flags = os.path.exists(stamp) and open(stamp).read() == flags_now
    if not force and same_flags and os.path.exists(LIB) and \
            all(os.path.getmtime(LIB) >= os.path.getmtime(d) for d in deps):
        return LIB
    _, nccl_lib = _nccl_dirs()
    tmp = LIB + f".tmp{os.getpid()}"
    cmd = ["nvcc", *nvcc_flags(), "-shared", "-cudart", "static", *SOURCES, "-o", tmp,
           "-L", nccl_lib, "-l:libnccl.so.2", "-Xlinker", f"-rpath,{nccl_lib}", "-ldl", "-lpthread"]
    if verbose:
        print(" ".join(cmd), file=sys.stderr)
    subprocess.check_call(cmd)
    os.replace(tmp, LIB)
    with open(stamp, "w") as f:
        f.write(flags_now)
    return LIB


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose=True))
