"""bench.py's JSON-line contract.  Without a GPU: the reference arm runs here
(the oracle on the host cores), the committed GPU line (profiles/bench_r02e.json,
the final round-2 line) carries every key the driver reads, and an N-GPU
request is never timed on fewer GPUs.  On a GPU (-m gpu): a small live run."""
import json
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
BASE_KEYS = {"metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better",
             "scaling", "vs_baseline", "dtype", "data", "config"}


def test_reference_arm_line():
    r = subprocess.run([sys.executable, "bench.py", "--impl", "reference", "--steps", "1", "--warmup", "0",
                        "--cpu-seconds", "1", "--n", "2048"], cwd=ROOT, capture_output=True, text=True,
                       timeout=600)
    assert r.returncode == 0, r.stderr[-2000:]
    line = json.loads(r.stdout.strip().splitlines()[-1])
    assert BASE_KEYS <= set(line)
    assert line["impl"] == "reference"
    assert line["value"] > 0 and line["unit"] == "TFLOP/s" and line["higher_is_better"] is True
    cb = line["cpu_baseline"]
    assert cb["kind"] == "oracle" and cb["cores"] >= 1 and cb["value"] == line["value"] and cb["sample"]
    assert line["e2e"] == {"value": line["value"], "unit": "TFLOP/s", "h2d_bytes_per_step": 0,
                           "d2h_bytes_per_step": 0}


def test_committed_gpu_line_has_every_key():
    line = json.load(open(os.path.join(ROOT, "profiles", "bench_r02e.json")))
    assert BASE_KEYS <= set(line)
    assert line["n_gpus"] == 1 and line["warmup"] >= 3
    assert line["config"]["workload"] and "l2" in line["config"]
    rf = line["roofline"]
    assert rf["bound"] == "tensor" and rf["unit"] == "TFLOP/s"
    assert abs(rf["frac"] - rf["achieved"] / rf["peak"]) < 1e-9 and rf["traffic"] > 0
    assert line["cpu_baseline"]["kind"] == "oracle" and line["cpu_baseline"]["cores"] >= 1
    e2e = line["e2e"]
    assert e2e["h2d_bytes_per_step"] == 2 * 4 * 16384 ** 2 and e2e["d2h_bytes_per_step"] == 4 * 16384 ** 2
    assert set(line["clocks"]) >= {"sm_mhz", "sm_max_mhz", "reasons"}
    assert line["gpu_launches"] > 0


def test_multi_gpu_request_is_never_silently_single():
    """`bench.py --gpus N` without a torchrun environment launches N ranks
    itself; with fewer visible GPUs than N it must fail loudly instead of
    timing one GPU under an N-GPU line."""
    import torch
    env = dict(os.environ)
    env.pop("WORLD_SIZE", None)
    if torch.cuda.device_count() >= 2:
        import pytest
        pytest.skip("enough GPUs: the launch itself is exercised by the driver's scaling run")
    r = subprocess.run([sys.executable, "bench.py", "--gpus", "2", "--steps", "1", "--warmup", "3"], cwd=ROOT,
                       capture_output=True, text=True, timeout=300, env=env)
    assert r.returncode != 0
    assert "--gpus 2" in r.stderr
    # a launched job whose WORLD_SIZE disagrees with --gpus is refused too
    env.update(WORLD_SIZE="1", RANK="0", LOCAL_RANK="0")
    r = subprocess.run([sys.executable, "bench.py", "--gpus", "2", "--steps", "1"], cwd=ROOT,
                       capture_output=True, text=True, timeout=300, env=env)
    assert r.returncode != 0 and "WORLD_SIZE=1" in r.stderr


def test_reference_arm_reports_requested_gpus():
    r = subprocess.run([sys.executable, "bench.py", "--impl", "reference", "--gpus", "4", "--steps", "1",
                        "--warmup", "0", "--cpu-seconds", "1", "--n", "1024"], cwd=ROOT, capture_output=True,
                       text=True, timeout=600)
    assert r.returncode == 0, r.stderr[-2000:]
    assert json.loads(r.stdout.strip().splitlines()[-1])["n_gpus"] == 4


@pytest.mark.gpu
def test_live_gpu_line_small():
    """bench.py on the GPU (small n so it takes seconds): one JSON line with
    every key the driver reads, our kernels counted in the timed region, the
    roofline of the GEMM kernel measured live and an e2e number through the
    host-buffer API."""
    import pytest
    import torch
    if not torch.cuda.is_available():
        pytest.skip("needs a GPU")
    r = subprocess.run([sys.executable, "bench.py", "--n", "2048", "--steps", "3", "--warmup", "3",
                        "--cpu-seconds", "1"], cwd=ROOT, capture_output=True, text=True, timeout=900)
    assert r.returncode == 0, r.stderr[-3000:]
    line = json.loads(r.stdout.strip().splitlines()[-1])
    assert BASE_KEYS <= set(line) and line["n_gpus"] == 1 and line["value"] > 0
    assert line["gpu_launches"] > 0
    rf = line["roofline"]
    assert rf["bound"] == "tensor" and 0 < rf["frac"] <= 1.5 and rf["achieved"] > 0
    assert line["e2e"]["value"] > 0 and line["e2e"]["h2d_bytes_per_step"] == 2 * 4 * 2048 ** 2
    assert line["cpu_baseline"]["kind"] == "oracle"
    assert {"sm_mhz", "sm_max_mhz", "reasons"} <= set(line["clocks"])
