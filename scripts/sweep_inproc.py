#!/usr/bin/env python
"""Interleaved A/B sweep of library env knobs inside one process.

    python scripts/sweep_inproc.py --n 16384 --rounds 4 --steps 5 \
        "LA_GROUP_M=16" "LA_GROUP_M=8"

Each round runs every variant for `steps` back-to-back la_gemm calls; the
variants alternate so thermal drift hits them equally.  Reports per variant
the median ms per call, TFLOP/s (2nmp/t), NVML energy per call (J) and mean
SM clock.  Knobs must be read by the library per call (getenv at launch).
"""
import argparse
import os
import statistics
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import inputs  # noqa: E402
import paper_1306_6192_b200 as la  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("variants", nargs="+")
    ap.add_argument("--n", type=int, default=16384)
    ap.add_argument("--rounds", type=int, default=4)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--mode", default="3xtf32")
    a = ap.parse_args()
    import pynvml
    pynvml.nvmlInit()
    h = pynvml.nvmlDeviceGetHandleByIndex(0)
    la.init(0)
    la.set_mode(a.mode)
    n = a.n
    A, B = inputs.pair(n, n, n, "random", device="cuda")
    C = torch.empty(n, n, device="cuda")
    for _ in range(3):
        la.gemm(A, B, out=C)
    torch.cuda.synchronize()
    res = {v: {"ms": [], "j": [], "clk": []} for v in a.variants}
    base_env = dict(os.environ)
    for r in range(a.rounds):
        for v in a.variants:
            os.environ.clear()
            os.environ.update(base_env)
            for kv in v.split(","):
                if "=" in kv:
                    k, val = kv.split("=", 1)
                    os.environ[k] = val
            la.gemm(A, B, out=C)            # one untimed call with the new knob
            torch.cuda.synchronize()
            e0 = pynvml.nvmlDeviceGetTotalEnergyConsumption(h)
            ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            ev0.record()
            for _ in range(a.steps):
                la.gemm(A, B, out=C)
            ev1.record()
            torch.cuda.synchronize()
            e1 = pynvml.nvmlDeviceGetTotalEnergyConsumption(h)
            clk = pynvml.nvmlDeviceGetClockInfo(h, pynvml.NVML_CLOCK_SM)
            ms = ev0.elapsed_time(ev1) / a.steps
            res[v]["ms"].append(ms)
            res[v]["j"].append((e1 - e0) / 1e3 / a.steps)
            res[v]["clk"].append(clk)
    os.environ.clear()
    os.environ.update(base_env)
    flops = 2.0 * n ** 3
    print(f"{'variant':40s} {'ms':>8s} {'TF/s':>7s} {'J/call':>7s} {'W':>6s} {'clk':>6s}")
    for v in a.variants:
        ms = statistics.median(res[v]["ms"])
        j = statistics.median(res[v]["j"])
        print(f"{v:40s} {ms:8.2f} {flops / ms / 1e9:7.1f} {j:7.2f} {j / ms * 1e3:6.0f} "
              f"{statistics.mean(res[v]['clk']):6.0f}")


if __name__ == "__main__":
    main()
