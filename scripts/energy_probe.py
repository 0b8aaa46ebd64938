#!/usr/bin/env python
"""Energy per issued TF32 flop at different problem sizes (same total work),
alternating, ~2 s per sample, NVML energy counter.  Tells how much of the
power budget data movement (DRAM / L2 traffic) costs."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import inputs  # noqa: E402
import paper_1306_6192_b200 as la  # noqa: E402
import pynvml  # noqa: E402

pynvml.nvmlInit()
h = pynvml.nvmlDeviceGetHandleByIndex(0)
la.init(0)
cases = {}
for n in [int(x) for x in (sys.argv[1:] or ["16384", "4096", "8192"])]:
    A, B = inputs.pair(n, n, n, "random", device="cuda")
    C = torch.empty(n, n, device="cuda")
    reps = max(1, int(2.0e13 * 3 // (6 * n ** 3)))   # ~ same issued flops per sample
    cases[n] = (A, B, C, reps)
    la.gemm(A, B, out=C)
torch.cuda.synchronize()
res = {n: [] for n in cases}
for rnd in range(3):
    for n, (A, B, C, reps) in cases.items():
        torch.cuda.synchronize()
        e0 = pynvml.nvmlDeviceGetTotalEnergyConsumption(h)
        ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        ev0.record()
        for _ in range(reps):
            la.gemm(A, B, out=C)
        ev1.record()
        torch.cuda.synchronize()
        e1 = pynvml.nvmlDeviceGetTotalEnergyConsumption(h)
        ms = ev0.elapsed_time(ev1)
        fl = 6.0 * n ** 3 * reps
        res[n].append((ms, (e1 - e0) / 1e3, fl, pynvml.nvmlDeviceGetClockInfo(h, pynvml.NVML_CLOCK_SM)))
for n, rs in res.items():
    for ms, j, fl, clk in rs:
        print(f"n={n:6d} {ms:8.1f} ms  {fl / ms / 1e9:7.1f} issued TF/s  {j:7.1f} J  {j / fl * 1e12:6.3f} pJ/flop  "
              f"{j / ms * 1e3:6.0f} W  clk {clk}")
