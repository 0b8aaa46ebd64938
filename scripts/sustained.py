#!/usr/bin/env python
"""Sustained la_gemm throughput: back-to-back n=16384 3xTF32 products for
`seconds`, throughput and SM clock per ~5-s window (NVML), and a final exact
check on integer inputs (no drift, no errors over the run).

    python scripts/sustained.py [seconds] [integer|random|stress]"""
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import inputs  # noqa: E402
import oracle  # noqa: E402
import paper_1306_6192_b200 as la  # noqa: E402
import pynvml  # noqa: E402

seconds = float(sys.argv[1]) if len(sys.argv) > 1 else 60
mode = sys.argv[2] if len(sys.argv) > 2 else "integer"   # input value mode (inputs.MODES)
n = 16384
pynvml.nvmlInit()
h = pynvml.nvmlDeviceGetHandleByIndex(0)
la.init(0)
A, B = inputs.pair(n, n, n, mode, device="cuda")
C = torch.empty(n, n, device="cuda")
la.gemm(A, B, out=C)
torch.cuda.synchronize()
t_end = time.time() + seconds
calls = 0
while time.time() < t_end:
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    j0 = pynvml.nvmlDeviceGetTotalEnergyConsumption(h)
    e0.record()
    k = 0
    t0 = time.time()
    while time.time() - t0 < 5.0:
        for _ in range(8):
            la.gemm(A, B, out=C)
        torch.cuda.synchronize()
        k += 8
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / k
    j = (pynvml.nvmlDeviceGetTotalEnergyConsumption(h) - j0) / 1e3 / k
    clk = pynvml.nvmlDeviceGetClockInfo(h, pynvml.NVML_CLOCK_SM)
    temp = pynvml.nvmlDeviceGetTemperature(h, pynvml.NVML_TEMPERATURE_GPU)
    calls += k
    print(f"{ms:7.2f} ms/GEMM  {2 * n ** 3 / ms / 1e9:6.1f} TFLOP/s  {j:5.1f} J/GEMM  {clk} MHz  {temp} C", flush=True)
if mode != "integer":
    sys.exit(0)
rows = np.array([0, 5000, n - 1])
cols = np.array([0, 7777, n - 1])
got = C[rows][:, cols].cpu().numpy()
ref = oracle.gemm(inputs.generate(n, n, 0, "integer", row_idx=rows).numpy(),
                  inputs.generate(n, n, 1, "integer", col_idx=cols).numpy())
print(f"{calls} calls, sampled integer result exact: {np.array_equal(got, ref)}")
