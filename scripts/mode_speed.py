#!/usr/bin/env python
"""la_gemm speed in both modes over sizes (device time per call, CUDA events)."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import inputs  # noqa: E402
import paper_1306_6192_b200 as la  # noqa: E402

la.init(0)
for n in (4096, 8192, 16384):
    A, B = inputs.pair(n, n, n, "random", device="cuda")
    C = torch.empty(n, n, device="cuda")
    for mode in ("3xtf32", "tf32"):
        la.set_mode(mode)
        for _ in range(3):
            la.gemm(A, B, out=C)
        torch.cuda.synchronize()
        reps = max(3, int(1e13 / (2 * n ** 3)))
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(reps):
            la.gemm(A, B, out=C)
        e1.record()
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / reps
        print(f"n={n:6d} {mode:7s} {ms:8.3f} ms  {2 * n ** 3 / ms / 1e9:7.1f} TF/s logical")
    la.set_mode("3xtf32")
