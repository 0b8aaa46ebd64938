#!/usr/bin/env python
"""Context only (never a backend): time torch.matmul (cuBLAS) on the bench
workload in FP32 (SIMT), TF32 (one pass) and, when CUBLAS_EMULATE_SINGLE_PRECISION=1
is set by the caller, cuBLAS's BF16x9 FP32 emulation; report TFLOP/s and the
max error against the oracle on sampled elements in units of 2^-20 sum|a||b|.

    python scripts/cublas_compare.py [n] [tf32|fp32]
"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import inputs  # noqa: E402
import oracle  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 16384
prec = sys.argv[2] if len(sys.argv) > 2 else "fp32"
torch.backends.cuda.matmul.allow_tf32 = prec == "tf32"
A, B = inputs.pair(n, n, n, "random", device="cuda")
C = torch.empty(n, n, device="cuda")
for _ in range(3):
    torch.matmul(A, B, out=C)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
steps = 10
e0.record()
for _ in range(steps):
    torch.matmul(A, B, out=C)
e1.record()
torch.cuda.synchronize()
ms = e0.elapsed_time(e1) / steps
rows = np.linspace(0, n - 1, 16).astype(np.int64)
cols = np.linspace(0, n - 1, 16).astype(np.int64)
As = inputs.generate(n, n, 0, "random", row_idx=rows).numpy()
Bs = inputs.generate(n, n, 1, "random", col_idx=cols).numpy()
ref = oracle.gemm(As, Bs, threads=8)
S = oracle.abs_scale(As, Bs)
err = float((np.abs(C[rows][:, cols].cpu().numpy().astype(np.float64) - ref) / S).max() / 2.0 ** -20)
print(f"cuBLAS {prec} emulate={os.environ.get('CUBLAS_EMULATE_SINGLE_PRECISION', '0')} n={n}: "
      f"{ms:.2f} ms  {2.0 * n ** 3 / ms / 1e9:.1f} TFLOP/s  max err {err:.3f} x 2^-20 S")
