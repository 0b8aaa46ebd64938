#!/usr/bin/env python
"""Run la_gemm a few times at size n (for ncu captures): python scripts/one_gemm.py 16384 [calls] [mode]"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import inputs  # noqa: E402
import paper_1306_6192_b200 as la  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 16384
calls = int(sys.argv[2]) if len(sys.argv) > 2 else 2
mode = sys.argv[3] if len(sys.argv) > 3 else "3xtf32"
la.init(0)
la.set_mode(mode)
A, B = inputs.pair(n, n, n, "random", device="cuda")
C = torch.empty(n, n, device="cuda")
for _ in range(calls):
    la.gemm(A, B, out=C)
torch.cuda.synchronize()
print("ok", n, calls, mode)
