#!/usr/bin/env python
"""Run la_gemm on one shape a few times (for ncu launch lists):
python scripts/one_shape.py n m p [calls] [mode]"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import inputs  # noqa: E402
import paper_1306_6192_b200 as la  # noqa: E402

n, m, p = (int(x) for x in sys.argv[1:4])
calls = int(sys.argv[4]) if len(sys.argv) > 4 else 3
la.init(0)
la.set_mode(sys.argv[5] if len(sys.argv) > 5 else "3xtf32")
A, B = inputs.pair(n, m, p, "random", device="cuda")
C = torch.empty(n, p, device="cuda")
for _ in range(calls):
    la.gemm(A, B, out=C)
torch.cuda.synchronize()
print("ok", n, m, p, calls, la.last_launch_count())
