#!/usr/bin/env python
"""la_dgemm then cuBLAS DGEMM (torch.matmul, float64) at size n, for ncu captures:
python scripts/one_dgemm.py 8192"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import inputs  # noqa: E402
import paper_1306_6192_b200 as la  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 8192
la.init(0)
A = inputs.generate_f64(n, n, 0, device="cuda")
B = inputs.generate_f64(n, n, 1, device="cuda")
C = la.dgemm(A, B)
R = torch.matmul(A, B)
torch.cuda.synchronize()
print("ok", n, float((C - R).abs().max()))
