#!/usr/bin/env python
"""la_cgemm at size n a few times (for ncu launch lists): python scripts/one_cgemm.py 4096"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import inputs  # noqa: E402
import paper_1306_6192_b200 as la  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 4096
la.init(0)
A = torch.view_as_complex(inputs.generate(n, 2 * n, 0, "random", device="cuda").view(n, n, 2)).contiguous()
B = torch.view_as_complex(inputs.generate(n, 2 * n, 1, "random", device="cuda").view(n, n, 2)).contiguous()
for _ in range(3):
    C = la.cgemm(A, B)
torch.cuda.synchronize()
print("ok", n)
