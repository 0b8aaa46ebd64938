#!/usr/bin/env python
"""One traced la_gemm_host call (LA_HOST_TRACE=1) at n=16384 after a warm-up."""
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import inputs  # noqa: E402
import paper_1306_6192_b200 as la  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 16384
la.init(0)
A, B = inputs.pair(n, n, n, "random", device="cuda")
Ah, Bh = A.cpu().pin_memory(), B.cpu().pin_memory()
Ch = torch.empty(n, n).pin_memory()
del A, B
la.gemm_host(Ah, Bh, out=Ch)
la.gemm_host(Ah, Bh, out=Ch)
os.environ["LA_HOST_TRACE"] = "1"
la.gemm_host(Ah, Bh, out=Ch)
