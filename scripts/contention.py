#!/usr/bin/env python
"""la_gemm at n=16384 while another stream keeps part of the GPU busy (a bf16
matmul loop): the persistent grid cannot be fully resident, so the K-phase wave
barrier must not stall (bounded wait, then give up for the launch)."""
import os
import sys
import time

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import inputs  # noqa: E402
import paper_1306_6192_b200 as la  # noqa: E402

n = 16384
la.init(0)
A, B = inputs.pair(n, n, n, "random", device="cuda")
C = torch.empty(n, n, device="cuda")
X = torch.randn(8192, 8192, device="cuda", dtype=torch.bfloat16)
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()


def timed(busy):
    torch.cuda.synchronize()
    if busy:
        with torch.cuda.stream(s2):
            for _ in range(40):
                X @ X
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with torch.cuda.stream(s1):
        e0.record(s1)
        la.gemm(A, B, out=C, stream=s1)
        e1.record(s1)
    torch.cuda.synchronize()
    return e0.elapsed_time(e1)


for tag in ("alone", "busy", "alone", "busy"):
    print(tag, f"{timed(tag == 'busy'):.1f} ms", flush=True)
