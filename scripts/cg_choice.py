#!/usr/bin/env python
"""Time la_gemm with LA_CTA_GROUP=1 vs 2 over mid-size shapes (kernel choice)."""
import os
import statistics
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import inputs  # noqa: E402
import paper_1306_6192_b200 as la  # noqa: E402

la.init(0)
shapes = [(1000, 2000, 1500), (1280, 2000, 1536), (1536, 1536, 1536), (1792, 1792, 1792), (2048, 2048, 2048)]
for (n, m, p) in shapes:
    A, B = inputs.pair(n, m, p, "random", device="cuda")
    C = torch.empty(n, p, device="cuda")
    res = {}
    for cg in ("1", "2"):
        os.environ["LA_CTA_GROUP"] = cg
        for _ in range(3):
            la.gemm(A, B, out=C)
        torch.cuda.synchronize()
        ts = []
        for _ in range(20):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            la.gemm(A, B, out=C)
            e1.record()
            torch.cuda.synchronize()
            ts.append(e0.elapsed_time(e1))
        res[cg] = statistics.median(ts)
    del os.environ["LA_CTA_GROUP"]
    pt = ((n + 255) // 256) * ((p + 255) // 256)
    print(f"{n}x{m}x{p}: pair tiles {pt:5d}  cg1 {res['1'] * 1e3:8.1f} us  cg2 {res['2'] * 1e3:8.1f} us  "
          f"best cg{'1' if res['1'] < res['2'] else '2'}")
