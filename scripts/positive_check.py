#!/usr/bin/env python
"""Accuracy on same-sign data vs the promotion interval: A, B uniform in [0, 1)
(|random| on the 2^-23 grid) and in [-1, 1), errors against the exact product
(fp64) and against the fp32 oracle, in units of 2^-20 * sum|a||b|.

    python scripts/positive_check.py [promote_k ...]"""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import inputs  # noqa: E402
import oracle  # noqa: E402
import paper_1306_6192_b200 as la  # noqa: E402

pks = [int(x) for x in sys.argv[1:]] or [256]
la.init(0)
os.environ["LA_SPLIT_K"] = "0"
for pk in pks:
    la.set_option("promote_k", pk)
    for m in (32, 64, 128, 256, 512, 2048, 16384):
        n = p = 256
        A0 = inputs.generate(n, m, 0, "random", seed=5)
        B0 = inputs.generate(m, p, 1, "random", seed=5)
        row = []
        for kind in ("random", "positive"):
            A, B = (A0.abs(), B0.abs()) if kind == "positive" else (A0, B0)
            C = la.gemm(A.cuda(), B.cuda()).cpu().numpy().astype(np.float64)
            S = oracle.abs_scale(A.numpy(), B.numpy())
            exact = A.numpy().astype(np.float64) @ B.numpy().astype(np.float64)
            ref = oracle.gemm(A.numpy(), B.numpy(), threads=16)
            row.append(f"{kind}: vs exact {float((np.abs(C - exact) / S).max() / 2 ** -20):6.3f} "
                       f"vs oracle {float((np.abs(C - ref) / S).max() / 2 ** -20):6.3f} "
                       f"(oracle vs exact {float((np.abs(ref - exact) / S).max() / 2 ** -20):6.3f})")
        print(f"promote_k={pk:5d} m={m:5d}  " + "   ".join(row), flush=True)
