#!/usr/bin/env python
"""Accuracy vs the promotion interval (LA_OPT_PROMOTE_K) on random-sign and
structured inputs (inputs.structured patterns with |B|), against the exact
product (int128 on the 2^-23 grid) and the fp32 oracle, in units of
2^-20 * sum|a||b|; split-K on (default) and off.  One 256 x m . m x 256
product per case.

    python scripts/promote_check.py [m ...]"""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import inputs  # noqa: E402
import oracle  # noqa: E402
import paper_1306_6192_b200 as la  # noqa: E402

ms = [int(x) for x in sys.argv[1:]] or [256, 512, 2048, 4096, 16384]
PKS = [int(x) for x in os.environ.get("PKS", "-1,256,64").split(",")]
la.init(0)
T = max(1, len(os.sched_getaffinity(0)))
n = p = 256
print("| m | inputs | oracle vs exact | " + " | ".join(
    f"{'auto' if pk < 0 else pk}, split-K {sk}: vs exact / vs oracle" for sk in ("on", "off") for pk in PKS) + " |")
print("|---" * (3 + 2 * len(PKS)) + "|")
for m in ms:
    A0 = inputs.generate(n, m, 0, "random", seed=11)
    B = inputs.generate(m, p, 1, "random", seed=11).abs()
    for pat in ("random",) + inputs.PATTERNS:
        A = A0 if pat == "random" else inputs.structured(A0, pat)
        An, Bn = A.numpy(), B.numpy()
        E = oracle.exact_grid(An, Bn, 23)
        S = oracle.abs_scale(An, Bn)
        O = oracle.gemm(An, Bn, threads=T).astype(np.float64)
        u = 2.0 ** -20
        row = [f"{float((np.abs(O - E) / S).max() / u):.3f}"]
        for sk in ("on", "off"):
            if sk == "off":
                os.environ["LA_SPLIT_K"] = "0"
            else:
                os.environ.pop("LA_SPLIT_K", None)
            for pk in PKS:
                la.set_option("promote_k", pk)
                C = la.gemm(A.cuda(), B.cuda()).cpu().numpy().astype(np.float64)
                row.append(f"{float((np.abs(C - E) / S).max() / u):.3f} / {float((np.abs(C - O) / S).max() / u):.3f}")
        print(f"| {m} | {pat} | " + " | ".join(row) + " |", flush=True)
la.set_option("promote_k", -1)
