#!/usr/bin/env python
"""Randomised accuracy sweep over structured inputs (inputs.PATTERNS: same-sign,
sign-flipped halves, signed blocks, ramped magnitudes, biased) and random
shapes, split-K on (default dispatch).  Checks reading C14' on every element:
|C - exact| / S <= |oracle - exact| / S + 2^-20 (max over the product), with
the exact product from int128 on the 2^-23 grid.  Prints the worst cases.

    python scripts/fuzz_structured.py [seconds] [seed]"""
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import inputs  # noqa: E402
import oracle  # noqa: E402
import paper_1306_6192_b200 as la  # noqa: E402

seconds = float(sys.argv[1]) if len(sys.argv) > 1 else 240
rng = np.random.default_rng(int(sys.argv[2]) if len(sys.argv) > 2 else 3)
T = max(1, len(os.sched_getaffinity(0)))
la.init(0)
t_end = time.time() + seconds
cases = fails = 0
worst = {}
u = 2.0 ** -20
while time.time() < t_end:
    n = int(rng.integers(1, 400))
    p = int(rng.integers(1, 400))
    m = int(np.exp(rng.uniform(np.log(16), np.log(12000))))
    pat = str(rng.choice(inputs.PATTERNS))
    seed = int(rng.integers(0, 2 ** 31))
    A = inputs.structured(inputs.generate(n, m, 0, "random", seed=seed), pat)
    B = inputs.generate(m, p, 1, "random", seed=seed).abs()
    An, Bn = A.numpy(), B.numpy()
    E = oracle.exact_grid(An, Bn, 23)
    S = oracle.abs_scale(An, Bn)
    O = oracle.gemm(An, Bn, threads=T).astype(np.float64)
    C = la.gemm(A.cuda(), B.cuda()).cpu().numpy().astype(np.float64)
    g = float((np.abs(C - E) / S).max()) / u
    o = float((np.abs(O - E) / S).max()) / u
    cases += 1
    ok = g <= o + 1.0
    fails += not ok
    key = (pat, "m<1024" if m < 1024 else "m>=1024")
    if g > worst.get(key, (0,))[0]:
        worst[key] = (g, o, (n, m, p, seed))
    if not ok:
        print(f"FAIL {pat} n={n} m={m} p={p} seed={seed}: gpu {g:.3f} oracle {o:.3f}", flush=True)
print(f"{cases} cases, {fails} C14' failures")
for k in sorted(worst):
    g, o, case = worst[k]
    print(f"  {k[0]:8s} {k[1]:8s} worst GPU vs exact {g:.3f} (oracle vs exact {o:.3f}) at {case}")
