#!/usr/bin/env python
"""Long randomized parity sweep (not part of the test suite): random shapes
(log-uniform, up to ~3000 per dimension, plus tile-boundary neighbours), random
inputs, both modes, every element checked against the oracle within the
tolerance; integer inputs exact.  Prints failures and a summary.

    python scripts/fuzz_long.py [seconds] [seed]"""
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import inputs  # noqa: E402
import oracle  # noqa: E402
import paper_1306_6192_b200 as la  # noqa: E402

seconds = float(sys.argv[1]) if len(sys.argv) > 1 else 300
rng = np.random.default_rng(int(sys.argv[2]) if len(sys.argv) > 2 else 7)
THREADS = max(1, len(os.sched_getaffinity(0)))
la.init(0)
t_end = time.time() + seconds
cases = fails = 0
worst = {"3xtf32": 0.0, "tf32": 0.0}
worst_case = {"3xtf32": None, "tf32": None}
kmin = int(os.environ.get("FUZZ_KMIN", "0"))
kmax = int(os.environ.get("FUZZ_KMAX", "0"))
while time.time() < t_end:
    dims = []
    for _ in range(3):
        if rng.random() < 0.3:
            d = int(rng.choice([128, 256, 512, 1024, 2048])) + int(rng.integers(-2, 3))
        else:
            d = int(np.exp(rng.uniform(0, np.log(3000))))
        dims.append(max(1, d))
    n, m, p = dims
    if kmax:  # targeted K range
        m = int(rng.integers(kmin, kmax + 1))
    seed = int(rng.integers(1, 2 ** 31))
    kind = rng.choice(["stress", "random", "integer"])
    mode = "tf32" if rng.random() < 0.25 else "3xtf32"
    if rng.random() < 0.2:  # complex product (per-component bound with the complex scales)
        n, m, p = max(1, n // 2), max(1, m // 2), max(1, p // 2)
        A = torch.view_as_complex(inputs.generate(n, 2 * m, 0, kind, seed=seed).view(n, m, 2)).contiguous()
        B = torch.view_as_complex(inputs.generate(m, 2 * p, 1, kind, seed=seed).view(m, p, 2)).contiguous()
        la.set_mode(mode)
        C = la.cgemm(A.cuda(), B.cuda()).cpu().numpy()
        la.set_mode("3xtf32")
        ref = oracle.cgemm(A.numpy(), B.numpy())
        cases += 1
        if kind == "integer":
            ok = np.array_equal(C, ref)
        else:
            Sr, Si = oracle.cabs_scale(A.numpy(), B.numpy())
            err = max(float((np.abs(C.real.astype(np.float64) - ref.real) / np.maximum(Sr, 1e-300)).max()),
                      float((np.abs(C.imag.astype(np.float64) - ref.imag) / np.maximum(Si, 1e-300)).max()))
            bound = 2.0 ** -20 if mode == "3xtf32" else 2.0 ** -9
            ok = err <= bound
            worst[mode] = max(worst[mode], err / bound)
        if not ok:
            fails += 1
            print(f"FAIL complex n={n} m={m} p={p} kind={kind} mode={mode} seed={seed}", flush=True)
        continue
    A = inputs.generate(n, m, 0, kind, seed=seed)
    B = inputs.generate(m, p, 1, kind, seed=seed)
    la.set_mode(mode)
    C = la.gemm(A.cuda(), B.cuda()).cpu().numpy()
    la.set_mode("3xtf32")
    ref = oracle.gemm(A.numpy(), B.numpy(), threads=THREADS)
    cases += 1
    if kind == "integer":
        ok = np.array_equal(C, ref)
        err = 0.0 if ok else float("inf")
    else:
        S = oracle.abs_scale(A.numpy(), B.numpy())
        err = float((np.abs(C.astype(np.float64) - ref) / np.maximum(S, 1e-300)).max())
        bound = 2.0 ** -20 if mode == "3xtf32" else 2.0 ** -9
        ok = err <= bound
        if err / bound > worst[mode]:
            worst[mode] = err / bound
            worst_case[mode] = (n, m, p, str(kind), seed)
    if not ok:
        fails += 1
        print(f"FAIL n={n} m={m} p={p} kind={kind} mode={mode} seed={seed} err={err}", flush=True)
print(f"{cases} cases, {fails} failures; worst error / bound: 3xtf32 {worst['3xtf32']:.3f} at {worst_case['3xtf32']}, "
      f"tf32 {worst['tf32']:.3f} at {worst_case['tf32']}")
