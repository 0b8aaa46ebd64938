#!/usr/bin/env python
"""Randomized cross-path sweep (not part of the test suite): random shapes
through la_dgemm (vs the binary64 oracle, 2 gamma_m bound), la_gemm_host /
la_gemm_host_batch and la_gemm_multi on a 1-rank communicator (bitwise vs
la_gemm without split-K), la_add (bitwise vs numpy).

    python scripts/fuzz_paths.py [seconds] [seed]"""
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
rng = np.random.default_rng(int(sys.argv[2]) if len(sys.argv) > 2 else 3)
la.init(0)
la.comm_init(la.get_unique_id(), 0, 1)
os.environ["LA_SPLIT_K"] = "0"
t_end = time.time() + seconds
stats = {"dgemm": 0, "host": 0, "batch": 0, "multi": 0, "add": 0}
fails = 0
worst_d = 0.0


def dim(hi=3000):
    if rng.random() < 0.3:
        return max(1, int(rng.choice([128, 256, 512, 1024, 2048, 2304])) + int(rng.integers(-2, 3)))
    return max(1, int(np.exp(rng.uniform(0, np.log(hi)))))


while time.time() < t_end:
    path = rng.choice(list(stats))
    n, m, p = dim(), dim(), dim()
    seed = int(rng.integers(1, 2 ** 31))
    try:
        if path == "dgemm":
            n, m, p = dim(1500), dim(1500), dim(1500)
            kind = rng.choice(["f64", "integer"])
            A = inputs.generate_f64(n, m, 0, kind, seed=seed)
            B = inputs.generate_f64(m, p, 1, kind, seed=seed)
            if rng.random() < 0.3:  # odd leading dimension / offset storage
                A = A[:, : max(1, m - 1)].contiguous() if m > 1 else A
                m = A.shape[1]
                B = B[:m].contiguous()
            C = la.dgemm(A.cuda(), B.cuda()).cpu().numpy()
            ref = oracle.dgemm(A.numpy(), B.numpy())
            if kind == "integer":
                ok = np.array_equal(C, ref)
            else:
                S = oracle.dabs_scale(A.numpy(), B.numpy())
                g = m * 2.0 ** -53 / (1 - m * 2.0 ** -53)
                r = float((np.abs(C - ref) / np.maximum(S, 1e-300)).max())
                worst_d = max(worst_d, r / (2 * g))
                ok = r <= 2 * g
        elif path == "add":
            A = inputs.generate(n, m, 0, "random", seed=seed, device="cuda")
            B = inputs.generate(n, m, 1, "random", seed=seed, device="cuda")
            sub = bool(rng.random() < 0.5)
            C = la.add(A, B, subtract=sub).cpu().numpy()
            ref = (A.cpu().numpy() - B.cpu().numpy()) if sub else (A.cpu().numpy() + B.cpu().numpy())
            ok = np.array_equal(C, ref)
        else:
            A = inputs.generate(n, m, 0, "stress", seed=seed, device="cuda")
            B = inputs.generate(m, p, 1, "stress", seed=seed, device="cuda")
            ref = la.gemm(A, B).cpu()
            if path == "host":
                os.environ["LA_HOST_PANELS"] = str(int(rng.choice([1, 3, 8, 12, 16])))
                C = torch.from_numpy(la.gemm_host(A.cpu().numpy(), B.cpu().numpy()))
                ok = torch.equal(C, ref)
            elif path == "batch":
                Ah, Bh = A.cpu().pin_memory(), B.cpu().pin_memory()
                k = int(rng.integers(2, 4))
                outs = la.gemm_host_batch([Ah] * k, [Bh] * k, [torch.empty(n, p).pin_memory() for _ in range(k)])
                ok = all(torch.equal(o, ref) for o in outs)
            else:
                la.set_option("panels", int(rng.integers(1, 6)))
                Cl = torch.empty(n, p, device="cuda")
                la.gemm_multi(n, m, p, A, B, Cl, None, root=0, ngpu=1)
                ok = torch.equal(Cl.cpu(), ref)
    except Exception as ex:  # report, keep going
        ok = False
        print(f"EXC {path} n={n} m={m} p={p}: {ex!r}", flush=True)
    stats[path] += 1
    if not ok:
        fails += 1
        print(f"FAIL {path} n={n} m={m} p={p} seed={seed}", flush=True)
print(f"{sum(stats.values())} cases {stats}, {fails} failures; dgemm worst error / (2 gamma_m) {worst_d:.3f}")
