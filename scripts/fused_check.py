#!/usr/bin/env python
"""Fused split (converter warps split the staged fp32 tiles in smem) against the
separate split pass: bitwise equality on integer and random inputs over a few
shapes (small first), the oracle on the small ones, then timings of both paths.

Kept for the record of profiles/fused_split_r02.md: it drives LA_FUSED_SPLIT,
which exists only in the experiment's commit ("Experiment: operand split fused
into the GEMM ..."); the fused path was removed in the next commit, so on
later builds both arms run the split pass.

    python scripts/fused_check.py [--quick|--probe|--debug-split]
"""
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import inputs  # noqa: E402
import oracle  # noqa: E402
import paper_1306_6192_b200 as la  # noqa: E402

la.init(0)
la.set_mode(os.environ.get("LA_MODE", "3xtf32"))


def run(A, B, fused):
    os.environ["LA_FUSED_SPLIT"] = "1" if fused else "0"
    C = la.gemm(A, B)
    torch.cuda.synchronize()
    return C


if "--probe" in sys.argv:
    # A = I (128 x 64), B[k][n] = 1000 k + n: C[i][j] should be 1000 i + j
    n, m, p = 128, 64, 128
    A = torch.zeros(n, m, device="cuda")
    A[torch.arange(m), torch.arange(m)] = 1.0
    kk = torch.arange(m, device="cuda", dtype=torch.float32)[:, None]
    nn = torch.arange(p, device="cuda", dtype=torch.float32)[None, :]
    B = 1000 * kk + nn
    Cs = run(A, B, False)
    print("split path exact:", torch.equal(Cs[:m], B))
    C = run(A, B, True)
    print("probe C[0:3, 0:8]:", C[0:3, 0:8].tolist())
    print("probe C[8, 0:8]:", C[8, 0:8].tolist(), "C[1, 32:36]", C[1, 32:36].tolist())
    ok = torch.equal(C[:m], B)
    print("probe exact:", ok)
    sys.exit(0)

shapes = [(128, 32, 128), (256, 256, 256), (300, 500, 200), (1000, 2000, 1500), (512, 64, 1024),
          (4096, 4096, 4096), (777, 1236, 260)]
for mode in ("3xtf32", "tf32"):
    la.set_mode(mode)
    for (n, m, p) in shapes:
        for kind in ("integer", "random"):
            A, B = inputs.pair(n, m, p, kind, device="cuda")
            t0 = time.time()
            Cf = run(A, B, True)
            Cs = run(A, B, False)
            same = torch.equal(Cf, Cs)
            msg = f"{mode} {n}x{m}x{p} {kind}: fused==split {same}"
            if n * m * p <= 2 ** 31 and mode == "3xtf32":
                ref = oracle.gemm(A.cpu().numpy(), B.cpu().numpy(), threads=16)
                if kind == "integer":
                    msg += f" oracle-exact {np.array_equal(Cf.cpu().numpy(), ref)}"
                else:
                    S = oracle.abs_scale(A.cpu().numpy(), B.cpu().numpy())
                    err = float((np.abs(Cf.cpu().numpy().astype(np.float64) - ref) / S).max()) * 2 ** 20
                    msg += f" err {err:.3f}"
            if not same:
                d = (Cf - Cs).abs()
                msg += f" maxdiff {float(d.max()):.3g} nbad {int((d > 0).sum())}"
            print(msg, flush=True)
la.set_mode("3xtf32")

if "--quick" in sys.argv:
    sys.exit(0)


def timeit(n, m, p, fused, reps=10, graph=False):
    A, B = inputs.pair(n, m, p, "random", device="cuda")
    C = torch.empty(n, p, device="cuda")
    os.environ["LA_FUSED_SPLIT"] = "1" if fused else "0"
    for _ in range(3):
        la.gemm(A, B, out=C)
    torch.cuda.synchronize()
    if graph:
        s = torch.cuda.Stream()
        s.wait_stream(torch.cuda.current_stream())
        g = torch.cuda.CUDAGraph()
        with torch.cuda.stream(s):
            la.gemm(A, B, out=C)
            with torch.cuda.graph(g, stream=s):
                for _ in range(20):
                    la.gemm(A, B, out=C)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(reps):
            g.replay()
        e1.record()
        torch.cuda.synchronize()
        return e0.elapsed_time(e1) / (reps * 20)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    ts = []
    for _ in range(reps):
        e0.record()
        la.gemm(A, B, out=C)
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    return float(np.median(ts))


if "--debug-split" in sys.argv:
    # converter cost breakdown (LA_TMP_DEBUG: 4 = skip the A split, 8 = skip B; results garbage)
    for mode in ("3xtf32", "tf32"):
        la.set_mode(mode)
        for dbg in ("0", "4", "8", "12"):
            os.environ["LA_TMP_DEBUG"] = dbg
            t = timeit(8192, 8192, 8192, True, 5)
            print(f"{mode} 8192 debug={dbg}: {t * 1e3:.1f} us ({2 * 8192 ** 3 / t / 1e9:.1f} TF)", flush=True)
        os.environ["LA_TMP_DEBUG"] = "0"
    sys.exit(0)

for mode in ("3xtf32", "tf32"):
    la.set_mode(mode)
    for (n, m, p, graph) in [(256, 256, 256, True), (1000, 2000, 1500, True), (4096, 4096, 4096, False),
                             (8192, 8192, 8192, False), (16384, 16384, 16384, False)]:
        reps = 10 if n < 16384 else 8
        tf = timeit(n, m, p, True, reps, graph)
        ts = timeit(n, m, p, False, reps, graph)
        fl = 2.0 * n * m * p
        print(f"{mode} {n}x{m}x{p} {'graph' if graph else 'events'}: fused {tf * 1e3:.1f} us "
              f"({fl / tf / 1e9:.1f} TF)  split {ts * 1e3:.1f} us ({fl / ts / 1e9:.1f} TF)  ratio {ts / tf:.3f}",
              flush=True)
