#!/usr/bin/env python
"""Fill the BASELINE.md rows: every BASELINE.json config that fits one GPU,
3xTF32 (and TF32 where the config asks), timed with CUDA events (and, up to
n = 2048, as a CUDA graph of 20 calls so the host is out of the loop; TFLOP/s
then come from the graph time), checked
against the oracle, with the oracle's own host time beside it.

    python scripts/bench_configs.py > profiles/configs_r01.md
"""
import os
import statistics
import sys
import time

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import inputs  # noqa: E402
import oracle  # noqa: E402
import paper_1306_6192_b200 as la  # noqa: E402

THREADS = max(1, len(os.sched_getaffinity(0)))
TF32_PEAK = 1125.0
CONFIGS = [  # (label, n, m, p, modes, full oracle?)
    ("C1 n=256", 256, 256, 256, ("3xtf32", "tf32"), True),
    ("C2 1000x2000.2000x1500", 1000, 2000, 1500, ("3xtf32", "tf32"), True),
    ("C3 n=4096", 4096, 4096, 4096, ("3xtf32", "tf32"), False),
    ("C4 n=16384", 16384, 16384, 16384, ("3xtf32", "tf32"), False),
]


def time_gemm(A, B, C, reps):
    for _ in range(3):
        la.gemm(A, B, out=C)
    torch.cuda.synchronize()
    ts = []
    for _ in range(reps):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        la.gemm(A, B, out=C)
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    return statistics.median(ts), min(ts)


def time_graph(A, B, C, calls=20, reps=5):
    """Device time per call with the host out of the loop: `calls` la_gemm
    captured in one CUDA graph, replayed `reps` times (median)."""
    s = torch.cuda.Stream()
    with torch.cuda.stream(s):
        la.gemm(A, B, out=C, stream=s)
    s.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=s):
        for _ in range(calls):
            la.gemm(A, B, out=C, stream=s)
    g.replay()
    torch.cuda.synchronize()
    ts = []
    for _ in range(reps):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        g.replay()
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1) / calls)
    return statistics.median(ts)


def main():
    la.init(0)
    print("| config | mode | median ms (events per call) | min ms | graph ms/call | logical TFLOP/s | % TF32 datasheet (issued) | max err / (2^-20 S) | integer exact | oracle (host) | oracle 1 thread | speedup vs oracle, 1 thr / all thr (Table 2 style) |")
    print("|---|---|---|---|---|---|---|---|---|---|---|---|")
    for label, n, m, p, modes, full in CONFIGS:
        A, B = inputs.pair(n, m, p, "stress", device="cuda")
        C = torch.empty(n, p, device="cuda")
        # oracle reference (full or sampled) and its host time
        if full:
            rows, cols = np.arange(n), np.arange(p)
        else:
            rows = np.unique(np.linspace(0, n - 1, 64).astype(np.int64))
            cols = np.unique(np.linspace(0, p - 1, 64).astype(np.int64))
        As = inputs.generate(n, m, 0, "stress", row_idx=rows).numpy()
        Bs = inputs.generate(m, p, 1, "stress", col_idx=cols).numpy()
        t0 = time.perf_counter()
        ref = oracle.gemm(As, Bs, threads=THREADS)
        t_or = time.perf_counter() - t0
        S = oracle.abs_scale(As, Bs)
        frac = (len(rows) * len(cols)) / (n * p)
        oracle_note = (f"{t_or:.2f} s full, {THREADS} thr" if full else
                       f"{t_or / frac:.0f} s extrapolated from {len(rows)}x{len(cols)} sample, {THREADS} thr")
        t_all = t_or / frac
        # single thread: full up to C2, else a 16 x 16 sample extrapolated
        if full:
            t0 = time.perf_counter()
            oracle.gemm(As, Bs, threads=1)
            t_one = time.perf_counter() - t0
            one_note = f"{t_one:.2f} s full"
        else:
            r1, c1 = rows[:16], cols[:16]
            t0 = time.perf_counter()
            oracle.gemm(As[:16], Bs[:, :16], threads=1)
            t_one = (time.perf_counter() - t0) * (n * p) / (len(r1) * len(c1))
            one_note = f"{t_one:.0f} s extrapolated from 16x16"
        Ai, Bi = inputs.pair(n, m, p, "integer", device="cuda")
        Ci = la.gemm(Ai, Bi)
        Ais = inputs.generate(n, m, 0, "integer", row_idx=rows).numpy()
        Bis = inputs.generate(m, p, 1, "integer", col_idx=cols).numpy()
        int_ok = np.array_equal(Ci[rows][:, cols].cpu().numpy(), oracle.gemm(Ais, Bis, threads=THREADS))
        for mode in modes:
            la.set_mode(mode)
            reps = 50 if n <= 2048 else (20 if n <= 4096 else 5)
            med, mn = time_gemm(A, B, C, reps)
            gms = time_graph(A, B, C) if n <= 2048 else None  # latency-bound sizes: host overhead out
            got = C[rows][:, cols].cpu().numpy().astype(np.float64)
            err = float((np.abs(got - ref) / S).max() / 2.0 ** -20)
            passes = 3 if mode == "3xtf32" else 1
            tf = 2.0 * n * m * p / ((gms if gms else med) * 1e-3) / 1e12
            gcol = f"{gms:.4f}" if gms else "-"
            t_gpu = (gms if gms else med) * 1e-3
            print(f"| {label} | {mode} | {med:.3f} | {mn:.3f} | {gcol} | {tf:.1f} | {100 * passes * tf / TF32_PEAK:.1f} | "
                  f"{err:.3f} | {int_ok if mode == '3xtf32' else '-'} | {oracle_note} | {one_note} | "
                  f"{t_one / t_gpu:,.0f} / {t_all / t_gpu:,.0f} |", flush=True)
        la.set_mode("3xtf32")


if __name__ == "__main__":
    main()
