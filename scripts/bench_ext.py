#!/usr/bin/env python
"""Measure the NEXT rows on one GPU: matrix add against the HBM
roofline, and the complex product (Table 2 "Complex Float") at the paper's
4096 x 4096 workload and larger.  Prints markdown rows."""
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

HBM = 6551.7


def timed(fn, reps):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    ts = []
    for _ in range(reps):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        fn()
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    return statistics.median(ts)


def main():
    la.init(0)
    th = max(1, len(os.sched_getaffinity(0)))
    print("| op | size | median ms | achieved | roofline | frac | oracle host time |")
    print("|---|---|---|---|---|---|---|")
    for n in (4096, 16384):
        A = inputs.generate(n, n, 0, "random", device="cuda")
        B = inputs.generate(n, n, 1, "random", device="cuda")
        C = torch.empty_like(A)
        ms = timed(lambda: la.add(A, B, out=C), 20)
        gbs = 12.0 * n * n / (ms * 1e-3) / 1e9
        An, Bn = A.cpu().numpy(), B.cpu().numpy()
        t0 = time.perf_counter()
        oracle.elementwise(An, Bn)
        to = time.perf_counter() - t0
        print(f"| add (C = A + B) | {n}x{n} ({n * n:,} ops) | {ms:.3f} | {gbs:.0f} GB/s | {HBM:.0f} GB/s (measured copy) "
              f"| {gbs / HBM:.2f} | {to * 1e3:.1f} ms (1 thread) |", flush=True)
    for n in (4096, 8192):
        re = inputs.generate(n, 2 * n, 0, "random", device="cuda")
        A = torch.view_as_complex(re.view(n, n, 2)).contiguous()
        re = inputs.generate(n, 2 * n, 1, "random", device="cuda")
        B = torch.view_as_complex(re.view(n, n, 2)).contiguous()
        C = torch.empty_like(A)
        ms = timed(lambda: la.cgemm(A, B, out=C), 10 if n <= 4096 else 5)
        tf = 8.0 * n ** 3 / (ms * 1e-3) / 1e12
        # sampled oracle
        rows = list(np.linspace(0, n - 1, 8).astype(int))
        cols = list(np.linspace(0, n - 1, 8).astype(int))
        As, Bs = A[rows].cpu().numpy(), B[:, cols].cpu().numpy()
        t0 = time.perf_counter()
        ref = oracle.cgemm(As, Bs)
        to = (time.perf_counter() - t0) * n * n / (len(rows) * len(cols))
        Sr, Si = oracle.cabs_scale(As, Bs)
        got = C[rows][:, cols].cpu().numpy()
        err = max((np.abs(got.real - ref.real) / Sr).max(), (np.abs(got.imag - ref.imag) / Si).max()) / 2.0 ** -20
        print(f"| cgemm 3xTF32 | {n}x{n} complex | {ms:.2f} | {tf:.1f} TFLOP/s (8n^3/t) | 1125 TFLOP/s TF32 x 1/3 pass "
              f"| {3 * tf / 1125:.2f} of datasheet (issued) | ~{to:.0f} s extrapolated, 1 thread; max err {err:.3f} x 2^-20 S |",
              flush=True)


def dgemm_rows():
    la.init(0)
    for n in (4096, 8192):
        A = inputs.generate_f64(n, n, 0, device="cuda")
        B = inputs.generate_f64(n, n, 1, device="cuda")
        C = torch.empty_like(A)
        ms = timed(lambda: la.dgemm(A, B, out=C), 10 if n <= 4096 else 5)
        tf = 2.0 * n ** 3 / (ms * 1e-3) / 1e12
        msc = timed(lambda: torch.matmul(A, B, out=C), 10 if n <= 4096 else 5)
        tfc = 2.0 * n ** 3 / (msc * 1e-3) / 1e12
        rows = list(np.linspace(0, n - 1, 8).astype(int))
        cols = list(np.linspace(0, n - 1, 8).astype(int))
        C2 = la.dgemm(A, B)
        As, Bs = A[rows].cpu().numpy(), B[:, cols].cpu().numpy()
        t0 = time.perf_counter()
        ref = oracle.dgemm(As, Bs)
        to = (time.perf_counter() - t0) * n * n / 64
        S = oracle.dabs_scale(As, Bs)
        err = (np.abs(C2[rows][:, cols].cpu().numpy() - ref) / S).max() / 2.0 ** -53
        print(f"| dgemm (DMMA) | {n}x{n} | {ms:.2f} | {tf:.1f} TFLOP/s | 40 TFLOP/s FP64 datasheet; cuBLAS DGEMM "
              f"{tfc:.1f} TFLOP/s ({msc:.2f} ms) on this box | {tf / 40:.2f} of datasheet, {tf / tfc:.2f} of cuBLAS "
              f"| ~{to:.0f} s extrapolated, 1 thread; max err {err:.1f} x 2^-53 S |", flush=True)


if __name__ == "__main__":
    if len(sys.argv) > 1 and sys.argv[1] == "dgemm":
        dgemm_rows()
        sys.exit(0)
    main()
