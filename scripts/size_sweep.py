#!/usr/bin/env python
"""Throughput of la_gemm (3xTF32 and plain TF32) over square sizes: device
time per call (CUDA graph of calls for small sizes, events for large),
logical TFLOP/s = 2n^3/t.  python scripts/size_sweep.py > profiles/size_sweep_r01.md"""
import os
import statistics
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import inputs  # noqa: E402
import paper_1306_6192_b200 as la  # noqa: E402

la.init(0)


def timed(A, B, C, n):
    calls = max(1, min(50, int(2e12 / (6 * n ** 3))))
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
    for _ in range(5):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        g.replay()
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1) / calls)
    return statistics.median(ts)


print("| n | 3xTF32 ms | 3xTF32 TFLOP/s | TF32 ms | TF32 TFLOP/s |")
print("|---|---|---|---|---|")
for n in (512, 1024, 1536, 2048, 3072, 4096, 6144, 8192, 12288, 16384):
    A, B = inputs.pair(n, n, n, "random", device="cuda")
    C = torch.empty(n, n, device="cuda")
    row = [str(n)]
    for mode in ("3xtf32", "tf32"):
        la.set_mode(mode)
        ms = timed(A, B, C, n)
        row += [f"{ms:.3f}", f"{2 * n ** 3 / ms / 1e9:.1f}"]
    la.set_mode("3xtf32")
    print("| " + " | ".join(row) + " |", flush=True)
    del A, B, C
