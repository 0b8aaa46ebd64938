#!/usr/bin/env python
"""Epilogue A/B of two library builds on output-heavy shapes (device time per
call in a CUDA graph).  python scripts/epi_ab.py TAG"""
import os
import statistics
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import inputs  # noqa: E402
import paper_1306_6192_b200 as la  # noqa: E402

la.init(0)


def graph_time(A, B, C, calls):
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
        ts.append(e0.elapsed_time(e1) / calls * 1e3)
    return statistics.median(ts)


out = []
for shape, calls in [((65536, 64, 65536), 2), ((32768, 128, 32768), 3), ((4096, 256, 4096), 10),
                     ((8192, 512, 8192), 5), ((4096, 4096, 4096), 5), ((16384, 16384, 16384), 1)]:
    A, B = inputs.pair(*shape, "random", device="cuda")
    C = torch.empty(shape[0], shape[2], device="cuda")
    out.append(f"{shape}: {graph_time(A, B, C, calls):9.1f} us")
    del A, B, C
    torch.cuda.empty_cache()
print(sys.argv[1], " | ".join(out), flush=True)
