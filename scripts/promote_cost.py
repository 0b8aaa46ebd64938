#!/usr/bin/env python
"""Device time per call (CUDA graph of 20 calls) for promotion intervals
(LA_OPT_PROMOTE_K) on short-K shapes, where the interval matters most.

    python scripts/promote_cost.py [pk ...]"""
import os
import statistics
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import inputs  # noqa: E402
import paper_1306_6192_b200 as la  # noqa: E402

la.init(0)
pks = [int(x) for x in sys.argv[1:]] or [-1, 64, 128, 256]


def graph_time(n, m, p, calls=20):
    A, B = inputs.pair(n, m, p, "random", device="cuda")
    C = torch.empty(n, p, device="cuda")
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
    for _ in range(7):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        g.replay()
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1) / calls * 1e3)
    return statistics.median(ts)


SHAPES = [(256, 256, 256), (2048, 256, 2048), (4096, 256, 4096), (8192, 256, 8192), (2048, 512, 2048),
          (4096, 512, 4096), (8192, 512, 8192), (4096, 1024, 4096)]
if os.environ.get("SHAPES"):  # e.g. SHAPES="4096x64x4096,1024x61x859"
    SHAPES = [tuple(int(v) for v in x.split("x")) for x in os.environ["SHAPES"].split(",")]
for shape in SHAPES:
    row = []
    for pk in pks:
        la.set_option("promote_k", pk)
        row.append(f"pk={pk}: {graph_time(*shape):8.1f} us")
    print(shape, " | ".join(row), flush=True)
la.set_option("promote_k", -1)
