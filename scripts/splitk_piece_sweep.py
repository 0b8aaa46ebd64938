#!/usr/bin/env python
"""Graph time per call vs the split-K minimum piece of single-CTA launches
(LA_SPLITK_MIN_PIECE1, diagnostics build; CTA pairs keep 8), configurations interleaved over rounds so clock drift
hits all of them alike; median per configuration.
    LA_BUILD_DIAGNOSTICS=1 python paper_1306_6192_b200/_build.py --force
    python scripts/splitk_piece_sweep.py [rounds]"""
import os
import statistics
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import inputs  # noqa: E402
import paper_1306_6192_b200 as la  # noqa: E402

la.init(0)
rounds = int(sys.argv[1]) if len(sys.argv) > 1 else 5


def graph_us(A, B, C, calls=40, reps=5):
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    g = torch.cuda.CUDAGraph()
    with torch.cuda.stream(s):
        la.gemm(A, B, out=C)
        with torch.cuda.graph(g, stream=s):
            for _ in range(calls):
                la.gemm(A, B, out=C)
    torch.cuda.synchronize()
    g.replay()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        g.replay()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / (calls * reps) * 1e3


shapes = [(256, 256, 256), (512, 512, 512), (256, 2048, 256), (128, 4096, 128), (777, 1236, 260),
          (1000, 2000, 1500), (512, 8192, 512), (300, 500, 200), (1024, 1024, 1024), (640, 3000, 700),
          (384, 1536, 384), (2000, 700, 300)]
pieces = [(8, 8), (4, 8)]   # (single CTA, CTA pair): (4, 8) = the default rule (4 while <= 3/4 of the SMs)
for (n, m, p) in shapes:
    A, B = inputs.pair(n, m, p, "random", device="cuda")
    C = torch.empty(n, p, device="cuda")
    res = {pc: [] for pc in pieces}
    for r in range(rounds):
        for pc in pieces:
            os.environ["LA_SPLITK_MIN_PIECE1"] = str(pc[0])
            res[pc].append(graph_us(A, B, C))
    print(f"{n}x{m}x{p}: " + "  ".join(f"pieces {pc}: {statistics.median(v):6.2f} us" for pc, v in res.items()),
          flush=True)
