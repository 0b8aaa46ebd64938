#!/usr/bin/env python
"""Per-kernel breakdown of small products (C1, C2, ...): CUDA-graph time per
call, and events around the split, GEMM and split-K reduce launches
(LA_OPT_KERNEL_TIMING; the events serialise the PDL overlap, so the parts sum
to more than the graph time).   python scripts/small_breakdown.py [n m p ...]"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import inputs  # noqa: E402
import paper_1306_6192_b200 as la  # noqa: E402

la.init(0)
shapes = [(256, 256, 256), (1000, 2000, 1500), (2048, 2048, 2048)]
if len(sys.argv) >= 4:
    v = [int(x) for x in sys.argv[1:]]
    shapes = [tuple(v[i:i + 3]) for i in range(0, len(v) - 2, 3)]
for (n, m, p) in shapes:
    A, B = inputs.pair(n, m, p, "random", device="cuda")
    C = torch.empty(n, p, device="cuda")
    for _ in range(3):
        la.gemm(A, B, out=C)
    torch.cuda.synchronize()
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    g = torch.cuda.CUDAGraph()
    with torch.cuda.stream(s):
        la.gemm(A, B, out=C)
        with torch.cuda.graph(g, stream=s):
            for _ in range(50):
                la.gemm(A, B, out=C)
    torch.cuda.synchronize()
    for _ in range(3):
        g.replay()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(10):
        g.replay()
    e1.record()
    torch.cuda.synchronize()
    graph_us = e0.elapsed_time(e1) / 500 * 1e3
    la.set_option("kernel_timing", 1)
    la.kernel_times()
    reps = 20
    for _ in range(reps):
        la.gemm(A, B, out=C)
    torch.cuda.synchronize()
    aux, gemm, nl = la.kernel_times()
    la.set_option("kernel_timing", 0)
    print(f"{n}x{m}x{p}: graph {graph_us:.1f} us/call ({2 * n * m * p / graph_us / 1e6:.1f} TF) | "
          f"events: split+reduce {aux / reps * 1e3:.1f} us, gemm {gemm / reps * 1e3:.1f} us, "
          f"launches/call {la.last_launch_count()}", flush=True)
