#!/usr/bin/env python
"""Small-problem overhead: la_gemm called directly vs replayed from a CUDA graph,
plus the device time of the split and GEMM kernels (LA_OPT_KERNEL_TIMING)."""
import os
import statistics
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import inputs  # noqa: E402
import paper_1306_6192_b200 as la  # noqa: E402

la.init(0)
for (n, m, p) in [(256, 256, 256), (1000, 2000, 1500), (2048, 2048, 2048), (4096, 4096, 4096)]:
    A, B = inputs.pair(n, m, p, "random", device="cuda")
    C = torch.empty(n, p, device="cuda")
    s = torch.cuda.Stream()
    reps = 200 if n <= 2048 else 50
    with torch.cuda.stream(s):
        for _ in range(5):
            la.gemm(A, B, out=C, stream=s)
        s.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(s)
        for _ in range(reps):
            la.gemm(A, B, out=C, stream=s)
        e1.record(s)
        s.synchronize()
        direct = e0.elapsed_time(e1) / reps
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=s):
            la.gemm(A, B, out=C, stream=s)
        g.replay()
        s.synchronize()
        e0.record(s)
        for _ in range(reps):
            g.replay()
        e1.record(s)
        s.synchronize()
        graph = e0.elapsed_time(e1) / reps
        la.set_option("kernel_timing", 1)
        la.kernel_times()
        for _ in range(20):
            la.gemm(A, B, out=C, stream=s)
        s.synchronize()
        sp, gm, ng = la.kernel_times()
        la.set_option("kernel_timing", 0)
    print(f"{n}x{m}x{p}: direct {direct * 1e3:8.1f} us  graph {graph * 1e3:8.1f} us  "
          f"split {sp / 20 * 1e3:7.1f} us  gemm {gm / ng * 1e3:8.1f} us  ({2 * n * m * p / graph / 1e9:.1f} TF/s graph)")
