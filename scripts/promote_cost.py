import os, sys, statistics, torch
sys.path.insert(0, os.getcwd())
import inputs, paper_1306_6192_b200 as la
la.init(0)
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
    g.replay(); torch.cuda.synchronize()
    ts = []
    for _ in range(7):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(); g.replay(); e1.record(); torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1) / calls * 1e3)
    return statistics.median(ts)
for shape in [(256, 256, 256), (4096, 256, 4096), (4096, 512, 4096), (4096, 1024, 4096), (8192, 1024, 8192)]:
    r = []
    for pk in (-1, 256):
        la.set_option("promote_k", pk)
        r.append(graph_time(*shape))
    print(shape, f"auto {r[0]:.1f} us  fixed-256 {r[1]:.1f} us  ({100 * (r[0] / r[1] - 1):+.1f}%)", flush=True)
