#!/usr/bin/env python
"""One GPU, 1-rank communicator: cost of la_gemm_multi without gather, with
ncclAllGather, and with the fused epilogue (peer stores into the symmetric
window), n = 16384."""
import os
import statistics
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import inputs  # noqa: E402
import paper_1306_6192_b200 as la  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 16384
la.init(0)
la.comm_init(la.get_unique_id(), 0, 1)
A, B = inputs.pair(n, n, n, "random", device="cuda")
Cl = torch.empty(n, n, device="cuda")
Cn = torch.empty(n, n, device="cuda")
Cf = la.gather_buffer(n, n)
variants = {"gemm": lambda: la.gemm(A, B, out=Cl),
            "multi, no gather": lambda: la.gemm_multi(n, n, n, A, B, Cl, None, 0, 1),
            "multi + ncclAllGather": lambda: la.gemm_multi(n, n, n, A, B, Cl, Cn, 0, 1),
            "multi + fused gather": lambda: la.gemm_multi(n, n, n, A, B, Cl, Cf, 0, 1)}
res = {k: [] for k in variants}
for _ in range(3):
    for k, f in variants.items():
        f()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(3):
            f()
        e1.record()
        torch.cuda.synchronize()
        res[k].append(e0.elapsed_time(e1) / 3)
for k, v in res.items():
    print(f"{k:28s} {statistics.median(v):8.2f} ms")
print("fused == gemm bitwise:", torch.equal(Cf, Cl), " nccl == gemm:", torch.equal(Cn, Cl))
