#!/usr/bin/env python
"""End-to-end (pinned host buffers -> la_gemm_host -> host C) time at n=16384
against the panel count of the 2-D transfer schedule (LA_HOST_PANELS).

    python scripts/e2e_sweep.py [n] [q[:tail_split] ...]
"""
import os
import sys
import time

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import inputs  # noqa: E402
import paper_1306_6192_b200 as la  # noqa: E402


def main():
    n = int(sys.argv[1]) if len(sys.argv) > 1 else 16384
    qs = sys.argv[2:] or ["1", "4", "8", "16", "32"]  # "q" or "q:tail_split"
    la.init(0)
    la.set_mode(os.environ.get("E2E_MODE", "3xtf32"))
    A, B = inputs.pair(n, n, n, "random", device="cuda")
    os.environ["LA_SPLIT_K"] = "0"
    ref = la.gemm(A, B)
    t0 = time.perf_counter()
    Ah, Bh = A.cpu().pin_memory(), B.cpu().pin_memory()
    Ch = torch.empty(n, n).pin_memory()
    refh = ref.cpu()
    print(f"# pinned staging {time.perf_counter() - t0:.1f} s")
    flops = 2.0 * n ** 3
    print("| panels[:tail split] | ms per call (median of 5) | min | e2e TFLOP/s | bitwise == la_gemm |")
    print("|---|---|---|---|---|")
    for q in qs:
        os.environ["LA_HOST_PANELS"] = q.split(":")[0]
        os.environ["LA_HOST_TAIL_SPLIT"] = q.split(":")[1] if ":" in q else "4"
        Ch.zero_()
        la.gemm_host(Ah, Bh, out=Ch)
        ok = torch.equal(Ch, refh)
        ts = []
        for _ in range(5):
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            la.gemm_host(Ah, Bh, out=Ch)
            e1.record()
            torch.cuda.synchronize()
            ts.append(e0.elapsed_time(e1))
        ts.sort()
        print(f"| {q} | {ts[2]:.2f} | {ts[0]:.2f} | {flops / (ts[2] * 1e-3) / 1e12:.1f} | {ok} |", flush=True)


if __name__ == "__main__":
    main()
