#!/usr/bin/env python
"""Config C5's size (n = 65536, A/B/C 16 GiB each) on ONE B200: la_gemm time
(3 timed calls after 1 warm-up) and the sampled error against the oracle.
The 8-GPU run of C5 needs a multi-GPU box; this is its 1-GPU baseline.

    python scripts/bench_c5.py >> profiles/configs_r01.md
"""
import os
import statistics
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import inputs  # noqa: E402
import oracle  # noqa: E402
import paper_1306_6192_b200 as la  # noqa: E402


def main():
    n = 65536
    la.init(0)
    A, B = inputs.pair(n, n, n, "random", device="cuda")
    C = torch.empty(n, n, device="cuda")
    la.gemm(A, B, out=C)
    torch.cuda.synchronize()
    ts = []
    for _ in range(3):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        la.gemm(A, B, out=C)
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    rows = np.unique(np.concatenate([np.linspace(0, n - 1, 16).astype(np.int64), [32767, 32768]]))
    cols = rows.copy()
    got = C[rows][:, cols].cpu().numpy().astype(np.float64)
    del A, B, C
    torch.cuda.empty_cache()
    As = inputs.generate(n, n, 0, "random", row_idx=rows).numpy()
    Bs = inputs.generate(n, n, 1, "random", col_idx=cols).numpy()
    ref = oracle.gemm(As, Bs, threads=max(1, len(os.sched_getaffinity(0))))
    S = oracle.abs_scale(As, Bs)
    err = float((np.abs(got - ref) / S).max() / 2.0 ** -20)
    med = statistics.median(ts)
    tf = 2.0 * n ** 3 / (med * 1e-3) / 1e12
    print(f"| C5 n=65536 (1 GPU) | 3xtf32 | {med:.1f} | {min(ts):.1f} | - | {tf:.1f} | {100 * 3 * tf / 1125.0:.1f} | "
          f"{err:.3f} | (integer: tests/test_parity.py::test_n65536_indexing_sampled) | "
          f"oracle on {len(rows)}x{len(cols)} sampled elements |", flush=True)


if __name__ == "__main__":
    main()
