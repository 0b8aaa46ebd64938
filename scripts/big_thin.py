#!/usr/bin/env python
"""Big, thin shapes (outputs of 4-16 GiB with short K, or long K with few
outputs): runs, sampled integer exactness, time."""
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import inputs  # noqa: E402
import oracle  # noqa: E402
import paper_1306_6192_b200 as la  # noqa: E402

la.init(0)
for (n, m, p) in [(65536, 64, 65536), (32768, 256, 32768), (64, 1 << 20, 64), (100000, 3, 20000)]:
    A, B = inputs.pair(n, m, p, "integer", device="cuda")
    C = la.gemm(A, B)
    torch.cuda.synchronize()
    t0 = time.time()
    la.gemm(A, B, out=C)
    torch.cuda.synchronize()
    dt = time.time() - t0
    rows = np.unique(np.array([0, n // 3, n - 1]))
    cols = np.unique(np.array([0, p // 2, p - 1]))
    got = C[rows][:, cols].cpu().numpy()
    ref = oracle.gemm(inputs.generate(n, m, 0, "integer", row_idx=rows).numpy(),
                      inputs.generate(m, p, 1, "integer", col_idx=cols).numpy())
    print(f"{n}x{m}x{p}: {dt * 1e3:.1f} ms, {2.0 * n * m * p / dt / 1e12:.1f} TFLOP/s, sampled exact "
          f"{np.array_equal(got, ref)}", flush=True)
    del A, B, C
    torch.cuda.empty_cache()
