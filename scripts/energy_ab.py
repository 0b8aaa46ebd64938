#!/usr/bin/env python
"""Energy A/B of library env knobs at n=16384 with ~3 s windows per sample
(NVML energy counter, 20 ms clock sampling), variants alternating.

    python scripts/energy_ab.py "LA_CLC=0" "LA_WAVE_SYNC=1" ...
"""
import os
import statistics
import sys
import threading
import time

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import inputs  # noqa: E402
import paper_1306_6192_b200 as la  # noqa: E402
import pynvml  # noqa: E402

variants = sys.argv[1:] or ["BASE=1"]
n = int(os.environ.get("N", "16384"))
seconds = float(os.environ.get("SECONDS_PER_SAMPLE", "3"))
rounds = int(os.environ.get("ROUNDS", "3"))
pynvml.nvmlInit()
h = pynvml.nvmlDeviceGetHandleByIndex(0)
la.init(0)
A, B = inputs.pair(n, n, n, "random", device="cuda")
C = torch.empty(n, n, device="cuda")
la.gemm(A, B, out=C)
torch.cuda.synchronize()
t0 = time.time()
la.gemm(A, B, out=C)
torch.cuda.synchronize()
reps = max(2, int(seconds / (time.time() - t0)))
base = dict(os.environ)
res = {v: [] for v in variants}
for r in range(rounds):
    for v in variants:
        os.environ.clear()
        os.environ.update(base)
        for kv in v.split(","):
            k, val = kv.split("=", 1)
            if k.startswith("opt:"):          # library option instead of an env knob
                la.set_option(k[4:], int(val))
            else:
                os.environ[k] = val
        la.gemm(A, B, out=C)
        torch.cuda.synchronize()
        clks, stop = [], [False]

        def sample():
            while not stop[0]:
                clks.append(pynvml.nvmlDeviceGetClockInfo(h, pynvml.NVML_CLOCK_SM))
                time.sleep(0.02)
        th = threading.Thread(target=sample)
        e0 = pynvml.nvmlDeviceGetTotalEnergyConsumption(h)
        ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        th.start()
        ev0.record()
        for _ in range(reps):
            la.gemm(A, B, out=C)
        ev1.record()
        torch.cuda.synchronize()
        stop[0] = True
        th.join()
        e1 = pynvml.nvmlDeviceGetTotalEnergyConsumption(h)
        ms = ev0.elapsed_time(ev1)
        res[v].append((ms / reps, (e1 - e0) / 1e3 / reps, (e1 - e0) / ms, statistics.median(clks)))
os.environ.clear()
os.environ.update(base)
print(f"n={n} reps/sample={reps} rounds={rounds}")
print(f"{'variant':36s} {'ms/gemm':>8s} {'TF/s':>7s} {'J/gemm':>7s} {'W':>6s} {'MHz':>6s}")
for v in variants:
    for ms, j, w, c in res[v]:
        print(f"  {v:34s} {ms:8.2f} {2 * n ** 3 / ms / 1e9:7.1f} {j:7.2f} {w:6.0f} {c:6.0f}")
    ms = statistics.median(x[0] for x in res[v])
    print(f"{v:36s} {ms:8.2f} {2 * n ** 3 / ms / 1e9:7.1f} {statistics.median(x[1] for x in res[v]):7.2f} "
          f"{statistics.median(x[2] for x in res[v]):6.0f} {statistics.median(x[3] for x in res[v]):6.0f}")
