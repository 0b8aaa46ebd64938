#!/usr/bin/env python
"""Interleaved sweep of schedule knobs of the diagnostics build (LA_GROUP_M,
LA_WAVE_SYNC) at one size: every configuration once per round, median over
rounds, each call in its own process (clock / power state shared fairly).
    LA_BUILD_DIAGNOSTICS=1 python paper_1306_6192_b200/_build.py --force
    python scripts/knob_sweep.py n rounds"""
import json
import os
import statistics
import subprocess
import sys

n, rounds = int(sys.argv[1]), int(sys.argv[2])
configs = [{"LA_GROUP_M": g, "LA_WAVE_SYNC": w} for g in ("8", "4", "16") for w in ("16", "8", "32")]
code = r'''
import json, os, sys, torch
sys.path.insert(0, os.getcwd())
import inputs, paper_1306_6192_b200 as la
n = int(sys.argv[1])
la.init(0)
A, B = inputs.pair(n, n, n, "random", device="cuda")
C = torch.empty(n, n, device="cuda")
for _ in range(3): la.gemm(A, B, out=C)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
reps = max(3, int(2e13 / (6 * n ** 3)))
e0.record()
for _ in range(reps): la.gemm(A, B, out=C)
e1.record(); torch.cuda.synchronize()
print(json.dumps({"ms": e0.elapsed_time(e1) / reps}))
'''
res = {i: [] for i in range(len(configs))}
for r in range(rounds):
    for i, cfg in enumerate(configs):
        env = dict(os.environ, **cfg)
        out = subprocess.run([sys.executable, "-c", code, str(n)], capture_output=True, text=True, env=env).stdout
        res[i].append(json.loads(out.strip().splitlines()[-1])["ms"])
for i, cfg in enumerate(configs):
    ms = statistics.median(res[i])
    print(f"n={n} group_m={cfg['LA_GROUP_M']:>2} wave_sync={cfg['LA_WAVE_SYNC']:>2}: {ms:.3f} ms "
          f"{2 * n ** 3 / ms / 1e9:.1f} TF/s  {['%.3f' % x for x in sorted(res[i])]}", flush=True)
