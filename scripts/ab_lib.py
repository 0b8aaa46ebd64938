#!/usr/bin/env python
"""A/B two builds of libla.so in one process-alternating run (each in its own
subprocess per round), n given: python scripts/ab_lib.py OLD.so NEW.so n rounds [mode]"""
import json
import os
import subprocess
import sys

old, new, n, rounds = sys.argv[1], sys.argv[2], int(sys.argv[3]), int(sys.argv[4])
mode = sys.argv[5] if len(sys.argv) > 5 else "3xtf32"
code = r'''
import os, sys, ctypes, json, torch
sys.path.insert(0, os.getcwd())
import paper_1306_6192_b200 as la
import inputs
n = %d
la.init(0)
la.set_mode("%s")
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
''' % (n, mode)
res = {"old": [], "new": []}
lib = os.path.join("paper_1306_6192_b200", "libla.so")
keep = lib + ".keep"
os.replace(lib, keep)
try:
    for r in range(rounds):
        for tag, path in (("old", old), ("new", new if new != "CUR" else keep)):
            subprocess.check_call(["cp", path, lib])
            out = subprocess.run([sys.executable, "-c", code], capture_output=True, text=True).stdout
            res[tag].append(json.loads(out.strip().splitlines()[-1])["ms"])
finally:
    os.replace(keep, lib)
for tag, v in res.items():
    v = sorted(v)
    print(f"{mode} n={n} {tag}: median {v[len(v) // 2]:.3f} ms  {2 * n ** 3 / v[len(v) // 2] / 1e9:.1f} TF/s  all {['%.3f' % x for x in v]}")
