#!/usr/bin/env python
"""A/B two libla.so builds on la_cgemm (alternating subprocesses):
python scripts/ab_cgemm.py OLD.so NEW.so n rounds"""
import json
import os
import subprocess
import sys

old, new, n, rounds = sys.argv[1], sys.argv[2], int(sys.argv[3]), int(sys.argv[4])
code = r'''
import os, sys, json, torch
sys.path.insert(0, os.getcwd())
import paper_1306_6192_b200 as la
import inputs
n = %d
la.init(0)
re = inputs.generate(n, 2 * n, 0, "random", device="cuda")
A = torch.view_as_complex(re.view(n, n, 2)).contiguous()
re = inputs.generate(n, 2 * n, 1, "random", device="cuda")
B = torch.view_as_complex(re.view(n, n, 2)).contiguous()
C = torch.empty_like(A)
for _ in range(3): la.cgemm(A, B, out=C)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
reps = max(3, int(2e13 / (24 * n ** 3)))
e0.record()
for _ in range(reps): la.cgemm(A, B, out=C)
e1.record(); torch.cuda.synchronize()
print(json.dumps({"ms": e0.elapsed_time(e1) / reps}))
''' % n
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
    print(f"cgemm n={n} {tag}: median {v[len(v) // 2]:.3f} ms  {8 * n ** 3 / v[len(v) // 2] / 1e9:.1f} TF/s  all {['%.3f' % x for x in v]}")
