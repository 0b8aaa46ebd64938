#!/usr/bin/env python
"""A/B libla.so builds through the raw C ABI (no binding, so builds with
different export lists compare): alternating subprocesses, median ms.
    python scripts/ab_raw.py OLD.so NEW.so n rounds [3xtf32|tf32]"""
import json
import os
import subprocess
import sys

old, new, n, rounds = sys.argv[1], sys.argv[2], int(sys.argv[3]), int(sys.argv[4])
mode = 1 if len(sys.argv) > 5 and sys.argv[5] == "tf32" else 0
code = r'''
import ctypes, json, os, sys, torch
sys.path.insert(0, os.getcwd())
import inputs
lib = ctypes.CDLL(sys.argv[1])
n, mode = int(sys.argv[2]), int(sys.argv[3])
assert lib.la_init(0) == 0 and lib.la_set_mode(mode) == 0
A, B = inputs.pair(n, n, n, "random", device="cuda")
C = torch.empty(n, n, device="cuda")
st = torch.cuda.current_stream().cuda_stream
f = lambda: lib.la_gemm(ctypes.c_int64(n), ctypes.c_int64(n), ctypes.c_int64(n), ctypes.c_void_p(A.data_ptr()),
                        ctypes.c_void_p(B.data_ptr()), ctypes.c_void_p(C.data_ptr()), ctypes.c_void_p(st))
for _ in range(3): assert f() == 0
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
reps = max(3, int(2e13 / ((6 if mode == 0 else 2) * n ** 3)))
e0.record()
for _ in range(reps): f()
e1.record(); torch.cuda.synchronize()
print(json.dumps({"ms": e0.elapsed_time(e1) / reps}))
'''
res = {"old": [], "new": []}
for r in range(rounds):
    for tag, path in (("old", old), ("new", new)):
        out = subprocess.run([sys.executable, "-c", code, os.path.abspath(path), str(n), str(mode)],
                             capture_output=True, text=True)
        res[tag].append(json.loads(out.stdout.strip().splitlines()[-1])["ms"])
for tag, v in res.items():
    v = sorted(v)
    fl = (6 if mode == 0 else 2) * n ** 3 / 3
    print(f"{'tf32' if mode else '3xtf32'} n={n} {tag}: median {v[len(v) // 2]:.3f} ms  "
          f"{2 * n ** 3 / v[len(v) // 2] / 1e9:.1f} TF/s  all {['%.3f' % x for x in v]}")
