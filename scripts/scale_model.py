#!/usr/bin/env python
"""Multi-GPU strong-scaling model at n = 16384 from single-GPU measurements.

This run has one B200, so the g-GPU time of la_gemm_multi is modelled from
what one GPU can measure -- each rank's own work -- plus the NVLink transfer
at the pool's measured rate (B200_PROFILING.md: 770 GB/s peer copy per
direction; 725 GB/s 8-rank all-reduce bus bandwidth):

  * per rank r: split of A_r (rows = n/g), then per B panel c: split of the
    panel + the GEMM A_r . B[:, panel c] on 148 - nccl_sms SMs (all SMs for the
    last panel) -- measured here with CUDA events (LA_OPT_KERNEL_TIMING spans)
    on exactly those shapes and SM caps;
  * the broadcast of panel c: 4 m w_c bytes at BW (+ a fixed per-call cost),
    on the comm stream, one panel after the other (the root's pack copy of
    the panel before it, at the measured D2D rate);
  * timeline: GEMM c starts when GEMM c-1 is done AND panel c has arrived.

Efficiency = T_1 / (g T_g), T_1 = la_gemm on the whole problem (measured).
Prints a table for several panel plans and writes profiles/scale_model_r02.json.

    python scripts/scale_model.py [n]
"""
import json
import os
import statistics
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import inputs  # noqa: E402
import paper_1306_6192_b200 as la  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 16384
m = p = n
BW = float(os.environ.get("NVLINK_GBS", "770")) * 1e9 * 0.9   # broadcast algorithm bandwidth (90% of peer copy)
CALL_US = 25.0                                                  # per-collective fixed cost
RESERVE = 8
os.environ["LA_SPLIT_K"] = "0"
la.init(0)
sms = torch.cuda.get_device_properties(0).multi_processor_count
A = inputs.generate(n, m, 0, "random", device="cuda")
B = inputs.generate(m, p, 1, "random", device="cuda")
C = torch.empty(n, p, device="cuda")


def timed(fn, reps=3):
    """median device ms of fn() split into (split_ms, gemm_ms) by the library's spans"""
    fn()
    torch.cuda.synchronize()
    la.set_option("kernel_timing", 1)
    la.kernel_times()
    out = []
    for _ in range(reps):
        fn()
        torch.cuda.synchronize()
        s, g, _ = la.kernel_times()
        out.append((s, g))
    la.set_option("kernel_timing", 0)
    return statistics.median(x[0] for x in out), statistics.median(x[1] for x in out)


def gemm_time(rows, w, capped):
    la.set_option("max_sms", sms - RESERVE if capped else 0)
    Ar = A[:rows]
    Bw = B[:, :w].contiguous()
    Cw = torch.empty(rows, w, device="cuda")
    s, g = timed(lambda: la.gemm(Ar, Bw, out=Cw))
    la.set_option("max_sms", 0)
    return s, g


# D2D pack rate (the root copies each panel contiguous before broadcasting it)
x = torch.empty(m, p // 4, device="cuda")
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(3):
    x.copy_(B[:, : p // 4])
e1.record()
torch.cuda.synchronize()
pack_gbs = 3 * 2 * x.numel() * 4 / (e0.elapsed_time(e1) * 1e-3) / 1e9
del x

# T_1
la.gemm(A, B, out=C)
torch.cuda.synchronize()
ts = []
for _ in range(3):
    e0.record()
    la.gemm(A, B, out=C)
    e1.record()
    torch.cuda.synchronize()
    ts.append(e0.elapsed_time(e1))
T1 = statistics.median(ts)


def plans(pw):
    """candidate panel plans (lists of widths, multiples of 256)"""
    out = {}
    for P in (1, 2, 4, 8):
        w = -(-p // P)
        w = -(-w // 256) * 256
        ws = []
        j = 0
        while j < p:
            ws.append(min(w, p - j))
            j += ws[-1]
        out[f"equal x{len(ws)}"] = ws
    for first, grow in ((512, 3), (1024, 3), (1024, 2), (2048, 2)):
        ws, j, w = [], 0, first
        while j < p:
            ww = min(w, p - j)
            if p - j - ww < first:   # no tiny last panel
                ww = p - j
            ws.append(ww)
            j += ww
            w = -(-(w * grow) // 256) * 256
        out[f"geometric {first}x{grow}"] = ws
    return out


def plans_for(g):
    out = plans(p)
    out["la_panel_plan (default)"] = la.panel_plan(n, m, p, g, sms, RESERVE)
    return out


cache = {}
result = {"n": n, "T1_ms": T1, "bw_model_gbs": BW / 1e9, "pack_gbs": pack_gbs, "nccl_sms": RESERVE, "g": {}}
print(f"n={n}: T1 = {T1:.2f} ms ({2 * n ** 3 / T1 / 1e9:.1f} TFLOP/s); broadcast modelled at {BW / 1e9:.0f} GB/s "
      f"+ {CALL_US:.0f} us/call; pack {pack_gbs:.0f} GB/s")
for g in (2, 4, 8):
    rows = n // g
    sa, _ = timed(lambda: la.gemm(A[:rows], B[:, :4].contiguous(), out=torch.empty(rows, 4, device="cuda")))
    best = None
    result["g"][g] = {}
    for name, ws in plans_for(g).items():
        for dist in (False, True):
            # dist: the root scatters 1/g of each raw panel, every rank splits
            # its slice and the hi/lo slices are all-gathered (8 bytes per
            # element arrive instead of 4; the split work per rank is 1/g)
            t_comm = 0.0
            t_comp = sa
            for c, w in enumerate(ws):
                last = c == len(ws) - 1
                key = (rows, w, not last)
                if key not in cache:
                    cache[key] = gemm_time(rows, w, not last)
                s, gm = cache[key]
                sb = max(0.0, s - sa)   # this launch also split A_r, which the multi path does once
                if dist:
                    raw = 4.0 * m * w
                    t_comm += (raw / pack_gbs / 1e9 + raw / g / BW + 8.0 * m * w * (g - 1) / g / BW +
                               2 * CALL_US * 1e-6 + sb / g * 1e-3) * 1e3
                    t_comp = max(t_comp, t_comm) + gm
                else:
                    bytes_ = 4.0 * m * w
                    t_comm += (bytes_ / pack_gbs / 1e9 + bytes_ / BW + CALL_US * 1e-6) * 1e3
                    t_comp = max(t_comp, t_comm) + sb + gm
            eff = T1 / (g * t_comp)
            label = name + (" dist-split" if dist else "")
            result["g"][g][label] = {"widths": ws, "ms": t_comp, "efficiency": eff}
            print(f"g={g} rows={rows:5d} {label:27s} panels={len(ws)} ms={t_comp:7.3f} eff={100 * eff:5.1f}%  {ws}",
                  flush=True)
            if best is None or eff > best[1]:
                best = (label, eff)
    result["g"][g]["best"] = best
out = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "gpurun_out", "scale_model.json")
os.makedirs(os.path.dirname(out), exist_ok=True)
json.dump(result, open(out, "w"), indent=1)
