#!/usr/bin/env python
"""Summarise an ncu report (--set full) and a launch-list CSV into profiles/.

    python scripts/ncu_summary.py gpurun_out/gemm_full.ncu-rep gpurun_out/launches.csv \
        --out profiles/ncu_r01_n16384 --n 16384 --mode 3xtf32

Writes <out>.md (human summary) and updates profiles/gemm_traffic.json (DRAM
bytes per GEMM launch, read by bench.py's roofline "traffic" field).
"""
import argparse
import csv
import io
import json
import os
import subprocess
import sys

KEYS = [
    "gpu__time_duration.sum",
    "sm__cycles_elapsed.avg.per_second",
    "sm__pipe_tensor_cycles_active_realtime.avg.pct_of_peak_sustained_elapsed",
    "sm__pipe_tensor_subpipe_hmma_cycles_active_realtime.avg",
    "sm__inst_executed_pipe_tc.sum",
    "sm__mem_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed",
    "l1tex__data_pipe_tc_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed",
    "dram__bytes_read.sum",
    "dram__bytes_write.sum",
    "dram__bytes_read.sum.per_second",
    "dram__throughput.avg.pct_of_peak_sustained_elapsed",
    "lts__t_bytes.sum",
    "lts__throughput.avg.pct_of_peak_sustained_elapsed",
    "lts__t_sector_hit_rate.pct",
    "launch__grid_size",
    "launch__cluster_size",
    "launch__registers_per_thread",
    "launch__shared_mem_per_block_dynamic",
    "sm__warps_active.avg.pct_of_peak_sustained_active",
]


def raw(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    rows = [r for r in rows if r and not r[0].startswith("==")]
    hdr, units = rows[0], rows[1]
    kernels = []
    for vals in rows[2:]:
        d = {}
        for h, u, v in zip(hdr, units, vals):
            d[h] = (v, u)
        kernels.append(d)
    return kernels


def to_bytes(v, u):
    f = float(v.replace(",", ""))
    scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12}.get(u, 1)
    return f * scale


def launches(path):
    rows = []
    for r in csv.reader(open(path)):
        if len(r) > 14 and r[0] != "ID" and not r[0].startswith("=="):
            rows.append((r[4], float(r[14])))
    tot = {}
    for name, ns in rows:
        key = name.split("(")[0]
        tot.setdefault(key, [0, 0.0])
        tot[key][0] += 1
        tot[key][1] += ns
    return rows, tot


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("rep")
    ap.add_argument("launch_csv", nargs="?")
    ap.add_argument("--out", required=True)
    ap.add_argument("--n", type=int, default=16384)
    ap.add_argument("--mode", default="3xtf32")
    ap.add_argument("--note", default="")
    a = ap.parse_args()
    ks = raw(a.rep)
    lines = [f"# ncu summary: {os.path.basename(a.rep)}", ""]
    if a.note:
        lines += [a.note, ""]
    lines += ["Captured with `ncu --set full --clock-control none --import-source on -k regex:gemm_tf32 -s 1 -c 1`",
              "under gpurun on one B200 (numbers taken under ncu are evidence, never bench values).", ""]
    traffic = None
    for i, k in enumerate(ks):
        name = k.get("Kernel Name", ("?", ""))[0]
        lines += [f"## kernel {i}: `{name}`", "", "| metric | value | unit |", "|---|---|---|"]
        for key in KEYS:
            hit = key if key in k else next((h for h in k if h.endswith("." + key) or h.endswith(key)), None)
            if hit:
                v, u = k[hit]
                lines.append(f"| {key} | {v} | {u} |")
        if "dram__bytes_read.sum" in k and "dram__bytes_write.sum" in k:
            rb = to_bytes(*k["dram__bytes_read.sum"])
            wb = to_bytes(*k["dram__bytes_write.sum"])
            traffic = rb + wb
            lines += ["", f"DRAM traffic per launch: {traffic / 1e9:.2f} GB (read {rb / 1e9:.2f}, write {wb / 1e9:.2f})"]
        lines.append("")
    if a.launch_csv and os.path.exists(a.launch_csv):
        rows, tot = launches(a.launch_csv)
        allns = sum(v[1] for v in tot.values())
        lines += ["## launch list (gpu__time_duration.sum, cold-cache, serialised)", "",
                  "| kernel | launches | total ms | share |", "|---|---|---|---|"]
        for key, (cnt, ns) in sorted(tot.items(), key=lambda x: -x[1][1]):
            lines.append(f"| `{key}` | {cnt} | {ns / 1e6:.3f} | {100 * ns / allns:.1f}% |")
        lines.append("")
    with open(a.out + ".md", "w") as f:
        f.write("\n".join(lines) + "\n")
    if traffic is not None:
        tp = os.path.join(os.path.dirname(a.out), "gemm_traffic.json")
        json.dump({"n": a.n, "mode": a.mode, "dram_bytes_per_launch": traffic,
                   "source": os.path.basename(a.out) + ".md"}, open(tp, "w"), indent=1)
    print("\n".join(lines))


if __name__ == "__main__":
    sys.exit(main())
