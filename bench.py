#!/usr/bin/env python
"""Benchmark of the hot path: fp32-accurate C = A.B (3xTF32 on tcgen05) at
n = 16384 (BASELINE.json metric), printed as ONE JSON line by rank 0.

    python bench.py [--gpus N --steps K --warmup W] [--impl reference]

A step is one la_gemm call (split of A, split of B, persistent tcgen05 GEMM)
on inputs already resident in HBM.  For N > 1 (torchrun, one process per GPU)
a step is one la_gemm_multi call: A and C row-sharded, B broadcast from rank 0
with ncclBroadcast in N-panels overlapped with the GEMM (strong scaling: the
total n = 16384 problem is fixed).  Timing: W untimed warm-up steps, then K
steps between CUDA events on the launching stream, bracketed by a barrier and
torch.cuda.synchronize(); the max over ranks is reported.  Every input is
1 GiB, larger than the 126 MB L2, so no flush is needed between steps.

Extra keys: roofline (the GEMM kernel's issued TF32 FLOP/s, measured with CUDA
events around each GEMM launch inside the timed region, against the measured
peak), cpu_baseline (the oracle, Listing 1 in C, on a bounded sample on the
host cores), e2e (same metric through la_gemm_host with pinned host buffers,
copies inside the timed region), clocks (nvidia-smi during the timed region),
gpu_launches (our kernels launched in the timed region).

--impl reference runs the only reference this paper has: the oracle (the
paper's Listing 1 loop) timed on the host cores, each step a bounded sample.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import tempfile
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "fp32 GEMM TFLOP/s (2nmp/t) at n=16384, 1/2/4/8 B200; % of tensor peak"
TF32_DATASHEET_TFLOPS = 1125.0   # 148 SM x 4096 flop/clk x 1.856 GHz (dense)
TF32_PER_BF16 = 0.5              # nominal tensor-core throughput ratio (guide: 1.1 vs 2.25 PF)


def _args():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--n", type=int, default=16384)
    ap.add_argument("--m", type=int, default=None)
    ap.add_argument("--p", type=int, default=None)
    ap.add_argument("--mode", choices=["3xtf32", "tf32"], default="3xtf32")
    ap.add_argument("--inputs", choices=["random", "stress", "integer"], default="random")
    ap.add_argument("--cpu-seconds", type=float, default=12.0)
    ap.add_argument("--gather", choices=["none", "nccl", "fused"], default="none",
                    help="N>1: also assemble C on every rank (ncclAllGather, or the fused epilogue)")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    a = ap.parse_args()
    a.m = a.m or a.n
    a.p = a.p or a.n
    return a


def _peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            pk = json.load(f)
        return pk, "measured"
    except Exception:
        return {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0, "bf16_tflops_sustained": 1400.0}, "fallback"


# ----------------------------------------------------------------- clocks
class Clocks:
    """Samples SM clock, power and throttle reasons every 20 ms during the timed
    region with NVML (the library nvidia-smi reads); falls back to nvidia-smi."""
    REASONS = {"hw_slowdown": 0x8, "sw_thermal_slowdown": 0x20, "hw_thermal_slowdown": 0x40,
               "sw_power_cap": 0x4, "hw_power_brake_slowdown": 0x80}

    def __init__(self, index: int):
        self.index = index
        self.samples = []
        self._stop = False
        self._thread = None

    def _run(self):
        import pynvml
        pynvml.nvmlInit()
        h = pynvml.nvmlDeviceGetHandleByIndex(self.index)
        self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(h, pynvml.NVML_CLOCK_SM)
        while not self._stop:
            try:
                sm = pynvml.nvmlDeviceGetClockInfo(h, pynvml.NVML_CLOCK_SM)
                pw = pynvml.nvmlDeviceGetPowerUsage(h) / 1000.0
                rs = pynvml.nvmlDeviceGetCurrentClocksEventReasons(h)
                self.samples.append((sm, pw, rs))
            except Exception:
                pass
            time.sleep(0.02)

    def __enter__(self):
        import threading
        self.max_mhz = None
        try:
            import pynvml  # noqa: F401
            self._thread = threading.Thread(target=self._run, daemon=True)
            self._thread.start()
            time.sleep(0.005)
        except Exception:
            self._thread = None
        return self

    def __exit__(self, *exc):
        self._stop = True
        if self._thread is not None:
            self._thread.join(timeout=2)

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unavailable"], "samples": 0}
        sm = [x[0] for x in self.samples]
        reasons = sorted({name for _, _, r in self.samples for name, bit in self.REASONS.items() if r & bit})
        return {"sm_mhz": statistics.median(sm), "sm_max_mhz": self.max_mhz, "reasons": reasons,
                "samples": len(self.samples), "power_w_max": max(x[1] for x in self.samples),
                "power_w_median": statistics.median(x[1] for x in self.samples), "source": "NVML, 20 ms"}


# ----------------------------------------------------------------- oracle sample (CPU)
def oracle_sample(n, m, p, kind, seconds, threads):
    """Time the oracle (Listing 1 in C) on a bounded sample of the n x m . m x p
    product: R rows x S columns, sized to take about `seconds` on `threads`."""
    import numpy as np
    import inputs
    import oracle
    S = min(p, 256)
    cols = np.linspace(0, p - 1, S).astype(np.int64)
    Bs = inputs.generate(m, p, inputs.ID_B, kind, col_idx=cols).numpy()
    # calibrate
    r0 = max(threads, 8)
    rows = np.arange(r0) * max(1, n // r0)
    As = inputs.generate(n, m, inputs.ID_A, kind, row_idx=rows).numpy()
    t = time.perf_counter()
    oracle.gemm(As, Bs, threads=threads)
    dt = time.perf_counter() - t
    R = int(min(n, max(r0, r0 * seconds / max(dt, 1e-3))))
    R = max(threads, R // threads * threads)
    rows = np.linspace(0, n - 1, R).astype(np.int64)
    As = inputs.generate(n, m, inputs.ID_A, kind, row_idx=rows).numpy()
    t = time.perf_counter()
    oracle.gemm(As, Bs, threads=threads)
    dt = time.perf_counter() - t
    flops = 2.0 * R * S * m
    return flops / dt / 1e12, dt, R, S


def _threads():
    return max(1, len(os.sched_getaffinity(0)))


# ----------------------------------------------------------------- reference arm
def run_reference(a, rank, world):
    if rank != 0:
        return 0
    import oracle
    oracle.build()
    threads = _threads()
    per_step = max(1.0, min(a.cpu_seconds, 150.0 / max(1, a.steps + a.warmup)))
    for _ in range(a.warmup):
        oracle_sample(a.n, a.m, a.p, a.inputs, min(per_step, 2.0), threads)
    vals, secs, last = [], [], None
    for _ in range(a.steps):
        v, dt, R, S = oracle_sample(a.n, a.m, a.p, a.inputs, per_step, threads)
        vals.append(v)
        secs.append(dt)
        last = (R, S)
    v = statistics.median(vals)
    sample = (f"{last[0]} rows x {last[1]} cols of the n={a.n} product per step "
              f"(2*R*S*m flop), Listing 1 in C (-O2 -ffp-contract=off), {threads} threads")
    line = {
        "impl": "reference", "metric": METRIC, "value": v, "unit": "TFLOP/s", "n_gpus": world,
        "steps": a.steps, "warmup": a.warmup, "ms_per_step": 1e3 * statistics.median(secs),
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f32",
        "data": "synthetic", "config": dict(_config(a, world), mode="oracle: Listing 1, binary32 mul+add"),
        "cpu_baseline": {"value": v, "unit": "TFLOP/s", "cores": threads, "kind": "oracle", "sample": sample},
        "e2e": {"value": v, "unit": "TFLOP/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "gpu_launches": 0,
    }
    print(json.dumps(line), flush=True)
    return 0


def _config(a, world):
    return {"workload": f"square fp32 C=A.B n={a.n} (BASELINE.json configs[3]; row-sharded over {world} GPU(s))"
            if a.n == a.m == a.p else f"fp32 C=A.B {a.n}x{a.m} . {a.m}x{a.p}",
            "n": a.n, "m": a.m, "p": a.p, "mode": a.mode,
            "inputs": f"{a.inputs} (counter-based generator, seed 13066192; inputs/)",
            "l2": "inputs larger than L2 (A, B, C 1 GiB each at n=16384); no flush needed",
            "parallelism": f"rows{world}" if world > 1 else "single-gpu",
            "gather": getattr(a, "gather", "none") if world > 1 else "n/a"}


# ----------------------------------------------------------------- our arm
def run_ours(a, rank, world, local_rank):
    import numpy as np
    import torch
    import torch.distributed as dist

    import inputs
    import paper_1306_6192_b200 as la

    torch.cuda.set_device(local_rank)
    la.init(local_rank)
    la.set_mode(a.mode)
    n, m, p = a.n, a.m, a.p
    passes = 3 if a.mode == "3xtf32" else 1
    stream = torch.cuda.current_stream()

    if world > 1:
        la.comm_init_from_process_group()
        row0, rows = la.shard_rows(n, rank, world)
    else:
        row0, rows = 0, n
    A = inputs.generate(n, m, inputs.ID_A, a.inputs, device="cuda", row_idx=list(range(row0, row0 + rows)))
    B = inputs.generate(m, p, inputs.ID_B, a.inputs, device="cuda") if (world == 1 or rank == 0) else None
    C = torch.empty(rows, p, device="cuda", dtype=torch.float32)
    C_full = None
    if a.gather != "none" and world > 1:
        C_full = la.gather_buffer(n, p) if a.gather == "fused" else torch.empty(n, p, device="cuda")

    def step():
        if world == 1:
            la.gemm(A, B, out=C, stream=stream)
        else:
            la.gemm_multi(n, m, p, A, B, C, C_full, root=0, ngpu=world, stream=stream)

    la.set_option("kernel_timing", 1)
    for _ in range(a.warmup):
        step()
    torch.cuda.synchronize()
    la.kernel_times()                        # forget warm-up spans
    if world > 1:
        dist.barrier()
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    with Clocks(local_rank) as clk:
        ev0.record(stream)
        for _ in range(a.steps):
            step()
        ev1.record(stream)
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
    launches = la.last_launch_count() * a.steps
    split_ms, gemm_ms, n_gemm = la.kernel_times()
    la.set_option("kernel_timing", 0)
    ms = ev0.elapsed_time(ev1) / a.steps
    if world > 1:
        t = torch.tensor([ms], device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())
    flops = 2.0 * n * m * p
    value = flops / (ms * 1e-3) / 1e12

    # N > 1: the same steps with C assembled on every rank (the
    # all-gather is reported in its own "with gather" row): ncclAllGather after
    # the GEMMs, and the fused epilogue storing into every rank's C_full
    comm = None
    gather = None
    if world > 1:
        nr, crank = la.comm_size()
        comm = {"ncclCommCount": nr, "rank0_user_rank": crank, "backend": "nccl (library communicator)"}
        gather = {}
        for kind in ("nccl", "fused"):
            # the main line above is already measured: a failing gather variant
            # is reported in its row instead of losing the line (every rank
            # agrees on success before the next variant)
            err = ""
            try:
                Cf = la.gather_buffer(n, p) if kind == "fused" else torch.empty(n, p, device="cuda")
                for _ in range(max(1, min(a.warmup, 2))):
                    la.gemm_multi(n, m, p, A, B, C, Cf, root=0, ngpu=world, stream=stream)
                torch.cuda.synchronize()
                dist.barrier()
                g0, g1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                g0.record(stream)
                for _ in range(a.steps):
                    la.gemm_multi(n, m, p, A, B, C, Cf, root=0, ngpu=world, stream=stream)
                g1.record(stream)
                torch.cuda.synchronize()
                gms = g0.elapsed_time(g1) / a.steps
                del Cf
            except Exception as ex:  # noqa: BLE001 -- reported, not fatal
                err, gms = f"{type(ex).__name__}: {ex}"[:300], float("nan")
            ok = torch.tensor([0.0 if err else 1.0], device="cuda")
            dist.all_reduce(ok, op=dist.ReduceOp.MIN)
            gt = torch.tensor([0.0 if err else gms], device="cuda")
            dist.all_reduce(gt, op=dist.ReduceOp.MAX)
            if ok.item() < 1.0:
                gather[kind] = {"error": err or "failed on another rank"}
                break
            gms = float(gt.item())
            gather[kind] = {"ms_per_step": gms, "value": flops / (gms * 1e-3) / 1e12, "unit": "TFLOP/s",
                            "api": "la_gemm_multi + " + ("ncclAllGather" if kind == "nccl" else
                                                         "fused epilogue stores into la_gather_alloc C_full")}

    # roofline of the dominant kernel (the GEMM), per launch, this rank
    pk, src = _peaks()
    # The GEMM is the only large kernel and is timed in a region of < 1 s, so the
    # burst figure applies (the 4-s sustained cuBLAS bf16 loop runs ~15% lower).
    tf32_peak = pk.get("bf16_tflops", 1590.0) * TF32_PER_BF16
    gemm_launch_ms = gemm_ms / max(1, n_gemm)
    issued_per_launch = passes * 2.0 * rows * m * p / max(1, n_gemm // a.steps)
    achieved = issued_per_launch / (gemm_launch_ms * 1e-3) / 1e12
    traffic = None
    tpath = os.path.join(ROOT, "profiles", "gemm_traffic.json")
    if os.path.exists(tpath):
        try:
            tj = json.load(open(tpath))
            if tj.get("n") == n and tj.get("mode") == a.mode and world == 1:
                traffic = tj.get("dram_bytes_per_launch")
        except Exception:
            pass
    roofline = {"bound": "tensor", "achieved": achieved, "peak": tf32_peak, "unit": "TFLOP/s",
                "frac": achieved / tf32_peak, "traffic": traffic,
                "kernel": f"gemm_tf32_sm100 ({passes} TF32 pass{'es' if passes > 1 else ''}, issued flops)",
                "peak_source": f"{src} bf16_tflops (burst) x {TF32_PER_BF16} (nominal TF32/BF16)",
                "frac_of_sustained_peak": achieved / (pk.get("bf16_tflops_sustained", 1400.0) * TF32_PER_BF16),
                "frac_of_tf32_datasheet": achieved / TF32_DATASHEET_TFLOPS,
                "gemm_ms_per_launch": gemm_launch_ms, "split_ms_per_step": split_ms / a.steps,
                "gemm_share_of_step": gemm_ms / a.steps / ms if world == 1 else None}

    # sampled parity of the timed output (oracle, a few elements)
    parity = None
    if rank == 0:
        try:
            import oracle
            rs = np.linspace(0, rows - 1, 8).astype(np.int64)
            cs = np.linspace(0, p - 1, 8).astype(np.int64)
            As = inputs.generate(n, m, inputs.ID_A, a.inputs, row_idx=(rs + row0).tolist()).numpy()
            Bs = inputs.generate(m, p, inputs.ID_B, a.inputs, col_idx=cs.tolist()).numpy()
            ref = oracle.gemm(As, Bs, threads=_threads())
            S = oracle.abs_scale(As, Bs)
            got = C[rs][:, cs].cpu().numpy().astype(np.float64)
            parity = float((np.abs(got - ref) / S).max() / 2.0 ** -20)
        except Exception as ex:  # report, never hide
            parity = f"failed: {ex}"

    # end to end through the public API with host buffers
    e2e = None
    if not a.no_e2e:
        torch.cuda.synchronize()
        Ah = A.cpu().pin_memory()
        Bh = B.cpu().pin_memory() if B is not None else None
        Ch = torch.empty(rows, p, dtype=torch.float32).pin_memory()
        ksteps = max(2, min(a.steps, 5))
        def e2e_step():
            if world == 1:
                la.gemm_host(Ah, Bh, out=Ch, stream=stream)
            else:
                A.copy_(Ah, non_blocking=True)
                if Bh is not None:
                    B.copy_(Bh, non_blocking=True)
                la.gemm_multi(n, m, p, A, B, C, None, root=0, ngpu=world, stream=stream)
                Ch.copy_(C, non_blocking=True)
                stream.synchronize()
        e2e_step()
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        for _ in range(ksteps):
            e2e_step()
        e1.record(stream)
        torch.cuda.synchronize()
        ems = e0.elapsed_time(e1) / ksteps
        if world > 1:
            t = torch.tensor([ems], device="cuda")
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            ems = float(t.item())
        h2d = 4 * rows * m + (4 * m * p if B is not None else 0)
        e2e = {"value": flops / (ems * 1e-3) / 1e12, "unit": "TFLOP/s", "h2d_bytes_per_step": h2d,
               "d2h_bytes_per_step": 4 * rows * p, "ms_per_step": ems,
               "api": "la_gemm_host (pinned host A, B -> device -> C back)" if world == 1
               else "H2D copies + la_gemm_multi + D2H copy"}
        if world == 1:
            # the same steps as one la_gemm_host_batch call: every step still
            # copies its A, B in and its C out inside the timed region, but the
            # copy-in of step i + 1 overlaps the compute / copy-out of step i
            # (two device staging slots; outputs alternate between two buffers)
            Ch2 = torch.empty(rows, p, dtype=torch.float32).pin_memory()
            outs = [Ch if i % 2 == 0 else Ch2 for i in range(ksteps)]
            la.gemm_host_batch([Ah, Ah], [Bh, Bh], [Ch, Ch2], stream=stream)   # warm-up: both slots
            torch.cuda.synchronize()
            e0.record(stream)
            la.gemm_host_batch([Ah] * ksteps, [Bh] * ksteps, outs, stream=stream)
            e1.record(stream)
            torch.cuda.synchronize()
            bms = e0.elapsed_time(e1) / ksteps
            e2e.update({"value": flops / (bms * 1e-3) / 1e12, "ms_per_step": bms,
                        "api": f"la_gemm_host_batch of {ksteps} steps (pinned host A, B -> device -> C back "
                               "each step; copy-in of step i+1 overlaps step i)",
                        "single_call": {"value": flops / (ems * 1e-3) / 1e12, "ms_per_step": ems,
                                        "api": "la_gemm_host, one synchronous call per step"}})

    if world > 1:
        dist.barrier()
    if rank != 0:
        return 0

    cpu = None
    if not a.no_cpu_baseline and world == 1:
        threads = _threads()
        v, dt, R, S = oracle_sample(n, m, p, a.inputs, a.cpu_seconds, threads)
        cpu = {"value": v, "unit": "TFLOP/s", "cores": threads, "kind": "oracle",
               "sample": f"{R} rows x {S} cols of the n={n} product (2*R*S*m = {2.0 * R * S * m:.3g} flop) "
                         f"in {dt:.1f} s, Listing 1 in C (-O2 -ffp-contract=off), {threads} threads"}

    clocks = clk.summary()
    if clocks.get("sm_mhz"):
        roofline["frac_of_clock_limited_tf32"] = achieved / (148 * 4096 * clocks["sm_mhz"] * 1e6 / 1e12)
    line = {
        "metric": METRIC, "value": value, "unit": "TFLOP/s", "n_gpus": world, "steps": a.steps,
        "warmup": a.warmup, "ms_per_step": ms, "higher_is_better": True, "scaling": "strong",
        "vs_baseline": None, "dtype": "tf32x3" if a.mode == "3xtf32" else "tf32", "data": "synthetic",
        "config": _config(a, world),
        "pct_tf32_datasheet": 100.0 * passes * flops / (ms * 1e-3) / 1e12 / TF32_DATASHEET_TFLOPS,
        "roofline": roofline, "cpu_baseline": cpu, "e2e": e2e, "clocks": clocks,
        "gpu_launches": launches, "parity_sample_max_err_units_2^-20": parity,
        "comm": comm, "gather": gather,
        "paper_context": PAPER_CONTEXT,
    }
    print(json.dumps(line), flush=True)
    return 0


# The paper's own figures (Table 2, 4096^3 fp32 product, wall seconds; GFLOP/s
# derived as 2n^3/t): context for the line above, other hardware, not a target.
PAPER_CONTEXT = [
    {"hardware": "NVIDIA Tesla C1060 (30 SM x 8 SP)", "kernel": "Listing 3 (global memory)",
     "workload": "4096^3 fp32", "time_s": 5.81, "gflops_derived": 23.7, "source": "PAPER.md:226, Table 2"},
    {"hardware": "NVIDIA Tesla C2050", "kernel": "Listing 4 (16x16 shared-memory tiles)",
     "workload": "4096^3 fp32", "time_s": 0.83, "gflops_derived": 165.6, "source": "PAPER.md:228, Table 2"},
    {"hardware": "Intel Xeon E7-4860", "kernel": "Listing 1 (sequential loop)",
     "workload": "4096^3 fp32", "time_s": 991.96, "gflops_derived": 0.139, "source": "PAPER.md:223, Table 2"},
]


def _self_launch(a):
    """--gpus N > 1 outside a torchrun environment: start the N ranks here (one
    process per GPU through torch.distributed.run, rendezvous on 127.0.0.1) and
    return the launcher's exit status; rank 0 prints the JSON line."""
    import socket
    import torch
    have = torch.cuda.device_count()
    if have < a.gpus:
        print(f"bench.py: --gpus {a.gpus} but only {have} CUDA device(s) are visible", file=sys.stderr)
        return 2
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={a.gpus}",
           "--master-addr=127.0.0.1", f"--master-port={port}", os.path.abspath(__file__)] + sys.argv[1:]
    return subprocess.call(cmd)


def main():
    a = _args()
    launched = "WORLD_SIZE" in os.environ
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))
    if a.impl == "reference":
        # the oracle runs on the host: rank 0 of a launched job, or this process
        return run_reference(a, rank, world if launched else a.gpus)
    if launched and world != a.gpus:
        print(f"bench.py: --gpus {a.gpus} but WORLD_SIZE={world}", file=sys.stderr)
        return 2
    if not launched and a.gpus > 1:
        return _self_launch(a)
    if world > 1:
        import torch
        import torch.distributed as dist
        torch.cuda.set_device(local_rank)
        dist.init_process_group("nccl", device_id=torch.device("cuda", local_rank))
        try:
            return run_ours(a, rank, world, local_rank)
        finally:
            dist.destroy_process_group()
    return run_ours(a, rank, world, local_rank)


if __name__ == "__main__":
    sys.exit(main())
