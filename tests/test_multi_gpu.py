"""Multi-GPU partition on real GPUs, one process
per GPU over NCCL, checked against the oracle.

Needs >= 2 GPUs and is skipped otherwise (this run's GPU boxes have one; the
host logic is covered by tests/test_multi.py's gloo world-2 test and the
device path by its 1-rank communicator tests).  With g = min(#GPUs, 8) ranks:
  * la_comm_size reports (g, rank);
  * integer inputs: every rank's C_local equals the oracle exactly on all its
    rows (sampled columns), the ncclAllGather C_full and the fused-gather C_full
    equal the oracle exactly on sampled rows of EVERY shard;
  * stress inputs: C_local within 2^-20 * sum|a||b| of the oracle;
  * C_local and C_full are bitwise equal to la_gemm on the full problem with
    split-K off (the multi path never splits K and keeps la_gemm's order).
"""
import os
import socket

import numpy as np
import pytest

import inputs

pytestmark = pytest.mark.gpu


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, q):
    try:
        import torch
        import torch.distributed as dist
        os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), LA_SPLIT_K="0")
        torch.cuda.set_device(rank)
        dist.init_process_group("nccl", rank=rank, world_size=world, device_id=torch.device("cuda", rank))
        import oracle
        import paper_1306_6192_b200 as la
        la.init(rank)
        la.set_option("panels", 3)
        la.comm_init_from_process_group()
        assert la.comm_size() == (world, rank)
        n, m, p = 128 * world + 256, 700, 900          # n % world == 0 (all-gather), ragged m, p
        row0, rows = la.shard_rows(n, rank, world)
        T = max(1, len(os.sched_getaffinity(0)) // world)
        cols = np.unique(np.linspace(0, p - 1, 40).astype(np.int64))
        samp = np.unique(np.concatenate([np.linspace(0, n - 1, 48).astype(np.int64),
                                         [la.shard_rows(n, r, world)[0] for r in range(world)]]))
        for kind in ("integer", "stress"):
            A = inputs.generate(n, m, 0, kind, device="cuda", row_idx=list(range(row0, row0 + rows)))
            B = inputs.generate(m, p, 1, kind, device="cuda") if rank == 0 else None
            Cl = torch.empty(rows, p, device="cuda")
            Cg = torch.empty(n, p, device="cuda")
            la.gemm_multi(n, m, p, A, B, Cl, Cg, root=0, ngpu=world)
            Cf = la.gather_buffer(n, p)
            Cf.fill_(-1.0)
            Cl2 = torch.empty(rows, p, device="cuda")
            la.gemm_multi(n, m, p, A, B, Cl2, Cf, root=0, ngpu=world)
            torch.cuda.synchronize()
            # oracle: this shard's rows x sampled columns; sampled rows of every shard
            As = inputs.generate(n, m, 0, kind, row_idx=list(range(row0, row0 + rows))).numpy()
            Bs = inputs.generate(m, p, 1, kind, col_idx=cols).numpy()
            ref = oracle.gemm(As, Bs, threads=T)
            got = Cl.cpu().numpy()[:, cols]
            Ar = inputs.generate(n, m, 0, kind, row_idx=samp).numpy()
            ref_all = oracle.gemm(Ar, Bs, threads=T)
            if kind == "integer":
                assert np.array_equal(got, ref), "C_local != oracle (integer)"
                assert np.array_equal(Cg.cpu().numpy()[samp][:, cols], ref_all), "ncclAllGather C != oracle"
                assert np.array_equal(Cf.cpu().numpy()[samp][:, cols], ref_all), "fused-gather C != oracle"
            else:
                S = oracle.abs_scale(As, Bs)
                assert float((np.abs(got.astype(np.float64) - ref) / S).max()) <= 2.0 ** -20
                S_all = oracle.abs_scale(Ar, Bs)
                for Cx in (Cg, Cf):
                    err = np.abs(Cx.cpu().numpy()[samp][:, cols].astype(np.float64) - ref_all) / S_all
                    assert float(err.max()) <= 2.0 ** -20
            # bitwise: la_gemm on the full problem (split-K off), on every rank
            Afull = inputs.generate(n, m, 0, kind, device="cuda")
            Bfull = inputs.generate(m, p, 1, kind, device="cuda")
            single = la.gemm(Afull, Bfull)
            torch.cuda.synchronize()
            assert torch.equal(Cl, single[row0:row0 + rows]) and torch.equal(Cl2, Cl)
            assert torch.equal(Cg, single) and torch.equal(Cf, single)
        dist.barrier()
        la.finalize()
        dist.destroy_process_group()
        q.put((rank, "ok"))
    except Exception as ex:  # reported to the parent
        import traceback
        q.put((rank, repr(ex) + traceback.format_exc()[-1500:]))


def test_multi_rank_against_oracle():
    import torch
    import torch.multiprocessing as mp
    world = min(torch.cuda.device_count(), 8)
    if world < 2:
        pytest.skip("needs >= 2 GPUs (one process per GPU); 1-rank device path in tests/test_multi.py")
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for pr in procs:
        pr.start()
    res = dict(q.get(timeout=600) for _ in procs)
    for pr in procs:
        pr.join(timeout=120)
    assert res == {r: "ok" for r in range(world)}, res
