"""Multi-GPU partition.

This run has one GPU, so:
  * the host-side logic of the partition runs in a world-size-2 gloo group on
    the CPU: the NCCL unique-id bootstrap, the row sharding (la_shard_rows) and
    the reassembly of C from row shards (each rank multiplies its shard with the
    oracle, the shards are all-gathered and must equal the full product);
  * the device path of la_gemm_multi (panel packing, ncclBroadcast of B,
    per-panel split + GEMM into column blocks of C, ncclAllGather) runs on one
    B200 with a 1-rank communicator and must be bitwise equal to la_gemm.
"""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import inputs


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, q):
    try:
        os.environ["MASTER_ADDR"] = "127.0.0.1"
        os.environ["MASTER_PORT"] = str(port)
        dist.init_process_group("gloo", rank=rank, world_size=world)
        import oracle
        import paper_1306_6192_b200 as la
        # 1. unique-id bootstrap: every rank sees rank 0's id
        uid = la.bootstrap_unique_id()
        ids = [None] * world
        dist.all_gather_object(ids, uid)
        assert all(x == ids[0] for x in ids) and len(uid) == 128 and any(uid)
        # 2. row sharding + reassembly of C, n not divisible by world
        n, m, p = 37, 50, 23
        row0, rows = la.shard_rows(n, rank, world)
        A = inputs.generate(n, m, 0, "integer", row_idx=list(range(row0, row0 + rows))).numpy()
        B = inputs.generate(m, p, 1, "integer").numpy()
        Cr = oracle.gemm(A, B)
        parts = [None] * world
        dist.all_gather_object(parts, (row0, Cr))
        full = np.concatenate([c for _, c in sorted(parts, key=lambda x: x[0])])
        Afull, _ = inputs.pair(n, m, p, "integer")
        assert np.array_equal(full, oracle.gemm(Afull.numpy(), B))
        # 3. max over ranks (bench timing rule)
        t = torch.tensor([float(rank + 1)])
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        assert t.item() == world
        dist.destroy_process_group()
        q.put((rank, "ok"))
    except Exception as ex:  # pragma: no cover - reported to the parent
        q.put((rank, repr(ex)))


def test_gloo_world2_host_logic():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for pr in procs:
        pr.start()
    res = dict(q.get(timeout=240) for _ in procs)
    for pr in procs:
        pr.join(timeout=60)
    assert res == {0: "ok", 1: "ok"}, res


@pytest.fixture(scope="module")
def la1():
    import paper_1306_6192_b200 as la
    la.init(0)
    la.comm_init(la.get_unique_id(), 0, 1)
    yield la
    la.set_option("panels", 0)


@pytest.mark.gpu
@pytest.mark.parametrize("n,m,p,g", [(4096, 2048, 8192, 2), (8192, 2048, 8192, 2), (2048, 8192, 8192, 8)])
def test_multi_model_panel_plan_bitwise(la1, n, m, p, g, monkeypatch):
    """The timeline model's unequal panels (narrow first panel, wider later
    ones: planned as for g ranks through LA_TEST_PLAN_NGPU) executed with one
    rank: bitwise equal to la_gemm without split-K, and integer inputs equal to
    the oracle on sampled elements."""
    import oracle
    la = la1
    la.set_option("panels", 0)
    ws = la.panel_plan(n, m, p, g)
    assert len(ws) > 1 and len(set(ws)) > 1, ws
    monkeypatch.setenv("LA_SPLIT_K", "0")
    monkeypatch.setenv("LA_TEST_PLAN_NGPU", str(g))
    for kind in ("stress", "integer"):
        A, B = inputs.pair(n, m, p, kind, device="cuda")
        ref = la.gemm(A, B)
        Cl = torch.empty(n, p, device="cuda")
        la.gemm_multi(n, m, p, A, B, Cl, None, root=0, ngpu=1)
        torch.cuda.synchronize()
        assert torch.equal(Cl, ref)
        if kind == "integer":
            rows = np.linspace(0, n - 1, 16).astype(np.int64)
            cols = np.unique(np.concatenate([np.cumsum([0] + ws[:-1]), np.linspace(0, p - 1, 24).astype(np.int64)]))
            got = Cl.cpu().numpy()[rows][:, cols]
            want = oracle.gemm(A.cpu().numpy()[rows], B.cpu().numpy()[:, cols], threads=8)
            assert np.array_equal(got, want)


@pytest.mark.gpu
@pytest.mark.parametrize("n,m,p,panels", [(512, 384, 640, 1), (512, 384, 640, 3), (300, 1000, 1500, 4),
                                          (4096, 2048, 4096, 4), (300, 1000, 1501, 4), (257, 70, 999, 2)])
def test_multi_one_rank_bitwise_equals_single(la1, n, m, p, panels, monkeypatch):
    la = la1
    la.set_option("panels", panels)
    monkeypatch.setenv("LA_SPLIT_K", "0")   # the multi path never splits K
    A, B = inputs.pair(n, m, p, "stress", device="cuda")
    ref = la.gemm(A, B)
    Cl = torch.empty(n, p, device="cuda")
    Cf = torch.empty(n, p, device="cuda")
    la.gemm_multi(n, m, p, A, B, Cl, Cf, root=0, ngpu=1)
    torch.cuda.synchronize()
    assert torch.equal(Cl, ref)
    assert torch.equal(Cf, ref)
    ws = la.panel_plan(n, m, p, 1, panels=panels)    # equal panels, multiples of 256 but the last
    assert len(ws) == -(-p // (-(-(-(-p // panels)) // 256) * 256))
    assert la.last_launch_count() == 1 + 2 * len(ws)  # split A, then split B + GEMM per panel


@pytest.mark.gpu
def test_multi_one_rank_tf32_mode(la1, monkeypatch):
    """Plain TF32 mode through the multi path equals la_gemm in the same mode."""
    la = la1
    la.set_option("panels", 3)
    monkeypatch.setenv("LA_SPLIT_K", "0")
    n, m, p = 640, 512, 1000
    A, B = inputs.pair(n, m, p, "stress", device="cuda")
    la.set_mode("tf32")
    try:
        ref = la.gemm(A, B)
        Cl = torch.empty(n, p, device="cuda")
        la.gemm_multi(n, m, p, A, B, Cl, None, root=0, ngpu=1)
        torch.cuda.synchronize()
    finally:
        la.set_mode("3xtf32")
    assert torch.equal(Cl, ref)


@pytest.mark.gpu
def test_multi_errors(la1):
    la = la1
    A = torch.zeros(8, 8, device="cuda")
    with pytest.raises(la.LaError):
        la.gemm_multi(8, 8, 8, A, A, torch.empty(8, 8, device="cuda"), None, root=0, ngpu=2)
    with pytest.raises(la.LaError):
        la.gemm_multi(8, 8, 8, A, None, torch.empty(8, 8, device="cuda"), None, root=0, ngpu=1)


@pytest.mark.gpu
@pytest.mark.parametrize("panels", [1, 3])
def test_fused_gather_one_rank_bitwise(la1, panels, monkeypatch):
    """Fused GEMM -> all-gather (la_gather_alloc + la_gemm_multi): with one rank
    the epilogue's peer stores land in this rank's own symmetric window, which
    must equal la_gemm bitwise; C_local is written as well."""
    la = la1
    la.set_option("panels", panels)
    monkeypatch.setenv("LA_SPLIT_K", "0")
    n, m, p = 700, 500, 900
    A, B = inputs.pair(n, m, p, "stress", device="cuda")
    ref = la.gemm(A, B)
    Cf = la.gather_buffer(n, p)
    Cf.fill_(-1.0)
    Cl = torch.empty(n, p, device="cuda")
    la.gemm_multi(n, m, p, A, B, Cl, Cf, root=0, ngpu=1)
    torch.cuda.synchronize()
    assert torch.equal(Cl, ref)
    assert torch.equal(Cf, ref)


@pytest.mark.gpu
def test_fused_gather_row_offset(la1, monkeypatch):
    """Exercise a non-zero destination row (rank r writes rows r*n/g...) on one
    GPU through the test hook LA_TEST_GATHER_ROW0: rows [7, 7+n) of a larger
    symmetric buffer receive C, every other element keeps its sentinel."""
    la = la1
    la.set_option("panels", 2)
    monkeypatch.setenv("LA_SPLIT_K", "0")
    n, m, p = 300, 130, 520
    A, B = inputs.pair(n, m, p, "integer", device="cuda")
    ref = la.gemm(A, B)
    Cf = la.gather_buffer(n + 20, p)
    Cf.fill_(-7.0)
    Cl = torch.empty(n, p, device="cuda")
    monkeypatch.setenv("LA_TEST_GATHER_ROW0", "7")
    la.gemm_multi(n, m, p, A, B, Cl, Cf, root=0, ngpu=1)
    torch.cuda.synchronize()
    assert torch.equal(Cf[7:7 + n], ref)
    assert torch.all(Cf[:7] == -7.0) and torch.all(Cf[7 + n:] == -7.0)


@pytest.mark.gpu
@pytest.mark.parametrize("g,kind", [(2, "integer"), (3, "stress"), (4, "integer"), (8, "stress")])
def test_fused_gather_emulated_ranks_vs_oracle(la1, g, kind, monkeypatch):
    """One GPU emulating g ranks of the fused GEMM -> all-gather (SURVEY 8(f)
    NEXT #1): every emulated rank r runs la_gemm_multi on its own rows of A
    (la_shard_rows) with the test hooks LA_TEST_GATHER_ROW0 = its first row and
    LA_TEST_GATHER_PEERS = g, so its epilogue stores its rows into g C_full
    copies (consecutive regions of one symmetric window, standing in for the g
    ranks' buffers).  The launches do not wait on one another.  After the g
    calls every copy must hold the whole product: the oracle exactly on
    integer inputs, within 2^-20 * sum|a||b| on stress inputs."""
    import oracle
    la = la1
    la.set_option("panels", 2)
    monkeypatch.setenv("LA_SPLIT_K", "0")
    n, m, p = 97 * g + 31, 300, 520
    A, B = inputs.pair(n, m, p, kind, device="cuda")
    Cf = la.gather_buffer(g * n, p)
    Cf.fill_(-3.0)
    monkeypatch.setenv("LA_TEST_GATHER_PEERS", str(g))
    monkeypatch.setenv("LA_TEST_GATHER_STRIDE", str(n * p))
    for r in range(g):
        row0, rows = la.shard_rows(n, r, g)
        monkeypatch.setenv("LA_TEST_GATHER_ROW0", str(row0))
        Cl = torch.empty(rows, p, device="cuda")
        la.gemm_multi(rows, m, p, A[row0:row0 + rows].contiguous(), B, Cl, Cf, root=0, ngpu=1)
    torch.cuda.synchronize()
    An, Bn = A.cpu().numpy(), B.cpu().numpy()
    ref = oracle.gemm(An, Bn, threads=8)
    S = oracle.abs_scale(An, Bn)
    copies = Cf.cpu().numpy().reshape(g, n, p)
    for pe in range(g):
        if kind == "integer":
            assert np.array_equal(copies[pe], ref), pe
        else:
            assert float((np.abs(copies[pe].astype(np.float64) - ref) / S).max()) <= 2.0 ** -20, pe
    assert np.array_equal(copies[0], copies[g - 1])


@pytest.mark.parametrize("n,m,p,g", [(16384, 16384, 16384, 2), (16384, 16384, 16384, 8), (65536, 65536, 65536, 8),
                                     (1000, 2000, 1500, 2), (4096, 300, 777, 4), (512, 512, 100, 8)])
def test_panel_plan_host(n, m, p, g):
    """la_panel_plan (host arithmetic, no GPU): the panels tile B's columns in
    order, widths are multiples of the 256-wide pair tile except the last, the
    model-chosen plan never starts with a panel wider than the next one (the
    first broadcast is the one nothing overlaps), one GPU gets one panel, and a
    forced count gives equal panels."""
    import paper_1306_6192_b200 as la
    ws = la.panel_plan(n, m, p, g)
    assert sum(ws) == p and all(w > 0 for w in ws)
    assert all(w % 256 == 0 for w in ws[:-1])
    if len(ws) > 1:
        assert ws[0] <= ws[1]
    assert la.panel_plan(n, m, p, 1) == [p]
    for P in (1, 3, 4):
        eq = la.panel_plan(n, m, p, g, panels=P)
        assert sum(eq) == p and len(eq) <= P and len(set(eq[:-1])) <= 1
    with pytest.raises(la.LaError):
        la.panel_plan(n, m, p, g, panels=-1)
    with pytest.raises(la.LaError):
        la.panel_plan(0, m, p, g)
