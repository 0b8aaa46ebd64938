"""Out-of-bounds write detection without compute-sanitizer (closed on this
pool): every output is placed inside a larger device buffer whose guard regions
hold a sentinel bit pattern; after the call the guards must be untouched and the
output exact (integer inputs) -- across ragged shapes that exercise every
predicated edge of the epilogues (tile tails, half-width tail items, column
stride 2 for complex, odd p for the DMMA paired stores)."""
import numpy as np
import pytest
import torch

import inputs
import oracle

pytestmark = pytest.mark.gpu
GUARD = 4096 + 3  # elements on each side (odd: also misaligns nothing, C stays at a 16-B offset below)
SENTINEL = -3.0e38


@pytest.fixture(scope="module")
def la():
    import paper_1306_6192_b200 as la
    la.init(0)
    la.set_mode("3xtf32")
    return la


def _guarded(count, dtype, align_elems):
    g = (GUARD // align_elems + 1) * align_elems
    buf = torch.full((g + count + g,), SENTINEL, dtype=dtype, device="cuda")
    return buf, g


def _check_guards(buf, g, count):
    lo, hi = buf[:g], buf[g + count:]
    assert torch.all(lo == SENTINEL), "write below the output"
    assert torch.all(hi == SENTINEL), "write above the output"


SHAPES = [(1, 1, 1), (17, 33, 5), (129, 257, 255), (257, 100, 383), (300, 70, 513), (1000, 64, 1500),
          (2305, 96, 2100), (4352, 64, 4360), (130, 3000, 250), (40, 16384, 70)]   # last two: split-K


@pytest.mark.parametrize("n,m,p", SHAPES)
@pytest.mark.parametrize("mode", ["3xtf32", "tf32"])
def test_gemm_guards(la, n, m, p, mode):
    A, B = inputs.pair(n, m, p, "integer", device="cuda")
    buf, g = _guarded(n * p, torch.float32, 4)
    C = buf[g:g + n * p].view(n, p)
    la.set_mode(mode)
    try:
        la.gemm(A, B, out=C)
    finally:
        la.set_mode("3xtf32")
    torch.cuda.synchronize()
    _check_guards(buf, g, n * p)
    rows = sorted({0, n // 2, n - 1})
    ref = oracle.gemm(A[rows].cpu().numpy(), B.cpu().numpy())
    assert np.array_equal(C[rows].cpu().numpy(), ref)


@pytest.mark.parametrize("n,m,p", [(1, 1, 1), (7, 33, 5), (130, 257, 513), (300, 40, 129)])
def test_cgemm_guards(la, n, m, p):
    re = inputs.generate(n, 2 * m, 0, "integer", device="cuda")
    A = torch.view_as_complex(re.view(n, m, 2)).contiguous()
    re = inputs.generate(m, 2 * p, 1, "integer", device="cuda")
    B = torch.view_as_complex(re.view(m, p, 2)).contiguous()
    buf, g = _guarded(2 * n * p, torch.float32, 4)
    C = torch.view_as_complex(buf[g:g + 2 * n * p].view(n, p, 2))
    la.cgemm(A, B, out=C)
    torch.cuda.synchronize()
    _check_guards(buf, g, 2 * n * p)
    assert np.array_equal(C.cpu().numpy(), oracle.cgemm(A.cpu().numpy(), B.cpu().numpy()))


@pytest.mark.parametrize("n,m,p", [(1, 1, 1), (5, 3, 7), (129, 17, 131), (200, 40, 255)])
def test_dgemm_guards(la, n, m, p):
    A = inputs.generate_f64(n, m, 0, "integer", device="cuda")
    B = inputs.generate_f64(m, p, 1, "integer", device="cuda")
    buf, g = _guarded(n * p, torch.float64, 2)
    C = buf[g:g + n * p].view(n, p)
    la.dgemm(A, B, out=C)
    torch.cuda.synchronize()
    _check_guards(buf, g, n * p)
    assert np.array_equal(C.cpu().numpy(), oracle.dgemm(A.cpu().numpy(), B.cpu().numpy()))


@pytest.mark.parametrize("rows,cols", [(1, 1), (3, 5), (33, 65), (64, 64)])
def test_add_guards(la, rows, cols):
    A = inputs.generate(rows, cols, 0, "integer", device="cuda")
    B = inputs.generate(rows, cols, 1, "integer", device="cuda")
    buf, g = _guarded(rows * cols, torch.float32, 4)
    C = buf[g:g + rows * cols].view(rows, cols)
    la.add(A, B, out=C)
    torch.cuda.synchronize()
    _check_guards(buf, g, rows * cols)
    assert torch.equal(C, A + B)


def test_multi_panel_guards(la, monkeypatch):
    la.comm_init(la.get_unique_id(), 0, 1)
    la.set_option("panels", 3)
    try:
        n, m, p = 300, 200, 700
        A, B = inputs.pair(n, m, p, "integer", device="cuda")
        buf, g = _guarded(n * p, torch.float32, 4)
        C = buf[g:g + n * p].view(n, p)
        la.gemm_multi(n, m, p, A, B, C, None, root=0, ngpu=1)
        torch.cuda.synchronize()
        _check_guards(buf, g, n * p)
        monkeypatch.setenv("LA_SPLIT_K", "0")
        assert torch.equal(C, la.gemm(A, B))
    finally:
        la.set_option("panels", 0)
