"""Seeded shape fuzz on the GPU: random (n, m, p), log-uniform in [1, 1200],
integer-valued inputs -> every product kind must equal its oracle exactly; and
the two GEMM kernels (single CTA 128x128 vs CTA pair 256x256) must agree
bitwise on the same inputs, because per-element accumulation order does not
depend on the tile shape."""
import os

import numpy as np
import pytest
import torch

import inputs
import oracle

pytestmark = pytest.mark.gpu
RNG = np.random.default_rng(20261018)
SHAPES = [tuple(int(x) for x in np.exp(RNG.uniform(0, np.log(1200), 3)).round().clip(1)) for _ in range(40)]


@pytest.fixture(scope="module")
def la():
    import paper_1306_6192_b200 as la
    la.init(0)
    la.set_mode("3xtf32")
    return la


@pytest.mark.parametrize("n,m,p", SHAPES)
def test_fuzz_gemm_integer_exact(la, n, m, p):
    A = inputs.generate(n, m, 0, "integer", seed=n * 7919 + m * 31 + p)
    B = inputs.generate(m, p, 1, "integer", seed=n * 7919 + m * 31 + p)
    C = la.gemm(A.cuda(), B.cuda()).cpu().numpy()
    assert np.array_equal(C, oracle.gemm(A.numpy(), B.numpy(), threads=8))


@pytest.mark.parametrize("n,m,p", SHAPES[:12])
def test_fuzz_kernels_agree_bitwise(la, n, m, p, monkeypatch):
    A, B = inputs.pair(n, m, p, "stress", device="cuda")
    monkeypatch.setenv("LA_SPLIT_K", "0")   # split factors depend on the tile count
    out = {}
    for cg in ("1", "2"):
        monkeypatch.setenv("LA_CTA_GROUP", cg)
        out[cg] = la.gemm(A, B)
    torch.cuda.synchronize()
    assert torch.equal(out["1"], out["2"])


@pytest.mark.parametrize("n,m,p", SHAPES[:10])
def test_fuzz_cgemm_dgemm_integer_exact(la, n, m, p):
    re = inputs.generate(n, 2 * m, 0, "integer")
    A = torch.view_as_complex(re.view(n, m, 2)).contiguous()
    re = inputs.generate(m, 2 * p, 1, "integer")
    B = torch.view_as_complex(re.view(m, p, 2)).contiguous()
    C = la.cgemm(A.cuda(), B.cuda()).cpu().numpy()
    assert np.array_equal(C, oracle.cgemm(A.numpy(), B.numpy()))
    Ad = inputs.generate_f64(n, m, 0, "integer")
    Bd = inputs.generate_f64(m, p, 1, "integer")
    D = la.dgemm(Ad.cuda(), Bd.cuda()).cpu().numpy()
    assert np.array_equal(D, oracle.dgemm(Ad.numpy(), Bd.numpy()))


# Degenerate aspect ratios: dot products, outer products, single rows/columns,
# very long K (split-K with many pieces), K = 1.  Integer inputs: exact.
EXTREME = [(1, 65536, 1), (1, 1, 4096), (4096, 1, 1), (2, 200000, 3), (4096, 1, 4096), (1, 70000, 1000),
           (1000, 70000, 1), (7, 3, 9000), (9000, 3, 7), (33, 123457, 65)]


@pytest.mark.parametrize("n,m,p", EXTREME)
@pytest.mark.parametrize("mode", ["3xtf32", "tf32"])
def test_extreme_shapes_integer_exact(la, n, m, p, mode):
    """Integer inputs in [-8, 8]: the product is exact in both modes (TF32
    represents these integers exactly, and every partial sum stays < 2^24)."""
    A = inputs.generate(n, m, 0, "integer", seed=n + 3 * m + 7 * p)
    B = inputs.generate(m, p, 1, "integer", seed=n + 3 * m + 7 * p)
    la.set_mode(mode)
    try:
        C = la.gemm(A.cuda(), B.cuda()).cpu().numpy()
    finally:
        la.set_mode("3xtf32")
    assert np.array_equal(C, oracle.gemm(A.numpy(), B.numpy(), threads=8))
