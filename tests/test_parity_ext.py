"""GPU parity for the NEXT rows: la_add and la_cgemm (Table 2
"Complex Float").  Add/subtract is one IEEE binary32 operation per element, so
it must be bitwise equal to the oracle.  The complex product is held to the
3xTF32 bound per component (scales sum|ar||br|+|ai||bi| and sum|ar||bi|+|ai||br|)
and must be exact on integer inputs."""
import os

import numpy as np
import pytest
import torch

import inputs
import oracle

pytestmark = pytest.mark.gpu
THREADS = max(1, len(os.sched_getaffinity(0)))


@pytest.fixture(scope="module")
def la():
    import paper_1306_6192_b200 as la
    la.init(0)
    la.set_mode("3xtf32")
    return la


@pytest.mark.parametrize("rows,cols", [(1, 1), (3, 5), (4096, 4096), (1000, 1500), (7, 4099)])
@pytest.mark.parametrize("sub", [False, True])
def test_add_bitwise(la, rows, cols, sub):
    A = inputs.generate(rows, cols, 0, "stress", device="cuda")
    B = inputs.generate(rows, cols, 1, "random", device="cuda")
    C = la.add(A, B, subtract=sub)
    torch.cuda.synchronize()
    ref = oracle.elementwise(A.cpu().numpy(), B.cpu().numpy(), sub)
    assert np.array_equal(C.cpu().numpy(), ref)


def test_add_in_place_and_unaligned(la):
    A = inputs.generate(33, 65, 0, "stress", device="cuda")
    B = inputs.generate(33, 65, 1, "stress", device="cuda")
    ref = oracle.elementwise(A.cpu().numpy(), B.cpu().numpy())
    la.add(A, B, out=A)                                   # in place
    assert np.array_equal(A.cpu().numpy(), ref)
    base = torch.zeros(33 * 65 + 1, device="cuda")
    X = base[1:].view(33, 65)                             # 4-byte aligned only: scalar path
    X.copy_(B)
    la.add(X, B, out=X, subtract=True)
    assert not X.any()
    # C partially overlapping A is rejected
    assert la._lib.la_add(33, 65, A.data_ptr(), B.data_ptr(), A.data_ptr() + 4, 0, None) == la.LA_ERR_INVALID_VALUE


def _cgen(n, m, mode, mid, device="cpu"):
    re = inputs.generate(n, 2 * m, mid, mode, device=device)
    return torch.view_as_complex(re.view(n, m, 2)).contiguous()


def _ccheck(A, B, C, kind):
    An, Bn = A.cpu().numpy(), B.cpu().numpy()
    ref = oracle.cgemm(An, Bn)
    if kind == "integer":
        assert np.array_equal(C, ref)
        return
    Sr, Si = oracle.cabs_scale(An, Bn)
    er = np.abs(C.real.astype(np.float64) - ref.real) / Sr
    ei = np.abs(C.imag.astype(np.float64) - ref.imag) / Si
    worst = max(er.max(), ei.max())
    assert worst <= 2.0 ** -20, f"{worst / 2.0 ** -20:.3f} x tol"


@pytest.mark.parametrize("kind", ["integer", "random", "stress"])
@pytest.mark.parametrize("n,m,p", [(1, 1, 1), (7, 33, 5), (256, 256, 256), (300, 1000, 129), (130, 257, 513)])
def test_cgemm_parity(la, kind, n, m, p):
    A, B = _cgen(n, m, kind, 0), _cgen(m, p, kind, 1)
    C = la.cgemm(A.cuda(), B.cuda()).cpu().numpy()
    _ccheck(A, B, C, kind)


@pytest.mark.parametrize("n,m,p", [(128, 4096, 128), (200, 2500, 96)])
def test_cgemm_same_sign_integer_exact(la, n, m, p):
    """Non-negative integer real and imaginary parts: the imaginary rows of the
    real embedding are same-sign sums, where sign-centred promotion chunks
    preload offsets (K spans >= 8 chunks here); integer partial sums stay
    exact, so the product equals the complex Listing 1 value for value."""
    A, B = _cgen(n, m, "integer", 0), _cgen(m, p, "integer", 1)
    A = torch.complex(A.real.abs(), A.imag.abs())
    B = torch.complex(B.real.abs(), B.imag.abs())
    C = la.cgemm(A.cuda(), B.cuda()).cpu().numpy()
    _ccheck(A, B, C, "integer")


def test_cgemm_4096_sampled(la):
    n = 4096
    A, B = _cgen(n, n, "random", 0, "cuda"), _cgen(n, n, "random", 1, "cuda")
    C = la.cgemm(A, B)
    rows = [0, 1, 255, 256, 2047, 2048, 4095]
    cols = [0, 127, 128, 4000, 4095]
    _ccheck(A[rows].cpu(), B[:, cols].cpu(), C[rows][:, cols].cpu().numpy(), "random")


def test_cgemm_real_inputs_match_la_gemm_bitwise(la, monkeypatch):
    """Zero imaginary parts: the real part is the real product computed with the
    same K-block order and promotion chunks (the embedding appends m zero
    columns), so it equals la_gemm without split-K bitwise and the imaginary
    part is exactly zero."""
    monkeypatch.setenv("LA_SPLIT_K", "0")
    A = inputs.generate(300, 500, 0, "stress", device="cuda")
    B = inputs.generate(500, 200, 1, "stress", device="cuda")
    C = la.cgemm(A.to(torch.complex64), B.to(torch.complex64))
    R = la.gemm(A, B)
    assert torch.equal(C.real.contiguous(), R)
    assert not C.imag.any()


def _dcheck(A, B, C, kind):
    An, Bn = A.cpu().numpy(), B.cpu().numpy()
    ref = oracle.dgemm(An, Bn)
    if kind == "integer":
        assert np.array_equal(C, ref)
        return
    S = oracle.dabs_scale(An, Bn)
    m = An.shape[1]
    u = 2.0 ** -53
    g = m * u / (1 - m * u)
    ratio = (np.abs(C - ref) / np.maximum(S, 1e-300)).max()
    assert ratio <= 2 * g, f"{ratio / g:.3f} x gamma_m"


@pytest.mark.parametrize("kind", ["integer", "f64"])
@pytest.mark.parametrize("n,m,p", [(1, 1, 1), (5, 3, 7), (128, 16, 128), (129, 17, 131), (300, 1000, 257),
                                   (1024, 1024, 1024), (2, 2, 2), (258, 66, 130), (1000, 2000, 1500),
                                   (131, 34, 18)])
def test_dgemm_parity(la, kind, n, m, p):
    """Even m and p with 16-byte aligned operands take the TMA kernel (ragged
    tiles in every dimension here), odd ones the cp.async kernel."""
    A = inputs.generate_f64(n, m, 0, kind)
    B = inputs.generate_f64(m, p, 1, kind)
    C = la.dgemm(A.cuda(), B.cuda()).cpu().numpy()
    _dcheck(A, B, C, kind)


@pytest.mark.parametrize("n,m,p", [(256, 512, 256), (300, 1000, 258), (64, 4096, 130)])
def test_dgemm_tma_and_cpasync_kernels_agree(la, n, m, p, monkeypatch):
    """The TMA kernel (K permuted inside each 8-wide group) and the cp.async
    kernel: identical on integer inputs, each within the binary64 bound."""
    Ai = inputs.generate_f64(n, m, 0, "integer", device="cuda")
    Bi = inputs.generate_f64(m, p, 1, "integer", device="cuda")
    A = inputs.generate_f64(n, m, 0, device="cuda")
    B = inputs.generate_f64(m, p, 1, device="cuda")
    out = {}
    for knob in ("0", "1"):
        monkeypatch.setenv("LA_DGEMM_CPASYNC", knob)
        out[knob] = (la.dgemm(Ai, Bi).cpu(), la.dgemm(A, B).cpu())
    assert torch.equal(out["0"][0], out["1"][0])
    for knob in ("0", "1"):
        _dcheck(A.cpu(), B.cpu(), out[knob][1].numpy(), "f64")


def test_dgemm_4096_sampled(la):
    n = 4096
    A = inputs.generate_f64(n, n, 0, device="cuda")
    B = inputs.generate_f64(n, n, 1, device="cuda")
    C = la.dgemm(A, B)
    rows, cols = [0, 127, 128, 2047, 4095], [0, 1, 128, 3000, 4095]
    _dcheck(A[rows].cpu(), B[:, cols].cpu(), C[rows][:, cols].cpu().numpy(), "f64")


def test_dgemm_odd_ldc_unaligned_pairs(la):
    """p odd: the epilogue's paired (16-byte) stores must fall back to scalars."""
    A = inputs.generate_f64(70, 33, 0, "integer").cuda()
    B = inputs.generate_f64(33, 45, 1, "integer").cuda()
    _dcheck(A.cpu(), B.cpu(), la.dgemm(A, B).cpu().numpy(), "integer")
