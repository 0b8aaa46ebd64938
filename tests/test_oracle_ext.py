"""Pins for the oracle's NEXT-row functions: matrix add/subtract and the
complex product (Table 2 "Complex Float").  No GPU needed."""
import os

import numpy as np
import pytest

import inputs
import oracle

GOLDEN = os.path.join(os.path.dirname(__file__), "golden", "complex_examples.txt")


def _read_complex_golden():
    lines = [l.split("#")[0].strip() for l in open(GOLDEN)]
    lines = [l for l in lines if l]
    out, cur, i = [], {}, 0
    while i < len(lines):
        tag, r, c = lines[i].split()
        r, c = int(r), int(c)
        rows = []
        for k in range(r):
            v = [float(x) for x in lines[i + 1 + k].split()]
            rows.append([complex(v[2 * j], v[2 * j + 1]) for j in range(c)])
        cur[tag] = np.array(rows, np.complex64)
        i += 1 + r
        if tag == "C":
            out.append(cur)
            cur = {}
    return out


def _cgen(n, m, mode, mid, seed=inputs.SEED):
    re = inputs.generate(n, 2 * m, mid, mode, seed).numpy()
    return (re[:, 0::2] + 1j * re[:, 1::2]).astype(np.complex64)


# ------------------------------------------------------------------ add/sub
def test_elementwise_identities():
    A = inputs.generate(37, 53, 0, "stress").numpy()
    Z = np.zeros_like(A)
    assert np.array_equal(oracle.elementwise(A, Z), A)
    assert np.array_equal(oracle.elementwise(A, A, subtract=True), Z)
    I = inputs.generate(37, 53, 1, "integer").numpy()
    Ai = inputs.generate(37, 53, 0, "integer").numpy()
    assert np.array_equal(oracle.elementwise(oracle.elementwise(Ai, I), I, subtract=True), Ai)


def test_elementwise_matches_numpy_binary32():
    A = inputs.generate(64, 70, 0, "stress").numpy()
    B = inputs.generate(64, 70, 1, "random").numpy()
    assert np.array_equal(oracle.elementwise(A, B), np.add(A, B, dtype=np.float32))
    assert np.array_equal(oracle.elementwise(A, B, True), np.subtract(A, B, dtype=np.float32))


def test_paper_add_op_count():
    """a 4096 x 4096 add is 16,777,216 elementary operations."""
    assert 4096 * 4096 == 16_777_216


# ------------------------------------------------------------------ complex
def test_complex_golden():
    for b in _read_complex_golden():
        assert np.array_equal(oracle.cgemm(b["A"], b["B"]), b["C"])


def test_complex_integer_bruteforce():
    rng = np.random.default_rng(9)
    for n in range(1, 6):
        for m in range(1, 6):
            for p in range(1, 6):
                A = (rng.integers(-8, 9, (n, m)) + 1j * rng.integers(-8, 9, (n, m))).astype(np.complex64)
                B = (rng.integers(-8, 9, (m, p)) + 1j * rng.integers(-8, 9, (m, p))).astype(np.complex64)
                ref = A.astype(np.complex128) @ B.astype(np.complex128)
                assert np.array_equal(oracle.cgemm(A, B).astype(np.complex128), ref), (n, m, p)


def test_complex_with_zero_imaginary_is_the_real_oracle():
    A = inputs.generate(9, 300, 0, "stress").numpy()
    B = inputs.generate(300, 7, 1, "stress").numpy()
    C = oracle.cgemm(A.astype(np.complex64), B.astype(np.complex64))
    assert np.array_equal(C.real, oracle.gemm(A, B)) and not C.imag.any()


def test_complex_conjugate_symmetry_bitwise():
    A, B = _cgen(11, 200, "stress", 0), _cgen(200, 13, "stress", 1)
    C = oracle.cgemm(A, B)
    Cc = oracle.cgemm(np.conj(A), np.conj(B))
    assert np.array_equal(Cc, np.conj(C))


@pytest.mark.parametrize("mode,shift", [("random", 23), ("stress", 24)])
def test_complex_error_vs_exact(mode, shift):
    n, m, p = 6, 700, 5
    A, B = _cgen(n, m, mode, 0), _cgen(m, p, mode, 1)
    C = oracle.cgemm(A, B)
    k = lambda x: np.rint(x.astype(np.float64) * 2.0 ** shift).astype(np.int64)
    ar, ai, br, bi = k(A.real), k(A.imag), k(B.real), k(B.imag)
    sc = 2.0 ** (-2 * shift)
    er = (ar @ br - ai @ bi).astype(np.float64) * sc
    ei = (ar @ bi + ai @ br).astype(np.float64) * sc
    Sr, Si = oracle.cabs_scale(A, B)
    assert np.allclose(Sr, (np.abs(ar) @ np.abs(br) + np.abs(ai) @ np.abs(bi)) * sc, rtol=2.0 ** -40, atol=0)
    u = 2.0 ** -24
    g = (2 * m + 1) * u / (1 - (2 * m + 1) * u)
    assert np.all(np.abs(C.real - er) <= g * Sr)
    assert np.all(np.abs(C.imag - ei) <= g * Si)
    assert np.max(np.abs(C.real - er) / Sr) <= 2.0 ** -21


# ------------------------------------------------------------------ double
def test_dgemm_integer_bruteforce():
    rng = np.random.default_rng(21)
    for n in range(1, 7):
        for m in range(1, 7):
            for p in range(1, 7):
                A = rng.integers(-(2 ** 20), 2 ** 20, (n, m))
                B = rng.integers(-(2 ** 20), 2 ** 20, (m, p))
                C = oracle.dgemm(A.astype(np.float64), B.astype(np.float64))
                assert np.array_equal(C.astype(np.int64), A @ B), (n, m, p)


def test_dgemm_binary64_ascending_semantics():
    A = inputs.generate_f64(5, 900, 0).numpy()
    B = inputs.generate_f64(900, 4, 1).numpy()
    C = oracle.dgemm(A, B)
    for i in range(5):
        for j in range(4):
            ref = np.cumsum(np.multiply(A[i], B[:, j]))[-1]
            assert C[i, j] == ref


def test_dgemm_error_vs_exact_python_integers():
    m = 300
    A = inputs.generate_f64(4, m, 0).numpy()
    B = inputs.generate_f64(m, 3, 1).numpy()
    C = oracle.dgemm(A, B)
    S = oracle.dabs_scale(A, B)
    ka = [[int(round(x * 2 ** 52)) for x in row] for row in A]
    kb = [[int(round(x * 2 ** 52)) for x in row] for row in B]
    u = 2.0 ** -53
    g = m * u / (1 - m * u)
    from fractions import Fraction
    for i in range(4):
        for j in range(3):
            exact = Fraction(sum(ka[i][r] * kb[r][j] for r in range(m)), 2 ** 104)
            assert abs(Fraction(C[i, j]) - exact) <= Fraction(g) * Fraction(S[i, j])


def test_dgemm_generator_matches_python():
    idx = [0, 7, 99999, 2 ** 33 + 1]
    t = inputs.generate_f64(1, 2 ** 35, 1, col_idx=idx)
    assert t.flatten().tolist() == [inputs.value_int_f64(inputs.SEED, 1, i) for i in idx]


# ------------------------------------------------------------------ tolerance scales, exact pins
def test_complex_abs_scales_exact_integers():
    """Both outputs of oracle_cabs_scale against exact Python integers (SURVEY
    8(c): the complex tolerance scales S_r = sum |ar||br| + |ai||bi| and
    S_i = sum |ar||bi| + |ai||br|).  Integer inputs up to 2^20 in magnitude keep
    every product (< 2^40) and every sum (< 2^47) exact in binary64, so each
    scale must equal the integer sum; mixed signs and unequal real/imaginary
    magnitudes make a swapped pairing (S_i computed with S_r's formula), a
    dropped |.| or a dropped term differ."""
    rng = np.random.default_rng(1306)
    n, m, p = 5, 40, 6
    ar, ai = rng.integers(-2 ** 20, 2 ** 20, (n, m)), rng.integers(-2 ** 10, 2 ** 10, (n, m))
    br, bi = rng.integers(-2 ** 20, 2 ** 20, (m, p)), rng.integers(-2 ** 12, 2 ** 12, (m, p))
    A = (ar + 1j * ai).astype(np.complex64)
    B = (br + 1j * bi).astype(np.complex64)
    Sr, Si = oracle.cabs_scale(A, B)
    for i in range(n):
        for j in range(p):
            er = sum(abs(int(ar[i, r])) * abs(int(br[r, j])) + abs(int(ai[i, r])) * abs(int(bi[r, j]))
                     for r in range(m))
            ei = sum(abs(int(ar[i, r])) * abs(int(bi[r, j])) + abs(int(ai[i, r])) * abs(int(br[r, j]))
                     for r in range(m))
            assert Sr[i, j] == er and Si[i, j] == ei, (i, j)
    # the two scales are different functions of the inputs here
    assert not np.array_equal(Sr, Si)


def test_double_abs_scale_exact():
    """oracle_dabs_scale against exact Python integers (integer inputs up to
    2^24: products < 2^48, m = 30 of them < 2^53, all exact) and,
    for 2^-52-grid inputs, against the exact rational sum within binary64
    accumulation error gamma_m * S (Higham) -- an overestimate (e.g. a doubled
    term) or a missing |.| fails both."""
    rng = np.random.default_rng(1307)
    n, m, p = 4, 30, 5
    A = rng.integers(-2 ** 24, 2 ** 24, (n, m))
    B = rng.integers(-2 ** 24, 2 ** 24, (m, p))
    S = oracle.dabs_scale(A.astype(np.float64), B.astype(np.float64))
    for i in range(n):
        for j in range(p):
            assert S[i, j] == sum(abs(int(A[i, r])) * abs(int(B[r, j])) for r in range(m)), (i, j)
    from fractions import Fraction
    m = 300
    Af = inputs.generate_f64(3, m, 0).numpy()
    Bf = inputs.generate_f64(m, 2, 1).numpy()
    S = oracle.dabs_scale(Af, Bf)
    u = 2.0 ** -53
    g = m * u / (1 - m * u)
    for i in range(3):
        for j in range(2):
            exact = sum(abs(Fraction(Af[i, r])) * abs(Fraction(Bf[r, j])) for r in range(m))
            assert abs(Fraction(S[i, j]) - exact) <= Fraction(g) * exact
