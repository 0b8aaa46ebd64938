"""Pins for the CPU oracle (oracle/oracle.c) -- no GPU needed.

Every test checks the oracle against something other than itself: worked
examples of P:47, closed forms the paper names (identity, the O(n) diagonal
product of P:51), the transpose identity, exact integer arithmetic done by
numpy/Python integers, a library routine with the same rounding semantics
(numpy float32 cumsum = ascending binary32 sums), and Higham's rigorous error
bound for recursive summation.  Each pin is chosen so that a plausible mistake
(a dropped term, a swapped index, a transposed operand, an FMA, a wrong
summation order or start value) fails at least one of them.
"""
import os

import numpy as np
import pytest

import inputs
import oracle

GOLDEN = os.path.join(os.path.dirname(__file__), "golden", "worked_examples.txt")


def _read_golden():
    blocks, cur, lines = [], {}, []
    for raw in open(GOLDEN):
        s = raw.split("#")[0].strip()
        if s:
            lines.append(s)
    i = 0
    while i < len(lines):
        tag, r, c = lines[i].split()
        r, c = int(r), int(c)
        mat = np.array([[float(v) for v in lines[i + 1 + k].split()] for k in range(r)], np.float32)
        assert mat.shape == (r, c)
        cur[tag] = mat
        i += 1 + r
        if tag == "C":
            blocks.append(cur)
            cur = {}
    return blocks


def _gen(n, m, p, mode, seed=inputs.SEED):
    A, B = inputs.pair(n, m, p, mode, seed)
    return A.numpy(), B.numpy()


def _grid_int(X, shift):
    k = X.astype(np.float64) * 2.0 ** shift
    ki = np.rint(k).astype(np.int64)
    assert np.array_equal(ki.astype(np.float64), k)
    return ki


# --------------------------------------------------------------------------- #
# Worked examples (tests/golden, hand expansions of P:47)
# --------------------------------------------------------------------------- #
def test_golden_worked_examples():
    blocks = _read_golden()
    assert len(blocks) == 2
    for b in blocks:
        C = oracle.gemm(b["A"], b["B"])
        assert np.array_equal(C, b["C"]), (C, b["C"])


# --------------------------------------------------------------------------- #
# Integer brute force: every (n, m, p) in {1..8}^3 vs exact int64 numpy matmul.
# Integer inputs in [-8, 8] keep every partial sum < 2^24, so the binary32
# result is unique and equals the exact integer.
# --------------------------------------------------------------------------- #
def test_integer_bruteforce_all_tiny_shapes():
    rng = np.random.default_rng(1306)
    for n in range(1, 9):
        for m in range(1, 9):
            for p in range(1, 9):
                Ai = rng.integers(-8, 9, size=(n, m))
                Bi = rng.integers(-8, 9, size=(m, p))
                C = oracle.gemm(Ai.astype(np.float32), Bi.astype(np.float32))
                assert np.array_equal(C.astype(np.int64), Ai @ Bi), (n, m, p)


@pytest.mark.parametrize("n,m,p", [(256, 256, 256), (37, 2000, 41), (5, 16384, 3)])
def test_integer_generator_inputs_exact(n, m, p):
    A, B = _gen(n, m, p, "integer")
    C = oracle.gemm(A, B, threads=4)
    exact = A.astype(np.int64) @ B.astype(np.int64)
    assert np.abs(exact).max() < 2 ** 24
    assert np.array_equal(C.astype(np.int64), exact)


# --------------------------------------------------------------------------- #
# Binary32 semantics: product rounded to fp32, then fp32 add, ascending r,
# starting from +0 (readings C1-C3).  numpy's float32 multiply is one
# IEEE RN product and float32 cumsum is the ascending left-to-right binary32
# accumulation -- a library routine with exactly the Listing 1 semantics.
# --------------------------------------------------------------------------- #
@pytest.mark.parametrize("mode", ["random", "stress"])
def test_binary32_ascending_semantics(mode):
    n, m, p = 9, 777, 11
    A, B = _gen(n, m, p, mode)
    C = oracle.gemm(A, B)
    for i in range(n):
        for j in range(p):
            prods = np.multiply(A[i, :], B[:, j], dtype=np.float32)
            ref = np.cumsum(prods, dtype=np.float32)[-1]
            assert C[i, j].tobytes() == np.float32(ref).tobytes(), (i, j)


def test_fma_witness_proves_no_contraction():
    """with K=4096 most elements differ between mul+add and fmaf;
    the oracle must be the mul+add one (equal to the cumsum reference above)."""
    A, B = _gen(4, 4096, 8, "stress")
    C = oracle.gemm(A, B)
    F = oracle.gemm_fma_witness(A, B)
    assert (C != F).sum() >= 8, "fmaf and mul+add agree: contraction is on or the witness is broken"
    prods = np.multiply(A[0, :], B[:, 0], dtype=np.float32)
    assert C[0, 0] == np.cumsum(prods, dtype=np.float32)[-1]


# --------------------------------------------------------------------------- #
# Rigorous error bound against the exact product (integers on the 2^-k grid,
# summed exactly by numpy int64): |c_hat - c| <= gamma_m * sum|a||b|,
# gamma_m = m u / (1 - m u), u = 2^-24 (Higham, recursive summation of m
# rounded products).  Also a statistical bound the GPU budget relies on.
# --------------------------------------------------------------------------- #
@pytest.mark.parametrize("mode,shift", [("random", 23), ("stress", 24)])
@pytest.mark.parametrize("n,m,p", [(17, 2000, 19), (3, 2048, 64)])
def test_error_vs_exact_within_higham(mode, shift, n, m, p):
    A, B = _gen(n, m, p, mode)
    C = oracle.gemm(A, B)
    Ai, Bi = _grid_int(A, shift), _grid_int(B, shift)
    exact = (Ai @ Bi).astype(np.float64) * 2.0 ** (-2 * shift)        # < 2^62, exact in int64
    absum = (np.abs(Ai) @ np.abs(Bi)).astype(np.float64) * 2.0 ** (-2 * shift)
    u = 2.0 ** -24
    gamma = m * u / (1 - m * u)
    err = np.abs(C.astype(np.float64) - exact)
    assert np.all(err <= gamma * absum)
    # statistical: the oracle's own error is far below the 2^-20 GPU tolerance
    assert np.max(err / absum) <= 2.0 ** -21


def test_exact_grid_matches_python_integers():
    A, B = _gen(6, 300, 5, "stress")
    E = oracle.exact_grid(A, B, 24)
    Ai, Bi = _grid_int(A, 24), _grid_int(B, 24)
    ref = [[sum(int(Ai[i, r]) * int(Bi[r, j]) for r in range(300)) for j in range(5)] for i in range(6)]
    for i in range(6):
        for j in range(5):
            assert E[i, j] == float(ref[i][j]) * 2.0 ** -48
    with pytest.raises(ValueError):
        oracle.exact_grid(A, B, 10)                      # not on the 2^-10 grid


def test_abs_scale_matches_exact_absolute_sum():
    A, B = _gen(7, 513, 9, "random")
    S = oracle.abs_scale(A, B)
    Ai, Bi = _grid_int(A, 23), _grid_int(B, 23)
    ref = (np.abs(Ai) @ np.abs(Bi)).astype(np.float64) * 2.0 ** -46
    assert np.allclose(S, ref, rtol=2.0 ** -40, atol=0)


# --------------------------------------------------------------------------- #
# Closed forms: identity, permutations (index mapping), the O(n)
# diagonal product of P:51, row/column scaling (one nonzero product per
# element => exactly fl(d*b)), and (AB)^T = B^T A^T (commutative products,
# same ascending order => bitwise).
# --------------------------------------------------------------------------- #
def test_identity_is_bitwise():
    A, _ = _gen(33, 47, 1, "stress")
    assert np.array_equal(oracle.gemm(A, np.eye(47, dtype=np.float32)), A)
    assert np.array_equal(oracle.gemm(np.eye(33, dtype=np.float32), A), A)


def test_permutation_rows_and_columns():
    rng = np.random.default_rng(7)
    A, _ = _gen(29, 31, 1, "stress")
    pr, pc = rng.permutation(29), rng.permutation(31)
    P = np.eye(29, dtype=np.float32)[pr]            # (P A)_i = A_{pr[i]}
    Q = np.eye(31, dtype=np.float32)[:, pc]         # (A Q)_{:,j} = A_{:, pc[j]}
    assert np.array_equal(oracle.gemm(P, A), A[pr])
    assert np.array_equal(oracle.gemm(A, Q), A[:, pc])


def test_diagonal_closed_form():
    rng = np.random.default_rng(11)
    d1 = rng.standard_normal(16).astype(np.float32)
    d2 = rng.standard_normal(16).astype(np.float32)
    C = oracle.gemm(np.diag(d1), np.diag(d2))
    assert np.array_equal(C, np.diag(np.multiply(d1, d2, dtype=np.float32)))
    B = rng.standard_normal((16, 23)).astype(np.float32)
    assert np.array_equal(oracle.gemm(np.diag(d1), B), np.multiply(d1[:, None], B, dtype=np.float32))
    A = rng.standard_normal((23, 16)).astype(np.float32)
    assert np.array_equal(oracle.gemm(A, np.diag(d2)), np.multiply(A, d2[None, :], dtype=np.float32))


def test_transpose_identity_bitwise():
    A, B = _gen(21, 301, 13, "stress")
    C = oracle.gemm(A, B)
    Ct = oracle.gemm(np.ascontiguousarray(B.T), np.ascontiguousarray(A.T))
    assert np.array_equal(Ct.T, C)


def test_thread_count_determinism():
    A, B = _gen(64, 500, 40, "random")
    C1 = oracle.gemm(A, B, threads=1)
    for t in (2, 7, 64, 200):
        assert np.array_equal(oracle.gemm(A, B, threads=t), C1)


def test_degenerate_inner_dimension_mismatch():
    with pytest.raises(ValueError):
        oracle.gemm(np.zeros((2, 3), np.float32), np.zeros((4, 2), np.float32))


# --------------------------------------------------------------------------- #
# Freivalds (exact int64) -- the check used at full size on integer inputs.
# --------------------------------------------------------------------------- #
def test_freivalds_accepts_and_rejects():
    A, B = _gen(50, 70, 60, "integer")
    Ai, Bi = A.astype(np.int64), B.astype(np.int64)
    C = (Ai @ Bi).astype(np.float32)
    x = np.ones(60, dtype=np.int64)
    assert oracle.freivalds(A, B, C, x) == 0
    C2 = C.copy()
    C2[17, 33] += 1.0
    assert oracle.freivalds(A, B, C2, x) == 1
    rng = np.random.default_rng(5)
    C3 = C.copy()
    C3[3, :] = C3[4, :]                                  # swapped-row style corruption
    x = rng.integers(-8, 9, size=60)
    assert oracle.freivalds(A, B, C3, x) >= 1 or np.array_equal(C3[3] @ x, C[3] @ x)
