"""CPU oracle for C = A.B -- TEST INFRASTRUCTURE ONLY.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s
``cpu_baseline`` / ``--impl reference`` leg may import this package.  The
product path (``paper_1306_6192_b200``) never imports, links or calls it, and
this package never imports the product path.  They share only the seeded input
generator in ``inputs/`` (which holds none of the method's arithmetic).

The arithmetic lives in ``oracle/oracle.c`` (plain C11, ``-O2
-ffp-contract=off -fno-fast-math``): it is the paper's Listing 1 triple loop
 computing the Cauchy product of P:47.  This module only
compiles it and marshals numpy arrays.

Functions
---------
gemm(A, B, threads)            Listing 1, fp32 multiply then fp32 add, ascending r.
gemm_fma_witness(A, B)         same loop with fmaf -- NOT the oracle, used to
                               prove the build does not contract (FMA witness).
abs_scale(A, B)                S_ij = sum_r |a_ir||b_rj| (binary64), the scale of
                               the north_star tolerance 2^-20 * S_ij.
exact_grid(A, B, shift)        exact c_ij for inputs on the 2^-shift grid (int128).
freivalds(A, B, C, x)          exact int64 Freivalds check C.x == A.(B.x).
elementwise(A, B, subtract)    C = A + B or A - B, one binary32 op per element.
cgemm(A, B)                    complex64 Listing 1 (Table 2 "Complex Float").
cabs_scale(A, B)               complex tolerance scales (real part, imaginary part).
dgemm(A, B)                    binary64 Listing 1 (Table 2 "Double").
dabs_scale(A, B)               binary64 tolerance scale for dgemm.
"""
from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "oracle.c")
_LIB = os.path.join(_HERE, "liboracle.so")
_CFLAGS = ["-O2", "-std=c11", "-ffp-contract=off", "-fno-fast-math", "-fPIC",
           "-shared", "-pthread"]

_lib = None


def build(force: bool = False) -> str:
    """Compile oracle.c into oracle/liboracle.so (gcc, no CUDA)."""
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        tmp = _LIB + f".tmp{os.getpid()}"
        subprocess.check_call(["gcc", *_CFLAGS, _SRC, "-o", tmp, "-lm"])
        os.replace(tmp, _LIB)
    return _LIB


def _load():
    global _lib
    if _lib is None:
        lib = ctypes.CDLL(build())
        i64, fp, dp = ctypes.c_int64, ctypes.c_void_p, ctypes.c_void_p
        lib.oracle_gemm.argtypes = [i64, i64, i64, fp, fp, fp, ctypes.c_int]
        lib.oracle_gemm.restype = ctypes.c_int
        lib.oracle_gemm_fma_witness.argtypes = [i64, i64, i64, fp, fp, fp]
        lib.oracle_gemm_fma_witness.restype = ctypes.c_int
        lib.oracle_abs_scale.argtypes = [i64, i64, i64, fp, fp, dp]
        lib.oracle_abs_scale.restype = ctypes.c_int
        lib.oracle_exact_grid.argtypes = [i64, i64, i64, fp, fp, ctypes.c_int, dp]
        lib.oracle_exact_grid.restype = ctypes.c_int
        lib.oracle_freivalds_i64.argtypes = [i64, i64, i64, fp, fp, fp, fp, fp]
        lib.oracle_freivalds_i64.restype = ctypes.c_int64
        lib.oracle_elementwise.argtypes = [i64, i64, fp, fp, fp, ctypes.c_int]
        lib.oracle_elementwise.restype = ctypes.c_int
        lib.oracle_cgemm.argtypes = [i64, i64, i64, fp, fp, fp]
        lib.oracle_cgemm.restype = ctypes.c_int
        lib.oracle_cabs_scale.argtypes = [i64, i64, i64, fp, fp, dp]
        lib.oracle_cabs_scale.restype = ctypes.c_int
        lib.oracle_dgemm.argtypes = [i64, i64, i64, fp, fp, fp]
        lib.oracle_dgemm.restype = ctypes.c_int
        lib.oracle_dabs_scale.argtypes = [i64, i64, i64, fp, fp, dp]
        lib.oracle_dabs_scale.restype = ctypes.c_int
        _lib = lib
    return _lib


def _f32(x) -> np.ndarray:
    a = np.ascontiguousarray(np.asarray(x), dtype=np.float32)
    if a.ndim != 2:
        raise ValueError("expected a 2-D matrix")
    return a


def _ptr(a: np.ndarray) -> int:
    return a.ctypes.data


def _dims(A, B):
    n, m = A.shape
    m2, p = B.shape
    if m != m2:
        raise ValueError(f"inner dimension mismatch: {A.shape} x {B.shape}")
    return n, m, p


def gemm(A, B, threads: int = 1) -> np.ndarray:
    """Listing 1: C = A.B in binary32, rows split over `threads`."""
    A, B = _f32(A), _f32(B)
    n, m, p = _dims(A, B)
    C = np.empty((n, p), dtype=np.float32)
    rc = _load().oracle_gemm(n, m, p, _ptr(A), _ptr(B), _ptr(C), int(threads))
    if rc != 0:
        raise RuntimeError(f"oracle_gemm failed ({rc})")
    return C


def gemm_fma_witness(A, B) -> np.ndarray:
    """NOT the oracle: Listing 1 with fmaf accumulation (FMA witness only)."""
    A, B = _f32(A), _f32(B)
    n, m, p = _dims(A, B)
    C = np.empty((n, p), dtype=np.float32)
    _load().oracle_gemm_fma_witness(n, m, p, _ptr(A), _ptr(B), _ptr(C))
    return C


def abs_scale(A, B) -> np.ndarray:
    """S_ij = sum_r |a_ir| |b_rj| in binary64 (tolerance scale)."""
    A, B = _f32(A), _f32(B)
    n, m, p = _dims(A, B)
    S = np.empty((n, p), dtype=np.float64)
    _load().oracle_abs_scale(n, m, p, _ptr(A), _ptr(B), _ptr(S))
    return S


def exact_grid(A, B, shift: int) -> np.ndarray:
    """Exact c_ij (rounded once to binary64) for inputs k * 2^-shift."""
    A, B = _f32(A), _f32(B)
    n, m, p = _dims(A, B)
    E = np.empty((n, p), dtype=np.float64)
    rc = _load().oracle_exact_grid(n, m, p, _ptr(A), _ptr(B), int(shift), _ptr(E))
    if rc != 0:
        raise ValueError(f"inputs are not on the 2^-{shift} grid")
    return E


def freivalds(A, B, C, x) -> int:
    """Exact int64 Freivalds check; returns the number of mismatching rows."""
    A, B, C = _f32(A), _f32(B), _f32(C)
    n, m, p = _dims(A, B)
    if C.shape != (n, p):
        raise ValueError("C has the wrong shape")
    x = np.ascontiguousarray(x, dtype=np.int64)
    if x.shape != (p,):
        raise ValueError("x must have length p")
    first = np.zeros(1, dtype=np.int64)
    bad = _load().oracle_freivalds_i64(n, m, p, _ptr(A), _ptr(B), _ptr(C), _ptr(x), _ptr(first))
    if bad < 0:
        raise ValueError("Freivalds needs integer-valued A, B and C")
    return int(bad)


def elementwise(A, B, subtract: bool = False) -> np.ndarray:
    """C = A + B (or A - B) elementwise in binary32."""
    A, B = _f32(A), _f32(B)
    if A.shape != B.shape:
        raise ValueError("shape mismatch")
    C = np.empty_like(A)
    _load().oracle_elementwise(A.shape[0], A.shape[1], _ptr(A), _ptr(B), _ptr(C), int(bool(subtract)))
    return C


def _c64(x) -> np.ndarray:
    a = np.ascontiguousarray(np.asarray(x), dtype=np.complex64)
    if a.ndim != 2:
        raise ValueError("expected a 2-D matrix")
    return a


def cgemm(A, B) -> np.ndarray:
    """Complex Listing 1: C = A.B for complex64 matrices (binary32 components)."""
    A, B = _c64(A), _c64(B)
    n, m = A.shape
    m2, p = B.shape
    if m != m2:
        raise ValueError("inner dimension mismatch")
    C = np.empty((n, p), dtype=np.complex64)
    _load().oracle_cgemm(n, m, p, _ptr(A), _ptr(B), _ptr(C))
    return C


def cabs_scale(A, B):
    """(Sr, Si): binary64 scales sum|ar||br|+|ai||bi| and sum|ar||bi|+|ai||br|."""
    A, B = _c64(A), _c64(B)
    n, m = A.shape
    _, p = B.shape
    S = np.empty((n, p, 2), dtype=np.float64)
    _load().oracle_cabs_scale(n, m, p, _ptr(A), _ptr(B), _ptr(S))
    return S[..., 0], S[..., 1]


def _f64(x) -> np.ndarray:
    a = np.ascontiguousarray(np.asarray(x), dtype=np.float64)
    if a.ndim != 2:
        raise ValueError("expected a 2-D matrix")
    return a


def dgemm(A, B) -> np.ndarray:
    """Binary64 Listing 1: C = A.B (mul then add, ascending r, no FMA)."""
    A, B = _f64(A), _f64(B)
    n, m, p = _dims(A, B)
    C = np.empty((n, p), dtype=np.float64)
    _load().oracle_dgemm(n, m, p, _ptr(A), _ptr(B), _ptr(C))
    return C


def dabs_scale(A, B) -> np.ndarray:
    A, B = _f64(A), _f64(B)
    n, m, p = _dims(A, B)
    S = np.empty((n, p), dtype=np.float64)
    _load().oracle_dabs_scale(n, m, p, _ptr(A), _ptr(B), _ptr(S))
    return S
