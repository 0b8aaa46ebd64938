"""Seeded synthetic inputs shared by the oracle side and the CUDA side.

This module holds NONE of the method's arithmetic (no products, no sums of
products): it only turns (seed, matrix id, element index) into a float32 value
with a counter-based generator, so that tests, ``smoke()`` and ``bench.py`` can
regenerate any row of A or column of B on the host without copying big
matrices back from the GPU.  It runs through torch integer ops, so the same
code produces bit-identical values on CPU and on CUDA (checked by
``tests/test_inputs.py`` against pure-Python integers and, on a GPU box,
CPU == CUDA).

Recipe (the paper fixes no values -- it uses dense square
4096x4096 matrices):

    h(id, idx) = splitmix64(splitmix64(seed ^ id) ^ idx),  idx = i*cols + j
    splitmix64(x): z = x + 0x9E3779B97F4A7C15
                   z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9
                   z = (z ^ (z >> 27)) * 0x94D049BB133111EB
                   return z ^ (z >> 31)            (uint64, wrapping)

    mode "random":  ((h >> 40) - 2^23) * 2^-23   uniform on the 2^-23 grid in [-1, 1)
    mode "stress":  ((h >> 39) - 2^24) * 2^-24   24-bit significands in [-1, 1)
    mode "integer": (h mod 17) - 8               uniform integers in [-8, 8]

A is matrix id 0, B is matrix id 1; the default seed is 13066192.
"""
from __future__ import annotations

import torch

SEED = 13066192
SEED_REPEAT = 13066193
ID_A, ID_B = 0, 1
MODES = ("random", "stress", "integer")
MODES_F64 = ("f64", "integer")
GRID_SHIFT = {"random": 23, "stress": 24, "integer": 0}

_M64 = (1 << 64) - 1


def _s64(u: int) -> int:
    """uint64 constant -> the int64 with the same bits."""
    u &= _M64
    return u - (1 << 64) if u >= (1 << 63) else u


_C0 = _s64(0x9E3779B97F4A7C15)
_C1 = _s64(0xBF58476D1CE4E5B9)
_C2 = _s64(0x94D049BB133111EB)


def _lsr(z: torch.Tensor, k: int) -> torch.Tensor:
    """Logical right shift of int64 bit patterns."""
    return (z >> k) & ((1 << (64 - k)) - 1)


def _splitmix64(z: torch.Tensor) -> torch.Tensor:
    z = z + _C0
    z = (z ^ _lsr(z, 30)) * _C1
    z = (z ^ _lsr(z, 27)) * _C2
    return z ^ _lsr(z, 31)


def splitmix64_int(x: int) -> int:
    """Pure-Python reference (used by the tests to pin the torch version)."""
    z = (x + 0x9E3779B97F4A7C15) & _M64
    z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & _M64
    z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & _M64
    return z ^ (z >> 31)


def value_int(seed: int, matrix_id: int, idx: int, mode: str) -> float:
    """Pure-Python reference for one element (tests only)."""
    h = splitmix64_int(splitmix64_int((seed ^ matrix_id) & _M64) ^ idx)
    if mode == "random":
        return ((h >> 40) - (1 << 23)) * 2.0 ** -23
    if mode == "stress":
        return ((h >> 39) - (1 << 24)) * 2.0 ** -24
    if mode == "integer":
        return float(h % 17 - 8)
    raise ValueError(mode)


def _values(idx: torch.Tensor, key: int, mode: str) -> torch.Tensor:
    h = _splitmix64(idx ^ key)
    if mode == "random":
        return ((_lsr(h, 40) - (1 << 23)).to(torch.float32)) * 2.0 ** -23
    if mode == "stress":
        return ((_lsr(h, 39) - (1 << 24)).to(torch.float32)) * 2.0 ** -24
    if mode == "integer":
        # unsigned h mod 17 from signed int64 bits: h_u = 2*(h_u >> 1) + (h_u & 1)
        r = (_lsr(h, 1) % 17 * 2 + (h & 1)) % 17
        return (r - 8).to(torch.float32)
    raise ValueError(f"unknown mode {mode!r}; expected one of {MODES}")


def _key(seed: int, matrix_id: int) -> int:
    return _s64(splitmix64_int((seed ^ matrix_id) & _M64))


def generate(rows: int, cols: int, matrix_id: int, mode: str = "random",
             seed: int = SEED, device="cpu", row_idx=None, col_idx=None,
             chunk: int = 1 << 24) -> torch.Tensor:
    """The (rows x cols) matrix `matrix_id`, or its sub-matrix at the given row
    and column indices (element (i, j) always has counter i*cols + j).
    Returns a contiguous float32 tensor on `device`."""
    device = torch.device(device)
    key = _key(seed, matrix_id)
    r = (torch.arange(rows, dtype=torch.int64, device=device) if row_idx is None
         else torch.as_tensor(row_idx, dtype=torch.int64, device=device))
    c = (torch.arange(cols, dtype=torch.int64, device=device) if col_idx is None
         else torch.as_tensor(col_idx, dtype=torch.int64, device=device))
    out = torch.empty((r.numel(), c.numel()), dtype=torch.float32, device=device)
    if out.numel() == 0:
        return out
    rows_per = max(1, chunk // max(1, c.numel()))
    for r0 in range(0, r.numel(), rows_per):
        rr = r[r0:r0 + rows_per]
        idx = rr[:, None] * cols + c[None, :]
        out[r0:r0 + rr.numel()] = _values(idx, key, mode)
    return out


def value_int_f64(seed: int, matrix_id: int, idx: int) -> float:
    """Pure-Python reference for one binary64 element (tests only)."""
    h = splitmix64_int(splitmix64_int((seed ^ matrix_id) & _M64) ^ idx)
    return ((h >> 11) - (1 << 52)) * 2.0 ** -52


def generate_f64(rows: int, cols: int, matrix_id: int, mode: str = "f64", seed: int = SEED, device="cpu",
                 row_idx=None, col_idx=None, chunk: int = 1 << 23) -> torch.Tensor:
    """Binary64 inputs for the double-precision product: mode "f64" draws
    ((h >> 11) - 2^52) * 2^-52 (53-bit significands, uniform on the 2^-52 grid in
    [-1, 1)); mode "integer" is the integer mode above, as float64."""
    device = torch.device(device)
    key = _key(seed, matrix_id)
    r = (torch.arange(rows, dtype=torch.int64, device=device) if row_idx is None
         else torch.as_tensor(row_idx, dtype=torch.int64, device=device))
    c = (torch.arange(cols, dtype=torch.int64, device=device) if col_idx is None
         else torch.as_tensor(col_idx, dtype=torch.int64, device=device))
    out = torch.empty((r.numel(), c.numel()), dtype=torch.float64, device=device)
    if out.numel() == 0:
        return out
    rows_per = max(1, chunk // max(1, c.numel()))
    for r0 in range(0, r.numel(), rows_per):
        rr = r[r0:r0 + rows_per]
        idx = rr[:, None] * cols + c[None, :]
        if mode == "f64":
            h = _splitmix64(idx ^ key)
            out[r0:r0 + rr.numel()] = (_lsr(h, 11) - (1 << 52)).to(torch.float64) * 2.0 ** -52
        else:
            out[r0:r0 + rr.numel()] = _values(idx, key, mode).to(torch.float64)
    return out


def pair(n: int, m: int, p: int, mode: str = "random", seed: int = SEED, device="cpu"):
    """(A, B) for the problem n x m by m x p."""
    return (generate(n, m, ID_A, mode, seed, device),
            generate(m, p, ID_B, mode, seed, device))


PATTERNS = ("positive", "mixed", "blocks", "ramp", "bias")


def structured(A: torch.Tensor, pattern: str, seed: int = SEED) -> torch.Tensor:
    """Structured variants of a "random"-mode A (n x m) along its K axis (the
    columns), for accuracy tests beyond symmetric random signs.  Every transform
    is exact in binary32 (sign flips, powers of two, or -1/4 on the 2^-23 grid),
    so the exact product stays computable on the 2^-23 grid:
      positive  |a|                          (same-sign products with |B|)
      mixed     |a|, negated in the second half of K (one sign change)
      blocks    |a| times a seeded sign per block of 1024 columns
      ramp      |a| * 2^floor(10 k / m)      (magnitudes growing along K)
      bias      a - 1/4                      (mostly negative, with noise)"""
    m = A.shape[1]
    k = torch.arange(m, device=A.device)
    if pattern == "positive":
        return A.abs()
    if pattern == "mixed":
        return torch.where(k >= m // 2, -A.abs(), A.abs())
    if pattern == "blocks":
        blk = (k // 1024).to(torch.int64)
        h = _splitmix64(blk ^ _key(seed, 7))
        sg = torch.where((h & 1) == 1, -1.0, 1.0).to(A.dtype)
        return A.abs() * sg[None, :]
    if pattern == "ramp":
        return A.abs() * torch.exp2(torch.floor(10.0 * k.to(torch.float64) / m)).to(A.dtype)[None, :]
    if pattern == "bias":
        return A - 0.25
    raise ValueError(f"unknown pattern {pattern!r}; expected one of {PATTERNS}")
