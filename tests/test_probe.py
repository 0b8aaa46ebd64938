"""tcgen05 kind::tf32 accumulator probes, run through la_gemm.

They classify how the tensor pipe rounds fp32 accumulation, which decides
whether accumulator promotion (LA_OPT_PROMOTE_K) is needed for the 2^-20
bound.  Every probe uses values exactly representable in TF32, so the split
(hi = tf32_rna(a)) leaves them unchanged and the single TF32 pass sees them
as given.  Results are printed and written to gpurun_out/probe.json when that
directory exists; the assertions only require that each outcome is one of the
candidate behaviours (so the probe documents the hardware instead of assuming
it), plus the end-to-end accuracy check that matters.
"""
import json
import os

import numpy as np
import pytest
import torch

import inputs
import oracle

pytestmark = pytest.mark.gpu

U = 2.0 ** -23   # ulp of 1.0 in fp32


@pytest.fixture(scope="module")
def la():
    import paper_1306_6192_b200 as la
    la.init(0)
    yield la
    la.set_mode("3xtf32")


def _row_dot(la, a_row, mode="tf32"):
    """c = a_row . ones via a 128 x K . K x 128 GEMM (one output tile)."""
    k = len(a_row)
    A = np.zeros((128, k), np.float32)
    A[0] = a_row
    B = np.ones((k, 128), np.float32)
    la.set_mode(mode)
    try:
        C = la.gemm(torch.from_numpy(A).cuda(), torch.from_numpy(B).cuda())
    finally:
        la.set_mode("3xtf32")
    return float(C[0, 0].item())


RESULTS = {}


def _record(name, value, table):
    label = next((k for k, v in table.items() if v == value), "other")
    RESULTS[name] = {"value": value.hex() if isinstance(value, float) else value, "class": label}
    print(f"probe {name}: {value!r} -> {label}")
    return label


def test_probe_within_one_mma(la):
    c = _row_dot(la, [1.0, 1.5 * 2.0 ** -24] + [0.0] * 6)
    lab = _record("within_mma", c, {"RN": 1 + U, "RZ": 1.0})
    assert lab in ("RN", "RZ")


def test_probe_across_mmas(la):
    c = _row_dot(la, [1.0] + [0.0] * 7 + [1.5 * 2.0 ** -24] + [0.0] * 7)
    lab = _record("across_mma", c, {"RN": 1 + U, "RZ": 1.0})
    assert lab in ("RN", "RZ")


def test_probe_alignment_width(la):
    c = _row_dot(la, [1.0] + [2.0 ** -24] * 7)
    lab = _record("seven_half_ulps", c, {"exact+RN": 1 + 4 * U, "exact+RZ": 1 + 3 * U,
                                          "per-term": 1.0, "2 guard bits": 1 + 2 * U})
    # measured on the B200: the 8 products are summed exactly, then truncated
    assert lab in ("exact+RN", "exact+RZ"), lab


def test_probe_negative(la):
    c = _row_dot(la, [-1.0, -1.5 * 2.0 ** -24] + [0.0] * 6)
    lab = _record("negative", c, {"RN/RD": -(1 + U), "RZ/RU": -1.0})
    assert lab in ("RN/RD", "RZ/RU")


# Accumulator against products: how a product sum below the accumulator's ulp
# is added (two MMAs: the first sets D, the second adds the small sum).
#   exact+RZ      : D + sum formed exactly, then rounded toward zero
#   sum-truncated : the sum aligned to D's ulp and truncated toward zero (its
#                   error has the sign of -sum, whatever D's sign), then added
#   floor         : two's-complement truncation (toward -inf) of the sum
def test_probe_accumulator_opposite_sign(la):
    d = 1.5 * 2.0 ** -24
    c1 = _row_dot(la, [-1.0] + [0.0] * 7 + [d] + [0.0] * 7)
    lab1 = _record("neg_acc_plus_small", c1, {"exact+RZ": -(1 - U), "sum-truncated/floor": -1.0})
    c2 = _row_dot(la, [1.0] + [0.0] * 7 + [-d] + [0.0] * 7)
    lab2 = _record("pos_acc_minus_small", c2, {"exact+RZ/floor": 1 - U, "sum-truncated": 1.0})
    c3 = _row_dot(la, [-1.0] + [0.0] * 7 + [-d] + [0.0] * 7)
    lab3 = _record("neg_acc_minus_small", c3, {"exact+RZ/sum-truncated": -1.0, "floor": -(1 + U)})
    c4 = _row_dot(la, [1.0] + [0.0] * 7 + [0.75 * U, 0.75 * U] + [0.0] * 6)
    lab4 = _record("two_sub_half_ulp_products", c4, {"sum-then-truncate": 1 + U, "per-product": 1.0})
    assert "other" not in (lab1, lab2, lab3, lab4), (c1, c2, c3, c4)


def test_probe_long_k_accuracy(la, monkeypatch):
    """3xTF32 at K = 16384 on 24-bit inputs: max error / (2^-20 S) without
    promotion and with promotion every 1024 / 256.  Split-K is off, so each
    output element is ONE accumulation over the whole K range and promote_k
    alone decides how much of it happens in the truncating TMEM accumulator
    (with split-K on, this one-tile shape would be cut into K = 256 pieces and
    the sweep would measure nothing)."""
    monkeypatch.setenv("LA_SPLIT_K", "0")
    n, m, p = 128, 16384, 128
    A, B = inputs.pair(n, m, p, "stress", device="cuda")
    Ah, Bh = A.cpu().numpy(), B.cpu().numpy()
    E = oracle.exact_grid(Ah[:16], Bh[:, :16], 24)
    S = oracle.abs_scale(Ah[:16], Bh[:, :16])
    out = {}
    old = la.get_option("promote_k")
    try:
        for pk in (0, 1024, 256):
            la.set_option("promote_k", pk)
            C = la.gemm(A, B)[:16, :16].cpu().numpy().astype(np.float64)
            out[pk] = float((np.abs(C - E) / S).max() / 2.0 ** -20)
    finally:
        la.set_option("promote_k", old)
    RESULTS["long_k_err_units_2^-20"] = out
    print("3xTF32 K=16384 max |C-exact|/S in units of 2^-20 by promote_k:", out)
    assert out[0] > 1.0, "whole-K TMEM accumulation should show the truncation bias (> 2^-20 S)"
    assert out[1024] < out[0] and out[256] <= out[1024]
    assert out[256] < 0.1


def test_zz_write_results():
    d = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "gpurun_out")
    if os.path.isdir(d):
        with open(os.path.join(d, "probe.json"), "w") as f:
            json.dump(RESULTS, f, indent=1)
