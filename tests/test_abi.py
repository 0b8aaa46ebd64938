"""C-ABI contract checks that need no GPU: the library loads, exports every
symbol include/la.h declares, and its host-side error paths behave (SURVEY
8(b)).  Compute calls are exercised only in the -m gpu tests."""
import ctypes
import os
import re

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _declared():
    src = open(os.path.join(ROOT, "include", "la.h")).read()
    return re.findall(r"^LA_API\s+[\w\s\*]*?\b(la_\w+)\s*\(", src, flags=re.M)


def test_header_and_binding_agree():
    import paper_1306_6192_b200 as la
    declared = _declared()
    assert len(declared) == 22
    assert sorted(declared) == sorted(la.EXPORTS)


def test_library_exports_every_declared_symbol():
    import paper_1306_6192_b200 as la
    lib = ctypes.CDLL(la.LIB_PATH)
    for name in _declared():
        assert hasattr(lib, name), name


def test_library_is_sm100a_only():
    """The fatbin carries sm_100a SASS and tcgen05/TMA instructions (no
    fallback architecture, no legacy mma.sync path)."""
    import subprocess
    import paper_1306_6192_b200 as la
    out = subprocess.run(["cuobjdump", "-lelf", la.LIB_PATH], capture_output=True, text=True).stdout
    assert "sm_100a" in out and "sm_90" not in out and "sm_80" not in out
    sass = subprocess.run(["cuobjdump", "-sass", la.LIB_PATH], capture_output=True, text=True).stdout
    assert "UTCHMMA" in sass      # tcgen05.mma
    assert "UTMALDG" in sass      # TMA tensor loads
    assert "LDTM" in sass         # tcgen05.ld
    assert re.search(r"\bHMMA\b", sass) is None


def test_status_strings():
    import paper_1306_6192_b200 as la
    names = [la.status_string(s) for s in range(7)]
    assert names == ["LA_OK", "LA_ERR_INVALID_VALUE", "LA_ERR_NOT_INITIALIZED", "LA_ERR_UNSUPPORTED",
                     "LA_ERR_OUT_OF_MEMORY", "LA_ERR_CUDA", "LA_ERR_NCCL"]


def test_not_initialized_and_argument_errors():
    import paper_1306_6192_b200 as la
    lib = la._lib
    if os.environ.get("CUDA_VISIBLE_DEVICES", None) != "" and _has_cuda():
        pytest.skip("a GPU is present; covered by tests/test_parity.py")
    assert lib.la_gemm(4, 4, 4, 16, 32, 64, None) == la.LA_ERR_NOT_INITIALIZED
    assert b"la_init" in lib.la_last_error()
    assert lib.la_gemm_host(4, 4, 4, 16, 32, 64, None) == la.LA_ERR_NOT_INITIALIZED
    assert lib.la_gemm_multi(4, 4, 4, 16, 32, 64, None, 0, 1, None) == la.LA_ERR_NOT_INITIALIZED
    assert lib.la_set_mode(7) == la.LA_ERR_INVALID_VALUE
    assert lib.la_set_option(99, 1) == la.LA_ERR_INVALID_VALUE
    assert lib.la_set_option(la.OPTIONS["panels"], -1) == la.LA_ERR_INVALID_VALUE
    # no device in this container: la_init reports it instead of crashing
    assert lib.la_init(0) in (la.LA_ERR_INVALID_VALUE, la.LA_ERR_CUDA)
    import ctypes
    a, b = ctypes.c_int(), ctypes.c_int()
    assert lib.la_comm_size(ctypes.byref(a), ctypes.byref(b)) == la.LA_ERR_NOT_INITIALIZED
    assert lib.la_comm_size(None, None) == la.LA_ERR_INVALID_VALUE
    assert la.finalize() is None


def test_options_roundtrip():
    import paper_1306_6192_b200 as la
    old = la.get_option("panels")
    la.set_option("panels", 6)
    assert la.get_option("panels") == 6
    la.set_option("panels", old)
    la.set_option("promote_k", -1)              # automatic by K (the default)
    assert la.get_option("promote_k") == -1
    with pytest.raises(la.LaError):
        la.set_option("promote_k", -2)
    assert la.get_option("nccl_sms") == 8
    with pytest.raises(la.LaError):
        la.set_option("nccl_sms", -1)


def test_shard_rows_partition():
    import paper_1306_6192_b200 as la
    for n in (1, 7, 8, 1000, 16384, 65536):
        for g in (1, 2, 3, 4, 8):
            if n < g:
                continue
            spans = [la.shard_rows(n, r, g) for r in range(g)]
            assert spans[0][0] == 0
            for (a0, a), (b0, _) in zip(spans, spans[1:]):
                assert a0 + a == b0
            assert spans[-1][0] + spans[-1][1] == n
            assert max(s for _, s in spans) - min(s for _, s in spans) <= 1
    with pytest.raises(la.LaError):
        la.shard_rows(10, 3, 2)


def _has_cuda():
    import torch
    return torch.cuda.is_available()
