"""Python binding of the C ABI in include/la.h (argument marshalling only).

Every step of the product runs in the CUDA kernels of ``libla.so``; this module
only converts torch tensors / numpy arrays to pointers and status codes to
exceptions.  There is no CPU fallback: if the shared library is missing the
import of the binding fails loudly (build it with ``__graft_entry__.build()``
or ``python paper_1306_6192_b200/_build.py``).

    import torch, paper_1306_6192_b200 as la
    la.init(0)
    C = la.gemm(A, B)          # A: n x m, B: m x p, float32 CUDA tensors
"""
from __future__ import annotations

import ctypes
import os

import numpy as np

_PKG = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_PKG, "libla.so")

LA_OK, LA_ERR_INVALID_VALUE, LA_ERR_NOT_INITIALIZED, LA_ERR_UNSUPPORTED, \
    LA_ERR_OUT_OF_MEMORY, LA_ERR_CUDA, LA_ERR_NCCL = range(7)
MODES = {"3xtf32": 0, "tf32": 1}
OPTIONS = {"promote_k": 0, "max_sms": 1, "panels": 2, "kernel_timing": 3, "nccl_sms": 4}

# every symbol include/la.h declares (checked by tests/test_abi.py)
EXPORTS = ("la_init", "la_set_mode", "la_set_option", "la_get_option", "la_gemm", "la_gemm_host",
           "la_get_unique_id", "la_comm_init", "la_gemm_multi", "la_shard_rows", "la_finalize",
           "la_status_string", "la_last_error", "la_last_launch_count", "la_kernel_times", "la_cgemm",
           "la_add", "la_dgemm", "la_gather_alloc", "la_gemm_host_batch", "la_comm_size",
           "la_panel_plan")


class LaError(RuntimeError):
    def __init__(self, status: int, func: str, detail: str):
        self.status = status
        super().__init__(f"{func}: {_lib.la_status_string(status).decode()} ({detail})")


def _load() -> ctypes.CDLL:
    if not os.path.exists(LIB_PATH):
        raise ImportError(f"{LIB_PATH} is not built; run `python -c 'import __graft_entry__ as g; g.build()'`")
    lib = ctypes.CDLL(LIB_PATH)
    i64, vp, st = ctypes.c_int64, ctypes.c_void_p, ctypes.c_int
    sig = {
        "la_init": ([ctypes.c_int], st),
        "la_set_mode": ([ctypes.c_int], st),
        "la_set_option": ([ctypes.c_int, i64], st),
        "la_get_option": ([ctypes.c_int, ctypes.POINTER(i64)], st),
        "la_gemm": ([i64, i64, i64, vp, vp, vp, vp], st),
        "la_gemm_host": ([i64, i64, i64, vp, vp, vp, vp], st),
        "la_gemm_host_batch": ([i64, i64, i64, i64, vp, vp, vp, vp], st),
        "la_cgemm": ([i64, i64, i64, vp, vp, vp, vp], st),
        "la_dgemm": ([i64, i64, i64, vp, vp, vp, vp], st),
        "la_gather_alloc": ([i64, ctypes.POINTER(ctypes.c_void_p)], st),
        "la_add": ([i64, i64, vp, vp, vp, ctypes.c_int, vp], st),
        "la_get_unique_id": ([vp], st),
        "la_comm_init": ([vp, ctypes.c_int, ctypes.c_int], st),
        "la_comm_size": ([ctypes.POINTER(ctypes.c_int), ctypes.POINTER(ctypes.c_int)], st),
        "la_gemm_multi": ([i64, i64, i64, vp, vp, vp, vp, ctypes.c_int, ctypes.c_int, vp], st),
        "la_shard_rows": ([i64, ctypes.c_int, ctypes.c_int, ctypes.POINTER(i64), ctypes.POINTER(i64)], st),
        "la_panel_plan": ([i64, i64, i64, ctypes.c_int, ctypes.c_int, ctypes.c_int, i64, ctypes.POINTER(i64),
                           ctypes.c_int, ctypes.POINTER(ctypes.c_int)], st),
        "la_finalize": ([], st),
        "la_status_string": ([ctypes.c_int], ctypes.c_char_p),
        "la_last_error": ([], ctypes.c_char_p),
        "la_last_launch_count": ([], ctypes.c_int),
        "la_kernel_times": ([ctypes.POINTER(ctypes.c_double), ctypes.POINTER(ctypes.c_double),
                             ctypes.POINTER(ctypes.c_int)], st),
    }
    for name, (args, res) in sig.items():
        f = getattr(lib, name)
        f.argtypes, f.restype = args, res
    return lib


_lib = _load()


def _check(status: int, func: str) -> None:
    if status != LA_OK:
        raise LaError(status, func, _lib.la_last_error().decode())


def status_string(status: int) -> str:
    return _lib.la_status_string(int(status)).decode()


def init(device: int | None = None) -> None:
    """la_init on `device` (default: torch's current CUDA device)."""
    if device is None:
        import torch
        device = torch.cuda.current_device()
    _check(_lib.la_init(int(device)), "la_init")


def finalize() -> None:
    _check(_lib.la_finalize(), "la_finalize")


def set_mode(mode: str) -> None:
    """'3xtf32' (default, fp32-accurate) or 'tf32'."""
    if mode not in MODES:
        raise ValueError(f"mode must be one of {sorted(MODES)}")
    _check(_lib.la_set_mode(MODES[mode]), "la_set_mode")


def set_option(name: str, value: int) -> None:
    _check(_lib.la_set_option(OPTIONS[name], int(value)), "la_set_option")


def get_option(name: str) -> int:
    v = ctypes.c_int64()
    _check(_lib.la_get_option(OPTIONS[name], ctypes.byref(v)), "la_get_option")
    return v.value


def last_launch_count() -> int:
    return _lib.la_last_launch_count()


def kernel_times():
    """(split_ms, gemm_ms, gemm_launches) summed over calls since the last query
    (needs set_option('kernel_timing', 1))."""
    a, b, c = ctypes.c_double(), ctypes.c_double(), ctypes.c_int()
    _check(_lib.la_kernel_times(ctypes.byref(a), ctypes.byref(b), ctypes.byref(c)), "la_kernel_times")
    return a.value, b.value, c.value


def _stream_ptr(stream):
    import torch
    if stream is None:
        stream = torch.cuda.current_stream()
    return ctypes.c_void_p(stream.cuda_stream)


def _check_dev(t, name, dtype=None, shape=None):
    """A contiguous 2-D CUDA tensor of `dtype` (default float32) and, if given,
    exactly `shape`: the library trusts the sizes it is passed, so a wrong-sized
    buffer must be rejected here, before it becomes an out-of-bounds write."""
    import torch
    dtype = torch.float32 if dtype is None else dtype
    if not isinstance(t, torch.Tensor) or not t.is_cuda or t.dtype != dtype:
        raise TypeError(f"{name} must be a {dtype} CUDA tensor")
    if t.dim() != 2 or not t.is_contiguous():
        raise ValueError(f"{name} must be a contiguous 2-D (row-major) matrix")
    if shape is not None and tuple(t.shape) != tuple(shape):
        raise ValueError(f"{name} has shape {tuple(t.shape)}, expected {tuple(shape)}")


def gemm(A, B, out=None, stream=None):
    """C = A . B (la_gemm) for float32 CUDA tensors; returns C (n x p)."""
    import torch
    _check_dev(A, "A")
    _check_dev(B, "B")
    n, m = A.shape
    m2, p = B.shape
    if m != m2:
        raise ValueError(f"inner dimension mismatch: {tuple(A.shape)} x {tuple(B.shape)}")
    if out is None:
        out = torch.empty((n, p), dtype=torch.float32, device=A.device)
    else:
        _check_dev(out, "out", shape=(n, p))
    _check(_lib.la_gemm(n, m, p, A.data_ptr(), B.data_ptr(), out.data_ptr(), _stream_ptr(stream)), "la_gemm")
    return out


def cgemm(A, B, out=None, stream=None):
    """C = A . B for complex64 CUDA tensors (la_cgemm, Table 2 "Complex Float")."""
    import torch
    _check_dev(A, "A", torch.complex64)
    _check_dev(B, "B", torch.complex64)
    n, m = A.shape
    m2, p = B.shape
    if m != m2:
        raise ValueError("inner dimension mismatch")
    if out is None:
        out = torch.empty((n, p), dtype=torch.complex64, device=A.device)
    else:
        _check_dev(out, "out", torch.complex64, (n, p))
    _check(_lib.la_cgemm(n, m, p, A.data_ptr(), B.data_ptr(), out.data_ptr(), _stream_ptr(stream)), "la_cgemm")
    return out


def dgemm(A, B, out=None, stream=None):
    """C = A . B for float64 CUDA tensors (la_dgemm, Table 2 "Double")."""
    import torch
    _check_dev(A, "A", torch.float64)
    _check_dev(B, "B", torch.float64)
    n, m = A.shape
    m2, p = B.shape
    if m != m2:
        raise ValueError("inner dimension mismatch")
    if out is None:
        out = torch.empty((n, p), dtype=torch.float64, device=A.device)
    else:
        _check_dev(out, "out", torch.float64, (n, p))
    _check(_lib.la_dgemm(n, m, p, A.data_ptr(), B.data_ptr(), out.data_ptr(), _stream_ptr(stream)), "la_dgemm")
    return out


def add(A, B, out=None, subtract=False, stream=None):
    """C = A + B (or A - B) for float32 CUDA matrices of equal shape (la_add)."""
    import torch
    _check_dev(A, "A")
    _check_dev(B, "B")
    if A.shape != B.shape:
        raise ValueError("shape mismatch")
    if out is None:
        out = torch.empty_like(A)
    else:
        _check_dev(out, "out", shape=tuple(A.shape))
    r, c = A.shape
    _check(_lib.la_add(r, c, A.data_ptr(), B.data_ptr(), out.data_ptr(), int(bool(subtract)),
                       _stream_ptr(stream)), "la_add")
    return out


def gemm_raw(n, m, p, a_ptr, b_ptr, c_ptr, stream_ptr=0):
    """la_gemm on raw device pointers (no checks beyond the library's)."""
    _check(_lib.la_gemm(n, m, p, a_ptr, b_ptr, c_ptr, ctypes.c_void_p(stream_ptr)), "la_gemm")


def gemm_host(A, B, out=None, stream=None):
    """End-to-end la_gemm_host on host float32 arrays (numpy, or CPU tensors,
    pinned or not); copies in, computes, copies out, synchronises."""
    import torch
    def arr(x):
        if isinstance(x, torch.Tensor):
            if x.device.type != "cpu" or x.dtype != torch.float32 or not x.is_contiguous():
                raise TypeError("host tensors must be contiguous float32 on the CPU")
            return x, x.data_ptr(), tuple(x.shape)
        x = np.ascontiguousarray(x, dtype=np.float32)
        return x, x.ctypes.data, x.shape
    A, pa, sa = arr(A)
    B, pb, sb = arr(B)
    n, m = sa
    m2, p = sb
    if m != m2:
        raise ValueError("inner dimension mismatch")
    if out is None:
        out = np.empty((n, p), dtype=np.float32)
    out, pc, sc = arr(out)
    if tuple(sc) != (n, p):
        raise ValueError("out has the wrong shape")
    _check(_lib.la_gemm_host(n, m, p, pa, pb, pc, _stream_ptr(stream)), "la_gemm_host")
    return out


def gemm_host_batch(As, Bs, outs=None, stream=None):
    """la_gemm_host_batch: C_i = A_i . B_i for equal-shape lists of host float32
    arrays (numpy or CPU tensors; pinned for overlap).  The copy-in of product
    i + 1 overlaps the compute and copy-out of product i.  Returns the outputs."""
    import torch
    if len(As) != len(Bs) or len(As) == 0:
        raise ValueError("As and Bs must be non-empty lists of equal length")
    def arr(x):
        if isinstance(x, torch.Tensor):
            if x.device.type != "cpu" or x.dtype != torch.float32 or not x.is_contiguous():
                raise TypeError("host tensors must be contiguous float32 on the CPU")
            return x, x.data_ptr(), tuple(x.shape)
        x = np.ascontiguousarray(x, dtype=np.float32)
        return x, x.ctypes.data, tuple(x.shape)
    a = [arr(x) for x in As]
    b = [arr(x) for x in Bs]
    n, m = a[0][2]
    m2, p = b[0][2]
    if m != m2 or any(x[2] != (n, m) for x in a) or any(x[2] != (m, p) for x in b):
        raise ValueError("all A must be n x m and all B m x p")
    if outs is None:
        outs = [np.empty((n, p), dtype=np.float32) for _ in As]
    c = [arr(x) for x in outs]
    if len(c) != len(a) or any(x[2] != (n, p) for x in c):
        raise ValueError("outs must be len(As) arrays of shape (n, p)")
    k = len(a)
    pa = (ctypes.c_void_p * k)(*[x[1] for x in a])
    pb = (ctypes.c_void_p * k)(*[x[1] for x in b])
    pc = (ctypes.c_void_p * k)(*[x[1] for x in c])
    _check(_lib.la_gemm_host_batch(k, n, m, p, pa, pb, pc, _stream_ptr(stream)), "la_gemm_host_batch")
    return [x[0] for x in c]


def shard_rows(n: int, rank: int, ngpu: int):
    """(row0, rows) owned by `rank` of `ngpu` (la_shard_rows)."""
    r0, r = ctypes.c_int64(), ctypes.c_int64()
    _check(_lib.la_shard_rows(int(n), int(rank), int(ngpu), ctypes.byref(r0), ctypes.byref(r)), "la_shard_rows")
    return r0.value, r.value


def panel_plan(n: int, m: int, p: int, ngpu: int, sms: int = 148, reserved: int = 8, panels: int = 0):
    """Column-panel widths la_gemm_multi broadcasts B in (la_panel_plan; host
    arithmetic, no GPU needed)."""
    cap = 64
    w = (ctypes.c_int64 * cap)()
    cnt = ctypes.c_int()
    _check(_lib.la_panel_plan(int(n), int(m), int(p), int(ngpu), int(sms), int(reserved), int(panels), w, cap,
                              ctypes.byref(cnt)), "la_panel_plan")
    return [w[i] for i in range(cnt.value)]


_COMM = {}   # this process's rank in the library communicator (binding-side shape checks)


def get_unique_id() -> bytes:
    buf = ctypes.create_string_buffer(128)
    _check(_lib.la_get_unique_id(buf), "la_get_unique_id")
    return buf.raw


def comm_init(uid: bytes, rank: int, ngpu: int) -> None:
    if len(uid) != 128:
        raise ValueError("the NCCL unique id is 128 bytes")
    buf = ctypes.create_string_buffer(uid, 128)
    _check(_lib.la_comm_init(buf, int(rank), int(ngpu)), "la_comm_init")
    _COMM.update(rank=int(rank), ngpu=int(ngpu))


def comm_size():
    """(nranks, rank) of the library's NCCL communicator (ncclCommCount,
    ncclCommUserRank)."""
    a, b = ctypes.c_int(), ctypes.c_int()
    _check(_lib.la_comm_size(ctypes.byref(a), ctypes.byref(b)), "la_comm_size")
    return a.value, b.value


def bootstrap_unique_id(group=None) -> bytes:
    """Rank 0 of an initialised torch.distributed group creates the NCCL unique
    id (la_get_unique_id); it is broadcast over the group; every rank returns
    the same 128 bytes."""
    import torch
    import torch.distributed as dist
    rank = dist.get_rank(group)
    uid = get_unique_id() if rank == 0 else bytes(128)
    dev = "cuda" if dist.get_backend(group) == "nccl" else "cpu"
    t = torch.tensor(list(uid), dtype=torch.uint8, device=dev)
    dist.broadcast(t, src=0, group=group)
    return bytes(t.cpu().tolist())


def comm_init_from_process_group(group=None) -> None:
    """Create the library's NCCL communicator over an initialised
    torch.distributed process group (one process per GPU)."""
    import torch.distributed as dist
    uid = bootstrap_unique_id(group)
    comm_init(uid, dist.get_rank(group), dist.get_world_size(group))


class _DeviceArray:
    """Minimal __cuda_array_interface__ holder so torch can view library memory."""

    def __init__(self, ptr, shape, typestr="<f4"):
        self.__cuda_array_interface__ = {"shape": tuple(shape), "typestr": typestr, "data": (int(ptr), False),
                                         "version": 3, "strides": None}


def gather_buffer(n: int, p: int):
    """la_gather_alloc: a symmetric n x p float32 C_full (collective); returns a
    torch CUDA tensor viewing the library-owned buffer (valid until the next
    gather_buffer / comm_init / finalize).  Passing it to gemm_multi as C_full
    selects the fused all-gather epilogue."""
    import torch
    ptr = ctypes.c_void_p()
    _check(_lib.la_gather_alloc(int(n) * int(p) * 4, ctypes.byref(ptr)), "la_gather_alloc")
    return torch.as_tensor(_DeviceArray(ptr.value, (n, p)), device="cuda")


def gemm_multi(n, m, p, A_local, B, C_local, C_full=None, root=0, ngpu=1, stream=None):
    """la_gemm_multi: row-sharded product; B is read on `root` only.  A_local
    and C_local hold this rank's rows (la_shard_rows), B is m x p (required on
    the root, ignored elsewhere), C_full (optional) is n x p."""
    # shapes are checked against this rank's shard when the call is consistent
    # with the communicator; an inconsistent call is left to the library to
    # reject (LA_ERR_INVALID_VALUE / NOT_INITIALIZED)
    rank = _COMM.get("rank")
    rows = shard_rows(n, rank, ngpu)[1] if rank is not None and ngpu == _COMM.get("ngpu") and n >= ngpu else None
    _check_dev(A_local, "A_local", shape=None if rows is None else (rows, m))
    _check_dev(C_local, "C_local", shape=None if rows is None else (rows, p))
    if B is not None:
        _check_dev(B, "B", shape=(m, p))
    if C_full is not None:   # n x p, or a larger symmetric buffer from gather_buffer (rows >= n)
        _check_dev(C_full, "C_full")
        if C_full.shape[1] != p or C_full.shape[0] < n:
            raise ValueError(f"C_full has shape {tuple(C_full.shape)}, expected ({n}, {p})")
    b = 0 if B is None else B.data_ptr()
    cf = 0 if C_full is None else C_full.data_ptr()
    _check(_lib.la_gemm_multi(n, m, p, A_local.data_ptr(), b, C_local.data_ptr(), cf, int(root), int(ngpu),
                              _stream_ptr(stream)), "la_gemm_multi")
    return C_full if C_full is not None else C_local
