"""paper_2211_10979_b200 — B200-native dense full-tableau simplex (libsimplex).

Thin Python binding over the C ABI in ``include/libsimplex.h``: argument
marshalling only.  Every step of the per-pivot loop (pricing, ratio test, pivot
update, loop control) runs in the sm_100a kernels of ``csrc/``; there is no CPU
fallback — importing this package without a built ``libsimplex.so`` raises, and
every call on a machine without a CUDA device returns SIMPLEX_E_CUDA.

PyTorch is used only for plumbing: a CUDA tensor may be passed as input or output
(its device pointer is handed to the library), the current torch stream orders
the library's work after the caller's, and a torch.distributed process group
carries the 128-byte NCCL id to all ranks.
"""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

_PKG = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_PKG, "libsimplex.so")

OK = 0
E_ARG, E_NONFINITE, E_NEG_RHS, E_OOM, E_CUDA, E_NCCL, E_STATE = -1, -2, -3, -4, -5, -6, -7
ERR_NAME = {E_ARG: "SIMPLEX_E_ARG", E_NONFINITE: "SIMPLEX_E_NONFINITE", E_NEG_RHS: "SIMPLEX_E_NEG_RHS",
            E_OOM: "SIMPLEX_E_OOM", E_CUDA: "SIMPLEX_E_CUDA", E_NCCL: "SIMPLEX_E_NCCL",
            E_STATE: "SIMPLEX_E_STATE"}
RUNNING, OPTIMAL, UNBOUNDED, INFEASIBLE, ITERATION_LIMIT = -1, 0, 2, 3, 4
DANTZIG, BLAND = 0, 1
STATUS_NAME = {RUNNING: "RUNNING", OPTIMAL: "OPTIMAL", UNBOUNDED: "UNBOUNDED",
               INFEASIBLE: "INFEASIBLE", ITERATION_LIMIT: "ITERATION_LIMIT"}

# every symbol declared in include/libsimplex.h
EXPORTS = ["simplex_default_options", "simplex_create", "simplex_reset", "simplex_iterate",
           "simplex_solve", "simplex_solve_lp", "simplex_get_solution", "simplex_get_trace", "simplex_get_tableau",
           "simplex_tableau_hash", "simplex_get_stats", "simplex_destroy", "simplex_last_error",
           "simplex_nccl_unique_id", "simplex_partition", "simplex_version"]


class Options(C.Structure):
    _fields_ = [("struct_size", C.c_uint32), ("tol_opt", C.c_double), ("tol_piv", C.c_double),
                ("max_pivots", C.c_int64), ("record_trace", C.c_int32), ("device", C.c_int32),
                ("nranks", C.c_int32), ("rank", C.c_int32), ("nccl_id", C.c_void_p),
                ("stream", C.c_void_p), ("virtual_ranks", C.c_int32), ("segment_pivots", C.c_int32),
                ("time_kernels", C.c_int32), ("lookahead", C.c_int32),
                ("pivot_rule", C.c_int32), ("phase1", C.c_int32), ("overlap", C.c_int32),
                ("exchange", C.c_int32), ("exchange_timeout_ms", C.c_int32),
                ("host_share", C.c_double), ("host_threads", C.c_int32)]


class Stats(C.Structure):
    _fields_ = [("pivots", C.c_int64), ("update_launches", C.c_int64), ("update_ms_total", C.c_double),
                ("loop_ms_total", C.c_double), ("graph_launches", C.c_int64),
                ("kernel_launches", C.c_int64), ("local_rows", C.c_int64), ("local_cols", C.c_int64),
                ("local_ld", C.c_int64), ("col_offset", C.c_int64), ("bytes_per_pivot", C.c_int64),
                ("path", C.c_int64), ("host_cols", C.c_int64), ("host_ms_total", C.c_double),
                ("host_wait_ms_total", C.c_double)]


class SimplexError(RuntimeError):
    def __init__(self, code, msg):
        super().__init__(f"{ERR_NAME.get(code, code)}: {msg}")
        self.code = code


_lib = None


def lib():
    """The loaded libsimplex.so (raises if it has not been built: no fallback)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(f"{LIB_PATH} not built; run `python -m paper_2211_10979_b200.build` "
                              "(there is no CPU fallback)")
        L = C.CDLL(LIB_PATH)
        vp, i64, pi64 = C.c_void_p, C.c_int64, C.POINTER(C.c_int64)
        pint = C.POINTER(C.c_int)
        L.simplex_default_options.argtypes = [C.POINTER(Options)]
        L.simplex_default_options.restype = None
        L.simplex_create.argtypes = [C.POINTER(vp), i64, i64, vp, vp, vp, C.POINTER(Options)]
        L.simplex_reset.argtypes = [vp, vp, vp, vp]
        L.simplex_iterate.argtypes = [vp, i64, pi64, pint]
        L.simplex_solve.argtypes = [vp, pint]
        L.simplex_solve_lp.argtypes = [vp, vp, vp, vp, vp, vp, C.POINTER(C.c_double), pi64, pint]
        L.simplex_get_solution.argtypes = [vp, vp, vp, C.POINTER(C.c_double), pi64, pint]
        L.simplex_get_trace.argtypes = [vp, vp, vp, i64, pi64]
        L.simplex_get_tableau.argtypes = [vp, vp, i64]
        L.simplex_tableau_hash.argtypes = [vp, C.POINTER(C.c_uint64)]
        L.simplex_get_stats.argtypes = [vp, C.POINTER(Stats)]
        L.simplex_destroy.argtypes = [vp]
        L.simplex_last_error.argtypes = []
        L.simplex_last_error.restype = C.c_char_p
        L.simplex_nccl_unique_id.argtypes = [vp]
        L.simplex_partition.argtypes = [i64, i64, i64, pi64, pi64]
        L.simplex_version.argtypes = []
        L.simplex_version.restype = C.c_char_p
        for name in EXPORTS:   # simplex_err-returning entry points
            if name not in ("simplex_default_options", "simplex_last_error", "simplex_version"):
                getattr(L, name).restype = C.c_int
        _lib = L
    return _lib


def use_library(path: str) -> None:
    """Experiment scripts only (scripts/_experiment.py): load `path` — a build with the
    SIMPLEX_* environment hooks compiled in — instead of the product libsimplex.so.
    Must be called before the library is first loaded."""
    global LIB_PATH
    if _lib is not None:
        raise RuntimeError("libsimplex is already loaded from " + LIB_PATH)
    LIB_PATH = path


def _check(code):
    if code != OK:
        raise SimplexError(code, lib().simplex_last_error().decode())


def default_options() -> Options:
    o = Options()
    lib().simplex_default_options(C.byref(o))
    return o


def nccl_unique_id() -> bytes:
    buf = C.create_string_buffer(128)
    _check(lib().simplex_nccl_unique_id(buf))
    return buf.raw


def partition(total_cols: int, nparts: int, part: int):
    """(c0, width) of column part `part` (simplex_partition)."""
    c0, w = C.c_int64(), C.c_int64()
    _check(lib().simplex_partition(int(total_cols), int(nparts), int(part), C.byref(c0), C.byref(w)))
    return c0.value, w.value


def share_nccl_id(group) -> bytes:
    """Rank 0 of the torch.distributed group draws a fresh ncclUniqueId; every rank
    returns the same 128 bytes (broadcast over the group's own backend)."""
    import torch.distributed as dist
    obj = [nccl_unique_id() if dist.get_rank(group) == 0 else None]
    dist.broadcast_object_list(obj, src=dist.get_global_rank(group, 0), group=group)
    assert isinstance(obj[0], (bytes, bytearray)) and len(obj[0]) == 128
    return bytes(obj[0])


def version() -> str:
    return lib().simplex_version().decode()


def _ptr(a, keep, numel, device=None):
    """Device pointer of a CUDA tensor (float64, contiguous, on the handle's device), or host
    pointer of a C-contiguous float64 copy of anything array-like; exactly `numel` elements."""
    if a is None:
        return None
    if hasattr(a, "is_cuda") and hasattr(a, "data_ptr"):
        import torch
        if a.is_cuda:
            if a.dtype != torch.float64 or not a.is_contiguous():
                raise ValueError("CUDA inputs must be contiguous float64 tensors")
            if a.numel() != numel:
                raise ValueError(f"expected {numel} elements, got {a.numel()}")
            if device is not None and device >= 0 and a.device.index != device:
                raise ValueError(f"CUDA input on device {a.device.index}, handle on device {device}")
            keep.append(a)
            return C.c_void_p(a.data_ptr())
        a = a.numpy()
    arr = np.ascontiguousarray(a, dtype=np.float64)
    if arr.size != numel:
        raise ValueError(f"expected {numel} elements, got {arr.size}")
    keep.append(arr)
    return C.c_void_p(arr.ctypes.data)


def _shape(a):
    return tuple(int(v) for v in a.shape)


def _current_stream(device):
    """torch's current stream ON THE HANDLE'S DEVICE (None without an initialised CUDA context)."""
    try:
        import torch
        if torch.cuda.is_available() and torch.cuda.is_initialized():
            dev = torch.cuda.current_device() if device is None or device < 0 else device
            return torch.cuda.current_stream(dev).cuda_stream
    except Exception:
        pass
    return None


class Simplex:
    """One libsimplex handle: maximize c^T x s.t. A x <= b, x >= 0 (Table I).

    A (m, n), b (m,), c (n,): float64 numpy arrays, CPU tensors, or CUDA tensors on
    the handle's device.  ``group`` (a torch.distributed process group) splits the
    columns over its ranks (one GPU per rank, NCCL); ``virtual_ranks`` splits them
    into slabs on one GPU (test path for the multi-GPU data flow)."""

    def __init__(self, A, b, c, *, tol_opt=1e-7, tol_piv=1e-10, max_pivots=0, record_trace=True,
                 device=None, group=None, virtual_ranks=1, segment_pivots=0, time_kernels=False,
                 lookahead=0, pivot_rule=DANTZIG, phase1=True, overlap=True, stream=None, exchange=0,
                 host_share=0.0, host_threads=0):
        L = lib()
        if len(_shape(A)) != 2:
            raise ValueError("A must be a 2-D (m, n) array")
        m, n = _shape(A)
        if _shape(b) != (m,) or _shape(c) != (n,):
            raise ValueError(f"b must have shape ({m},) and c shape ({n},); got {_shape(b)}, {_shape(c)}")
        o = default_options()
        o.tol_opt, o.tol_piv, o.max_pivots = tol_opt, tol_piv, max_pivots
        o.record_trace = 1 if record_trace else 0
        o.device = -1 if device is None else int(device)
        o.virtual_ranks = int(virtual_ranks)
        o.segment_pivots = int(segment_pivots)
        o.time_kernels = 1 if time_kernels else 0
        o.lookahead = int(lookahead)
        o.pivot_rule = int(pivot_rule)
        o.phase1 = 1 if phase1 else 0
        o.overlap = 1 if overlap else 0
        o.exchange = int(exchange)
        o.host_share = float(host_share)
        o.host_threads = int(host_threads)
        s = stream if stream is not None else _current_stream(o.device)
        o.stream = s if s else None
        self._idbuf = None
        if group is not None:
            import torch.distributed as dist
            o.nranks = dist.get_world_size(group)
            o.rank = dist.get_rank(group)
            if o.nranks > 1:
                self._idbuf = C.create_string_buffer(share_nccl_id(group), 128)
                o.nccl_id = C.cast(self._idbuf, C.c_void_p)
        self.m, self.n = m, n
        self.nranks, self.rank = o.nranks, o.rank
        keep = []
        h = C.c_void_p()
        _check(L.simplex_create(C.byref(h), m, n, _ptr(A, keep, m * n, o.device), _ptr(b, keep, m, o.device),
                                _ptr(c, keep, n, o.device), C.byref(o)))
        self._h = h
        self.device = self._device_of_handle(o.device)

    # --------------------------------------------------------------- lifecycle
    def close(self):
        if getattr(self, "_h", None):
            lib().simplex_destroy(self._h)
            self._h = None

    __del__ = close

    def __enter__(self):
        return self

    def __exit__(self, *exc):
        self.close()

    # --------------------------------------------------------------- calls
    @staticmethod
    def _device_of_handle(device):
        if device is not None and device >= 0:
            return device
        try:
            import torch
            return torch.cuda.current_device()
        except Exception:
            return -1

    def reset(self, A, b, c):
        """Rebuild from new data of the SAME shape (simplex_reset)."""
        m, n = self.m, self.n
        if _shape(A) != (m, n) or _shape(b) != (m,) or _shape(c) != (n,):
            raise ValueError(f"reset needs A ({m}, {n}), b ({m},), c ({n},)")
        keep = []
        _check(lib().simplex_reset(self._h, _ptr(A, keep, m * n, self.device), _ptr(b, keep, m, self.device),
                                   _ptr(c, keep, n, self.device)))

    def solve(self) -> int:
        st = C.c_int()
        _check(lib().simplex_solve(self._h, C.byref(st)))
        return st.value

    def solve_lp(self, A, b, c, x=None, y=None):
        """reset(A, b, c) + solve() + solution(x, y) in ONE library call (simplex_solve_lp: one
        launch and one synchronisation on the small-tableau path).  Returns (x, y, objective,
        pivots, status) like solution()."""
        m, n = self.m, self.n
        if _shape(A) != (m, n) or _shape(b) != (m,) or _shape(c) != (n,):
            raise ValueError(f"solve_lp needs A ({m}, {n}), b ({m},), c ({n},)")
        xo = np.empty(n) if x is None else x
        yo = np.empty(m) if y is None else y
        keep = []
        obj, piv, st = C.c_double(), C.c_int64(), C.c_int()
        _check(lib().simplex_solve_lp(self._h, _ptr(A, keep, m * n, self.device), _ptr(b, keep, m, self.device),
                                      _ptr(c, keep, n, self.device), _out_ptr(xo, keep, n, self.device),
                                      _out_ptr(yo, keep, m, self.device), C.byref(obj), C.byref(piv), C.byref(st)))
        return xo, yo, obj.value, piv.value, st.value

    def iterate(self, max_pivots: int):
        done, st = C.c_int64(), C.c_int()
        _check(lib().simplex_iterate(self._h, int(max_pivots), C.byref(done), C.byref(st)))
        return done.value, st.value

    def solution(self, x=None, y=None):
        """(x, y, objective, pivots, status); x / y may be preallocated outputs (numpy or CUDA)."""
        xo = np.empty(self.n) if x is None else x
        yo = np.empty(self.m) if y is None else y
        keep = []
        obj, piv, st = C.c_double(), C.c_int64(), C.c_int()
        _check(lib().simplex_get_solution(self._h, _out_ptr(xo, keep, self.n, self.device),
                                          _out_ptr(yo, keep, self.m, self.device), C.byref(obj),
                                          C.byref(piv), C.byref(st)))
        return xo, yo, obj.value, piv.value, st.value

    def trace(self):
        st = self.stats()
        cap = st.pivots
        k = np.zeros(max(cap, 1), dtype=np.int32)
        r = np.zeros(max(cap, 1), dtype=np.int32)
        ln = C.c_int64()
        _check(lib().simplex_get_trace(self._h, C.c_void_p(k.ctypes.data), C.c_void_p(r.ctypes.data), cap,
                                       C.byref(ln)))
        return k[:ln.value].copy(), r[:ln.value].copy()

    def tableau(self):
        """This rank's logical slab (all columns on 1 GPU / with virtual ranks): (T, col_offset)."""
        st = self.stats()
        T = np.empty((st.local_rows, st.local_cols))
        _check(lib().simplex_get_tableau(self._h, C.c_void_p(T.ctypes.data), st.local_cols))
        return T, st.col_offset

    def tableau_hash(self) -> int:
        h = C.c_uint64()
        _check(lib().simplex_tableau_hash(self._h, C.byref(h)))
        return h.value

    def stats(self) -> Stats:
        s = Stats()
        _check(lib().simplex_get_stats(self._h, C.byref(s)))
        return s


def _out_ptr(a, keep, numel, device):
    """An output buffer: float64, contiguous, exactly `numel` elements (CUDA: on the handle's
    device).  Anything else raises ValueError instead of becoming an out-of-bounds write."""
    if hasattr(a, "is_cuda") and hasattr(a, "data_ptr"):
        import torch
        if a.dtype != torch.float64 or not a.is_contiguous() or a.numel() != numel:
            raise ValueError(f"output must be a contiguous float64 tensor of {numel} elements")
        if a.is_cuda and device is not None and device >= 0 and a.device.index != device:
            raise ValueError(f"output on device {a.device.index}, handle on device {device}")
        keep.append(a)
        return C.c_void_p(a.data_ptr())
    if not (isinstance(a, np.ndarray) and a.dtype == np.float64 and a.flags.c_contiguous and a.size == numel):
        raise ValueError(f"output must be a C-contiguous float64 array of {numel} elements")
    return C.c_void_p(a.ctypes.data)


__all__ = ["Simplex", "SimplexError", "lib", "default_options", "nccl_unique_id", "share_nccl_id",
           "partition", "version",
           "OPTIMAL", "UNBOUNDED", "ITERATION_LIMIT", "RUNNING", "STATUS_NAME", "EXPORTS"]
