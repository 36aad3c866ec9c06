"""Thin ctypes binding of libesnmf.so (include/esnmf.h).  Argument marshalling only:
every step of the method runs in the library's CUDA kernels.  There is no CPU
fallback -- if the extension is missing or cannot load, import fails loudly.

Functions keep the C names (esnmf_create, esnmf_iterate, ...); ``ESNMF`` is a
small convenience wrapper owning one handle.
"""
from __future__ import annotations

import ctypes
import os

import numpy as np

from . import _build

c_i32, c_i64, c_u64, c_dbl, c_p = ctypes.c_int32, ctypes.c_int64, ctypes.c_uint64, ctypes.c_double, ctypes.c_void_p

ESNMF_OK, ESNMF_EINVAL, ESNMF_ENOMEM, ESNMF_ECUDA, ESNMF_ECOMM = 0, 1, 2, 3, 4
ESNMF_ESINGULAR, ESNMF_EDEGENERATE, ESNMF_ESTATE, ESNMF_ETRUNC = 5, 6, 7, 8
ESNMF_T_UNLIMITED = -1
ESNMF_T_SAME = -2
ESNMF_ENFORCE_COLUMN, ESNMF_ENFORCE_MATRIX = 0, 1
ESNMF_SIDE_V, ESNMF_SIDE_U = 0, 1

ALLGATHER_FN = ctypes.CFUNCTYPE(ctypes.c_int, c_p, c_p, c_p, c_i64, c_p)
ALLREDUCE_FN = ctypes.CFUNCTYPE(ctypes.c_int, c_p, ctypes.POINTER(c_dbl), c_i64, c_p)


class esnmf_comm(ctypes.Structure):
    _fields_ = [("ctx", c_p), ("allgather", ALLGATHER_FN), ("allreduce_sum_f64", ALLREDUCE_FN)]


class esnmf_options(ctypes.Structure):
    _fields_ = [
        ("seed", c_u64), ("ridge_scale", c_dbl), ("device", c_i32), ("stream", c_p),
        ("world", c_i32), ("rank", c_i32), ("comm", ctypes.POINTER(esnmf_comm)),
        ("inputs_on_device", c_i32),
        ("at_row_ptr", c_p), ("at_col_idx", c_p), ("at_val", c_p), ("U0", c_p),
        ("head_terms", c_i32), ("t_u", c_i64), ("t_v", c_i64), ("enforce", c_i32), ("init_nnz", c_i64),
        ("seq_k2", c_i32), ("seq_iters", c_i32), ("row_normalize", c_i32), ("keep_ls", c_i32),
    ]


class esnmf_record(ctypes.Structure):
    _fields_ = [("it", c_i32), ("R", c_dbl), ("E", c_dbl), ("nnz_u", c_i64), ("nnz_v", c_i64),
                ("dead_u", c_i32), ("dead_v", c_i32), ("active_u", c_i64), ("active_v", c_i64),
                ("peak_u", c_i64), ("peak_v", c_i64)]

    def as_dict(self) -> dict:
        return {f: getattr(self, f) for f, _ in self._fields_}


class esnmf_info(ctypes.Structure):
    _fields_ = [("n", c_i64), ("m", c_i64), ("nnz", c_i64), ("k", c_i32), ("t", c_i64), ("world", c_i32),
                ("rank", c_i32), ("v_row0", c_i64), ("v_rows", c_i64), ("u_row0", c_i64), ("u_rows", c_i64),
                ("iterations", c_i64), ("device_bytes", c_i64), ("normA2", c_dbl), ("launches", c_i64),
                ("head_terms", c_i32), ("head_dense", c_i32),
                ("ls_cols", c_i32), ("seq_block", c_i32)]


class esnmf_cost(ctypes.Structure):
    _fields_ = [("v_tail_products", c_dbl), ("v_tail_gather_fma", c_dbl), ("v_tail_active", c_dbl),
                ("v_head_products", c_dbl), ("v_head_mma_flops", c_dbl), ("v_yw_mma_flops", c_dbl),
                ("u_products", c_dbl), ("head_terms", c_i32), ("v_tail_gather", c_i32),
                ("v_gather_by_cost", c_i32), ("paper_order_tail", c_i32)]

    def as_dict(self) -> dict:
        return {f: getattr(self, f) for f, _ in self._fields_}


class esnmf_phase(ctypes.Structure):
    _fields_ = [("name", ctypes.c_char * 32), ("calls", c_i64), ("ms", c_dbl)]


class ESNMFError(RuntimeError):
    def __init__(self, status: int, where: str, msg: str):
        super().__init__(f"{where}: status {status} ({msg})")
        self.status = status


_LIB = None

# symbol name -> (restype, argtypes); the complete exported C ABI
SIGNATURES = {
    "esnmf_options_init": (ctypes.c_int, [ctypes.POINTER(esnmf_options)]),
    "esnmf_create": (ctypes.c_int, [ctypes.POINTER(c_p), c_i64, c_i64, c_i32, c_i64, c_p, c_p, c_p,
                                    ctypes.POINTER(esnmf_options)]),
    "esnmf_iterate": (ctypes.c_int, [c_p, c_i32]),
    "esnmf_half_step": (ctypes.c_int, [c_p, c_i32]),
    "esnmf_residual": (ctypes.c_int, [c_p, ctypes.POINTER(c_dbl)]),
    "esnmf_error": (ctypes.c_int, [c_p, ctypes.POINTER(c_dbl)]),
    "esnmf_records": (ctypes.c_int, [c_p, c_i64, ctypes.POINTER(c_i64), ctypes.POINTER(esnmf_record)]),
    "esnmf_get_U": (ctypes.c_int, [c_p, c_i64, ctypes.POINTER(c_i64), c_p, c_p, c_p]),
    "esnmf_get_V": (ctypes.c_int, [c_p, c_i64, ctypes.POINTER(c_i64), c_p, c_p, c_p]),
    "esnmf_set_factor": (ctypes.c_int, [c_p, c_i32, c_i64, c_p, c_p, c_p]),
    "esnmf_get_ls": (ctypes.c_int, [c_p, c_i32, ctypes.POINTER(c_i64), ctypes.POINTER(c_i64), c_p]),
    "esnmf_get_gram": (ctypes.c_int, [c_p, c_i32, c_p, ctypes.POINTER(c_dbl)]),
    "esnmf_get_info": (ctypes.c_int, [c_p, ctypes.POINTER(esnmf_info)]),
    "esnmf_profile": (ctypes.c_int, [c_p, c_i32]),
    "esnmf_cost_model": (ctypes.c_int, [c_p, ctypes.POINTER(esnmf_cost)]),
    "esnmf_nccl_unique_id": (ctypes.c_int, [c_p]),
    "esnmf_nccl_comm_create": (ctypes.c_int, [c_i32, c_i32, c_p, c_i32, ctypes.POINTER(ctypes.POINTER(esnmf_comm))]),
    "esnmf_nccl_comm_destroy": (None, [ctypes.POINTER(esnmf_comm)]),
    "esnmf_phase_times": (ctypes.c_int, [c_p, c_i64, ctypes.POINTER(c_i64), ctypes.POINTER(esnmf_phase)]),
    "esnmf_destroy": (None, [c_p]),
    "esnmf_strerror": (ctypes.c_char_p, [ctypes.c_int]),
    "esnmf_last_error": (ctypes.c_char_p, []),
    "esnmf_partition_rows": (ctypes.c_int, [c_i64, c_p, c_i32, c_p]),
    "esnmf_truncate": (ctypes.c_int, [c_p, c_i32, c_i64, c_i32]),
    "esnmf_topic_accuracy": (ctypes.c_int, [c_p, c_p, c_i32, c_p]),
    "esnmf_version": (ctypes.c_char_p, []),
}


def lib():
    """Load libesnmf.so (building it first if the sources are newer)."""
    global _LIB
    if _LIB is None:
        path = _build.build()
        if not os.path.exists(path):
            raise ImportError(f"libesnmf.so missing at {path}")
        L = ctypes.CDLL(path)
        for name, (res, args) in SIGNATURES.items():
            f = getattr(L, name)
            f.restype = res
            f.argtypes = args
        _LIB = L
    return _LIB


def _check(st: int, where: str):
    if st != ESNMF_OK:
        L = lib()
        raise ESNMFError(st, where, (L.esnmf_last_error() or L.esnmf_strerror(st) or b"").decode())


def _ptr(x):
    """(pointer, on_device) of a numpy array or torch tensor (contiguous)."""
    if x is None:
        return None, None
    if isinstance(x, np.ndarray):
        if not x.flags.c_contiguous:
            raise ValueError("array must be C-contiguous")
        return x.ctypes.data, False
    # torch tensor
    if not x.is_contiguous():
        raise ValueError("tensor must be contiguous")
    return x.data_ptr(), x.is_cuda


# ----------------------------------------------------------------- C-name API

def esnmf_options_init() -> esnmf_options:
    o = esnmf_options()
    _check(lib().esnmf_options_init(ctypes.byref(o)), "esnmf_options_init")
    return o


def esnmf_create(n, m, k, t, row_ptr, col_idx, val, opt: esnmf_options | None = None):
    """Returns an opaque handle (int).  Host numpy or device torch inputs."""
    o = opt if opt is not None else esnmf_options_init()
    p0, d0 = _ptr(row_ptr)
    p1, d1 = _ptr(col_idx)
    p2, d2 = _ptr(val)
    if not (d0 == d1 == d2):
        raise ValueError("row_ptr, col_idx, val must all be host or all device")
    if d0:
        o.inputs_on_device = 1
    h = c_p()
    _check(lib().esnmf_create(ctypes.byref(h), int(n), int(m), int(k), int(t), p0, p1, p2, ctypes.byref(o)),
           "esnmf_create")
    return h.value


def esnmf_iterate(h, iters: int):
    _check(lib().esnmf_iterate(h, int(iters)), "esnmf_iterate")


def esnmf_half_step(h, side: int):
    _check(lib().esnmf_half_step(h, int(side)), "esnmf_half_step")


def esnmf_residual(h) -> float:
    r = c_dbl()
    _check(lib().esnmf_residual(h, ctypes.byref(r)), "esnmf_residual")
    return r.value


def esnmf_error(h) -> float:
    e = c_dbl()
    _check(lib().esnmf_error(h, ctypes.byref(e)), "esnmf_error")
    return e.value


def esnmf_records(h) -> list[dict]:
    cnt = c_i64()
    st = lib().esnmf_records(h, 0, ctypes.byref(cnt), None)
    if st not in (ESNMF_OK, ESNMF_ETRUNC):
        _check(st, "esnmf_records")
    buf = (esnmf_record * max(1, cnt.value))()
    _check(lib().esnmf_records(h, cnt.value, ctypes.byref(cnt), buf), "esnmf_records")
    return [buf[i].as_dict() for i in range(cnt.value)]


def _get_factor(fn, h, name):
    nnz = c_i64()
    st = fn(h, 0, ctypes.byref(nnz), None, None, None)
    if st not in (ESNMF_OK, ESNMF_ETRUNC):
        _check(st, name)
    n = nnz.value
    row = np.empty(max(n, 1), np.int32)
    col = np.empty(max(n, 1), np.int32)
    val = np.empty(max(n, 1), np.float32)
    _check(fn(h, n, ctypes.byref(nnz), row.ctypes.data, col.ctypes.data, val.ctypes.data), name)
    return row[:n], col[:n], val[:n]


def esnmf_get_U(h):
    """(row, col, val) canonical column-major COO of U."""
    return _get_factor(lib().esnmf_get_U, h, "esnmf_get_U")


def esnmf_get_V(h):
    return _get_factor(lib().esnmf_get_V, h, "esnmf_get_V")


def esnmf_set_factor(h, side: int, row, col, val):
    row = np.ascontiguousarray(row, np.int32)
    col = np.ascontiguousarray(col, np.int32)
    val = np.ascontiguousarray(val, np.float32)
    _check(lib().esnmf_set_factor(h, int(side), len(row), row.ctypes.data, col.ctypes.data, val.ctypes.data),
           "esnmf_set_factor")


def esnmf_get_ls(h, side: int):
    """(row0, LS rows x k float32) of this rank's shard for the last half-step of `side`."""
    r0, rows = c_i64(), c_i64()
    _check(lib().esnmf_get_ls(h, int(side), ctypes.byref(r0), ctypes.byref(rows), None), "esnmf_get_ls")
    k = esnmf_get_info(h)["ls_cols"]   # k, or k2 (the current block) in sequential mode
    out = np.empty((rows.value, k), np.float32)
    _check(lib().esnmf_get_ls(h, int(side), ctypes.byref(r0), ctypes.byref(rows), out.ctypes.data), "esnmf_get_ls")
    return r0.value, out


def esnmf_get_gram(h, side: int):
    k = esnmf_get_info(h)["ls_cols"]
    G = np.empty((k, k), np.float64)
    eps = c_dbl()
    _check(lib().esnmf_get_gram(h, int(side), G.ctypes.data, ctypes.byref(eps)), "esnmf_get_gram")
    return G, eps.value


def esnmf_topic_accuracy(h, labels, n_journals: int, k: int) -> np.ndarray:
    lab = np.ascontiguousarray(labels, np.int32)
    acc = np.empty(k, np.float64)
    _check(lib().esnmf_topic_accuracy(h, lab.ctypes.data, int(n_journals), acc.ctypes.data), "esnmf_topic_accuracy")
    return acc


def esnmf_get_info(h) -> dict:
    i = esnmf_info()
    _check(lib().esnmf_get_info(h, ctypes.byref(i)), "esnmf_get_info")
    return {f: getattr(i, f) for f, _ in i._fields_}


def esnmf_cost_model(h) -> dict:
    """The last V side's cost model and tail order, and the U side's product count
    (esnmf_cost_model in include/esnmf.h)."""
    c = esnmf_cost()
    _check(lib().esnmf_cost_model(h, ctypes.byref(c)), "esnmf_cost_model")
    return c.as_dict()


ESNMF_NCCL_ID_BYTES = 128


def esnmf_nccl_unique_id() -> bytes:
    """A fresh NCCL unique id (rank 0 draws it; every rank needs the same bytes)."""
    buf = ctypes.create_string_buffer(ESNMF_NCCL_ID_BYTES)
    _check(lib().esnmf_nccl_unique_id(buf), "esnmf_nccl_unique_id")
    return buf.raw


class NcclComm:
    """The library's own NCCL communicator (esnmf_nccl_comm_create): pass ``.struct``
    as ESNMF(comm=...).  Collective: every rank constructs it with the same id."""

    def __init__(self, world: int, rank: int, uid: bytes, device: int):
        if len(uid) != ESNMF_NCCL_ID_BYTES:
            raise ValueError("NCCL unique id must be 128 bytes")
        self.world, self.rank = world, rank
        self._ptr = ctypes.POINTER(esnmf_comm)()
        buf = ctypes.create_string_buffer(uid, ESNMF_NCCL_ID_BYTES)
        _check(lib().esnmf_nccl_comm_create(int(world), int(rank), buf, int(device), ctypes.byref(self._ptr)),
               "esnmf_nccl_comm_create")
        self.struct = self._ptr.contents

    def close(self):
        if self._ptr:
            lib().esnmf_nccl_comm_destroy(self._ptr)
            self._ptr = ctypes.POINTER(esnmf_comm)()


def esnmf_profile(h, enable: bool):
    _check(lib().esnmf_profile(h, 1 if enable else 0), "esnmf_profile")


def esnmf_phase_times(h) -> dict:
    """{phase name: (calls, total ms)} since profiling was enabled."""
    buf = (esnmf_phase * 32)()
    cnt = c_i64()
    _check(lib().esnmf_phase_times(h, 32, ctypes.byref(cnt), buf), "esnmf_phase_times")
    return {buf[i].name.decode(): (buf[i].calls, buf[i].ms) for i in range(cnt.value)}


def esnmf_truncate(h, side: int, t: int, whole: bool = False):
    _check(lib().esnmf_truncate(h, int(side), int(t), ESNMF_ENFORCE_MATRIX if whole else ESNMF_ENFORCE_COLUMN),
           "esnmf_truncate")


def esnmf_destroy(h):
    if h:
        lib().esnmf_destroy(h)


def esnmf_partition_rows(row_ptr: np.ndarray, world: int) -> np.ndarray:
    row_ptr = np.ascontiguousarray(row_ptr, np.int64)
    b = np.empty(world + 1, np.int64)
    _check(lib().esnmf_partition_rows(len(row_ptr) - 1, row_ptr.ctypes.data, int(world), b.ctypes.data),
           "esnmf_partition_rows")
    return b


def esnmf_version() -> str:
    return lib().esnmf_version().decode()


# ------------------------------------------------------------- convenience

class ESNMF:
    """One solver handle.  ``inputs``: dict with a_ptr/a_col/a_val (+ optional
    at_ptr/at_col/at_val), numpy (host) or torch CUDA tensors (device)."""

    def __init__(self, n, m, k, t, inputs: dict, seed: int = 0, ridge_scale: float = 1e-10, stream=None,
                 device: int = -1, use_at: bool = True, U0=None, world: int = 1, rank: int = 0, comm=None,
                 head_terms: int = -1, t_u="same", t_v="same", whole: bool = False, init_nnz: int = 0,
                 seq_k2: int = 0, seq_iters: int = 0, row_normalize: bool = False, keep_ls: bool = False):
        """t_u / t_v: separate budgets ("same" = t, None = unlimited); whole: whole-factor
        enforcement (Alg. 2 as printed) instead of per column; init_nnz: sparse U_0
        (reading C18); seq_k2 > 0: sequential ALS (Alg. 3) in blocks of seq_k2 topics,
        seq_iters iterations per block; row_normalize: divide each row of A by its nnz
        on the device; keep_ls: esnmf_iterate always writes the V side's LS buffer
        (esnmf_get_ls after esnmf_iterate; esnmf_half_step always writes it)."""
        o = esnmf_options_init()
        o.head_terms = head_terms
        o.t_u = ESNMF_T_SAME if t_u == "same" else (ESNMF_T_UNLIMITED if t_u is None else int(t_u))
        o.t_v = ESNMF_T_SAME if t_v == "same" else (ESNMF_T_UNLIMITED if t_v is None else int(t_v))
        o.enforce = ESNMF_ENFORCE_MATRIX if whole else ESNMF_ENFORCE_COLUMN
        o.init_nnz = int(init_nnz)
        o.seq_k2, o.seq_iters = int(seq_k2), int(seq_iters)
        o.row_normalize = 1 if row_normalize else 0
        o.keep_ls = 1 if keep_ls else 0
        o.seed = seed
        o.ridge_scale = ridge_scale
        o.device = device
        self._keep = []
        if world > 1 and comm is None:
            raise ValueError("world > 1 needs a comm (paper_1510_05237_b200.comm)")
        if comm is not None:
            o.world, o.rank = world, rank
            self._keep.append(comm)
            o.comm = ctypes.pointer(comm)
        if stream is not None:
            o.stream = stream
        if use_at and inputs.get("at_ptr") is not None:
            o.at_row_ptr = _ptr(inputs["at_ptr"])[0]
            o.at_col_idx = _ptr(inputs["at_col"])[0]
            o.at_val = _ptr(inputs["at_val"])[0]
        if U0 is not None:
            U0 = np.ascontiguousarray(U0, np.float32) if isinstance(U0, np.ndarray) else U0
            self._keep.append(U0)
            o.U0 = _ptr(U0)[0]
        self.k, self.n, self.m, self.t = k, n, m, t
        self.h = esnmf_create(n, m, k, ESNMF_T_UNLIMITED if t is None else t, inputs["a_ptr"], inputs["a_col"],
                              inputs["a_val"], o)

    def iterate(self, iters: int = 1):
        esnmf_iterate(self.h, iters)

    def half_step(self, side: int):
        esnmf_half_step(self.h, side)

    def residual(self) -> float:
        return esnmf_residual(self.h)

    def error(self) -> float:
        return esnmf_error(self.h)

    def records(self) -> list[dict]:
        return esnmf_records(self.h)

    def get_U(self):
        return esnmf_get_U(self.h)

    def get_V(self):
        return esnmf_get_V(self.h)

    def set_factor(self, side, row, col, val):
        esnmf_set_factor(self.h, side, row, col, val)

    def get_ls(self, side):
        return esnmf_get_ls(self.h, side)

    def get_gram(self, side):
        return esnmf_get_gram(self.h, side)

    def truncate(self, side: int, t: int, whole: bool = False):
        esnmf_truncate(self.h, side, t, whole)

    def topic_accuracy(self, labels, n_journals: int) -> np.ndarray:
        """Eq. (3)-(4) per topic column of V (esnmf_topic_accuracy)."""
        return esnmf_topic_accuracy(self.h, labels, n_journals, self.k)

    def info(self) -> dict:
        return esnmf_get_info(self.h)

    def cost_model(self) -> dict:
        return esnmf_cost_model(self.h)

    def profile(self, enable: bool = True):
        esnmf_profile(self.h, enable)

    def phase_times(self) -> dict:
        return esnmf_phase_times(self.h)

    def close(self):
        if self.h:
            esnmf_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def __enter__(self):
        return self

    def __exit__(self, *a):
        self.close()
