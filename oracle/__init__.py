"""oracle -- plain, slow fp64 CPU oracle of enforced-sparse ALS (arXiv 1510.05237).

TEST INFRASTRUCTURE ONLY.  Only ``tests/``, ``__graft_entry__.smoke()`` and
``bench.py``'s ``cpu_baseline`` / ``--impl reference`` legs may import this
package.  It shares no code with the CUDA path (paper_1510_05237_b200/); the
two meet only in the seeded inputs from ``synth/``.

The arithmetic lives in ``esnmf_oracle.c`` (fp64, OpenMP); this module only
marshals arrays and strings the paper's steps together in the paper's order
(Alg. 2, with per-column enforcement):

    V  = A^T U (U^T U + eps I)^{-1}, clamp, keep t per column
    U' = A V (V^T V + eps I)^{-1},   clamp, keep t per column
    R  = ||U' - U||_F / ||U'||_F
    E  = ||A - U' V^T||_F / ||A||_F  (trace identity)

``oracle.bruteforce`` is a dense numpy twin used to pin this module on tiny
inputs.  Parity status of every function: DESIGN.md section 4.
"""
from __future__ import annotations

import ctypes
import functools
import os
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
_SO = os.path.join(HERE, "liboracle.so")
RHO_DEFAULT = 1e-10   # ridge scale, reading C6


def build(verbose: bool = False) -> None:
    src = os.path.join(HERE, "esnmf_oracle.c")
    cmd = ["gcc", "-O2", "-fopenmp", "-shared", "-fPIC", src, "-o", _SO, "-lm"]
    subprocess.run(cmd, check=True, capture_output=not verbose)


@functools.lru_cache(None)
def _lib():
    if not os.path.exists(_SO) or os.path.getmtime(_SO) < os.path.getmtime(os.path.join(HERE, "esnmf_oracle.c")):
        build()
    lib = ctypes.CDLL(_SO)
    i64, i32, u64, p, d = ctypes.c_int64, ctypes.c_int32, ctypes.c_uint64, ctypes.c_void_p, ctypes.c_double
    lib.or_u0.argtypes = [i64, i32, u64, p]
    lib.or_u0_sparsify.argtypes = [i64, i32, u64, i64, p]
    lib.or_splitmix64_pub.argtypes = [u64]
    lib.or_splitmix64_pub.restype = u64
    lib.or_gram.argtypes = [i64, i32, p, p]
    lib.or_cholesky.argtypes = [i32, p, d, p, p]
    lib.or_cholesky.restype = ctypes.c_int
    lib.or_solve_rows.argtypes = [i64, i32, p, p, p]
    lib.or_spmm.argtypes = [i64, i32, p, p, p, p, p]
    lib.or_spmm_rows.argtypes = [i64, p, i32, p, p, p, p, p]
    lib.or_clamp_top_t.argtypes = [i64, i32, i64, p, p]
    lib.or_clamp_top_t_whole.argtypes = [i64, i32, i64, p, p]
    lib.or_residual.argtypes = [i64, i32, p, p]
    lib.or_residual.restype = d
    lib.or_error.argtypes = [i64, i32, p, p, p, p, d]
    lib.or_error.restype = d
    lib.or_frob2_f32.argtypes = [i64, p]
    lib.or_frob2_f32.restype = d
    return lib


def _p(a: np.ndarray) -> int:
    assert a.flags.c_contiguous
    return a.ctypes.data


def _c(a, dtype):
    return np.ascontiguousarray(a, dtype=dtype)


# ----------------------------------------------------------------- primitives

def splitmix64(x: int) -> int:
    return int(_lib().or_splitmix64_pub(x))


def u0(n: int, k: int, seed: int = 0, init_nnz: int = 0) -> np.ndarray:
    """Initial guess U_0 (reading C10): dense uniform(0,1), fp32-exact.
    init_nnz > 0: each entry kept with probability init_nnz / n by a hash draw
    (reading C18; the nnz of U_0 varied in P:289-298)."""
    out = np.empty((n, k), np.float32)
    _lib().or_u0(n, k, seed, _p(out))
    if init_nnz > 0:
        _lib().or_u0_sparsify(n, k, seed, int(init_nnz), _p(out))
    return out


def gram(F: np.ndarray) -> np.ndarray:
    """F^T F in fp64."""
    F = _c(F, np.float64)
    rows, k = F.shape
    G = np.empty((k, k), np.float64)
    _lib().or_gram(rows, k, _p(F), _p(G))
    return G


def cholesky(G: np.ndarray, rho: float = RHO_DEFAULT):
    """L with L L^T = G + eps I, eps = rho (tr G / k + 1) (C6).
    Raises np.linalg.LinAlgError if not positive definite."""
    G = _c(G, np.float64)
    k = G.shape[0]
    L = np.empty((k, k), np.float64)
    eps = ctypes.c_double(0.0)
    rc = _lib().or_cholesky(k, _p(G), rho, _p(L), ctypes.byref(eps))
    if rc != 0:
        raise np.linalg.LinAlgError("G + eps I is not positive definite")
    return L, eps.value


def solve_rows(L: np.ndarray, Y: np.ndarray, out: np.ndarray | None = None) -> np.ndarray:
    """X = Y (L L^T)^{-1}, row by row (two triangular solves).  out=Y solves in
    place (each row's solve reads y_i before it writes x_i: or_solve_row)."""
    Y = _c(Y, np.float64)
    X = np.empty_like(Y) if out is None else out
    assert X.shape == Y.shape and X.dtype == np.float64 and X.flags.c_contiguous
    _lib().or_solve_rows(Y.shape[0], Y.shape[1], _p(_c(L, np.float64)), _p(Y), _p(X))
    return X


def solve_gram(G: np.ndarray, rho: float = RHO_DEFAULT) -> np.ndarray:
    """(G + eps I)^{-1} (SPEC solve_gram)."""
    L, _ = cholesky(G, rho)
    return solve_rows(L, np.eye(G.shape[0]))


def spmm(ptr, idx, val, F: np.ndarray) -> np.ndarray:
    """Y = T F with T in CSR (rows = output rows), F dense (P:63 A^T U, P:64 A V)."""
    F = _c(F, np.float64)
    rows_out = len(ptr) - 1
    k = F.shape[1]
    Y = np.empty((rows_out, k), np.float64)
    _lib().or_spmm(rows_out, k, _p(_c(ptr, np.int64)), _p(_c(idx, np.int32)), _p(_c(val, np.float32)), _p(F), _p(Y))
    return Y


def spmm_rows(sel, ptr, idx, val, F: np.ndarray) -> np.ndarray:
    """Rows ``sel`` of T F only (sampled parity at full size)."""
    F = _c(F, np.float64)
    sel = _c(sel, np.int64)
    Y = np.empty((len(sel), F.shape[1]), np.float64)
    _lib().or_spmm_rows(len(sel), _p(sel), F.shape[1], _p(_c(ptr, np.int64)), _p(_c(idx, np.int32)),
                        _p(_c(val, np.float32)), _p(F), _p(Y))
    return Y


def clamp_top_t(X: np.ndarray, t: int | None, whole: bool = False, inplace: bool = False):
    """Projection + enforcement (P:63 clamp; P:134,146 keep t largest).
    whole=False: per column (C4 ties -> lower row); returns (X', kept per column).
    whole=True: of the whole matrix, Alg. 2 as printed (C17 ties ->
    lower column, then row); returns (X', [kept total]).  inplace=True overwrites
    X (fp64, C order) instead of a copy."""
    if inplace:
        assert X.dtype == np.float64 and X.flags.c_contiguous
    else:
        X = np.array(X, dtype=np.float64, order="C", copy=True)
    rows, k = X.shape
    if whole:
        kept = np.empty(1, np.int64)
        _lib().or_clamp_top_t_whole(rows, k, -1 if t is None else int(t), _p(X), _p(kept))
        return X, kept
    kept = np.empty(k, np.int64)
    _lib().or_clamp_top_t(rows, k, -1 if t is None else int(t), _p(X), _p(kept))
    return X, kept


def residual(Unew: np.ndarray, Uold: np.ndarray) -> float:
    """R = ||U_i - U_{i-1}|| / ||U_i||.  ValueError if ||U_i|| = 0."""
    a, b = _c(Unew, np.float64), _c(Uold, np.float64)
    r = _lib().or_residual(a.shape[0], a.shape[1], _p(a), _p(b))
    if r < 0:
        raise ValueError("residual undefined: ||U_i||_F == 0")
    return float(r)


def error(U, AV, GU, GV, normA2: float) -> float:
    """E = ||A - U V^T||_F / ||A||_F via the trace identity (BJ:5)."""
    U, AV = _c(U, np.float64), _c(AV, np.float64)
    return float(_lib().or_error(U.shape[0], U.shape[1], _p(U), _p(AV), _p(_c(GU, np.float64)),
                                 _p(_c(GV, np.float64)), normA2))


def frob2(val) -> float:
    v = _c(val, np.float32)
    return float(_lib().or_frob2_f32(len(v), _p(v)))


# ------------------------------------------------------------------ the method

def half_step(ptr, idx, val, F: np.ndarray, t: int | None, rho: float = RHO_DEFAULT, whole: bool = False,
              lean: bool = False) -> dict:
    """One ALS half-step in the paper's order (P:133-134 for the V side with
    T = A^T and F = U; P:135-136 for the U side with T = A and F = V):
        G = F^T F; L L^T = G + eps I; Y = T F; LS = Y (G + eps I)^{-1};
        F' = keep_top_t_per_column(max(LS, 0)).
    All dense fp64.  peak = positives of LS (SPEC peak_nnz).  lean=True (memory
    only, the same operations in the same order): LS overwrites Y and F'
    overwrites LS in one buffer; Y and LS are not returned (the Box golden,
    whose 8M x 200 fp64 buffers would not fit three at a time)."""
    G = gram(F)
    L, eps = cholesky(G, rho)
    Y = spmm(ptr, idx, val, F)
    if lean:
        LS = solve_rows(L, Y, out=Y)
        peak = int(np.count_nonzero(LS > 0))
        Fn, kept = clamp_top_t(LS, t, whole, inplace=True)
        return dict(G=G, eps=eps, L=L, Y=None, LS=None, F=Fn, kept=kept, peak=peak)
    LS = solve_rows(L, Y)
    Fn, kept = clamp_top_t(LS, t, whole)
    return dict(G=G, eps=eps, L=L, Y=Y, LS=LS, F=Fn, kept=kept, peak=int(np.count_nonzero(LS > 0)))


_SAME = object()


def run(inp: dict, k: int, t: int | None, iters: int, seed: int = 0, rho: float = RHO_DEFAULT,
        U_init: np.ndarray | None = None, keep_states: bool = False, t_u=_SAME, t_v=_SAME,
        whole: bool = False, init_nnz: int = 0, lean: bool = False, on_record=None) -> dict:
    """Alg. 2 for ``iters`` iterations: per-column enforcement
    (BJ:5) or, whole=True, of the whole matrix (Alg. 2 as printed).
    t_u / t_v (default t; None = unlimited) are the separate budgets of P:124
    (U-only / V-only enforcement).  Returns the per-iteration records
    {it, R, E, nnz_u, nnz_v, dead_u, dead_v} (IterationRecord) and
    the final dense U, V.  lean=True: the V side in one buffer (half_step lean)
    and the previous V freed before the next V side -- memory only; on_record
    is called with each record as it is made (long runs)."""
    tu = t if t_u is _SAME else t_u
    tv = t if t_v is _SAME else t_v
    n, m = inp["n"], inp["m"]
    U = (u0(n, k, seed, init_nnz) if U_init is None else U_init).astype(np.float64)
    normA2 = frob2(inp["a_val"])
    recs, states = [], []
    V = hv = None
    for it in range(1, iters + 1):
        if lean:
            V = hv = None  # freed before the next V side's buffer is made
        hv = half_step(inp["at_ptr"], inp["at_col"], inp["at_val"], U, tv, rho, whole, lean)
        V = hv["F"]
        hu = half_step(inp["a_ptr"], inp["a_col"], inp["a_val"], V, tu, rho, whole)
        Un = hu["F"]
        R = residual(Un, U)
        GU = gram(Un)
        E = error(Un, hu["Y"], GU, hu["G"], normA2)
        recs.append(dict(it=it, R=R, E=E, nnz_u=int(np.count_nonzero(Un)), nnz_v=int(np.count_nonzero(V)),
                         dead_u=int(np.sum(~Un.any(axis=0))), dead_v=int(np.sum(~V.any(axis=0))),
                         peak_u=hu["peak"], peak_v=hv["peak"]))
        if on_record is not None:
            on_record(recs[-1])
        if keep_states:
            states.append(dict(U_prev=U, V=V, U=Un, LS_V=hv["LS"], LS_U=hu["LS"], G_U=hv["G"], G_V=hu["G"]))
        U = Un
    return dict(records=recs, U=U, V=V, states=states, normA2=normA2)


def seq_half_step(ptr, idx, val, F: np.ndarray, O1: np.ndarray, b0: int, k2: int, t: int | None,
                  rho: float = RHO_DEFAULT, whole: bool = False) -> dict:
    """One half-step of sequential ALS (Alg. 3) for the block columns
    [b0, b0 + k2), in the order of Eq. (7) / Eq. (8):
        V side (T = A^T, F = U, O1 = V_1):  V_2 = (A^T U_2 - V_1 U_1^T U_2)(U_2^T U_2)^{-1}
        U side (T = A,   F = V, O1 = U_1):  U_2 = (A V_2 - U_1 V_1^T V_2)(V_2^T V_2)^{-1}
    with F_1 = F[:, :b0] (converged topics), F_2 = F[:, b0:b0+k2], the ridge of
    reading C6 on the block Gram (reading C19), then clamp and keep t per column
    of the block (whole=True: t over the block, Alg. 3 step 2/4 as printed).
    Returns LS2 (rows x k2, before the clamp) and F2 (after)."""
    F = _c(F, np.float64)
    F1, F2 = F[:, :b0], np.ascontiguousarray(F[:, b0:b0 + k2])
    G22 = gram(F2)
    L, eps = cholesky(G22, rho)
    Y = spmm(ptr, idx, val, F2)                       # A^T U_2  /  A V_2
    if b0 > 0:
        Y = Y - _c(O1, np.float64) @ (F1.T @ F2)      # - V_1 (U_1^T U_2)  /  - U_1 (V_1^T V_2)
    LS2 = solve_rows(L, Y)                            # (.)(F_2^T F_2 + eps I)^{-1}
    F2n, kept = clamp_top_t(LS2, t, whole)
    return dict(G22=G22, eps=eps, Y=Y, LS2=LS2, F2=F2n, kept=kept, peak=int(np.sum(LS2 > 0)))


def run_sequential(inp: dict, k: int, k2: int, t: int | None, iters: int, seed: int = 0,
                   rho: float = RHO_DEFAULT, t_u=_SAME, t_v=_SAME, whole: bool = False,
                   init_nnz: int = 0) -> dict:
    """Sequential ALS NMF (Alg. 3): eta = k / k2 blocks of k2 topics;
    every block starts from U_2 = U_0 (n x k2; the same U_0 for every
    block), runs ``iters`` iterations ("do until convergence", fixed count as
    reading C12; the START block is Alg. 2 with U_0, which is this update with no
    converged topics), then is appended to U_1, V_1.  One record per
    iteration over the whole factors U = [U_1 U_2 0], V = [V_1 V_2 0]: R on the
    full U (the block's first iteration compares with [U_1 U_0 0]), E the true
    relative error of the current U V^T, peak = nnz(F_1) + positives of LS_2."""
    tu = t if t_u is _SAME else t_u
    tv = t if t_v is _SAME else t_v
    n, m = inp["n"], inp["m"]
    if k2 <= 0 or k % k2:
        raise ValueError("k must be a multiple of k2")
    U = np.zeros((n, k))
    V = np.zeros((m, k))
    U0 = u0(n, k2, seed, init_nnz).astype(np.float64)
    normA2 = frob2(inp["a_val"])
    recs = []
    for b in range(k // k2):
        b0 = b * k2
        U[:, b0:b0 + k2] = U0                                              # P:336 Set U_2 = U_0
        for _ in range(iters):
            Uprev = U.copy()
            hv = seq_half_step(inp["at_ptr"], inp["at_col"], inp["at_val"], U, V[:, :b0], b0, k2, tv, rho, whole)
            V[:, b0:b0 + k2] = hv["F2"]                                    # steps 1-2
            hu = seq_half_step(inp["a_ptr"], inp["a_col"], inp["a_val"], V, U[:, :b0], b0, k2, tu, rho, whole)
            U[:, b0:b0 + k2] = hu["F2"]                                    # steps 3-4
            R = residual(U, Uprev)                                         # P:160 on the whole U
            AV = spmm(inp["a_ptr"], inp["a_col"], inp["a_val"], V)
            E = error(U, AV, gram(U), gram(V), normA2)                     # P:161 on the whole U V^T
            recs.append(dict(it=len(recs) + 1, R=R, E=E, nnz_u=int(np.count_nonzero(U)),
                             nnz_v=int(np.count_nonzero(V)), dead_u=int(np.sum(~U.any(axis=0))),
                             dead_v=int(np.sum(~V.any(axis=0))),
                             peak_u=int(np.count_nonzero(U[:, :b0])) + hu["peak"],
                             peak_v=int(np.count_nonzero(V[:, :b0])) + hv["peak"], block=b))
    return dict(records=recs, U=U, V=V, normA2=normA2)


# ------------------------------------------------ NEXT-4: preprocessing, accuracy

def normalize_rows(inp: dict) -> dict:
    """P:153 "divide each row of the data matrix by the number of nonzero entries
    in that row": a_ij / nnz(row i of A), rounded to fp32 (the stored data type,
    reading C24).  Returns a copy of ``inp`` with a_val and at_val (column index =
    term) replaced."""
    ln = np.diff(np.asarray(inp["a_ptr"], np.int64)).astype(np.float32)
    out = dict(inp)
    out["a_val"] = np.asarray(inp["a_val"], np.float32) / np.repeat(ln, np.diff(inp["a_ptr"]))
    if inp.get("at_val") is not None:
        out["at_val"] = np.asarray(inp["at_val"], np.float32) / ln[np.asarray(inp["at_col"], np.int64)]
    return out


def topic_accuracy(V: np.ndarray, labels, n_journals: int) -> np.ndarray:
    """Eq. (3)-(4) per topic column c of V: the documents "belonging"
    to the topic are the nonzero entries of column c (n_D of them);
        Acc = (sum_{i<k} Jnl(i,k)) / (beta - alpha) - alpha / (beta - alpha),
        alpha = floor(n_D/n_J) (n_J (floor(n_D/n_J) - 1) / 2 + n_D mod n_J),
        beta = n_D (n_D - 1) / 2,
    and Acc = 1 for n_D <= 1.  The same-journal pair count is
    sum_j C(count_j, 2) over the topic's documents of journal j (the pairs
    grouped by journal); n_J = 1 gives beta = alpha: Acc = 1 (reading C25)."""
    labels = np.asarray(labels, np.int64)
    nJ = int(n_journals)
    acc = np.ones(V.shape[1])
    for c in range(V.shape[1]):
        docs = np.nonzero(V[:, c])[0]
        nD = len(docs)
        if nD <= 1:
            continue
        cnt = np.bincount(labels[docs], minlength=nJ).astype(np.int64)
        same = int(np.sum(cnt * (cnt - 1) // 2))
        q = nD // nJ
        alpha = q * (nJ * (q - 1) + 2 * (nD % nJ)) // 2   # an integer: the pairs of the most even spread
        beta = nD * (nD - 1) // 2
        acc[c] = 1.0 if beta == alpha else (same - alpha) / (beta - alpha)
    return acc


# ------------------------------------------------------------- format helpers

def dense_to_coo(F: np.ndarray):
    """Canonical column-major COO (ascending column, then row)."""
    rows, cols = np.nonzero(F.T)   # over F^T: first index = column of F
    return cols.astype(np.int32), rows.astype(np.int32), F[cols, rows]


def coo_to_dense(shape, row, col, val, dtype=np.float64) -> np.ndarray:
    F = np.zeros(shape, dtype)
    F[np.asarray(row, np.int64), np.asarray(col, np.int64)] = val
    return F
