"""oracle.bruteforce -- dense numpy twin of the oracle, for tiny inputs only.

TEST INFRASTRUCTURE ONLY.  Independent of ``esnmf_oracle.c``: it uses LAPACK
solves (numpy.linalg.solve / pinv) instead of the oracle's Cholesky, a stable
lexsort instead of qsort, and materialises A - U V^T instead of the trace
identity.  Its job is to pin the oracle (tests/test_oracle.py).
"""
from __future__ import annotations

import numpy as np


def dense(ptr, idx, val, ncols: int) -> np.ndarray:
    rows = len(ptr) - 1
    D = np.zeros((rows, ncols), np.float64)
    for r in range(rows):
        s, e = int(ptr[r]), int(ptr[r + 1])
        D[r, np.asarray(idx[s:e], np.int64)] = np.asarray(val[s:e], np.float64)
    return D


def ridge_eps(G: np.ndarray, rho: float) -> float:
    return rho * (np.trace(G) / G.shape[0] + 1.0)


def ls_step(T: np.ndarray, F: np.ndarray, rho: float) -> np.ndarray:
    """T F (F^T F + eps I)^{-1}: the least-squares solve of Alg. 1 step 1/2."""
    G = F.T @ F
    Gr = G + ridge_eps(G, rho) * np.eye(G.shape[0])
    return np.linalg.solve(Gr, (T @ F).T).T


def top_t_per_column(X: np.ndarray, t: int | None) -> np.ndarray:
    """clamp, then keep per column the t largest positives, ties -> lower row (C4, C5)."""
    Y = np.where(X > 0, X, 0.0)
    if t is None:
        return Y
    out = np.zeros_like(Y)
    rows = np.arange(Y.shape[0])
    for c in range(Y.shape[1]):
        pos = rows[Y[:, c] > 0]
        order = np.lexsort((pos, -Y[pos, c]))   # primary: value desc; secondary: row asc
        keep = pos[order[:t]]
        out[keep, c] = Y[keep, c]
    return out


def top_t_whole(X: np.ndarray, t: int | None) -> np.ndarray:
    """clamp, then keep the t largest positives of the whole matrix, ties -> lower
    column, then lower row (Alg. 2 as printed; reading C17)."""
    Y = np.where(X > 0, X, 0.0)
    if t is None:
        return Y
    r, c = np.nonzero(Y)
    order = np.lexsort((r, c, -Y[r, c]))   # primary value desc, then column, then row
    keep = order[:t]
    out = np.zeros_like(Y)
    out[r[keep], c[keep]] = Y[r[keep], c[keep]]
    return out


def projected_als(A: np.ndarray, U0: np.ndarray, t: int | None, iters: int, rho: float):
    """Alg. 2 (t given) / Alg. 1 (t None), per-column enforcement, dense."""
    U = U0.astype(np.float64)
    recs = []
    nA = np.linalg.norm(A)
    for _ in range(iters):
        V = top_t_per_column(ls_step(A.T, U, rho), t)
        Un = top_t_per_column(ls_step(A, V, rho), t)
        R = np.linalg.norm(Un - U) / np.linalg.norm(Un)
        E = np.linalg.norm(A - Un @ V.T) / nA
        recs.append((R, E))
        U = Un
    return U, V, recs


def projected_als_budgets(A: np.ndarray, U0: np.ndarray, t_u: int | None, t_v: int | None, iters: int,
                          rho: float, whole: bool):
    """Alg. 2 as printed with separate budgets and whole-matrix or
    per-column enforcement, dense."""
    top = top_t_whole if whole else top_t_per_column
    U = U0.astype(np.float64)
    recs = []
    nA = np.linalg.norm(A)
    for _ in range(iters):
        V = top(ls_step(A.T, U, rho), t_v)
        Un = top(ls_step(A, V, rho), t_u)
        recs.append((np.linalg.norm(Un - U) / np.linalg.norm(Un), np.linalg.norm(A - Un @ V.T) / nA))
        U = Un
    return U, V, recs


def sequential_als(A: np.ndarray, U0: np.ndarray, k: int, t_u: int | None, t_v: int | None, iters: int,
                   rho: float, whole: bool = False):
    """Alg. 3, dense: the block of k2 = U0.shape[1] topics found by
    Eq. (7) / (8) with the converged topics subtracted from A explicitly
    (A - U_1 V_1^T, materialised), every block from U_0.  Returns U, V and
    (R, E) per iteration over the whole factors."""
    top = top_t_whole if whole else top_t_per_column
    n, m = A.shape
    k2 = U0.shape[1]
    U, V = np.zeros((n, k)), np.zeros((m, k))
    nA = np.linalg.norm(A)
    recs = []
    for b0 in range(0, k, k2):
        U[:, b0:b0 + k2] = U0
        R1 = A - U[:, :b0] @ V[:, :b0].T           # the residual the new topics fit
        for _ in range(iters):
            Uprev = U.copy()
            V[:, b0:b0 + k2] = top(ls_step(R1.T, U[:, b0:b0 + k2], rho), t_v)
            U[:, b0:b0 + k2] = top(ls_step(R1, V[:, b0:b0 + k2], rho), t_u)
            recs.append((np.linalg.norm(U - Uprev) / np.linalg.norm(U), np.linalg.norm(A - U @ V.T) / nA))
    return U, V, recs


def topic_accuracy_pairs(V: np.ndarray, labels, n_journals: int) -> np.ndarray:
    """Eq. (3)-(4) with the double sum over document pairs written out (tiny only)."""
    acc = np.ones(V.shape[1])
    nJ = n_journals
    for c in range(V.shape[1]):
        docs = [j for j in range(V.shape[0]) if V[j, c] != 0]
        nD = len(docs)
        if nD <= 1:
            continue
        same = sum(1 for a in range(nD - 1) for b in range(a + 1, nD) if labels[docs[a]] == labels[docs[b]])
        alpha = (nD // nJ) * (nJ * ((nD // nJ) - 1) / 2 + nD % nJ)
        beta = nD * (nD - 1) / 2
        acc[c] = 1.0 if beta == alpha else same / (beta - alpha) - alpha / (beta - alpha)
    return acc
