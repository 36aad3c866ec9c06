"""Pins for the fp64 oracle (oracle/), independent of the oracle itself.

Each test fixes the oracle against something other than its own formula:
published values (SPEC examples, the splitmix64 reference vector), closed
forms (planted exact factorisations, 2x2 inverses, k = 1 division), library
routines that implement a different algorithm (LAPACK solve / pinv, SVD,
stable lexsort, materialised norms), brute force on tiny inputs, and
invariants.  A dropped term, wrong sign / index or transposed operand in any
oracle function fails at least one of these.
"""
import numpy as np
import pytest

import oracle
from oracle import bruteforce as bf
import synth


def csr(D):
    D = np.asarray(D, np.float64)
    ptr, idx, val = [0], [], []
    for r in D:
        nz = np.nonzero(r)[0]
        idx += list(nz)
        val += list(r[nz])
        ptr.append(len(idx))
    return np.array(ptr, np.int64), np.array(idx, np.int32), np.array(val, np.float32)


def rand_sparse(rng, rows, cols, density, integer=False):
    M = (rng.random((rows, cols)) < density) * (rng.integers(1, 5, (rows, cols)) if integer else rng.lognormal(0, 1, (rows, cols)))
    return M.astype(np.float32).astype(np.float64)


# ------------------------------------------------------------ published values

def test_splitmix64_reference_vector():
    # splitmix64 seeded with 0: first three outputs of the reference generator
    assert oracle.splitmix64(0) == 0xE220A8397B1DCDAF
    assert oracle.splitmix64(0x9E3779B97F4A7C15) == 0x6E789E6AA1B965F4
    assert oracle.splitmix64((2 * 0x9E3779B97F4A7C15) % 2**64) == 0x06C45D188009454F


def test_u0_structure():
    U = oracle.u0(1000, 7, 0)
    assert U.dtype == np.float32 and U.shape == (1000, 7)
    assert U.min() > 0 and U.max() < 1
    s = U.astype(np.float64) * 2.0**24        # (2j+1) 2^-24: an odd integer
    assert np.all(s == np.round(s)) and np.all(np.round(s) % 2 == 1)
    assert abs(U.mean() - 0.5) < 0.02
    assert np.array_equal(U, oracle.u0(1000, 7, 0))
    assert not np.array_equal(U, oracle.u0(1000, 7, 1))
    # counter layout: element (i, c) depends on i*k + c only
    assert oracle.u0(10, 5, 3).ravel()[7] == oracle.u0(35, 1, 3)[7, 0]


def test_spec_gram_examples():
    assert np.array_equal(oracle.gram([[1, 2], [3, 4]]), [[10, 14], [14, 20]])
    assert np.array_equal(oracle.gram(np.eye(2)), np.eye(2))
    G = oracle.gram([[1, 0], [2, 0], [0, 0]])
    assert G[1].tolist() == [0, 0] and G[:, 1].tolist() == [0, 0]


def test_spec_solve_gram_examples():
    assert np.allclose(oracle.solve_gram(np.array([[10.0, 14], [14, 20]]), 0.0), [[5, -3.5], [-3.5, 2.5]], rtol=1e-12)
    assert np.allclose(oracle.solve_gram(np.diag([2.0, 4.0]), 0.0), np.diag([0.5, 0.25]), rtol=1e-15)
    assert np.array_equal(oracle.solve_gram(np.eye(3), 0.0), np.eye(3))
    # ridge reading C6: eps = rho (tr G / k + 1)
    _, eps = oracle.cholesky(np.diag([2.0, 4.0]), 1e-3)
    assert eps == pytest.approx(1e-3 * (3.0 + 1.0), rel=1e-15)
    with pytest.raises(np.linalg.LinAlgError):
        oracle.cholesky(np.zeros((2, 2)), 0.0)


def test_spec_matmul_example():
    ptr, idx, val = csr([[1, 2], [3, 4]])
    Y = oracle.spmm(ptr, idx, val, np.array([[5.0, 6], [7, 8]]))
    assert np.array_equal(Y, [[19, 22], [43, 50]])
    ptr, idx, val = csr(np.eye(3))
    F = np.arange(6.0).reshape(3, 2)
    assert np.array_equal(oracle.spmm(ptr, idx, val, F), F)


def test_spec_clamp_and_top_t_examples():
    X, kept = oracle.clamp_top_t(np.array([[1.0, -2], [-3, 4]]), None)
    assert np.array_equal(X, [[1, 0], [0, 4]]) and kept.tolist() == [1, 1]
    X2, _ = oracle.clamp_top_t(X, None)
    assert np.array_equal(X2, X)                                                       # idempotent
    col = np.array([[3.0], [2.0], [1.0], [0.5]])
    X, kept = oracle.clamp_top_t(col, 2)
    assert X[:, 0].tolist() == [3, 2, 0, 0] and kept[0] == 2
    X, _ = oracle.clamp_top_t(col, 10)
    assert np.array_equal(X, col)
    X, kept = oracle.clamp_top_t(col, 0)
    assert not X.any() and kept[0] == 0
    two = np.array([[5.0, 4], [1, 3], [0, 2]])
    X, _ = oracle.clamp_top_t(two, 1)
    assert X.tolist() == [[5, 4], [0, 0], [0, 0]]
    g = np.array([[9.0, 1], [8, 0.5], [7, 0.25], [6, 0.125]])
    X, kept = oracle.clamp_top_t(g, 2)
    assert kept.tolist() == [2, 2] and X[:, 0].tolist() == [9, 8, 0, 0] and X[:, 1].tolist() == [1, 0.5, 0, 0]


def test_spec_residual_examples():
    U = np.array([[1.0, 0], [2, 3]])
    assert oracle.residual(U, U) == 0.0
    assert oracle.residual(U, np.zeros_like(U)) == 1.0
    assert oracle.residual(U, 2 * U) == pytest.approx(1.0, rel=1e-15)
    with pytest.raises(ValueError):
        oracle.residual(np.zeros_like(U), U)


def test_spec_als_step_v_identity():
    ptr, idx, val = csr(np.diag([2.0, 3.0]))          # A^T = diag(2,3)
    h = oracle.half_step(ptr, idx, val, np.eye(2), None, rho=0.0)
    assert np.allclose(h["LS"], np.diag([2.0, 3.0]), rtol=1e-15)


# ---------------------------------------------------- closed forms / library

def test_gram_psd_and_against_numpy():
    rng = np.random.default_rng(0)
    F = rand_sparse(rng, 200, 9, 0.3)
    G = oracle.gram(F)
    assert np.allclose(G, F.T @ F, rtol=1e-13, atol=0)
    assert np.array_equal(G, G.T)
    assert np.linalg.eigvalsh(G).min() >= -1e-12 * np.trace(G)


def test_solve_matches_lapack_and_pinv():
    """V_ls = A^T pinv(U)^T for full-column-rank U (normal equations = pseudoinverse)."""
    rng = np.random.default_rng(1)
    A = rand_sparse(rng, 60, 40, 0.2)
    U = rand_sparse(rng, 60, 4, 0.5) + 0.01 * rng.random((60, 4))
    ptr, idx, val = csr(A.T)
    h = oracle.half_step(ptr, idx, val, U, None, rho=0.0)
    ref_pinv = A.T @ np.linalg.pinv(U).T
    assert np.allclose(h["LS"], ref_pinv, rtol=1e-9, atol=1e-9 * np.abs(ref_pinv).max())
    ref_solve = bf.ls_step(bf.dense(ptr, idx, val, 60), U, 0.0)
    assert np.allclose(h["LS"], ref_solve, rtol=1e-11, atol=1e-12 * np.abs(ref_solve).max())
    # with the ridge: LAPACK solve of (G + eps I)
    h2 = oracle.half_step(ptr, idx, val, U, None, rho=1e-3)
    ref2 = bf.ls_step(A.T, U, 1e-3)
    assert np.allclose(h2["LS"], ref2, rtol=1e-11, atol=1e-12 * np.abs(ref2).max())


def test_rank_one_is_a_division():
    """k = 1: (u^T u + eps)^{-1} is a scalar division."""
    rng = np.random.default_rng(2)
    A = rand_sparse(rng, 30, 20, 0.3)
    u = rng.random((30, 1)) + 0.1
    ptr, idx, val = csr(A.T)
    rho = 1e-6
    h = oracle.half_step(ptr, idx, val, u, None, rho=rho)
    g = float(u[:, 0] @ u[:, 0])
    ref = (A.T @ u[:, 0]) / (g + rho * (g + 1.0))
    assert np.allclose(h["LS"][:, 0], ref, rtol=1e-13)


def test_error_trace_identity_vs_materialised():
    rng = np.random.default_rng(3)
    A = rand_sparse(rng, 25, 18, 0.3)
    U = rand_sparse(rng, 25, 3, 0.5)
    V = rand_sparse(rng, 18, 3, 0.5)
    E = oracle.error(U, A @ V, U.T @ U, V.T @ V, float(np.sum(A * A)))
    ref = np.linalg.norm(A - U @ V.T) / np.linalg.norm(A)
    assert E == pytest.approx(ref, rel=1e-12)
    assert oracle.error(np.zeros_like(U), A @ np.zeros_like(V), np.zeros((3, 3)), np.zeros((3, 3)),
                        float(np.sum(A * A))) == pytest.approx(1.0, rel=1e-15)


def test_planted_exact_factorisation_is_a_fixed_point():
    """A = U* V*^T with sparse, non-negative, full-column-rank factors holding exactly
    t entries per column: one iteration from U = U* returns V*, U*, so E = R = 0."""
    rng = np.random.default_rng(4)
    n, m, k, t = 40, 30, 3, 6
    Us, Vs = np.zeros((n, k)), np.zeros((m, k))
    for c in range(k):
        Us[rng.choice(n, t, replace=False), c] = rng.integers(1, 5, t)
        Vs[rng.choice(m, t, replace=False), c] = rng.integers(1, 5, t)
    assert np.linalg.matrix_rank(Us) == k and np.linalg.matrix_rank(Vs) == k
    A = Us @ Vs.T                                   # small integers: exact in fp32
    p, i, v = csr(A)
    pt, it, vt = csr(A.T)
    inp = dict(n=n, m=m, a_ptr=p, a_col=i, a_val=v, at_ptr=pt, at_col=it, at_val=vt)
    r = oracle.run(inp, k, t, 1, U_init=Us)
    assert np.allclose(r["V"], Vs, rtol=1e-8, atol=0)
    assert np.allclose(r["U"], Us, rtol=1e-8, atol=0)
    assert np.array_equal(r["V"] != 0, Vs != 0) and np.array_equal(r["U"] != 0, Us != 0)
    assert r["records"][0]["E"] < 1e-7 and r["records"][0]["R"] < 1e-8


def test_planted_block_corpus_converges():
    """Heuristic convergence quorum: noise-free planted blocks, t >= the
    planted column support -> E <= 1e-3 within 200 iterations for >= 8/10 seeds."""
    k, terms, docs = 5, 10, 20
    n, m = k * terms, k * docs
    rng = np.random.default_rng(5)
    A = np.zeros((n, m))
    for c in range(k):
        A[c * terms:(c + 1) * terms, c * docs:(c + 1) * docs] = np.outer(rng.integers(1, 4, terms), rng.integers(1, 4, docs))
    p, i, v = csr(A)
    pt, it, vt = csr(A.T)
    inp = dict(n=n, m=m, a_ptr=p, a_col=i, a_val=v, at_ptr=pt, at_col=it, at_val=vt)
    ok = 0
    for seed in range(10):
        r = oracle.run(inp, k, docs, 200, seed=seed)
        ok += min(x["E"] for x in r["records"]) <= 1e-3
    assert ok >= 8


# ---------------------------------------------------------- brute force (tiny)

def test_top_t_invariants_and_ties():
    rng = np.random.default_rng(6)
    X = rng.normal(size=(300, 7))
    X[10:20, 3] = 0.75          # forced exact ties inside column 3
    X[:, 5] = -1.0              # all-negative column
    for t in (0, 1, 5, 13, 50, 299, 1000):
        Y, kept = oracle.clamp_top_t(X, t)
        ref = bf.top_t_per_column(X, t)
        assert np.array_equal(Y, ref)
        for c in range(X.shape[1]):
            pos = X[:, c] > 0
            assert kept[c] == min(t, pos.sum()) == np.count_nonzero(Y[:, c])
            kv, dv = Y[Y[:, c] > 0, c], X[pos & (Y[:, c] == 0), c]
            if len(kv) and len(dv):
                assert kv.min() >= dv.max()
        assert np.array_equal(oracle.clamp_top_t(Y, t)[0], Y)                           # idempotent
        assert np.all(Y >= 0)
    Y, _ = oracle.clamp_top_t(X, 15)   # ties at 0.75 resolved by lower row first
    col = X[:, 3]
    above = np.sum(col > 0.75)
    if 0 < 15 - above < 10:
        kept_rows = np.nonzero(Y[10:20, 3])[0]
        assert kept_rows.tolist() == list(range(15 - above))


@pytest.mark.parametrize("t", [None, 4, 9])
def test_oracle_run_matches_bruteforce(t):
    rng = np.random.default_rng(7)
    n, m, k = 40, 30, 3
    A = rand_sparse(rng, n, m, 0.25)
    p, i, v = csr(A)
    pt, it, vt = csr(A.T)
    inp = dict(n=n, m=m, a_ptr=p, a_col=i, a_val=v, at_ptr=pt, at_col=it, at_val=vt)
    rho = 1e-10
    r = oracle.run(inp, k, t, 8, seed=3, rho=rho)
    U0 = oracle.u0(n, k, 3)
    U, V, recs = bf.projected_als(A, U0, t, 8, rho)
    assert np.allclose(r["U"], U, rtol=1e-9, atol=1e-12 * np.abs(U).max())
    assert np.allclose(r["V"], V, rtol=1e-9, atol=1e-12 * np.abs(V).max())
    for rec, (R, E) in zip(r["records"], recs):
        assert rec["R"] == pytest.approx(R, rel=1e-8, abs=1e-12)
        assert rec["E"] == pytest.approx(E, rel=1e-10)
        if t is not None:
            assert rec["nnz_u"] <= k * t and rec["nnz_v"] <= k * t


@pytest.mark.parametrize("t", [None, 4])
def test_oracle_lean_mode_is_the_same_run(t):
    """run(lean=True) (the Box golden's memory mode: LS and the new factor
    overwrite Y in place) makes the same records and factors as the plain run,
    and on_record sees every record; pinned by the brute-force twin above."""
    rng = np.random.default_rng(8)
    n, m, k = 40, 30, 3
    A = rand_sparse(rng, n, m, 0.25)
    p, i, v = csr(A)
    pt, it, vt = csr(A.T)
    inp = dict(n=n, m=m, a_ptr=p, a_col=i, a_val=v, at_ptr=pt, at_col=it, at_val=vt)
    seen = []
    a = oracle.run(inp, k, t, 6, seed=3)
    b = oracle.run(inp, k, t, 6, seed=3, lean=True, on_record=seen.append)
    assert seen == b["records"]
    # (or_gram sums its per-thread partials in arrival order: equal to rounding)
    for F in ("U", "V"):
        assert np.array_equal(a[F] != 0, b[F] != 0)
        assert np.allclose(a[F], b[F], rtol=1e-12, atol=0)
    for x, y in zip(a["records"], b["records"]):
        assert {q: x[q] for q in x if q not in ("R", "E")} == {q: y[q] for q in y if q not in ("R", "E")}
        assert x["R"] == pytest.approx(y["R"], rel=1e-12) and x["E"] == pytest.approx(y["E"], rel=1e-12)
    U0 = oracle.u0(n, k, 3)
    U, V, _ = bf.projected_als(A, U0, t, 6, 1e-10)
    assert np.allclose(b["V"], V, rtol=1e-9, atol=1e-12 * np.abs(V).max())


def test_oracle_tiny_config_records_sane():
    cfg = synth.CONFIGS["tiny"]
    g = synth.generate(cfg)
    r = oracle.run(g, cfg.k, cfg.t, 5, seed=cfg.seed)
    for x in r["records"]:
        assert 0 <= x["E"] <= 1.0 + 1e-12
        assert x["nnz_u"] <= cfg.k * cfg.t and x["nnz_v"] <= cfg.k * cfg.t
    assert r["records"][0]["R"] > 0.5   # U_1 differs from the dense U_0
    assert r["records"][-1]["E"] < r["records"][0]["E"]


# ---- Alg. 2 as printed: whole-matrix enforcement, separate budgets (NEXT-1) ----

def test_whole_matrix_top_t_against_bruteforce_and_invariants():
    rng = np.random.default_rng(11)
    X = rng.normal(size=(200, 6))
    X[5:15, 2] = 0.5            # exact ties inside a column
    X[5:15, 4] = 0.5            # ... and across columns
    X[:, 1] = -1.0              # all-negative column
    npos = int(np.sum(X > 0))
    for t in (0, 1, 7, 40, 333, npos, npos + 10, None):
        Y, kept = oracle.clamp_top_t(X, t, whole=True)
        assert np.array_equal(Y, bf.top_t_whole(X, t))
        want = npos if t is None else min(t, npos)
        assert kept[0] == want == np.count_nonzero(Y)
        kv, dv = Y[Y > 0], X[(X > 0) & (Y == 0)]
        if len(kv) and len(dv):
            assert kv.min() >= dv.max()                       # nothing dropped beats a kept entry
        assert np.array_equal(oracle.clamp_top_t(Y, t, whole=True)[0], Y)   # idempotent
    # ties at 0.5: lower column first, then lower row
    above = int(np.sum(X > 0.5))
    t = above + 12
    Y, _ = oracle.clamp_top_t(X, t, whole=True)
    assert np.count_nonzero(Y[5:15, 2]) == 10 and np.count_nonzero(Y[5:15, 4]) == 2
    assert np.nonzero(Y[5:15, 4])[0].tolist() == [0, 1]


def test_whole_matrix_reduces_to_per_column_for_one_column():
    rng = np.random.default_rng(12)
    X = rng.normal(size=(500, 1))
    for t in (0, 3, 100, 499, None):
        assert np.array_equal(oracle.clamp_top_t(X, t, whole=True)[0], oracle.clamp_top_t(X, t)[0])


@pytest.mark.parametrize("t_u,t_v,whole", [(10, 25, True), (None, 6, False), (6, None, False), (15, None, True)])
def test_oracle_budgets_match_bruteforce(t_u, t_v, whole):
    """Separate t_u / t_v, U-only / V-only enforcement,
    whole-matrix (Alg. 2 as printed) against the dense numpy twin."""
    rng = np.random.default_rng(13)
    n, m, k = 40, 30, 3
    A = rand_sparse(rng, n, m, 0.25)
    p, i, v = csr(A)
    pt, it, vt = csr(A.T)
    inp = dict(n=n, m=m, a_ptr=p, a_col=i, a_val=v, at_ptr=pt, at_col=it, at_val=vt)
    rho = 1e-10
    r = oracle.run(inp, k, 999, 6, seed=5, rho=rho, t_u=t_u, t_v=t_v, whole=whole)
    U, V, recs = bf.projected_als_budgets(A, oracle.u0(n, k, 5), t_u, t_v, 6, rho, whole)
    assert np.allclose(r["U"], U, rtol=1e-9, atol=1e-12 * np.abs(U).max())
    assert np.allclose(r["V"], V, rtol=1e-9, atol=1e-12 * np.abs(V).max())
    for rec, (R, E) in zip(r["records"], recs):
        assert rec["E"] == pytest.approx(E, rel=1e-10)
        if whole and t_u is not None:
            assert rec["nnz_u"] <= t_u
        if whole and t_v is not None:
            assert rec["nnz_v"] <= t_v


def test_sparse_u0_mask():
    """Reading C18: init_nnz >= n keeps the dense U_0; otherwise only zeroes are
    introduced, each entry independently with probability init_nnz / n (binomial
    count per column), and the kept values are U_0's."""
    n, k = 4000, 6
    dense = oracle.u0(n, k, 3)
    assert np.array_equal(oracle.u0(n, k, 3, n), dense)
    assert np.array_equal(oracle.u0(n, k, 3, 10 * n), dense)
    for nnz in (10, 200, 1000):
        s = oracle.u0(n, k, 3, nnz)
        kept = s != 0
        assert np.array_equal(s[kept], dense[kept])
        p = nnz / n
        cnt = kept.sum(axis=0)
        sd = np.sqrt(n * p * (1 - p))
        assert np.all(np.abs(cnt - nnz) <= 5 * sd + 1), (nnz, cnt)
    # independent of the value stream: the same mask for another seed differs
    assert not np.array_equal(oracle.u0(n, k, 3, 200) != 0, oracle.u0(n, k, 4, 200) != 0)


# ---- NEXT-2: sequential ALS (Alg. 3) ----

def _inp(A):
    p, i, v = csr(A)
    pt, it, vt = csr(A.T)
    return dict(n=A.shape[0], m=A.shape[1], a_ptr=p, a_col=i, a_val=v, at_ptr=pt, at_col=it, at_val=vt)


@pytest.mark.parametrize("k,k2,t_u,t_v,whole", [(4, 1, 8, 10, False), (6, 2, None, 7, False), (6, 3, 9, 12, False),
                                                 (4, 2, 15, 18, True)])
def test_sequential_matches_bruteforce(k, k2, t_u, t_v, whole):
    """Eq. (7)/(8) with the deflation term against the dense twin that fits the
    materialised residual A - U_1 V_1^T (a dropped term, a wrong sign or a
    transposed U_1^T U_2 fails here)."""
    rng = np.random.default_rng(21)
    n, m = 40, 30
    A = rand_sparse(rng, n, m, 0.3)
    rho = 1e-10
    r = oracle.run_sequential(_inp(A), k, k2, 999, 5, seed=2, rho=rho, t_u=t_u, t_v=t_v, whole=whole)
    U, V, recs = bf.sequential_als(A, oracle.u0(n, k2, 2).astype(np.float64), k, t_u, t_v, 5, rho, whole)
    assert np.allclose(r["U"], U, rtol=1e-8, atol=1e-11 * np.abs(U).max())
    assert np.allclose(r["V"], V, rtol=1e-8, atol=1e-11 * np.abs(V).max())
    assert len(r["records"]) == len(recs) == 5 * (k // k2)
    for rec, (R, E) in zip(r["records"], recs):
        assert rec["R"] == pytest.approx(R, rel=1e-7, abs=1e-12)
        assert rec["E"] == pytest.approx(E, rel=1e-9)


def test_sequential_single_block_is_alg2():
    """eta = 1 (k2 = k): Alg. 3 is its START step, i.e. Alg. 2 from U_0."""
    cfg = synth.CONFIGS["tiny"]
    g = synth.generate(cfg)
    a = oracle.run(g, cfg.k, cfg.t, 4, seed=cfg.seed)
    b = oracle.run_sequential(g, cfg.k, cfg.k, cfg.t, 4, seed=cfg.seed)
    assert np.allclose(a["U"], b["U"], rtol=1e-12, atol=0) and np.allclose(a["V"], b["V"], rtol=1e-12, atol=0)
    for x, y in zip(a["records"], b["records"]):
        assert x["nnz_u"] == y["nnz_u"] and x["nnz_v"] == y["nnz_v"] and x["peak_u"] == y["peak_u"]
        assert x["E"] == pytest.approx(y["E"], rel=1e-10) and x["R"] == pytest.approx(y["R"], rel=1e-10)


def test_sequential_one_topic_is_a_division():
    """k2 = 1: (U_2^T U_2)^{-1} is a scalar: the V side is
    (A^T u - V_1 (U_1^T u)) / (u^T u + eps), written out by hand."""
    rng = np.random.default_rng(22)
    n, m = 30, 25
    A = rand_sparse(rng, n, m, 0.3)
    inp = _inp(A)
    U = rng.random((n, 3))
    V1 = rng.random((m, 2))
    h = oracle.seq_half_step(inp["at_ptr"], inp["at_col"], inp["at_val"], U, V1, 2, 1, None, rho=0.0)
    u = U[:, 2]
    want = (A.T @ u - V1 @ (U[:, :2].T @ u)) / (u @ u)
    assert np.allclose(h["LS2"][:, 0], want, rtol=1e-12, atol=1e-12)
    assert np.array_equal(h["F2"][:, 0], np.maximum(h["LS2"][:, 0], 0))


def test_sequential_planted_disjoint_topics_recovered():
    """A = sum of k rank-one blocks with disjoint supports and distinct scales:
    sequential rank-one ALS finds them one by one (power iteration on the
    deflated residual), so the final error is ~0 and every U column is
    supported on one planted block (t = the block's size)."""
    k, terms, docs = 3, 8, 10
    n, m = k * terms, k * docs
    rng = np.random.default_rng(23)
    A = np.zeros((n, m))
    for c, s in enumerate((8.0, 4.0, 2.0)):
        A[c * terms:(c + 1) * terms, c * docs:(c + 1) * docs] = s * np.outer(rng.integers(1, 4, terms),
                                                                                rng.integers(1, 4, docs))
    r = oracle.run_sequential(_inp(A), k, 1, None, 30, seed=1, t_u=terms, t_v=docs)
    assert r["records"][-1]["E"] < 1e-6
    u = oracle.run_sequential(_inp(A), k, 1, None, 30, seed=1)          # unlimited: same fit, up to decayed leakage
    assert np.abs(u["U"] @ u["V"].T - A).max() <= 1e-6 * A.max()
    for c in range(k):
        blocks = {i // terms for i in np.nonzero(r["U"][:, c])[0]}
        assert blocks == {c}    # largest block first (the top singular pair of the residual)
    # the error drops as each block is appended
    E = [x["E"] for x in r["records"]]
    assert E[29] > E[59] > E[89]


# ---- NEXT-4: row normalisation, clustering accuracy Eq. (3)-(4) ----

def test_normalize_rows_divides_by_row_nnz():
    A = np.array([[2.0, 0, 4.0], [0, 3.0, 0], [0, 0, 0], [1.0, 1.0, 1.0]])
    inp = _inp(A)
    out = oracle.normalize_rows(inp)
    want = np.array([[1.0, 0, 2.0], [0, 3.0, 0], [0, 0, 0], [1 / 3, 1 / 3, 1 / 3]], np.float32)
    D = bf.dense(out["a_ptr"], out["a_col"], out["a_val"], 3)
    assert np.array_equal(D.astype(np.float32), want)
    Dt = bf.dense(out["at_ptr"], out["at_col"], out["at_val"], 4)
    assert np.array_equal(Dt.T, D)                       # A^T normalised by the same (term) rows


def test_accuracy_closed_cases():
    """1 when all of a topic's documents share a journal, 0 when they are spread as
    evenly as possible (alpha), 1 for <= 1 document."""
    nJ = 5
    labels = np.arange(40) % nJ                         # doc j in journal j mod 5
    V = np.zeros((40, 5))
    V[[0, 5, 10, 15], 0] = 1                            # all journal 0
    V[:10, 1] = 1                                       # 2 per journal: uniform
    V[:7, 2] = 1                                        # counts (2,2,1,1,1): most even for 7
    V[3, 3] = 1                                         # one document
    acc = oracle.topic_accuracy(V, labels, nJ)
    assert acc[0] == 1.0 and acc[1] == 0.0 and acc[2] == 0.0 and acc[3] == 1.0 and acc[4] == 1.0
    V2 = np.zeros((40, 1))
    V2[[0, 5, 1], 0] = 1                                # 1 same pair of 3; alpha = 0, beta = 3
    assert oracle.topic_accuracy(V2, labels, nJ)[0] == pytest.approx(1 / 3)


def test_accuracy_against_pair_loops():
    rng = np.random.default_rng(31)
    for nJ in (2, 3, 5):
        labels = rng.integers(0, nJ, 60)
        V = (rng.random((60, 6)) < 0.3) * rng.random((60, 6))
        assert np.allclose(oracle.topic_accuracy(V, labels, nJ), bf.topic_accuracy_pairs(V, labels, nJ),
                           rtol=1e-12, atol=1e-12)


def test_planted_corpus_shape_and_labels():
    from synth.planted import planted_corpus
    g = planted_corpus(n_terms=3000, n_docs=600, n_journals=5, tokens=60, topic_terms=300, seed=4)
    assert np.bincount(g["labels"]).tolist() == [120] * 5
    A = bf.dense(g["a_ptr"], g["a_col"], g["a_val"], 600)
    assert np.array_equal(A.T, bf.dense(g["at_ptr"], g["at_col"], g["at_val"], 3000))
    assert np.all(A.sum(axis=1)[A.sum(axis=1) > 0] >= 2)     # no term occurring once
    assert np.all(A == np.round(A)) and A.min() >= 0         # occurrence counts
