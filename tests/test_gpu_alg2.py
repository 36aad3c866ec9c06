"""GPU parity of Alg. 2 as printed: whole-factor enforcement
(`whole=True`, reading C17) and the separate budgets t_u / t_v of P:124,
including U-only / V-only enforcement -- SURVEY 8(f) NEXT-1.

Same bar as tests/test_gpu_parity.py (reading C15): LS products 1e-5
column-relative, kept entries 1e-5 relative, supports identical except
near-ties, trajectories within 1e-3 relative in E.
"""
import numpy as np
import pytest

import oracle
import synth
from paper_1510_05237_b200 import ESNMF, ESNMF_SIDE_U, ESNMF_SIDE_V, ESNMFError
from parity import PROD_TOL, TIE_TOL, TRAJ_TOL, check_canonical, check_products, coo_dense

pytestmark = pytest.mark.gpu
TINY, MEDIUM = synth.CONFIGS["tiny"], synth.CONFIGS["medium"]


def check_whole_selection(gpu_F, ref_F, ref_ls, t):
    """Whole-factor top-t: same count, kept values match, support differences only
    between near-ties of the global threshold."""
    assert np.all(gpu_F >= 0)
    g, r = gpu_F > 0, ref_F > 0
    assert g.sum() == r.sum(), (g.sum(), r.sum())
    if t is not None:
        assert g.sum() <= t
    scale = max(np.abs(ref_ls).max(), 1e-300)
    only_g, only_r = g & ~r, r & ~g
    if only_g.any():
        thr = ref_F[r].min()
        assert np.all(np.abs(ref_ls[only_g] - thr) <= TIE_TOL * scale)
        assert np.all(np.abs(ref_ls[only_r] - thr) <= TIE_TOL * scale)
    both = g & r   # entries: 1e-5 relative + 1e-6 of the factor's scale (near-zero keeps, reading C15)
    assert np.all(np.abs(gpu_F[both] - ref_F[both]) <= 1e-5 * np.abs(ref_F[both]) + TIE_TOL * scale)


def factor(s, side, rows, k):
    r, c, v = s.get_U() if side == ESNMF_SIDE_U else s.get_V()
    check_canonical(r, c, k)
    return coo_dense((rows, k), r, c, v)


def half_steps(s, g, cfg, k, t_u, t_v, whole):
    for side in (ESNMF_SIDE_V, ESNMF_SIDE_U):
        if side == ESNMF_SIDE_V:
            F, T, rows, t = factor(s, ESNMF_SIDE_U, cfg.n, k), ("at_ptr", "at_col", "at_val"), cfg.m, t_v
        else:
            F, T, rows, t = factor(s, ESNMF_SIDE_V, cfg.m, k), ("a_ptr", "a_col", "a_val"), cfg.n, t_u
        ref = oracle.half_step(g[T[0]], g[T[1]], g[T[2]], F, t, whole=whole)
        s.half_step(side)
        _, ls = s.get_ls(side)
        check_products(ls, ref["LS"])
        out = factor(s, side, rows, k)
        if whole:
            check_whole_selection(out, ref["F"], ref["LS"], t)
        else:
            assert np.array_equal((out > 0).sum(axis=0), (ref["F"] > 0).sum(axis=0))


CASES = [
    # (t_u, t_v, whole)
    (300, 400, True),       # Alg. 2 as printed, separate budgets
    (None, 450, True),      # V-only, whole factor
    (50, None, False),      # U-only, per column
    (None, 50, False),      # V-only, per column
    (20, 35, False),        # separate per-column budgets
]


@pytest.mark.parametrize("t_u,t_v,whole", CASES)
def test_tiny_trajectory_and_half_steps(t_u, t_v, whole):
    cfg = TINY
    g = synth.generate(cfg)
    ref = oracle.run(g, cfg.k, cfg.t, cfg.iters, seed=cfg.seed, t_u=t_u, t_v=t_v, whole=whole)
    s = ESNMF(cfg.n, cfg.m, cfg.k, cfg.t, g, seed=cfg.seed, t_u=t_u, t_v=t_v, whole=whole)
    s.iterate(cfg.iters)
    recs = s.records()
    for a, b in zip(recs, ref["records"]):
        assert abs(a["E"] - b["E"]) <= TRAJ_TOL * b["E"], (a["it"], a["E"], b["E"])
        assert a["nnz_u"] == b["nnz_u"] and a["nnz_v"] == b["nnz_v"], a["it"]
    if whole:
        if t_u is not None:
            assert all(r["nnz_u"] <= t_u for r in recs)
        if t_v is not None:
            assert all(r["nnz_v"] <= t_v for r in recs)
    half_steps(s, g, cfg, cfg.k, t_u, t_v, whole)


def test_medium_whole_matrix_half_steps():
    cfg = MEDIUM
    g = synth.generate(cfg)
    s = ESNMF(cfg.n, cfg.m, cfg.k, cfg.t, g, seed=cfg.seed, t_u=cfg.k * 300, t_v=cfg.k * 500, whole=True)
    s.iterate(4)
    half_steps(s, g, cfg, cfg.k, cfg.k * 300, cfg.k * 500, True)


def test_whole_matrix_large_budget_uses_three_pass_select():
    """t > 8192 (kSelFastT): the exact multi-pass selection over the flat factor."""
    cfg = MEDIUM
    g = synth.generate(cfg)
    s = ESNMF(cfg.n, cfg.m, cfg.k, cfg.t, g, seed=cfg.seed, t_u=20000, t_v=30000, whole=True)
    s.iterate(2)
    half_steps(s, g, cfg, cfg.k, 20000, 30000, True)


def test_bad_budgets_rejected():
    g = synth.generate(TINY)
    with pytest.raises(ESNMFError):
        ESNMF(TINY.n, TINY.m, TINY.k, TINY.t, g, t_u=-5)


# ---- NEXT-3: enforce-after, sparse initial guess, peak nnz telemetry ----

@pytest.mark.parametrize("whole", [False, True])
def test_enforce_after_truncation(whole):
    """Alg. 1 (t unlimited) then one truncation of U and V: the
    factors equal the oracle's truncation of the same (GPU) factors."""
    cfg = TINY
    g = synth.generate(cfg)
    s = ESNMF(cfg.n, cfg.m, cfg.k, None, g, seed=cfg.seed)
    s.iterate(5)
    U = factor(s, ESNMF_SIDE_U, cfg.n, cfg.k)
    V = factor(s, ESNMF_SIDE_V, cfg.m, cfg.k)
    t = 300 if whole else 40
    s.truncate(ESNMF_SIDE_U, t, whole)
    s.truncate(ESNMF_SIDE_V, t, whole)
    Ut = factor(s, ESNMF_SIDE_U, cfg.n, cfg.k)
    Vt = factor(s, ESNMF_SIDE_V, cfg.m, cfg.k)
    assert np.array_equal(Ut, oracle.clamp_top_t(U, t, whole)[0])   # same values in, exact selection out
    assert np.array_equal(Vt, oracle.clamp_top_t(V, t, whole)[0])
    # the truncated state iterates on (the next V side starts from the truncated U)
    s.half_step(ESNMF_SIDE_V)
    ref = oracle.half_step(g["at_ptr"], g["at_col"], g["at_val"], Ut, None)
    _, ls = s.get_ls(ESNMF_SIDE_V)
    check_products(ls, ref["LS"])


@pytest.mark.parametrize("init_nnz", [50, 400])
def test_sparse_initial_guess_and_peak_nnz(init_nnz):
    """U_0 with ~init_nnz entries per column (reading C18) bitwise equal to the
    oracle's, the trajectory from it, and the records' peak nnz (positives of the
    clamped least-squares factor before truncation)."""
    cfg = TINY
    g = synth.generate(cfg)
    s = ESNMF(cfg.n, cfg.m, cfg.k, cfg.t, g, seed=cfg.seed, init_nnz=init_nnz)
    U0 = factor(s, ESNMF_SIDE_U, cfg.n, cfg.k)
    ref0 = oracle.u0(cfg.n, cfg.k, cfg.seed, init_nnz)
    assert np.array_equal(U0.astype(np.float32), ref0)
    assert abs(np.count_nonzero(U0) / cfg.k - init_nnz) < 5 * np.sqrt(init_nnz) + 5
    ref = oracle.run(g, cfg.k, cfg.t, 8, seed=cfg.seed, init_nnz=init_nnz)
    s.iterate(8)
    for a, b in zip(s.records(), ref["records"]):
        assert abs(a["E"] - b["E"]) <= TRAJ_TOL * b["E"], (a["it"], a["E"], b["E"])
        assert a["nnz_u"] == b["nnz_u"] and a["nnz_v"] == b["nnz_v"]
        # a positive near zero may flip sign with rounding: allow 1e-4 relative
        assert abs(a["peak_u"] - b["peak_u"]) <= 1e-4 * b["peak_u"] + 1
        assert abs(a["peak_v"] - b["peak_v"]) <= 1e-4 * b["peak_v"] + 1


@pytest.mark.parametrize("whole,t", [(True, 3000), (True, 200_000), (False, 6000), (False, 9000), (False, 300)])
def test_selection_with_huge_tie_buckets(whole, t):
    """Three distinct values only: the threshold bucket holds far more than the
    4,096 keys sorted on chip, so the exact multi-block radix levels (value,
    then row bits) decide K*; the result is the oracle's selection exactly
    (ties -> lower column, then row; per column -> lower row, readings C4 / C17)."""
    cfg = MEDIUM
    g = synth.generate(cfg)
    k = 20
    s = ESNMF(cfg.n, cfg.m, k, cfg.t, g, seed=cfg.seed)
    rng = np.random.default_rng(5)
    U = (rng.random((cfg.n, k)) < 0.3) * rng.choice(np.float32([0.25, 0.5, 1.0]), size=(cfg.n, k))
    r, c = np.nonzero(U.T)                        # canonical: column, then row
    s.set_factor(ESNMF_SIDE_U, c.astype(np.int32), r.astype(np.int32), U[c, r].astype(np.float32))
    s.truncate(ESNMF_SIDE_U, t, whole)
    got = factor(s, ESNMF_SIDE_U, cfg.n, k)
    assert np.array_equal(got, oracle.clamp_top_t(U.astype(np.float64), t, whole)[0])
