"""GPU parity of sequential ALS (Alg. 3).

The GPU runs the k2-column pipeline on the current block and subtracts the
converged topics' term O_1 (H_1^T H_2) W_22 of Eq. (7) / (8) after the
product (csrc/k_seq.cuh); the converged columns sit in frozen factors.  Same
bar as tests/test_gpu_parity.py (reading C15): block LS 1e-5 column-relative against oracle.seq_half_step, supports
identical except near-ties, trajectories within 1e-3 relative in E.
"""
import numpy as np
import pytest

import oracle
import synth
from paper_1510_05237_b200 import ESNMF, ESNMF_SIDE_U, ESNMF_SIDE_V, ESNMFError
from parity import TRAJ_TOL, check_canonical, check_products, check_selection, check_topt_property, coo_dense

pytestmark = pytest.mark.gpu
TINY, MEDIUM = synth.CONFIGS["tiny"], synth.CONFIGS["medium"]


def factor(s, side, rows, k):
    r, c, v = s.get_U() if side == ESNMF_SIDE_U else s.get_V()
    check_canonical(r, c, k)
    return coo_dense((rows, k), r, c, v)


def seq_half_steps(s, g, cfg, k, k2, b0, t_u, t_v):
    """One V side and one U side of block b0 / k2 against oracle.seq_half_step."""
    for side in (ESNMF_SIDE_V, ESNMF_SIDE_U):
        U = factor(s, ESNMF_SIDE_U, cfg.n, k)
        V = factor(s, ESNMF_SIDE_V, cfg.m, k)
        if side == ESNMF_SIDE_V:
            ref = oracle.seq_half_step(g["at_ptr"], g["at_col"], g["at_val"], U, V[:, :b0], b0, k2, t_v)
            frozen, rows, t = V[:, :b0], cfg.m, t_v
        else:
            ref = oracle.seq_half_step(g["a_ptr"], g["a_col"], g["a_val"], V, U[:, :b0], b0, k2, t_u)
            frozen, rows, t = U[:, :b0], cfg.n, t_u
        s.half_step(side)
        _, ls = s.get_ls(side)
        assert ls.shape[1] == k2 == s.info()["ls_cols"]
        check_products(ls, ref["LS2"])
        out = factor(s, side, rows, k)
        assert np.array_equal(out[:, :b0], frozen)                 # converged topics untouched
        assert not out[:, b0 + k2:].any()                           # later blocks still empty
        check_selection(out[:, b0:b0 + k2], ref["F2"], ref["LS2"], t)
        check_topt_property(ls, out[:, b0:b0 + k2], t)


@pytest.mark.parametrize("k2,iters", [(1, 3), (2, 4), (5, 3)])
def test_tiny_sequential_trajectory(k2, iters):
    cfg = TINY
    g = synth.generate(cfg)
    nb = cfg.k // k2
    ref = oracle.run_sequential(g, cfg.k, k2, cfg.t, iters, seed=cfg.seed)
    s = ESNMF(cfg.n, cfg.m, cfg.k, cfg.t, g, seed=cfg.seed, seq_k2=k2, seq_iters=iters)
    s.iterate(nb * iters)
    recs = s.records()
    assert len(recs) == nb * iters == len(ref["records"])
    for a, b in zip(recs, ref["records"]):
        assert abs(a["E"] - b["E"]) <= TRAJ_TOL * b["E"], (a["it"], a["E"], b["E"])
        assert a["nnz_u"] == b["nnz_u"] and a["nnz_v"] == b["nnz_v"], a["it"]
        assert a["dead_u"] == b["dead_u"] and a["dead_v"] == b["dead_v"], a["it"]
        assert abs(a["R"] - b["R"]) <= 1e-3 * b["R"] + 1e-6, (a["it"], a["R"], b["R"])
        assert abs(a["peak_u"] - b["peak_u"]) <= 1e-4 * b["peak_u"] + 1
    # every column holds <= t entries and the schedule is complete
    U = factor(s, ESNMF_SIDE_U, cfg.n, cfg.k)
    assert np.all((U > 0).sum(axis=0) <= cfg.t)
    with pytest.raises(ESNMFError):
        s.iterate(1)


@pytest.mark.parametrize("k2", [1, 2, 5])
def test_tiny_sequential_half_steps_mid_block(k2):
    """Half-steps of block 1 and of the last block against the oracle's Eq. (7)/(8)."""
    cfg = TINY
    g = synth.generate(cfg)
    iters = 3
    s = ESNMF(cfg.n, cfg.m, cfg.k, cfg.t, g, seed=cfg.seed, seq_k2=k2, seq_iters=iters)
    s.iterate(iters + 1)                       # block 1, one iteration in
    seq_half_steps(s, g, cfg, cfg.k, k2, k2, cfg.t, cfg.t)
    last = cfg.k // k2 - 1
    s2 = ESNMF(cfg.n, cfg.m, cfg.k, cfg.t, g, seed=cfg.seed, seq_k2=k2, seq_iters=iters)
    s2.iterate(last * iters + 2)
    seq_half_steps(s2, g, cfg, cfg.k, k2, last * k2, cfg.t, cfg.t)


def test_single_block_equals_alg2():
    """k2 = k: Alg. 3 is Alg. 2 from U_0 -- same factors as the standard mode."""
    cfg = TINY
    g = synth.generate(cfg)
    a = ESNMF(cfg.n, cfg.m, cfg.k, cfg.t, g, seed=cfg.seed)
    b = ESNMF(cfg.n, cfg.m, cfg.k, cfg.t, g, seed=cfg.seed, seq_k2=cfg.k, seq_iters=6)
    a.iterate(6)
    b.iterate(6)
    for x, y in zip(a.records(), b.records()):
        assert x["nnz_u"] == y["nnz_u"] and x["nnz_v"] == y["nnz_v"]
        assert x["E"] == y["E"] and x["R"] == y["R"]          # no frozen columns: the same arithmetic
    for x, y in zip(a.get_U(), b.get_U()):
        assert np.array_equal(x, y)


@pytest.mark.parametrize("k2", [2, 5])
def test_sequential_whole_block_budgets(k2):
    """Alg. 3 steps 2 and 4 as printed: t_v / t_u over the whole block V_2 / U_2."""
    cfg = TINY
    g = synth.generate(cfg)
    ref = oracle.run_sequential(g, cfg.k, k2, None, 3, seed=cfg.seed, t_u=20 * k2, t_v=30 * k2, whole=True)
    s = ESNMF(cfg.n, cfg.m, cfg.k, None, g, seed=cfg.seed, seq_k2=k2, seq_iters=3, t_u=20 * k2, t_v=30 * k2,
              whole=True)
    s.iterate(cfg.k // k2 * 3)
    for a, b in zip(s.records(), ref["records"]):
        assert abs(a["E"] - b["E"]) <= TRAJ_TOL * b["E"], (a["it"], a["E"], b["E"])
        assert a["nnz_u"] == b["nnz_u"] and a["nnz_v"] == b["nnz_v"], a["it"]


def test_sequential_budgets_sparse_u0_and_whole_k2_1():
    cfg = TINY
    g = synth.generate(cfg)
    ref = oracle.run_sequential(g, cfg.k, 1, None, 3, seed=cfg.seed, t_u=30, t_v=None, init_nnz=300)
    s = ESNMF(cfg.n, cfg.m, cfg.k, None, g, seed=cfg.seed, seq_k2=1, seq_iters=3, t_u=30, t_v=None, init_nnz=300)
    s.iterate(cfg.k * 3)
    for a, b in zip(s.records(), ref["records"]):
        assert abs(a["E"] - b["E"]) <= TRAJ_TOL * b["E"]
        assert a["nnz_u"] == b["nnz_u"] and a["nnz_v"] == b["nnz_v"]
    # whole-matrix with k2 = 1 is the per-column selection of the one block column
    w = ESNMF(cfg.n, cfg.m, cfg.k, cfg.t, g, seed=cfg.seed, seq_k2=1, seq_iters=2, whole=True)
    c = ESNMF(cfg.n, cfg.m, cfg.k, cfg.t, g, seed=cfg.seed, seq_k2=1, seq_iters=2)
    w.iterate(5)
    c.iterate(5)
    assert [r["E"] for r in w.records()] == [r["E"] for r in c.records()]


def test_sequential_bad_options():
    g = synth.generate(TINY)
    for kw in (dict(seq_k2=3, seq_iters=2), dict(seq_k2=2, seq_iters=0), dict(seq_k2=-1, seq_iters=2),
               dict(seq_k2=2, seq_iters=2, U0=np.ones((TINY.n, TINY.k), np.float32))):
        with pytest.raises(ESNMFError):
            ESNMF(TINY.n, TINY.m, TINY.k, TINY.t, g, **kw)


def test_medium_sequential_half_steps():
    cfg = MEDIUM
    g = synth.generate(cfg)
    k2 = 10
    s = ESNMF(cfg.n, cfg.m, cfg.k, cfg.t, g, seed=cfg.seed, seq_k2=k2, seq_iters=2)
    s.iterate(2 * 2 + 1)                      # block 2, one iteration in
    seq_half_steps(s, g, cfg, cfg.k, k2, 2 * k2, cfg.t, cfg.t)
