"""GPU parity of SURVEY 8(f) NEXT-4: row normalisation of A and the
clustering accuracy of Eq. (3)-(4) on a planted-topic corpus with
journal labels (synth/planted.py stands in for the PubMed journals).
"""
import numpy as np
import pytest

import oracle
import synth
from synth.planted import planted_corpus
from paper_1510_05237_b200 import ESNMF, ESNMF_SIDE_U, ESNMF_SIDE_V, ESNMFError
from parity import TRAJ_TOL, check_canonical, check_products, check_selection, coo_dense

pytestmark = pytest.mark.gpu
TINY = synth.CONFIGS["tiny"]


def factor(s, side, rows, k):
    r, c, v = s.get_U() if side == ESNMF_SIDE_U else s.get_V()
    check_canonical(r, c, k)
    return coo_dense((rows, k), r, c, v)


@pytest.mark.parametrize("use_at", [True, False])
def test_row_normalised_trajectory_and_half_steps(use_at):
    """A row-normalised on the device (given A^T normalised by column, or A^T built
    from the normalised A) against the oracle on oracle.normalize_rows(A)."""
    cfg = TINY
    g = synth.generate(cfg)
    gn = oracle.normalize_rows(g)
    s = ESNMF(cfg.n, cfg.m, cfg.k, cfg.t, g, seed=cfg.seed, row_normalize=True, use_at=use_at)
    assert s.info()["normA2"] == pytest.approx(oracle.frob2(gn["a_val"]), rel=1e-12)
    ref = oracle.run(gn, cfg.k, cfg.t, cfg.iters, seed=cfg.seed)
    s.iterate(cfg.iters)
    for a, b in zip(s.records(), ref["records"]):
        assert abs(a["E"] - b["E"]) <= TRAJ_TOL * b["E"], (a["it"], a["E"], b["E"])
        assert a["nnz_u"] == b["nnz_u"] and a["nnz_v"] == b["nnz_v"]
    for side in (ESNMF_SIDE_V, ESNMF_SIDE_U):
        if side == ESNMF_SIDE_V:
            F, T, rows = factor(s, ESNMF_SIDE_U, cfg.n, cfg.k), ("at_ptr", "at_col", "at_val"), cfg.m
        else:
            F, T, rows = factor(s, ESNMF_SIDE_V, cfg.m, cfg.k), ("a_ptr", "a_col", "a_val"), cfg.n
        h = oracle.half_step(gn[T[0]], gn[T[1]], gn[T[2]], F, cfg.t)
        s.half_step(side)
        _, ls = s.get_ls(side)
        check_products(ls, h["LS"])
        check_selection(factor(s, side, rows, cfg.k), h["F"], h["LS"], cfg.t)


def small_corpus():
    return planted_corpus(n_terms=4000, n_docs=1500, n_journals=5, tokens=80, topic_terms=400, seed=7)


@pytest.mark.parametrize("seq,norm", [(False, True), (True, True), (False, False)])
def test_accuracy_matches_oracle(seq, norm):
    """esnmf_topic_accuracy on the GPU's V equals Eq. (3)-(4) evaluated by the oracle
    on the same V (exact integer counts), for Alg. 2 and for sequential ALS (k2 = 1,
    converged columns included); and the run itself tracks the oracle's."""
    g = small_corpus()
    k, t, iters = 5, 150, 30
    kw = dict(seq_k2=1, seq_iters=iters // 5) if seq else {}
    s = ESNMF(g["n"], g["m"], k, t, g, seed=1, row_normalize=norm, **kw)
    s.iterate(iters)
    V = factor(s, ESNMF_SIDE_V, g["m"], k)
    acc = s.topic_accuracy(g["labels"], g["n_journals"])
    ref_acc = oracle.topic_accuracy(V, g["labels"], g["n_journals"])
    assert np.allclose(acc, ref_acc, rtol=1e-12, atol=1e-12), (acc, ref_acc)
    gn = oracle.normalize_rows(g) if norm else g
    ref = (oracle.run_sequential(gn, k, 1, t, iters // 5, seed=1) if seq else oracle.run(gn, k, t, iters, seed=1))
    for a, b in zip(s.records(), ref["records"]):
        assert abs(a["E"] - b["E"]) <= TRAJ_TOL * b["E"], (a["it"], a["E"], b["E"])
    if not norm:  # raw counts: the planted journals are found (heuristic, as S:464)
        assert acc.min() > 0.9, acc


def test_accuracy_bad_labels():
    g = small_corpus()
    s = ESNMF(g["n"], g["m"], 5, 100, g, seed=1)
    s.iterate(1)
    bad = g["labels"].copy()
    bad[3] = 5
    with pytest.raises(ESNMFError):
        s.topic_accuracy(bad, 5)
