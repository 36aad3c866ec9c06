"""GPU parity of the V-side tensor-core head (csrc/k_vhead.cuh).

The V-side product A^T Z is split by term: the `head_terms` most frequent terms
run as a dense fp16-split GEMM on tcgen05, the rest as the sparse row gather.
The split changes only the summation order, so every check here is the same
oracle parity as tests/test_gpu_parity.py (reading C15: products 1e-5
column-relative, near-tie-only support differences), for several head sizes,
plus head-on versus head-off agreement on the same state.
"""
import numpy as np
import pytest

import oracle
import synth
from paper_1510_05237_b200 import ESNMF, ESNMF_SIDE_U, ESNMF_SIDE_V
from parity import PROD_TOL, check_canonical, check_products, check_selection, check_topt_property, coo_dense

pytestmark = pytest.mark.gpu
TINY, MEDIUM = synth.CONFIGS["tiny"], synth.CONFIGS["medium"]


def dense(s, side, rows, k):
    r, c, v = s.get_U() if side == ESNMF_SIDE_U else s.get_V()
    check_canonical(r, c, k)
    return coo_dense((rows, k), r, c, v)


def v_side_parity(s, g, cfg, k, t):
    F = dense(s, ESNMF_SIDE_U, cfg.n, k)
    ref = oracle.half_step(g["at_ptr"], g["at_col"], g["at_val"], F, t)
    s.half_step(ESNMF_SIDE_V)
    _, ls = s.get_ls(ESNMF_SIDE_V)
    out = dense(s, ESNMF_SIDE_V, cfg.m, k)
    err = check_products(ls, ref["LS"])
    check_selection(out, ref["F"], ref["LS"], t)
    check_topt_property(ls, out, t)
    return err


@pytest.mark.parametrize("head,dense", [(64, 0), (64, 1), (192, 4), (1024, 2), (1024, 0), (1984, 0)])
def test_tiny_head_sizes_first_and_late(head, dense, monkeypatch):
    """dense = chunks stored as dense tiles (the rest built on chip from entry runs)."""
    monkeypatch.setenv("ESNMF_HEAD_DENSE", str(dense))
    g = synth.generate(TINY)
    s = ESNMF(TINY.n, TINY.m, TINY.k, TINY.t, g, seed=TINY.seed, head_terms=head)
    assert s.info()["head_terms"] == head
    v_side_parity(s, g, TINY, TINY.k, TINY.t)      # from dense U0
    s.half_step(ESNMF_SIDE_U)
    s.iterate(5)
    v_side_parity(s, g, TINY, TINY.k, TINY.t)      # from a sparse late U


@pytest.mark.parametrize("k", [1, 16, 33, 100, 200, 256])
def test_tiny_head_odd_ranks(k):
    """kn = k rounded up to 16: padding columns of the MMA must not leak."""
    g = synth.generate(TINY)
    s = ESNMF(TINY.n, TINY.m, k, 37, g, seed=TINY.seed, head_terms=128)
    v_side_parity(s, g, TINY, k, 37)
    s.half_step(ESNMF_SIDE_U)
    v_side_parity(s, g, TINY, k, 37)


def test_medium_auto_head_late_state():
    g = synth.generate(MEDIUM)
    s = ESNMF(MEDIUM.n, MEDIUM.m, MEDIUM.k, MEDIUM.t, g, seed=MEDIUM.seed)
    assert s.info()["head_terms"] >= 64
    s.iterate(4)
    err = v_side_parity(s, g, MEDIUM, MEDIUM.k, MEDIUM.t)
    assert err < PROD_TOL


def test_head_on_off_agree():
    """Same state, head on vs off: LS within fp32 rounding, identical trajectory."""
    g = synth.generate(MEDIUM)
    a = ESNMF(MEDIUM.n, MEDIUM.m, MEDIUM.k, MEDIUM.t, g, seed=MEDIUM.seed, head_terms=512)
    b = ESNMF(MEDIUM.n, MEDIUM.m, MEDIUM.k, MEDIUM.t, g, seed=MEDIUM.seed, head_terms=0)
    assert b.info()["head_terms"] == 0
    a.iterate(3)
    b.iterate(3)
    ea = [r["E"] for r in a.records()]
    eb = [r["E"] for r in b.records()]
    assert np.allclose(ea, eb, rtol=1e-6, atol=0)
    # same U in both, then one V side each
    r, c, v = a.get_U()
    b.set_factor(ESNMF_SIDE_U, r, c, v)
    a.half_step(ESNMF_SIDE_V)
    b.half_step(ESNMF_SIDE_V)
    _, la = a.get_ls(ESNMF_SIDE_V)
    _, lb = b.get_ls(ESNMF_SIDE_V)
    check_products(la, lb.astype(np.float64), tol=5e-6)


def test_head_deterministic():
    g = synth.generate(TINY)
    outs = []
    for _ in range(2):
        s = ESNMF(TINY.n, TINY.m, TINY.k, TINY.t, g, seed=TINY.seed, head_terms=192, keep_ls=True)
        s.iterate(4)
        _, ls = s.get_ls(ESNMF_SIDE_V)
        outs.append((ls, s.get_U()))
    assert np.array_equal(outs[0][0], outs[1][0])
    for x, y in zip(outs[0][1], outs[1][1]):
        assert np.array_equal(x, y)


def test_deferred_ls_buffer_same_run(monkeypatch):
    """esnmf_iterate without keep_ls: the head kernel's epilogue selects from its
    candidates and writes no LS buffer; the buffer is written by a gated re-run of
    the head only when a column's predicted threshold fails (iteration 1 always:
    no prediction yet; graph replays later).  The run is bitwise the run that
    writes the buffer every time, and esnmf_get_ls(V) refuses the stale buffer."""
    monkeypatch.setenv("ESNMF_PRED_MIN_ROWS", "1")  # the predicted path at Medium's size
    g = synth.generate(MEDIUM)
    runs = []
    for keep in (False, True):
        s = ESNMF(MEDIUM.n, MEDIUM.m, MEDIUM.k, MEDIUM.t, g, seed=MEDIUM.seed, keep_ls=keep)
        s.iterate(8)
        if keep:
            s.get_ls(ESNMF_SIDE_V)
        else:
            with pytest.raises(RuntimeError, match="keep_ls"):
                s.get_ls(ESNMF_SIDE_V)
        s.get_ls(ESNMF_SIDE_U)  # the U side's buffer is always written (E reads it)
        runs.append((s.records(), s.get_U(), s.get_V()))
        s.half_step(ESNMF_SIDE_V)  # explicit half-steps always write it
        s.get_ls(ESNMF_SIDE_V)
        s.close()
    assert runs[0][0] == runs[1][0]
    for x, y in zip(runs[0][1] + runs[0][2], runs[1][1] + runs[1][2]):
        assert np.array_equal(x, y)


def test_large_k_paths_medium():
    """k = 200 (Box's rank): 2-float4-per-lane tail gather, kn = 208 MMA with 256-column
    accumulators, the packed fp64 sweep and the 2-chunk U-side register tiles."""
    cfg = MEDIUM.with_(k=200, t=300)
    g = synth.generate(MEDIUM)
    s = ESNMF(cfg.n, cfg.m, cfg.k, cfg.t, g, seed=cfg.seed)
    assert s.info()["head_terms"] >= 64
    s.iterate(2)
    v_side_parity(s, g, cfg, cfg.k, cfg.t)


@pytest.mark.parametrize("cfg_name,head", [("tiny", 128), ("medium", 512)])
def test_fused_selection_in_head_epilogue(cfg_name, head, monkeypatch):
    """V-side selection pass 1 fused into the head kernel's epilogue (opt-in
    ESNMF_FUSED_SELECT=1; positives per column + candidates above the predicted
    threshold; k_sel_pred_sort): the same factors, bit for bit, as the unfused
    path, and the oracle's trajectory."""
    cfg = synth.CONFIGS[cfg_name]
    g = synth.generate(cfg)
    monkeypatch.setenv("ESNMF_PRED_MIN_ROWS", "1")
    a = ESNMF(cfg.n, cfg.m, cfg.k, cfg.t, g, seed=cfg.seed, head_terms=head)
    b = ESNMF(cfg.n, cfg.m, cfg.k, cfg.t, g, seed=cfg.seed, head_terms=head)
    iters = 8 if cfg_name == "tiny" else 4
    monkeypatch.setenv("ESNMF_FUSED_SELECT", "1")   # read at every V side
    a.iterate(iters)
    monkeypatch.delenv("ESNMF_FUSED_SELECT")
    b.iterate(iters)
    for x, y in zip(a.get_V(), b.get_V()):
        assert np.array_equal(x, y)
    for x, y in zip(a.get_U(), b.get_U()):
        assert np.array_equal(x, y)
    ra, rb = a.records(), b.records()
    assert [r["E"] for r in ra] == [r["E"] for r in rb]
    assert [r["peak_v"] for r in ra] == [r["peak_v"] for r in rb]
    if cfg_name == "tiny":
        ref = oracle.run(g, cfg.k, cfg.t, iters, seed=cfg.seed)
        for x, y in zip(ra, ref["records"]):
            assert abs(x["E"] - y["E"]) <= 1e-3 * y["E"] and x["nnz_v"] == y["nnz_v"]
    # and a late (fused) V side against the oracle directly
    monkeypatch.setenv("ESNMF_FUSED_SELECT", "1")
    v_side_parity(a, g, cfg, cfg.k, cfg.t)


@pytest.mark.parametrize("k", [1, 2, 3, 5, 8])
def test_narrow_v_side(k):
    """kpad <= 8: the V side is the narrow SpMM with a compact z (no head); its LS,
    selection and trajectory match the oracle."""
    g = synth.generate(TINY)
    s = ESNMF(TINY.n, TINY.m, k, 40, g, seed=TINY.seed)
    assert s.info()["head_terms"] == 0
    v_side_parity(s, g, TINY, k, 40)
    s.half_step(ESNMF_SIDE_U)
    s.iterate(4)
    v_side_parity(s, g, TINY, k, 40)
    ref = oracle.run(g, k, 40, 4, seed=TINY.seed)
    t = ESNMF(TINY.n, TINY.m, k, 40, g, seed=TINY.seed)
    t.iterate(4)
    for a, b in zip(t.records(), ref["records"]):
        assert abs(a["E"] - b["E"]) <= 1e-3 * b["E"] and a["nnz_v"] == b["nnz_v"]
