"""CUDA-graph replay of steady-state iterations (esnmf_iterate captures one
iteration per U-slot parity and replays it): identical results to eager
launches, records numbered and filled on every replay, state changes between
calls honoured."""
import numpy as np
import pytest

import oracle
import synth
from paper_1510_05237_b200 import ESNMF, ESNMF_SIDE_U, ESNMF_SIDE_V
from parity import TRAJ_TOL

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("cfg_name", ["tiny", "medium"])
def test_graph_replay_equals_eager(cfg_name, monkeypatch):
    cfg = synth.CONFIGS[cfg_name]
    g = synth.generate(cfg)
    a = ESNMF(cfg.n, cfg.m, cfg.k, cfg.t, g, seed=cfg.seed)
    monkeypatch.setenv("ESNMF_NO_GRAPH", "1")
    b = ESNMF(cfg.n, cfg.m, cfg.k, cfg.t, g, seed=cfg.seed)
    b.iterate(11)
    monkeypatch.delenv("ESNMF_NO_GRAPH")
    a.iterate(5)       # 2 eager, then one capture per U-slot parity, then replays
    a.iterate(6)       # replays only
    ra, rb = a.records(), b.records()
    assert [r["it"] for r in ra] == list(range(1, 12))
    for x, y in zip(ra, rb):
        assert x == y
    for x, y in zip(a.get_U(), b.get_U()):
        assert np.array_equal(x, y)
    for x, y in zip(a.get_V(), b.get_V()):
        assert np.array_equal(x, y)
    assert a.info()["launches"] == b.info()["launches"]


def test_graph_state_changes_between_calls():
    """half_step / set_factor / truncate between iterate calls drop the graphs;
    the trajectory still matches the oracle from the changed state."""
    cfg = synth.CONFIGS["tiny"]
    g = synth.generate(cfg)
    s = ESNMF(cfg.n, cfg.m, cfg.k, cfg.t, g, seed=cfg.seed)
    s.iterate(6)
    r, c, v = s.get_U()
    U = np.zeros((cfg.n, cfg.k))
    U[r, c] = v
    s.truncate(ESNMF_SIDE_U, 20)
    Ut = oracle.clamp_top_t(U, 20)[0]
    s.iterate(7)
    ref = oracle.run(g, cfg.k, cfg.t, 7, U_init=Ut)
    for x, y in zip(s.records()[6:], ref["records"]):
        assert abs(x["E"] - y["E"]) <= TRAJ_TOL * y["E"] and x["nnz_u"] == y["nnz_u"]
    assert [x["it"] for x in s.records()] == list(range(1, 14))
    s.half_step(ESNMF_SIDE_V)
    s.half_step(ESNMF_SIDE_U)
    s.iterate(4)
    assert len(s.records()) == 17


def test_graph_replay_sequential_blocks(monkeypatch):
    """Sequential ALS (Alg. 3) replays graphs inside a block; block changes run
    eagerly: the same records and factors as without graphs."""
    cfg = synth.CONFIGS["tiny"]
    g = synth.generate(cfg)
    a = ESNMF(cfg.n, cfg.m, cfg.k, cfg.t, g, seed=cfg.seed, seq_k2=2, seq_iters=7)
    monkeypatch.setenv("ESNMF_NO_GRAPH", "1")
    b = ESNMF(cfg.n, cfg.m, cfg.k, cfg.t, g, seed=cfg.seed, seq_k2=2, seq_iters=7)
    b.iterate(35)
    monkeypatch.delenv("ESNMF_NO_GRAPH")
    a.iterate(12)
    a.iterate(23)
    for x, y in zip(a.records(), b.records()):
        assert x == y
    for x, y in zip(a.get_U(), b.get_U()):
        assert np.array_equal(x, y)
