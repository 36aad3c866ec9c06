"""Checkpoint / resume (paper_1510_05237_b200/checkpoint.py):
the file format round-trips on the host, and on the GPU a run saved after 3
iterations and resumed on a fresh handle continues exactly like the uninterrupted run."""
import numpy as np
import pytest

import synth
from paper_1510_05237_b200 import ESNMF, checkpoint


class _FakeSolver:
    n, m, k, t = 7, 5, 2, 3

    def get_U(self):
        return np.array([0, 4, 1], np.int32), np.array([0, 0, 1], np.int32), np.array([0.5, 1.5, 2.0], np.float32)

    def get_V(self):
        return np.array([3], np.int32), np.array([1], np.int32), np.array([0.25], np.float32)

    def records(self):
        return [{"it": 1, "R": 0.5, "E": 0.9, "nnz_u": 3, "nnz_v": 1}]


def test_checkpoint_files_round_trip(tmp_path):
    man = checkpoint.save(_FakeSolver(), str(tmp_path), seed=11)
    man2, fac = checkpoint.load(str(tmp_path))
    assert man2 == man and man["iterations"] == 1 and man["E"] == 0.9 and man["seed"] == 11
    for name, ref in (("U", _FakeSolver().get_U()), ("V", _FakeSolver().get_V())):
        for a, b in zip(fac[name], ref):
            assert a.dtype == b.dtype and np.array_equal(a, b)
    (tmp_path / "manifest.json").write_text('{"format": "other"}')
    with pytest.raises(ValueError):
        checkpoint.load(str(tmp_path))


@pytest.mark.gpu
def test_resume_continues_the_run(tmp_path):
    cfg = synth.CONFIGS["tiny"]
    g = synth.generate(cfg)
    full = ESNMF(cfg.n, cfg.m, cfg.k, cfg.t, g, seed=cfg.seed)
    full.iterate(6)
    ref = full.records()
    part = ESNMF(cfg.n, cfg.m, cfg.k, cfg.t, g, seed=cfg.seed)
    part.iterate(3)
    checkpoint.save(part, str(tmp_path), seed=cfg.seed)
    part.close()
    s, man = checkpoint.resume(str(tmp_path), g)
    assert man["iterations"] == 3
    s.iterate(3)
    got = s.records()
    for a, b in zip(got, ref[3:]):
        for key in ("E", "R", "nnz_u", "nnz_v"):
            assert a[key] == b[key], (key, a, b)
    for fa, fb in ((s.get_U(), full.get_U()), (s.get_V(), full.get_V())):
        for x, y in zip(fa, fb):
            assert np.array_equal(x, y)
