"""Synthetic input generator (synth/): shape, determinism, Zipf structure.

The generator is input plumbing; these tests check it produces the workload
BASELINE.json describes (BJ:7-11) and that the GPU twin is bitwise identical.
"""
import numpy as np
import pytest

import synth

TINY = synth.CONFIGS["tiny"]


def test_tiny_shape_and_rows():
    g = synth.generate(TINY)
    n, m, d = TINY.n, TINY.m, TINY.d
    assert g["at_ptr"][-1] == m * d == g["a_ptr"][-1]
    cols = g["at_col"].reshape(m, d)
    # d distinct terms per document, strictly increasing (canonical CSR)
    assert np.all(np.diff(cols, axis=1) > 0)
    assert cols.min() >= 0 and cols.max() < n
    assert np.all(g["at_val"] > 0) and np.all(np.isfinite(g["at_val"]))


def test_transpose_consistent():
    g = synth.generate(TINY)
    n, m = TINY.n, TINY.m
    A = np.zeros((n, m), np.float32)
    for i in range(n):
        s, e = g["a_ptr"][i], g["a_ptr"][i + 1]
        assert np.all(np.diff(g["a_col"][s:e]) > 0)
        A[i, g["a_col"][s:e]] = g["a_val"][s:e]
    At = np.zeros((m, n), np.float32)
    for j in range(m):
        s, e = g["at_ptr"][j], g["at_ptr"][j + 1]
        At[j, g["at_col"][s:e]] = g["at_val"][s:e]
    assert np.array_equal(A, At.T)


def test_deterministic_and_seeded():
    a = synth.generate(TINY)
    synth.generate.cache_clear()
    b = synth.generate(TINY)
    assert np.array_equal(a["at_col"], b["at_col"]) and np.array_equal(a["at_val"], b["at_val"])
    c = synth.generate(TINY.with_(seed=1))
    assert not np.array_equal(a["at_col"], c["at_col"])


def test_zipf_head_and_lognormal():
    cfg = synth.CONFIGS["medium"]
    g = synth.generate(cfg)
    L = np.diff(g["a_ptr"])
    # rank-0 term appears in (almost) every document (SURVEY 8(d) shape facts)
    assert L[0] > 0.99 * cfg.m
    assert L.argmax() == 0
    # term frequency decreasing in rank on average (Zipf)
    assert L[:10].mean() > L[100:110].mean() > L[10_000:10_010].mean()
    logv = np.log(g["a_val"].astype(np.float64))
    assert abs(logv.mean()) < 0.01 and abs(logv.std() - cfg.sigma) < 0.01


def test_cdf_and_vtab_tables():
    c = synth.zipf_cdf(1000, 1.1)
    assert c[-1] == 1.0 and np.all(np.diff(c) > 0)
    p0 = 1.0 / np.sum(np.arange(1, 1001) ** -1.1)
    assert abs(c[0] - p0) < 1e-15
    v = synth.lognormal_vtab(1.0)
    assert len(v) == 65537 and np.all(np.diff(v) > 0)
    assert abs(v[32768] - 1.0) < 1e-12  # median knot (p = 32769/65538) of lognormal(0, s) is exp(0)


@pytest.mark.gpu
def test_gpu_generator_bitwise_equal_cpu():
    import torch

    for cfg in (TINY, synth.CONFIGS["medium"]):
        h = synth.generate(cfg)
        d = synth.generate_device(cfg)
        torch.cuda.synchronize()
        for key in ("at_col", "at_val", "a_ptr", "a_col", "a_val"):
            assert np.array_equal(d[key].cpu().numpy(), h[key]), (cfg.name, key)
