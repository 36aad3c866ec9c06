"""Multi-rank path.

CPU (gloo, world_size 2): the sharding math -- nnz-balanced term shards and
equal document shards (esnmf_partition_rows), local per-column top-t on each
shard, allgather of the candidates and the merge rule -- reproduces the
unsharded oracle half-step exactly; and the comm adapter moves the library's
exchange buffers correctly.
GPU (one device): P logical ranks as P handles driven from P threads through
the loopback group -- the same library code path as P processes over NCCL --
give the same factors for P = 2 and 3, matching P = 1 and the oracle.
"""
import os
import threading

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import oracle
import synth
from parity import TRAJ_TOL, check_products, check_selection, check_topt_property, coo_dense, r_close
import paper_1510_05237_b200 as pk
from paper_1510_05237_b200 import ESNMF, ESNMF_SIDE_U, ESNMF_SIDE_V

TINY = synth.CONFIGS["tiny"]


def merge_rule(cands, t):
    """Global top-t of the union of local top-t candidate lists (value desc, row asc)."""
    rows = np.concatenate([c[0] for c in cands])
    vals = np.concatenate([c[1] for c in cands])
    if t is not None and len(rows) > t:
        order = np.lexsort((rows, -vals))[:t]
        keep = np.zeros(len(rows), bool)
        keep[order] = True
        rows, vals = rows[keep], vals[keep]
    o = np.argsort(rows, kind="stable")
    return rows[o], vals[o]


def local_topt(LS, row0, t):
    out = []
    for c in range(LS.shape[1]):
        col = LS[:, c]
        pos = np.nonzero(col > 0)[0]
        if t is not None and len(pos) > t:
            order = np.lexsort((pos, -col[pos]))[:t]
            pos = np.sort(pos[order])
        out.append((pos + row0, col[pos]))
    return out


def _shard_worker(rank, world, port, result):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    g = synth.generate(TINY)
    k, t = TINY.k, TINY.t
    U = oracle.u0(TINY.n, k, 0).astype(np.float64)
    # V side: equal document shards
    m0, m1 = TINY.m * rank // world, TINY.m * (rank + 1) // world
    L, _ = oracle.cholesky(oracle.gram(U))
    LS = oracle.solve_rows(L, oracle.spmm_rows(np.arange(m0, m1), g["at_ptr"], g["at_col"], g["at_val"], U))
    loc = local_topt(LS, m0, t)
    # allgather the candidates (padded to t per column, like the library buffer)
    cap = t
    buf = np.zeros((k, 2, cap + 1), np.float64)
    for c, (r, v) in enumerate(loc):
        buf[c, 0, 0] = len(r)
        buf[c, 0, 1:len(r) + 1] = r
        buf[c, 1, 1:len(r) + 1] = v
    gathered = [torch.zeros_like(torch.from_numpy(buf)) for _ in range(world)]
    dist.all_gather(gathered, torch.from_numpy(buf))
    merged = []
    for c in range(k):
        cands = []
        for p in range(world):
            b = gathered[p].numpy()
            n = int(b[c, 0, 0])
            cands.append((b[c, 0, 1:n + 1].astype(np.int64), b[c, 1, 1:n + 1]))
        merged.append(merge_rule(cands, t))
    # U side: nnz-balanced term shards, T of the error by allreduce
    bounds = pk.esnmf_partition_rows(g["a_ptr"], world)
    result[rank] = dict(merged=merged, bounds=bounds)
    dist.destroy_process_group()


def test_sharded_topt_merge_equals_unsharded_gloo():
    world = 2
    mgr = mp.Manager()
    result = mgr.dict()
    mp.spawn(_shard_worker, args=(world, 29541, result), nprocs=world, join=True)
    g = synth.generate(TINY)
    ref = oracle.half_step(g["at_ptr"], g["at_col"], g["at_val"], oracle.u0(TINY.n, TINY.k, 0), TINY.t)["F"]
    for rank in range(world):
        merged = result[rank]["merged"]
        for c in range(TINY.k):
            rows, vals = merged[c]
            want = np.nonzero(ref[:, c])[0]
            assert np.array_equal(rows, want)
            assert np.allclose(vals, ref[want, c], rtol=1e-12, atol=0)
        b = result[rank]["bounds"]
        assert b[0] == 0 and b[-1] == TINY.n and np.all(np.diff(b) >= 0)


# ------------------------------------------------------------------ GPU


def run_loopback(world, cfg, g, iters, t="cfg", post=None, k=None, **kw):
    """P logical ranks in P threads; ``post(rank, handle)`` (optional) runs in the
    rank's thread after the iterations (half-steps there are collective too)."""
    tval = cfg.t if t == "cfg" else t
    grp = pk.comm.LoopbackGroup(world)
    handles = [None] * world
    errs = []

    def worker(r):
        try:
            stream = torch.cuda.Stream()
            handles[r] = ESNMF(cfg.n, cfg.m, k or cfg.k, tval, g, seed=cfg.seed, world=world, rank=r,
                               comm=grp.comms[r], stream=stream.cuda_stream, **kw)
            handles[r].iterate(iters)
            handles[r].records()
            if post is not None:
                post(r, handles[r])
        except Exception as e:  # pragma: no cover
            errs.append(e)
            grp.barrier.abort()

    th = [threading.Thread(target=worker, args=(r,)) for r in range(world)]
    for x in th:
        x.start()
    for x in th:
        x.join(timeout=600)
    assert not errs, errs
    return handles


@pytest.mark.gpu
@pytest.mark.parametrize("world", [2, 3])
def test_loopback_ranks_match_single_gpu(world):
    import paper_1510_05237_b200.comm  # noqa: F401

    g = synth.generate(TINY)
    hs = run_loopback(world, TINY, g, 4)
    one = ESNMF(TINY.n, TINY.m, TINY.k, TINY.t, g, seed=TINY.seed)
    one.iterate(4)
    r1 = one.records()
    u1, v1 = one.get_U(), one.get_V()
    ref = oracle.run(g, TINY.k, TINY.t, 4, seed=TINY.seed)["records"]
    for h in hs:
        recs = h.records()
        for a, b, o in zip(recs, r1, ref):
            assert abs(a["E"] - b["E"]) <= 1e-6 * b["E"]
            assert a["nnz_u"] == b["nnz_u"] and a["nnz_v"] == b["nnz_v"]
            # peak nnz summed over ranks (the single GPU's count, >= nnz)
            assert a["peak_u"] == b["peak_u"] and a["peak_v"] == b["peak_v"]
            assert a["peak_u"] >= a["nnz_u"] and a["peak_v"] >= a["nnz_v"]
            # and the oracle's run from the same U_0 (BJ:5; reading C15)
            assert abs(a["E"] - o["E"]) <= TRAJ_TOL * o["E"] and r_close(a["R"], o["R"])
            assert (a["nnz_u"], a["nnz_v"], a["peak_u"], a["peak_v"]) == (o["nnz_u"], o["nnz_v"], o["peak_u"],
                                                                          o["peak_v"])
        ur, vr = h.get_U(), h.get_V()
        for x, y in zip(ur[:2] + vr[:2], u1[:2] + v1[:2]):
            assert np.array_equal(x, y)        # same supports
        assert np.allclose(ur[2], u1[2], rtol=1e-5) and np.allclose(vr[2], v1[2], rtol=1e-5)
    # every rank holds the same replicated factors, bitwise
    for h in hs[1:]:
        for x, y in zip(h.get_U() + h.get_V(), hs[0].get_U() + hs[0].get_V()):
            assert np.array_equal(x, y)


@pytest.mark.gpu
def test_loopback_two_vs_three_ranks_bitwise():
    import paper_1510_05237_b200.comm  # noqa: F401

    g = synth.generate(TINY)
    a = run_loopback(2, TINY, g, 3)[0]
    b = run_loopback(3, TINY, g, 3)[0]
    for x, y in zip(a.get_U() + a.get_V(), b.get_U() + b.get_V()):
        assert np.array_equal(x, y)          # shard layout does not change the factors
    for ra, rb in zip(a.records(), b.records()):
        assert ra["R"] == rb["R"]            # computed on the replicated U
        assert ra["E"] == pytest.approx(rb["E"], rel=1e-12)  # T is a sum over ranks


@pytest.mark.gpu
def test_loopback_options_match_single_gpu():
    """The §8(f) options on the sharded path: row normalisation (each rank scales
    its term rows and its documents' A^T entries by the global row nnz), separate
    budgets, sparse U_0; the accuracy of a rank's replicated V equals the single
    GPU's."""
    import paper_1510_05237_b200.comm  # noqa: F401

    g = synth.generate(TINY)
    kw = dict(row_normalize=True, t_u=30, t_v=45, init_nnz=400)
    hs = run_loopback(2, TINY, g, 4, **kw)
    one = ESNMF(TINY.n, TINY.m, TINY.k, TINY.t, g, seed=TINY.seed, **kw)
    one.iterate(4)
    for a, b in zip(hs[0].records(), one.records()):
        assert abs(a["E"] - b["E"]) <= 1e-6 * b["E"]
        assert a["nnz_u"] == b["nnz_u"] and a["nnz_v"] == b["nnz_v"]
    labels = np.arange(TINY.m) % 3
    assert np.allclose(hs[1].topic_accuracy(labels, 3), one.topic_accuracy(labels, 3), rtol=0, atol=1e-12)


def _sharded_half_steps(world, cfg, g, iters, k=None, t="cfg"):
    """Run P ranks for ``iters`` iterations, then one V and one U half-step on every
    rank; returns the replicated state before (U), the assembled LS of each side
    (every rank's shard of rows, placed at its row0) and the factors after."""
    k = k or cfg.k
    shards = {ESNMF_SIDE_V: [None] * world, ESNMF_SIDE_U: [None] * world}
    state = {}

    def post(r, h):
        if r == 0:
            state["U"] = h.get_U()
        for side in (ESNMF_SIDE_V, ESNMF_SIDE_U):
            h.half_step(side)
            row0, ls = h.get_ls(side)
            shards[side][r] = (row0, ls)
            if r == 0 and side == ESNMF_SIDE_V:
                state["V"] = h.get_V()
        if r == 0:
            state["U_after"] = h.get_U()

    hs = run_loopback(world, cfg, g, iters, t=t, post=post, k=k)
    full = {}
    for side, n_rows in ((ESNMF_SIDE_V, cfg.m), (ESNMF_SIDE_U, cfg.n)):
        LS = np.zeros((n_rows, k), np.float32)
        covered = 0
        for row0, ls in shards[side]:
            LS[row0:row0 + len(ls)] = ls
            covered += len(ls)
        assert covered == n_rows              # the shards partition the rows
        full[side] = LS
    return hs, state, full


@pytest.mark.gpu
@pytest.mark.parametrize("world", [2, 3])
def test_loopback_half_steps_match_oracle(world):
    """The sharded path (local top-t, allgather, merge: a6) against the ORACLE's
    half-steps from the same state: every rank's LS rows and the merged factors."""
    import paper_1510_05237_b200.comm  # noqa: F401

    cfg = TINY
    g = synth.generate(cfg)
    hs, st, LS = _sharded_half_steps(world, cfg, g, 3)
    U = coo_dense((cfg.n, cfg.k), *st["U"])
    ref = oracle.half_step(g["at_ptr"], g["at_col"], g["at_val"], U, cfg.t)
    check_products(LS[ESNMF_SIDE_V], ref["LS"])
    V = coo_dense((cfg.m, cfg.k), *st["V"])
    check_selection(V, ref["F"], ref["LS"], cfg.t)
    ref = oracle.half_step(g["a_ptr"], g["a_col"], g["a_val"], V, cfg.t)
    check_products(LS[ESNMF_SIDE_U], ref["LS"])
    check_selection(coo_dense((cfg.n, cfg.k), *st["U_after"]), ref["F"], ref["LS"], cfg.t)


@pytest.mark.gpu
@pytest.mark.slow
def test_loopback_large_p8_matches_oracle_and_single_gpu():
    """P = 8 at Large (BJ:9, t = 1,000; the 8-GPU configuration of north_star) on
    one device: records equal the single GPU's; LS rows of every shard, sampled
    (the head term rows and 1,500 documents), against the oracle row by row; the
    top-t property of the merged factors on the assembled LS."""
    import paper_1510_05237_b200.comm  # noqa: F401

    cfg = synth.CONFIGS["large"]
    g = synth.generate(cfg)
    hs, st, LS = _sharded_half_steps(8, cfg, g, 2)
    recs = hs[0].records()
    for h in hs:
        h.close()
    one = ESNMF(cfg.n, cfg.m, cfg.k, cfg.t, g, seed=cfg.seed)
    one.iterate(2)
    for a, b in zip(recs, one.records()):
        assert abs(a["E"] - b["E"]) <= 1e-6 * b["E"] and (a["nnz_u"], a["nnz_v"]) == (b["nnz_u"], b["nnz_v"])
        # the positives of the LS buffers: the sharded U side's products are fp64
        # (k_spmm_terms), the single GPU's fp16 hi/lo on tcgen05, so an entry within
        # rounding of zero may fall on either side
        assert abs(a["peak_u"] - b["peak_u"]) <= 1e-6 * b["peak_u"] and a["peak_v"] == b["peak_v"]
    one.close()
    rng = np.random.default_rng(0)
    U = coo_dense((cfg.n, cfg.k), *st["U"])
    L, _ = oracle.cholesky(oracle.gram(U))
    docs = np.sort(rng.choice(cfg.m, 1500, replace=False))
    ref = oracle.solve_rows(L, oracle.spmm_rows(docs, g["at_ptr"], g["at_col"], g["at_val"], U))
    scale = np.abs(LS[ESNMF_SIDE_V]).max(axis=0).astype(np.float64)
    assert (np.abs(LS[ESNMF_SIDE_V][docs] - ref) / scale).max() <= 1e-5
    Vr, Vc, Vv = st["V"]
    V = coo_dense((cfg.m, cfg.k), Vr, Vc, Vv)
    check_topt_property(LS[ESNMF_SIDE_V], V, cfg.t)
    L, _ = oracle.cholesky(oracle.gram(V))
    terms = np.unique(np.concatenate([np.arange(20), rng.choice(cfg.n, 1500, replace=False)]))
    ref = oracle.solve_rows(L, oracle.spmm_rows(terms, g["a_ptr"], g["a_col"], g["a_val"], V))
    scale = np.abs(LS[ESNMF_SIDE_U]).max(axis=0).astype(np.float64)
    assert (np.abs(LS[ESNMF_SIDE_U][terms] - ref) / scale).max() <= 1e-5
    check_topt_property(LS[ESNMF_SIDE_U], coo_dense((cfg.n, cfg.k), *st["U_after"]), cfg.t)


@pytest.mark.gpu
@pytest.mark.slow
def test_loopback_box_shaped_merge_matches_oracle():
    """The merge at Box's shape (BJ:10: k = 200, t = 5,000, P = 8: up to 40,000
    candidate keys per column) on the Medium matrix: the merged factors equal the
    oracle's clamp + top-t of the full LS from the same state (check_selection)."""
    import paper_1510_05237_b200.comm  # noqa: F401

    cfg = synth.CONFIGS["medium"]
    g = synth.generate(cfg)
    hs, st, LS = _sharded_half_steps(8, cfg, g, 2, k=200, t=5000)
    for h in hs:
        h.close()
    U = coo_dense((cfg.n, 200), *st["U"])
    ref = oracle.half_step(g["at_ptr"], g["at_col"], g["at_val"], U, 5000)
    check_products(LS[ESNMF_SIDE_V], ref["LS"])
    V = coo_dense((cfg.m, 200), *st["V"])
    check_selection(V, ref["F"], ref["LS"], 5000)
    ref = oracle.half_step(g["a_ptr"], g["a_col"], g["a_val"], V, 5000)
    check_products(LS[ESNMF_SIDE_U], ref["LS"])
    check_selection(coo_dense((cfg.n, 200), *st["U_after"]), ref["F"], ref["LS"], 5000)


# ------------------------------------------------------- built-in NCCL

def _nccl_id_worker(rank, world, port, result):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    uid = pk.comm.broadcast_nccl_id()
    result[rank] = uid
    dist.destroy_process_group()


def test_nccl_unique_id_broadcast_gloo():
    """Host logic of the library's NCCL communicator (no GPU needed): rank 0 draws
    the 128-byte NCCL unique id through the C ABI (esnmf_nccl_unique_id) and the
    process group hands every rank the same bytes."""
    world = 2
    mgr = mp.Manager()
    result = mgr.dict()
    mp.spawn(_nccl_id_worker, args=(world, 29553, result), nprocs=world, join=True)
    ids = [result[r] for r in range(world)]
    assert len(ids[0]) == 128 and ids[0] == ids[1]
    assert any(ids[0])  # not all zero
    assert pk.esnmf.esnmf_nccl_unique_id() != ids[0]  # a fresh id each time


def _forced_sharded(cfg, g, iters, **kw):
    """One rank through the multi-rank code path (local top-t, allgather + merge,
    the term-row U side, T allreduced) with the library's OWN NCCL communicator of
    size 1 -- the plumbing of an 8-GPU run exercised on one device."""
    os.environ["ESNMF_FORCE_SHARDED"] = "1"
    try:
        uid = pk.esnmf.esnmf_nccl_unique_id()
        comm = pk.esnmf.NcclComm(1, 0, uid, 0)
        s = ESNMF(cfg.n, cfg.m, cfg.k, cfg.t, g, seed=cfg.seed, world=1, rank=0, comm=comm.struct, **kw)
    finally:
        del os.environ["ESNMF_FORCE_SHARDED"]
    s.iterate(iters)
    return s, comm


@pytest.mark.gpu
def test_builtin_nccl_sharded_path_matches_oracle():
    """The sharded path on the library's NCCL communicator, CUDA graphs on (the
    collectives are captured with the iteration): the Tiny trajectory against the
    oracle's golden run (E, nnz, R_1), the factors against the single-GPU path."""
    import json

    from parity import TRAJ_TOL, r_close

    cfg = TINY
    g = synth.generate(cfg)
    s, comm = _forced_sharded(cfg, g, cfg.iters)
    gold = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "traj_tiny.json")))["records"]
    recs = s.records()
    assert len(recs) == len(gold)
    for a, b in zip(recs, gold):
        assert abs(a["E"] - b["E"]) <= TRAJ_TOL * b["E"], (a["it"], a["E"], b["E"])
        assert (a["nnz_u"], a["nnz_v"]) == (b["nnz_u"], b["nnz_v"])
    assert r_close(recs[0]["R"], gold[0]["R"])
    one = ESNMF(cfg.n, cfg.m, cfg.k, cfg.t, g, seed=cfg.seed)
    one.iterate(cfg.iters)
    for a, b in zip(recs, one.records()):
        assert abs(a["E"] - b["E"]) <= 1e-6 * b["E"] and (a["nnz_u"], a["nnz_v"]) == (b["nnz_u"], b["nnz_v"])
    for x, y in zip(s.get_U()[:2] + s.get_V()[:2], one.get_U()[:2] + one.get_V()[:2]):
        assert np.array_equal(x, y)
    s.close()
    one.close()
    comm.close()


@pytest.mark.gpu
@pytest.mark.slow
def test_builtin_nccl_sharded_large_half_steps():
    """Large through the sharded path on the library's NCCL communicator: sampled LS
    rows of both sides against the oracle row by row, the selection property."""
    cfg = synth.CONFIGS["large"]
    g = synth.generate(cfg)
    s, comm = _forced_sharded(cfg, g, 3)
    rng = np.random.default_rng(1)
    for side in (ESNMF_SIDE_V, ESNMF_SIDE_U):
        F = coo_dense((cfg.n, cfg.k), *s.get_U()) if side == ESNMF_SIDE_V else coo_dense((cfg.m, cfg.k), *s.get_V())
        ptr, idx, val, rows = ((g["at_ptr"], g["at_col"], g["at_val"], cfg.m) if side == ESNMF_SIDE_V
                               else (g["a_ptr"], g["a_col"], g["a_val"], cfg.n))
        L, _ = oracle.cholesky(oracle.gram(F))
        s.half_step(side)
        _, ls = s.get_ls(side)
        sel = np.unique(np.concatenate([np.arange(20), rng.choice(rows, 1500, replace=False)]))
        ref = oracle.solve_rows(L, oracle.spmm_rows(sel, ptr, idx, val, F))
        scale = np.abs(ls).max(axis=0).astype(np.float64)
        assert (np.abs(ls[sel].astype(np.float64) - ref) / scale).max() <= 1e-5
        out = coo_dense((cfg.m, cfg.k), *s.get_V()) if side == ESNMF_SIDE_V else coo_dense((cfg.n, cfg.k), *s.get_U())
        check_topt_property(ls, out, cfg.t)
    s.close()
    comm.close()
