"""Per-iteration device time of the method's variants on one config (one GPU).

    python tools/bench_variants.py [--config large] [--iters 40] [--out profiles/X.json]

Variants (all through the C ABI, inputs resident, CUDA events on the library's
stream after warm-up):
  alg2_column   Alg. 2 with per-column enforcement (the north_star path)
  alg2_whole    Alg. 2 as printed, whole-factor budgets t_u = t_v = k t
  seq_k2_1      sequential ALS (Alg. 3), one topic per block (the paper's timing case)
  seq_k2_10     sequential ALS, blocks of 10 topics
For the sequential variants the timed region covers whole blocks (block
appends and restarts included): ms/iteration = total / iterations.  The
paper's comparison (P:398, 100 iterations of a five-topic PubMed NMF) is the
ratio column-wise : sequential, which this prints on synthetic data.
"""
import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    import torch

    import synth
    from paper_1510_05237_b200 import ESNMF

    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="large")
    ap.add_argument("--iters", type=int, default=40)
    ap.add_argument("--out", default=None)
    ap.add_argument("--pubmed", action="store_true",
                    help="the paper's timing case (P:398): 100 iterations of a 5-topic NMF of a PubMed-sized "
                         "planted corpus (synth/planted.py), row-normalised, with clustering accuracy")
    a = ap.parse_args()
    if a.pubmed:
        return pubmed(a)
    cfg = synth.CONFIGS[a.config]
    dev = torch.device("cuda", 0)
    g = synth.generate_device(cfg, device=dev)
    stream = torch.cuda.Stream(dev)
    torch.cuda.set_stream(stream)
    variants = {
        "alg2_column": dict(),
        "alg2_whole": dict(whole=True, t_u=cfg.k * cfg.t, t_v=cfg.k * cfg.t),
        "seq_k2_1": dict(seq_k2=1, seq_iters=2),
        "seq_k2_4": dict(seq_k2=4, seq_iters=4),
        "seq_k2_10": dict(seq_k2=10, seq_iters=4),
    }
    out = {}
    for name, kw in variants.items():
        s = ESNMF(cfg.n, cfg.m, cfg.k, cfg.t, g, seed=cfg.seed, stream=stream.cuda_stream, **kw)
        if "seq_k2" in kw:
            warm = kw["seq_iters"]                       # block 0
            steps = min(cfg.k // kw["seq_k2"] - 1, max(1, a.iters // kw["seq_iters"])) * kw["seq_iters"]
        else:
            warm, steps = 5, a.iters
        s.iterate(warm)
        torch.cuda.synchronize()
        s.profile(True)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        s.iterate(steps)
        e1.record(stream)
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1)
        ph = s.phase_times()
        s.profile(False)
        rec = s.records()[-1]
        top = sorted(((k, v[1] / steps) for k, v in ph.items() if v[0]), key=lambda kv: -kv[1])[:5]
        out[name] = {"ms_per_iter": round(ms / steps, 4), "iters_timed": steps, "E_last": rec["E"],
                     "nnz_u": rec["nnz_u"], "nnz_v": rec["nnz_v"],
                     "top_phases_ms_per_iter": {k: round(v, 4) for k, v in top}}
        print(name, json.dumps(out[name]), flush=True)
        s.close()
        torch.cuda.empty_cache()
    res = {"config": cfg.name, "variants": out,
           "column_over_seq_k2_1": round(out["alg2_column"]["ms_per_iter"] / out["seq_k2_1"]["ms_per_iter"], 2)}
    print(json.dumps(res))
    if a.out:
        with open(a.out, "w") as f:
            json.dump(res, f, indent=1)


def pubmed(a):
    """P:398's comparison on a PubMed-sized planted corpus (20,112 terms x 7,510
    documents, 5 journals): 100 iterations of a 5-topic NMF with whole-matrix,
    column-wise and sequential (k2 = 1, 20 iterations per topic) enforcement;
    device time per iteration and the mean clustering accuracy (Eq. (3)-(4))."""
    import torch

    from synth.planted import planted_corpus
    from paper_1510_05237_b200 import ESNMF

    g = planted_corpus()
    k, t, iters = 5, 200, 100
    stream = torch.cuda.Stream()
    torch.cuda.set_stream(stream)
    variants = {
        "alg2_whole": dict(whole=True, t_u=k * t, t_v=k * t),
        "alg2_column": dict(),
        "seq_k2_1": dict(seq_k2=1, seq_iters=iters // k),
        "alg2_column_raw_counts": dict(row_normalize=False),
    }
    out = {}
    for name, kw in variants.items():
        kw = dict(dict(row_normalize=True), **kw)
        s = ESNMF(g["n"], g["m"], k, t, g, seed=0, stream=stream.cuda_stream, **kw)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        s.iterate(iters)
        e1.record(stream)
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1)
        acc = s.topic_accuracy(g["labels"], g["n_journals"])
        out[name] = {"ms_per_iter": round(ms / iters, 4), "ms_100_iters": round(ms, 2),
                     "E_last": s.records()[-1]["E"], "accuracy": [round(x, 4) for x in acc],
                     "accuracy_mean": round(float(acc.mean()), 4)}
        print(name, json.dumps(out[name]), flush=True)
        s.close()
    res = {"config": "pubmed_like 20112x7510, k=5, t=200 per column (1000 per factor), 100 iterations",
           "variants": out}
    print(json.dumps(res))
    if a.out:
        with open(a.out, "w") as f:
            json.dump(res, f, indent=1)


if __name__ == "__main__":
    main()
