"""Quick steady-state timing of one config (development; bench.py is the contract):
ms per iteration over K graph-replayed iterations (CUDA events on the library's
stream), then a profiled eager pass with the per-phase times.  One GPU.

    python tools/quick_time.py [--config large] [--steps 20] [--warmup 6] [--head N]
"""
import argparse
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    import torch

    import synth
    from paper_1510_05237_b200 import ESNMF

    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="large")
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=6)
    ap.add_argument("--head", type=int, default=-1)
    ap.add_argument("--t", default="cfg")
    ap.add_argument("--k", type=int, default=0)
    ap.add_argument("--tag", default="")
    a = ap.parse_args()
    cfg = synth.CONFIGS[a.config]
    t = cfg.t if a.t == "cfg" else (None if a.t == "inf" else int(a.t))
    k = a.k or cfg.k
    gd = synth.generate_device(cfg)
    st = torch.cuda.Stream()
    t0 = time.time()
    s = ESNMF(cfg.n, cfg.m, k, t, gd, seed=cfg.seed, stream=st.cuda_stream, head_terms=a.head)
    torch.cuda.synchronize()
    create_s = time.time() - t0
    del gd
    torch.cuda.empty_cache()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(st)
    s.iterate(1)
    e1.record(st)
    torch.cuda.synchronize()
    it1 = e0.elapsed_time(e1)
    s.iterate(a.warmup - 1)
    torch.cuda.synchronize()
    e0.record(st)
    s.iterate(a.steps)
    e1.record(st)
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / a.steps
    recs = s.records()
    s.profile(True)
    s.iterate(min(a.steps, 10))
    torch.cuda.synchronize()
    ph = {k_: round(v[1] / max(1, v[0]), 4) for k_, v in s.phase_times().items() if v[0]}
    info = s.info()
    print(json.dumps(dict(tag=a.tag, config=a.config, k=k, t=t, head=info["head_terms"], ms=round(ms, 4),
                          it1_ms=round(it1, 3), create_s=round(create_s, 2), phases=ph, E=recs[-1]["E"],
                          R=recs[-1]["R"], nnz_u=recs[-1]["nnz_u"], nnz_v=recs[-1]["nnz_v"],
                          env={k_: v for k_, v in os.environ.items() if k_.startswith("ESNMF_")})))


if __name__ == "__main__":
    main()
