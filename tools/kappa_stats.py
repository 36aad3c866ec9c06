"""Condition numbers of the two Gram systems (G + eps I) along a run, per
iteration (the precision of a product taken as Y W with W = (G + eps I)^{-1}
depends on them).  One GPU.

    python tools/kappa_stats.py [--config large] [--iters 12]
"""
import argparse
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    import synth
    from paper_1510_05237_b200 import ESNMF, ESNMF_SIDE_U, ESNMF_SIDE_V

    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="large")
    ap.add_argument("--iters", type=int, default=12)
    ap.add_argument("--t", default="cfg")
    a = ap.parse_args()
    cfg = synth.CONFIGS[a.config]
    t = cfg.t if a.t == "cfg" else (None if a.t == "inf" else int(a.t))
    g = synth.generate_device(cfg) if cfg.nnz > 2e7 else synth.generate(cfg)
    s = ESNMF(cfg.n, cfg.m, cfg.k, t, g, seed=cfg.seed)
    out = []
    for it in range(a.iters):
        row = {"it": it + 1}
        for side, nm in ((ESNMF_SIDE_V, "GU"), (ESNMF_SIDE_U, "GV")):
            s.half_step(side)
            G, eps = s.get_gram(side)
            M = G + eps * np.eye(G.shape[0])
            W = np.linalg.inv(M)
            row[nm + "_kinf"] = float(np.abs(M).sum(1).max() * np.abs(W).sum(1).max())
            row[nm + "_k2"] = float(np.linalg.cond(M))
            # amplification of a relative operand error in Y W, per column: max_j-sum |W_jc| / |W_cc|
            row[nm + "_wamp"] = float((np.abs(W).sum(0) / np.abs(np.diag(W))).max())
        out.append(row)
    print(json.dumps(dict(config=a.config, t=t, rows=out)))


if __name__ == "__main__":
    main()
