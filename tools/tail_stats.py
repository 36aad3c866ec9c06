"""Statistics of the V-side tail at Large steady state (planning the next design):
active tail entries (term rows of U with a nonzero, outside the head), U nonzeros
per active entry, per document.  One GPU.

    python tools/tail_stats.py [--config large] [--iters 10]
"""
import argparse
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    import torch

    import synth
    from paper_1510_05237_b200 import ESNMF

    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="large")
    ap.add_argument("--iters", type=int, default=10)
    a = ap.parse_args()
    cfg = synth.CONFIGS[a.config]
    gd = synth.generate_device(cfg)
    s = ESNMF(cfg.n, cfg.m, cfg.k, cfg.t, gd, seed=cfg.seed)
    s.iterate(a.iters)
    h = s.info()["head_terms"]
    r, c, v = s.get_U()
    nnz_row = np.bincount(np.asarray(r, np.int64), minlength=cfg.n)
    at_col = gd["at_col"].to(torch.int64)
    nr = torch.from_numpy(nnz_row).cuda()
    tail = at_col >= h            # the head is the first h term ids (Zipf order)
    act = tail & (nr[at_col] > 0)
    n_tail, n_act = int(tail.sum()), int(act.sum())
    unnz = int(nr[at_col][act].sum())
    per_doc = act.view(cfg.m, cfg.d).sum(1).float()
    out = dict(config=cfg.name, head_terms=h, entries=int(at_col.numel()), tail_entries=n_tail,
               active_tail_entries=n_act, u_nnz_over_active=unnz, u_nnz_per_active=unnz / max(1, n_act),
               active_per_doc_mean=float(per_doc.mean()), active_per_doc_max=int(per_doc.max()),
               u_rows_nonzero=int((nnz_row > 0).sum()), u_rows_nonzero_tail=int((nnz_row[h:] > 0).sum()),
               u_nnz=int(len(r)), z_row_bytes_if_gathered=n_act * 4 * cfg.k)
    # coverage of the active tail entries by a static band of the next C terms after
    # the head (a shared-memory Z cache candidate; terms are generated in Zipf order)
    band = {}
    for C in (64, 128, 256, 384, 512, 1024, 2048):
        band[C] = round(float((act & (at_col < h + C)).sum()) / max(1, n_act), 4)
    out["active_coverage_by_band"] = band
    print(json.dumps(out))


if __name__ == "__main__":
    main()
