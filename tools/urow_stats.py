"""U-row density by term rank at steady state (planning the paper-order V side).

For the V-side product Y = A^T U taken in the paper's order, an entry
(doc j, term i) of A^T costs r_i = nnz(U row i) products.  This prints, per band
of 64 term ranks (term id = Zipf rank - 1, synth/), the A^T entries in the band,
the entries whose U row is nonzero, and the paper-order products sum r_i, next
to the dense-tile tensor-core cost of the same band (3 fp16 passes over 128-doc
tiles).  One GPU.

    python tools/urow_stats.py [--config large] [--iters 10]
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
    ap.add_argument("--bands", type=int, default=48)
    a = ap.parse_args()
    cfg = synth.CONFIGS[a.config]
    gd = synth.generate_device(cfg)
    s = ESNMF(cfg.n, cfg.m, cfg.k, cfg.t, gd, seed=cfg.seed)
    s.iterate(a.iters)
    h = s.info()["head_terms"]
    r, c, v = s.get_U()
    nnz_row = torch.from_numpy(np.bincount(np.asarray(r, np.int64), minlength=cfg.n)).cuda()
    at_col = gd["at_col"]
    B = 64
    band = (at_col // B).to(torch.int64)
    nb = (cfg.n + B - 1) // B
    ent = torch.bincount(band, minlength=nb)
    ri = nnz_row[at_col.to(torch.int64)]
    act = torch.bincount(band, weights=(ri > 0).to(torch.float64), minlength=nb)
    prod = torch.bincount(band, weights=ri.to(torch.float64), minlength=nb)
    del ri, band
    urow = torch.bincount(torch.arange(cfg.n, device="cuda") // B, weights=nnz_row.to(torch.float64), minlength=nb)
    ntiles = (cfg.m + 127) // 128
    kn = (cfg.k + 15) // 16 * 16
    tc_flops_band = ntiles * 128 * B * kn * 2 * 3
    rows = []
    for q in range(min(a.bands, nb)):
        rows.append(dict(band=q, entries=int(ent[q]), active=int(act[q]), products=int(prod[q]),
                         u_nnz=int(urow[q]), density=float(ent[q]) / (cfg.m * B)))
    tail = dict(entries=int(ent[a.bands:].sum()), active=int(act[a.bands:].sum()),
                products=int(prod[a.bands:].sum()), u_nnz=int(urow[a.bands:].sum()))
    out = dict(config=cfg.name, iters=a.iters, head_terms=h, u_nnz=int(len(r)), tc_flops_per_band=tc_flops_band,
               bands=rows, beyond=tail, total_products=int(prod.sum()), total_entries=int(ent.sum()))
    print(json.dumps(out))


if __name__ == "__main__":
    main()
