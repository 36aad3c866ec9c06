"""Write oracle trajectories to tests/golden/ (calls only oracle/ and synth/).

    python tests/golden/make_golden.py [tiny medium sweep large box]

Each file records, per iteration, the oracle's R, E and factor nnz for one
BASELINE.json config (BJ:7-11) from U_0 (reading C10, seed 0).  The GPU
trajectory tests compare against these files (E within 1e-3 relative, BJ:5).
"""
import json
import os
import sys
import time

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))

import oracle  # noqa: E402
import synth   # noqa: E402


def run(cfg, t, iters, tag, lean=False):
    """lean (Box): the oracle's memory-lean mode, and the file rewritten after
    every iteration, so a run stopped early still leaves a valid shorter
    trajectory (its "iters" = the records written)."""
    g = synth.generate(cfg)
    normA2 = oracle.frob2(g["a_val"])
    path = os.path.join(HERE, f"traj_{tag}.json")
    t0 = time.time()
    recs = []

    def write():
        out = dict(config=cfg.name, n=cfg.n, m=cfg.m, d=cfg.d, s=cfg.s, sigma=cfg.sigma, k=cfg.k, t=t,
                   iters=len(recs), seed=cfg.seed, rho=oracle.RHO_DEFAULT, normA2=normA2, records=recs,
                   oracle_seconds=time.time() - t0,
                   source="tests/golden/make_golden.py -> oracle.run (fp64 C oracle, Alg. 2 per-column, "
                          "P:122-144, P:304)" + (", lean memory mode" if lean else ""))
        with open(path + ".tmp", "w") as f:
            json.dump(out, f, indent=1)
        os.replace(path + ".tmp", path)
        print(path, len(recs), f"{out['oracle_seconds']:.1f}s", "E", recs[-1]["E"], flush=True)

    def on_record(rec):
        recs.append(rec)
        if lean:
            write()

    oracle.run(g, cfg.k, t, iters, seed=cfg.seed, lean=lean, on_record=on_record)
    write()


def main(which):
    C = synth.CONFIGS
    if "tiny" in which:
        run(C["tiny"], C["tiny"].t, C["tiny"].iters, "tiny")
    if "medium" in which:
        run(C["medium"], C["medium"].t, C["medium"].iters, "medium")
    if "sweep" in which:
        for t in synth.SWEEP_T:
            run(C["medium"], t, C["medium"].iters, f"sweep_t{'inf' if t is None else t}")
    if "large" in which:
        run(C["large"], C["large"].t, C["large"].iters, "large")
    if "box" in which:  # as many iterations as the host's time allows (the file grows per iteration)
        run(C["box"], C["box"].t, int(os.environ.get("BOX_ITERS", C["box"].iters)), "box", lean=True)


if __name__ == "__main__":
    main(sys.argv[1:] or ["tiny", "medium", "sweep"])
