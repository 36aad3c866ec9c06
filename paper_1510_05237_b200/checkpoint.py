"""Checkpoint / resume of a solver run ("Checkpoint / resume").

The state an ALS run carries from one iteration to the next is the factor U
(Alg. 2: the next V side is computed from U alone) plus the telemetry
of the iterations so far.  ``save`` writes U and V as canonical column-major COO
``.npy`` arrays (row, col, val) and a JSON manifest (n, m, k, t, seed,
iterations, the last R and E, the records); ``resume`` creates a handle on the
same matrix and sets U, so the next ``iterate`` continues the run: its V side
starts from the saved U and its residual R is measured against it.

Host-side file handling only: the factors cross the C ABI through
``esnmf_get_U/V`` and ``esnmf_set_factor`` (include/esnmf.h)."""
from __future__ import annotations

import json
import os

import numpy as np

from .esnmf import ESNMF, ESNMF_SIDE_U

FORMAT = "esnmf-checkpoint-1"


def save(solver: ESNMF, path: str, seed: int | None = None) -> dict:
    """Write ``path``/U_{row,col,val}.npy, V_{...}.npy and manifest.json; returns the manifest."""
    os.makedirs(path, exist_ok=True)
    for name, (row, col, val) in (("U", solver.get_U()), ("V", solver.get_V())):
        np.save(os.path.join(path, f"{name}_row.npy"), np.asarray(row, np.int32))
        np.save(os.path.join(path, f"{name}_col.npy"), np.asarray(col, np.int32))
        np.save(os.path.join(path, f"{name}_val.npy"), np.asarray(val, np.float32))
    recs = solver.records()
    man = {
        "format": FORMAT,
        "n": int(solver.n), "m": int(solver.m), "k": int(solver.k),
        "t": None if solver.t is None else int(solver.t),
        "seed": seed,
        "iterations": len(recs),
        "R": recs[-1]["R"] if recs else None,
        "E": recs[-1]["E"] if recs else None,
        "records": recs,
    }
    with open(os.path.join(path, "manifest.json"), "w") as f:
        json.dump(man, f, indent=1)
    return man


def load(path: str) -> tuple[dict, dict]:
    """(manifest, {"U": (row, col, val), "V": (row, col, val)})."""
    with open(os.path.join(path, "manifest.json")) as f:
        man = json.load(f)
    if man.get("format") != FORMAT:
        raise ValueError(f"{path}: not an {FORMAT} checkpoint")
    fac = {}
    for name in ("U", "V"):
        fac[name] = tuple(np.load(os.path.join(path, f"{name}_{p}.npy")) for p in ("row", "col", "val"))
    return man, fac


def resume(path: str, inputs: dict, **kw) -> tuple[ESNMF, dict]:
    """A handle on ``inputs`` (the same matrix) whose U is the checkpoint's; the next
    ``iterate`` continues the saved run.  ``kw`` go to ``ESNMF`` (seed defaults to the
    manifest's).  Returns (solver, manifest)."""
    man, fac = load(path)
    kw.setdefault("seed", man["seed"] if man["seed"] is not None else 0)
    s = ESNMF(man["n"], man["m"], man["k"], man["t"], inputs, **kw)
    s.set_factor(ESNMF_SIDE_U, *fac["U"])
    return s, man
