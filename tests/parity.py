"""Comparison rules for GPU-vs-oracle parity (BJ:5, reading C15).

* products (pre-clamp LS rows): per column c,
      max_j |gpu[j,c] - ref[j,c]| <= PROD_TOL * max_j |ref[j,c]|
* retained factor entries: per entry |gpu - ref| <= ENTRY_TOL * |ref|; in a
  column that keeps ALL its positives (#positive <= t, or t unlimited) entries
  near zero are kept too, and there the bar is
  ENTRY_TOL * |ref| + TIE_TOL * max_j |ref[j,c]| (an fp32 LS entry carries an
  absolute error ~1e-7 of its column's scale, reading C15)
* retained support: identical, except swaps between entries whose oracle
  values differ by <= TIE_TOL * max_j |ref[j,c]| (near-ties); in a column that
  keeps all its positives the threshold is zero, and an entry within
  TIE_TOL * max_j |ref[j,c]| of zero may be kept on one side only
* trajectory: |E_gpu - E_ref| <= TRAJ_TOL * E_ref per iteration (BJ:5).
* residual R FROM THE SAME STATE (one iteration from the GPU's factor):
  |R_gpu - R_ref| <= TRAJ_TOL * R_ref + 2 * ENTRY_TOL * (1 + R_ref): R is a
  difference of two factors that each carry the per-entry ENTRY_TOL, so
  ||U_i - U_{i-1}|| may move by ENTRY_TOL (||U_i|| + ||U_{i-1}||); late
  iterations have R ~ 1e-4, where that term, not 1e-3 R, is the bound.
* residual along a whole TRAJECTORY (50 iterations from U_0): not a parity
  quantity.  The two runs' supports may differ by near-tie swaps (the selection
  rule above), and late in a run, where R is small, a swapped threshold entry is
  a large part of ||U_i - U_{i-1}||: the GPU's R differed from the oracle's run
  by up to 41 % on the Medium sweep (t = 10,000, R ~ 3e-3, iteration 32;
  DESIGN.md section 4) while E -- BJ:5's trajectory criterion -- stayed within
  1e-3.  So R_1 (both runs start from U_0) and R one iteration past the end of
  every trajectory, from the GPU's state, are the R checks (r_close).
"""
import numpy as np

PROD_TOL = 1e-5
ENTRY_TOL = 1e-5
TIE_TOL = 1e-6
TRAJ_TOL = 1e-3


def r_close(r_gpu: float, r_ref: float) -> bool:
    """Residual R of one iteration from the same state (module doc)."""
    return abs(r_gpu - r_ref) <= TRAJ_TOL * r_ref + 2 * ENTRY_TOL * (1 + r_ref)


def coo_dense(shape, row, col, val):
    F = np.zeros(shape, np.float64)
    F[np.asarray(row, np.int64), np.asarray(col, np.int64)] = val
    return F


def check_products(gpu: np.ndarray, ref: np.ndarray, tol: float = PROD_TOL) -> float:
    """Returns the worst column-relative error; asserts it is <= tol."""
    scale = np.abs(ref).max(axis=0)
    scale[scale == 0] = 1.0
    err = (np.abs(gpu.astype(np.float64) - ref) / scale).max()
    assert err <= tol, f"LS column-relative error {err:.3e} > {tol:.0e}"
    return float(err)


def check_canonical(row, col, k):
    row, col = np.asarray(row), np.asarray(col)
    key = col.astype(np.int64) * (1 << 32) + row
    assert np.all(np.diff(key) > 0), "factor COO not in canonical (column, row) order"
    assert col.min(initial=0) >= 0 and col.max(initial=0) < k


def check_selection(gpu_F: np.ndarray, ref_F: np.ndarray, ref_ls: np.ndarray, t: int | None):
    """gpu_F, ref_F dense factors after clamp + top-t; ref_ls the oracle's pre-clamp LS."""
    assert np.all(gpu_F >= 0)
    swaps = 0
    worst = 0.0
    for c in range(ref_F.shape[1]):
        scale = max(np.abs(ref_ls[:, c]).max(), 1e-300)
        g, r = gpu_F[:, c] > 0, ref_F[:, c] > 0
        if t is not None:
            assert g.sum() <= t
        keeps_all = t is None or int((ref_ls[:, c] > 0).sum()) <= t
        if keeps_all:
            # the threshold is zero: an entry within an fp32 LS entry's error of zero
            # (TIE_TOL of the column scale, reading C15) may take either sign
            differ = np.nonzero(g != r)[0]
            assert np.all(np.abs(ref_ls[differ, c]) <= TIE_TOL * scale), f"column {c}: kept set differs off zero"
            swaps += len(differ)
            g = r = g & r
        assert g.sum() == r.sum(), f"column {c}: {g.sum()} kept vs oracle {r.sum()}"
        only_g = np.nonzero(g & ~r)[0]
        only_r = np.nonzero(r & ~g)[0]
        if len(only_g):
            # every swap must be a near-tie around the oracle's threshold
            thr = ref_F[r, c].min()
            assert np.all(np.abs(ref_ls[only_g, c] - thr) <= TIE_TOL * scale + 1e-300), f"column {c}: non-tie swap"
            assert np.all(np.abs(ref_ls[only_r, c] - thr) <= TIE_TOL * scale + 1e-300), f"column {c}: non-tie swap"
            swaps += len(only_g)
        both = g & r
        if both.any():
            slack = (TIE_TOL / ENTRY_TOL) * scale if keeps_all else 0.0
            rel = np.abs(gpu_F[both, c] - ref_F[both, c]) / (ref_F[both, c] + slack)
            worst = max(worst, float(rel.max()))
    assert worst <= ENTRY_TOL, f"retained entry relative error {worst:.3e} > {ENTRY_TOL:.0e}"
    return swaps, worst


def assert_kept_values(kept_vals, ls_vals, col_scale):
    """A kept factor entry is its LS entry: bitwise, or -- on the paper-order V
    side, whose kept values are recomputed exactly after the selection
    (k_polish_v) -- within the product tolerance of the
    tensor-core LS value the selection used: the LS value's own tolerance,
    PROD_TOL of its column's scale."""
    kv = np.asarray(kept_vals, np.float64)
    lv = np.asarray(ls_vals, np.float64)
    assert np.all(np.abs(kv - lv) <= ENTRY_TOL * np.abs(lv) + PROD_TOL * col_scale), "kept value != its LS entry"


def check_topt_property(ls: np.ndarray, F: np.ndarray, t: int | None):
    """Selection validity on the GPU's own LS values (any size): exactly
    min(t, #positive) kept per column, kept values are the LS values
    (assert_kept_values), every kept LS value >= every dropped positive, ties at
    the threshold -> lower rows."""
    for c in range(ls.shape[1]):
        x = ls[:, c]
        pos = x > 0
        kept = F[:, c] > 0
        npos = int(pos.sum())
        want = npos if t is None else min(t, npos)
        assert kept.sum() == want, f"column {c}: kept {kept.sum()} want {want}"
        assert_kept_values(F[kept, c], x[kept], np.abs(x).max())
        dropped = pos & ~kept
        if kept.any() and dropped.any():
            kmin = x[kept].min()
            assert kmin >= x[dropped].max()     # on the values the selection used
            tie_dropped = np.nonzero(dropped & (x == kmin))[0]
            tie_kept = np.nonzero(kept & (x == kmin))[0]
            if len(tie_dropped):
                assert tie_kept.max() < tie_dropped.min(), f"column {c}: tie not broken toward lower rows"


def check_topt_property_coo(ls: np.ndarray, row, col, val, t: int | None):
    """check_topt_property for a factor given as canonical COO (rows x k too large
    to densify on the host, e.g. Box's 8M x 200 V): the same four conditions."""
    row = np.asarray(row, np.int64)
    col = np.asarray(col, np.int64)
    val = np.asarray(val)
    order = np.argsort(col, kind="stable")
    bounds = np.searchsorted(col[order], np.arange(ls.shape[1] + 1))
    for c in range(ls.shape[1]):
        sel = order[bounds[c]:bounds[c + 1]]
        kr, kv = row[sel], val[sel]
        x = np.ascontiguousarray(ls[:, c])
        npos = int(np.count_nonzero(x > 0))
        want = npos if t is None else min(t, npos)
        assert len(kr) == want, f"column {c}: kept {len(kr)} want {want}"
        assert np.all(kv > 0)
        assert_kept_values(kv, x[kr], np.abs(x).max())
        if len(kr) and want < npos:
            kl = x[kr]                         # the LS values the selection used
            kmin = kl.min()
            x[kr] = -np.inf
            assert kmin >= x.max(), f"column {c}: dropped positive above the kept minimum"
            tie_dropped = np.nonzero(x == kmin)[0]
            if len(tie_dropped):
                assert kr[kl == kmin].max() < tie_dropped.min(), f"column {c}: tie not broken toward lower rows"
