"""Rounding-sensitivity band of the oracle (test infrastructure).

On ill-conditioned members of the config-4/5 family (reaction band, nb = 8)
GMRES's iteration count is itself sensitive to rounding: perturbing b by
1e-15 (relative, N(0,1)) moves the oracle's first solve_system attempt on
g60x60_nb8_band_s1 anywhere in 87..100 iterations.  A GPU run -- whose sums
associate differently (warp reductions, the Gram form of MGS, the LS sweep
programs) -- is a rounding-level perturbation of the same kind, so it is held
to the oracle's own band: iterations within [min - 1, max + 1] of the
ensemble {unperturbed, K perturbed} and, per history entry, a deviation from
the unperturbed oracle no larger than the ensemble's own spread (times a
margin) or a floor.
"""
import numpy as np

PERTURB = 1e-15


def perturbed(b, seed):
    return b * (1.0 + PERTURB * np.random.default_rng(1000 + seed).standard_normal(b.size))


def oracle_ensemble(orc, a, b, method, k=6, **setup_kw):
    """[unperturbed, k perturbed] oracle SolveResults of solve_system."""
    runs = [orc.system(a).setup(method, b, **setup_kw).solve()]
    for s in range(k):
        runs.append(orc.system(a).setup(method, perturbed(b, s), **setup_kw).solve())
    return runs


def iteration_band(runs, attr="attempt_iterations"):
    vals = np.array([list(getattr(r, attr)) for r in runs if len(getattr(r, attr)) == len(getattr(runs[0], attr))])
    return vals.min(axis=0), vals.max(axis=0)


def history_spread(hists):
    """Per-entry relative spread of an ensemble of histories (over the common length)."""
    m = min(len(h) for h in hists)
    h0 = np.asarray(hists[0][:m])
    dev = np.zeros(m)
    for h in hists[1:]:
        dev = np.maximum(dev, np.abs(np.asarray(h[:m]) - h0) / np.maximum(np.abs(h0), 1e-300))
    return dev


def check_history(hg, hists, margin=100.0, floor=1e-8):
    """The GPU history deviates from the unperturbed oracle by no more than
    margin x the ensemble's own spread (running max, so the bound never
    shrinks along the solve) or floor; returns the worst ratio."""
    spread = np.maximum.accumulate(history_spread(hists))
    h0 = np.asarray(hists[0])
    m = min(len(hg), len(h0), len(spread))
    dev = np.abs(np.asarray(hg[:m]) - h0[:m]) / np.maximum(np.abs(h0[:m]), 1e-300)
    bound = np.maximum(margin * spread[:m], floor)
    bad = np.nonzero(dev > bound)[0]
    assert bad.size == 0, (f"history entry {bad[0]}: gpu {hg[bad[0]]!r} oracle {h0[bad[0]]!r} "
                           f"dev {dev[bad[0]]:.3e} > bound {bound[bad[0]]:.3e}")
    return float(np.max(dev / bound)) if m else 0.0
