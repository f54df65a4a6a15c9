"""Setup digests + solve record of one BASELINE config on one implementation
(shared by scripts/big_digest.py, tests/golden/make_big_golden.py and
tests/test_gpu_big.py).

The record holds sha256 digests of the scaled system, the ILU(0) factors and
every AMG level (C/F splitting, A_l, P_l, R_l) -- equal digests mean a bitwise
equal setup -- plus the solve: per-attempt data, the residual history of the
last attempt, strided samples of x and (optionally) of M r and of every
stage's output for a seeded r.
"""
import hashlib

import numpy as np

from paper_1912_04385_b200 import gen

X_STRIDE = 97
APPLY_STRIDE = 997
SCALARS = ("setup_s", "solve_s", "iterations", "total_iterations", "attempts", "converged", "breakdown",
           "final_true_residual", "x_norm", "x_err_vs_xstar", "apply_norm", "perturb_seed")


def digest(a) -> str:
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def setup_digests(s) -> dict:
    out = {}
    abar, bbar = s.scaled()
    out["scaled"] = digest(abar) + digest(bbar)
    del abar
    out["ilu"] = digest(s.ilu_values())
    for st in range(s.n_stages() - 1):
        try:
            h = s.stage_amg(st)
        except Exception:  # -direct stage: no hierarchy
            continue
        nl = h.n_levels
        out[f"s{st}/sizes"] = np.array([h.level_info(l) for l in range(nl)], np.int64)
        for l in range(nl):
            for which in ([0] if l == 0 else [0, 1, 2]):
                rp, ci, v = h.level_csr(l, which)
                out[f"s{st}/l{l}/w{which}"] = digest(rp) + digest(ci) + digest(v)
            if l + 1 < nl:
                out[f"s{st}/l{l}/cf"] = digest(h.cf(l))
    return out


def levelset_digests(s) -> dict:
    """Digests of the level sets of every sequential sweep: the ILU(0) block DAG
    (ilu0.cpp:48-57) and Gauss-Seidel on every smoothed AMG level (amg.cpp:31-42),
    both directions, with the depths."""
    out = {}
    for d in (1, -1):
        lv, nl = s.levelsets(d)
        out[f"ilu/d{d}"] = digest(lv) + f":{nl}"
    for st in range(s.n_stages() - 1):
        try:
            h = s.stage_amg(st)
        except Exception:  # -direct stage
            continue
        for l in range(h.n_levels - 1):
            for d in (1, -1):
                lv, nl = h.levelsets(l, d)
                out[f"s{st}/l{l}/d{d}"] = digest(lv) + f":{nl}"
    return out


def run_case(api, cid, iters=500, method=None, setup_digest=True, apply_sample=False, perturb_seed=None, log=print):
    import time
    method = method or gen.CONFIG_METHODS[cid][-1]
    a, b, xs = gen.generate(cid)
    blob = {"input": digest(a.values) + digest(b), "method": method}
    if perturb_seed is not None:  # rounding-level perturbation of b (tests/ensemble.py)
        from tests.ensemble import perturbed
        b = perturbed(b, perturb_seed)
        blob["perturb_seed"] = perturb_seed
    s = api.system(a)
    a.values = None  # the implementation holds its own copy (host RAM for the oracle at c5)
    t0 = time.time()
    s.setup(method, b)
    blob["setup_s"] = time.time() - t0
    log(f"setup {blob['setup_s']:.1f}s")
    if setup_digest:
        blob.update(setup_digests(s))
    if apply_sample:
        r = np.random.default_rng(2024).uniform(-1.0, 1.0, s.a.dim)
        z = s.apply(r)
        blob["apply_norm"] = float(np.linalg.norm(z))
        blob["apply_sample"] = z[::APPLY_STRIDE].copy()
        for st in range(s.n_stages()):
            z = s.apply_stage(st, r)
            blob[f"stage{st}_norm"] = float(np.linalg.norm(z))
            blob[f"stage{st}_sample"] = z[::APPLY_STRIDE].copy()
        del z, r
    t0 = time.time()
    res = s.solve(1e-8, iters)
    blob["solve_s"] = time.time() - t0
    blob.update(iterations=res.iterations, total_iterations=res.total_iterations, attempts=res.attempts,
                converged=int(res.converged), breakdown=int(res.breakdown),
                final_true_residual=res.final_true_residual, history=res.residual_history,
                attempt_iterations=np.array(res.attempt_iterations),
                attempt_converged=np.array(res.attempt_converged, np.int8),
                attempt_tol=np.array(res.attempt_tol), attempt_true_residual=np.array(res.attempt_true_residual),
                x_norm=float(np.linalg.norm(res.x)), x_sample=res.x[::X_STRIDE].copy(),
                x_err_vs_xstar=float(np.linalg.norm(res.x - xs) / np.linalg.norm(xs)))
    log(f"solve {blob['solve_s']:.1f}s: iterations {res.iterations} (attempts {res.attempt_iterations}) "
        f"converged {res.converged} true {res.final_true_residual:.3e} last rel {res.residual_history[-1]:.8e}")
    return blob
