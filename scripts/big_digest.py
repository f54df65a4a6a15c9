"""Setup digests + GMRES history of one BASELINE config on one implementation.

    python scripts/big_digest.py IMPL CID [--iters K] [--out PATH] [--method M]

IMPL = gpu | oracle | ref.  Writes an .npz with sha256 digests of the scaled
system, the ILU(0) factors and every AMG level (C/F splitting, A_l, P_l, R_l),
the level sizes, and the solve result (history of the last attempt, per-attempt
data, a strided sample of x and its norm).  The digests of two implementations
are equal iff the setup is bitwise equal; tests/golden/make_big_golden.py turns
the oracle's file into the committed fixture.
"""
import argparse
import hashlib
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from paper_1912_04385_b200 import gen  # noqa: E402

X_STRIDE = 97


def digest(a) -> str:
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def bind(impl):
    if impl == "gpu":
        from paper_1912_04385_b200.api import gpu
        return gpu()
    import oracle
    return oracle.api() if impl == "oracle" else oracle.ref_api()


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("impl")
    ap.add_argument("cid", type=int)
    ap.add_argument("--iters", type=int, default=500)
    ap.add_argument("--method", default=None)
    ap.add_argument("--out", default=None)
    ap.add_argument("--no-setup-digest", action="store_true")
    args = ap.parse_args()
    api = bind(args.impl)
    method = args.method or gen.CONFIG_METHODS[args.cid][-1]
    out = args.out or os.path.join(ROOT, "gpurun_out", f"digest_{args.impl}_c{args.cid}_{method}.npz")
    os.makedirs(os.path.dirname(out), exist_ok=True)
    t0 = time.time()
    a, b, xs = gen.generate(args.cid)
    blob = {"input": digest(a.values) + digest(b), "method": method}
    print(f"generated c{args.cid} in {time.time() - t0:.1f}s", flush=True)
    s = api.system(a)
    a.values = None  # the implementation holds its own copy; keep host RAM for the oracle at c5
    t0 = time.time()
    s.setup(method, b)
    blob["setup_s"] = time.time() - t0
    print(f"{args.impl} setup {blob['setup_s']:.1f}s", flush=True)
    if not args.no_setup_digest:
        abar, bbar = s.scaled()
        blob["scaled"] = digest(abar) + digest(bbar)
        del abar
        blob["ilu"] = digest(s.ilu_values())
        for st in range(s.n_stages() - 1):
            try:
                h = s.stage_amg(st)
            except Exception:
                continue
            nl = h.n_levels
            blob[f"s{st}/sizes"] = np.array([h.level_info(l) for l in range(nl)], np.int64)
            for l in range(nl):
                for which in ([0] if l == 0 else [0, 1, 2]):
                    rp, ci, v = h.level_csr(l, which)
                    blob[f"s{st}/l{l}/w{which}"] = digest(rp) + digest(ci) + digest(v)
                if l + 1 < nl:
                    blob[f"s{st}/l{l}/cf"] = digest(h.cf(l))
        print(f"digests done", flush=True)
    t0 = time.time()
    r = s.solve(1e-8, args.iters)
    blob["solve_s"] = time.time() - t0
    blob["iterations"] = r.iterations
    blob["total_iterations"] = r.total_iterations
    blob["attempts"] = r.attempts
    blob["converged"] = int(r.converged)
    blob["breakdown"] = int(r.breakdown)
    blob["final_true_residual"] = r.final_true_residual
    blob["history"] = r.residual_history
    for key in ("attempt_iterations", "attempt_true_residual", "attempt_tol"):
        if hasattr(r, key):
            blob[key] = np.array(getattr(r, key))
    blob["x_norm"] = float(np.linalg.norm(r.x))
    blob["x_sample"] = r.x[::X_STRIDE].copy()
    blob["x_err_vs_xstar"] = float(np.linalg.norm(r.x - xs) / np.linalg.norm(xs))
    print(f"{args.impl} solve {blob['solve_s']:.1f}s: iterations {r.iterations} (total {r.total_iterations}, "
          f"attempts {r.attempts}) converged {r.converged} true {r.final_true_residual:.3e} "
          f"last rel {r.residual_history[-1]:.8e}", flush=True)
    np.savez_compressed(out, **blob)
    print("wrote", out)


if __name__ == "__main__":
    main()
