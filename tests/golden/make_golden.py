"""Generates tests/golden/oracle_golden.npz: oracle results on small members of
the BASELINE generator family and config 1 (iteration counts, residual
histories, C/F splittings, level sizes, digests of the scaled system and ILU
factors).  The reference cannot be built here, so these fixtures
pin the ORACLE across hosts (this container vs the GPU box) and give the GPU
parity tests a committed target; the oracle itself is pinned by the
reference's known-answer tests (tests/test_kat.py).

    python tests/golden/make_golden.py
"""
import hashlib
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)

from paper_1912_04385_b200 import gen  # noqa: E402
import oracle  # noqa: E402

CASES = {
    "c1_cpr": (1, "cpr-amg", {}),
    "g12x10_cpr": (dict(nx=12, ny=10, nb=4, kappa=1.0, perm_sigma=1.0, band=True, seed=7), "cpr-amg",
                   dict(max_coarse_size=40)),
    "g12x10_cptr3": (dict(nx=12, ny=10, nb=4, kappa=1.0, perm_sigma=1.0, band=True, seed=7), "cptr3-amg",
                     dict(max_coarse_size=40)),
    "g20x20_cptr3_hiPe": (dict(nx=20, ny=20, nb=4, kappa=1e-3, perm_sigma=2.0, band=False, seed=2), "cptr3-amg",
                          dict(max_coarse_size=40)),
    "g16x16_nb8_cptr3": (dict(nx=16, ny=16, nb=8, kappa=1.0, perm_sigma=1.5, band=True, seed=4), "cptr3-amg",
                         dict(max_coarse_size=40)),
}


def digest(a: np.ndarray) -> str:
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def system(spec):
    return gen.generate(spec if isinstance(spec, int) else gen.make_spec(**spec))


def run_case(api, spec, method, amg):
    a, b, xs = system(spec)
    s = api.system(a).setup(method, b, **amg)
    r = s.solve()
    out = {"iterations": r.iterations, "total_iterations": r.total_iterations, "attempts": r.attempts,
           "converged": int(r.converged), "history": r.residual_history, "x": r.x,
           "input_digest": digest(a.values) + digest(b)}
    abar, bbar = s.scaled()
    out["scaled_digest"] = digest(abar) + digest(bbar)
    out["ilu_digest"] = digest(s.ilu_values())
    cfs, sizes = [], []
    for st in range(s.n_stages() - 1):
        h = s.stage_amg(st)
        sizes.append([h.level_info(l) for l in range(h.n_levels)])
        cfs.append([np.packbits(h.cf(l).astype(np.uint8)) for l in range(h.n_levels - 1)])
    out["level_sizes"] = sizes
    out["cf"] = cfs
    return out


def main():
    o = oracle.api()
    blob = {}
    for name, (spec, method, amg) in CASES.items():
        r = run_case(o, spec, method, amg)
        for k, v in r.items():
            if k == "cf":
                for st, levels in enumerate(v):
                    for l, bits in enumerate(levels):
                        blob[f"{name}/cf/{st}/{l}"] = bits
            elif k == "level_sizes":
                for st, lv in enumerate(v):
                    blob[f"{name}/sizes/{st}"] = np.array(lv, np.int64)
            else:
                blob[f"{name}/{k}"] = np.array(v)
        print(name, r["iterations"], r["converged"])
    np.savez_compressed(os.path.join(os.path.dirname(os.path.abspath(__file__)), "oracle_golden.npz"), **blob)


if __name__ == "__main__":
    main()
