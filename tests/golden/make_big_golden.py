"""Generates tests/golden/big_c4.npz and big_c5.npz: the CPU oracle's record
(tests/bigcase.py) of BASELINE configs 4 and 5 -- setup digests (scaled
system, ILU(0) factors, every AMG level), the solve_system attempts and
histories, strided samples of x and of the preconditioner / stage outputs --
the committed target of tests/test_gpu_big.py.  The oracle is pinned to the
reference's own execution by tests/test_ref_pin.py.

    python tests/golden/make_big_golden.py [4] [5]

Cost in this container (1 core): c4 ~4 min (three attempts of ~75
iterations); c5 ~12 min (67 s setup, 40 iterations of ~15 s, ~45 GB RAM), plus
the same c5 run with b perturbed by 1e-15 (N(0,1) relative): the history's own
sensitivity to rounding-level changes.
"""
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)

import oracle  # noqa: E402
from tests.bigcase import run_case  # noqa: E402

C5_ITERS = 40


def main(cids):
    o = oracle.api()
    for cid in cids:
        if cid == 4:
            blob = run_case(o, 4, 500, apply_sample=True)
        else:
            blob = run_case(o, 5, C5_ITERS, apply_sample=True)
            pert = run_case(o, 5, C5_ITERS, setup_digest=False, perturb=1e-15)
            blob["perturbed_history"] = pert["history"]
        np.savez_compressed(os.path.join(HERE, f"big_c{cid}.npz"), **blob)
        print(f"c{cid}: iterations {blob['iterations']} attempts {blob['attempts']}", flush=True)


if __name__ == "__main__":
    main([int(a) for a in sys.argv[1:]] or [4, 5])
