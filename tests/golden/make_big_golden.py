"""Generates tests/golden/big_c4.npz and big_c5.npz: the CPU oracle's record
(tests/bigcase.py) of BASELINE configs 4 and 5 -- setup digests (scaled
system, ILU(0) factors, every AMG level), the solve_system attempts and
histories, strided samples of x and of the preconditioner / stage outputs --
the committed target of tests/test_gpu_big.py.  The oracle is pinned to the
reference's own execution by tests/test_ref_pin.py.

    python tests/golden/make_big_golden.py [4] [5]

Each record also holds the same solve with b perturbed by 1e-15 (N(0,1)
relative; tests/ensemble.py) -- 3 runs at c4, 1 at c5 --: the oracle's own
sensitivity to rounding-level changes, the band the GPU is held to.
Cost in this container (1 core): c4 ~16 min (4 x three attempts of ~75
iterations); c5 ~25 min (2 x (67 s setup + 40 iterations of ~15 s), ~45 GB RAM).
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
C4_PERTURBED = 3
C5_PERTURBED = 1


def main(cids):
    o = oracle.api()
    for cid in cids:
        iters, npert = (500, C4_PERTURBED) if cid == 4 else (C5_ITERS, C5_PERTURBED)
        blob = run_case(o, cid, iters, apply_sample=True)
        # the oracle's own rounding band (tests/ensemble.py): the same solve with
        # b perturbed by 1e-15
        for s in range(npert):
            pert = run_case(o, cid, iters, setup_digest=False, perturb_seed=s)
            blob[f"pert{s}_history"] = pert["history"]
            blob[f"pert{s}_attempt_iterations"] = pert["attempt_iterations"]
            blob[f"pert{s}_final_true_residual"] = pert["final_true_residual"]
            blob[f"pert{s}_attempt_true_residual"] = pert["attempt_true_residual"]
            blob[f"pert{s}_x_sample"] = pert["x_sample"]
        if cid == 5:  # keep the committed record small: every 970th entry of x
            for key in [k for k in blob if k.endswith("x_sample")]:
                blob[key] = blob[key][::10]
            blob["x_sample_stride"] = np.int64(970)
        np.savez_compressed(os.path.join(HERE, f"big_c{cid}.npz"), **blob)
        print(f"c{cid}: iterations {blob['iterations']} attempts {blob['attempts']}", flush=True)


if __name__ == "__main__":
    main([int(a) for a in sys.argv[1:]] or [4, 5])
