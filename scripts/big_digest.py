"""Setup digests + solve record of one BASELINE config on one implementation.

    python scripts/big_digest.py IMPL CID [--iters K] [--out PATH] [--method M]
                                 [--apply-sample] [--perturb-seed S] [--no-setup-digest]

IMPL = gpu | oracle | ref.  Writes the record of tests/bigcase.py as .npz.
"""
import argparse
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from tests.bigcase import run_case  # noqa: E402


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
    ap.add_argument("--apply-sample", action="store_true")
    ap.add_argument("--perturb-seed", type=int, default=None)
    args = ap.parse_args()
    blob = run_case(bind(args.impl), args.cid, args.iters, args.method, not args.no_setup_digest,
                    args.apply_sample, args.perturb_seed, log=lambda m: print(f"{args.impl}: {m}", flush=True))
    out = args.out or os.path.join(ROOT, "gpurun_out", f"digest_{args.impl}_c{args.cid}_{blob['method']}.npz")
    os.makedirs(os.path.dirname(out), exist_ok=True)
    np.savez_compressed(out, **blob)
    print("wrote", out)


if __name__ == "__main__":
    main()
