"""Generates tests/golden/levelsets_c45.npz: digests (and depths) of the oracle's
level sets of every sequential sweep at BASELINE configs 4 and 5 -- the ILU(0)
block DAG and Gauss-Seidel on every smoothed level of both AMG hierarchies, both
directions (tests/bigcase.py:levelset_digests) -- the bit-exact target of
tests/test_gpu_big.py::test_levelsets_c4_c5.  Cost here: c4 ~5 s, c5 ~80 s setup
and ~45 GB of RAM.

    python tests/golden/make_levelset_golden.py
"""
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))

import oracle  # noqa: E402
from paper_1912_04385_b200 import gen  # noqa: E402
from tests.bigcase import levelset_digests  # noqa: E402


def main():
    o = oracle.api()
    blob = {}
    for cid in (4, 5):
        a, b, _ = gen.generate(cid)
        s = o.system(a)
        a.values = None
        s.setup(gen.CONFIG_METHODS[cid][-1], b)
        for k, v in levelset_digests(s).items():
            blob[f"c{cid}/{k}"] = v
        print(f"c{cid}: {sum(1 for k in blob if k.startswith(f'c{cid}/'))} level-set digests", flush=True)
        del s
    np.savez_compressed(os.path.join(HERE, "levelsets_c45.npz"), **blob)


if __name__ == "__main__":
    main()
