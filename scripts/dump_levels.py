"""Dump the AMG level operators and their sweep level sets of one config from the
CPU oracle (input of scripts/ls_sim.py).  python scripts/dump_levels.py CID STAGE OUTDIR"""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import oracle  # noqa: E402
from paper_1912_04385_b200 import gen  # noqa: E402

cid, st, out = int(sys.argv[1]), int(sys.argv[2]), sys.argv[3]
os.makedirs(out, exist_ok=True)
o = oracle.api()
a, b, _ = gen.generate(cid)
s = o.system(a).setup(gen.CONFIG_METHODS[cid][-1], b)
h = s.stage_amg(st)
for l in range(h.n_levels - 1):
    rp, ci, v = h.level_csr(l, 0)
    lf, nf = h.levelsets(l, 1)
    lb, nb = h.levelsets(l, -1)
    np.savez(os.path.join(out, f"c{cid}_s{st}_l{l}.npz"), rp=rp, ci=ci, v=v, lf=lf, lb=lb)
    print(l, len(rp) - 1, len(ci), nf, nb, flush=True)
