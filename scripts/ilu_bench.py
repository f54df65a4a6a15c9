"""Diagnostics: ILU(0) apply timing, warp-per-block-row kernel vs the level-synchronous
programs (MPREC_ILU_LS=<groups>).  python scripts/ilu_bench.py CID"""
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1912_04385_b200 import gen  # noqa: E402
from paper_1912_04385_b200.api import gpu  # noqa: E402

cid = int(sys.argv[1]) if len(sys.argv) > 1 else 5
api = gpu()
a, b, _ = gen.generate(cid)
s = api.system(a).setup("ilu0", b)
r = np.random.default_rng(3).standard_normal(a.dim)
y0 = s.apply(r)
t0 = time.perf_counter()
for _ in range(5):
    y = s.apply(r)
dt = (time.perf_counter() - t0) / 5
print(f"config {cid} ilu0 apply ({os.environ.get('MPREC_ILU_LS', '0')} groups): {1e3 * dt:.2f} ms per apply (host round trip incl.)")
np.save(f"/tmp/ilu_y_{os.environ.get('MPREC_ILU_LS', '0')}.npy", y)
