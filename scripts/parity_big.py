"""Diagnostics: GPU vs oracle on a BASELINE config at full size (setup bitwise,
preconditioner apply, first GMRES iterations).  python scripts/parity_big.py CID [method] [iters]"""
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1912_04385_b200 import gen  # noqa: E402
from paper_1912_04385_b200.api import gpu  # noqa: E402
import oracle  # noqa: E402

cid = int(sys.argv[1])
method = sys.argv[2] if len(sys.argv) > 2 else "cptr3-amg"
iters = int(sys.argv[3]) if len(sys.argv) > 3 else 3
a, b, xs = gen.generate(cid)
g, o = gpu(), oracle.api()
t0 = time.time(); sg = g.system(a).setup(method, b); print(f"gpu setup {time.time()-t0:.1f}s", flush=True)
t0 = time.time(); so = o.system(a).setup(method, b); print(f"orc setup {time.time()-t0:.1f}s", flush=True)
ag, bg = sg.scaled(); ao, bo = so.scaled()
print("scaled bitwise:", np.array_equal(ag, ao), np.array_equal(bg, bo), flush=True)
del ag, ao
for st in range(so.n_stages() - 1):
    hg, ho = sg.stage_amg(st), so.stage_amg(st)
    same = hg.n_levels == ho.n_levels and all(np.array_equal(hg.cf(l), ho.cf(l)) for l in range(ho.n_levels - 1))
    print(f"stage {st}: levels {hg.n_levels}/{ho.n_levels} C/F bitwise {same}", flush=True)
print("ilu bitwise:", np.array_equal(sg.ilu_values(), so.ilu_values()), flush=True)
r = np.random.default_rng(1).uniform(-1, 1, a.dim)
t0 = time.time(); zg = sg.apply(r); tg = time.time() - t0
t0 = time.time(); zo = so.apply(r); to = time.time() - t0
print(f"apply rel diff {np.linalg.norm(zg-zo)/np.linalg.norm(zo):.3e}  gpu {tg:.3f}s orc {to:.1f}s", flush=True)
for st in range(so.n_stages()):
    d = np.linalg.norm(sg.apply_stage(st, r) - so.apply_stage(st, r)) / np.linalg.norm(so.apply_stage(st, r))
    print(f"  stage {st} rel diff {d:.3e}", flush=True)
t0 = time.time(); rg = sg.solve(1e-8, iters); tg = time.time() - t0
t0 = time.time(); ro = so.solve(1e-8, iters); to = time.time() - t0
print("gpu hist", rg.residual_history, f"{tg:.2f}s")
print("orc hist", ro.residual_history, f"{to:.2f}s")
print("x rel diff", np.linalg.norm(rg.x - ro.x) / max(np.linalg.norm(ro.x), 1e-300))
