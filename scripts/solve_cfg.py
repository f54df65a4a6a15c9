"""Diagnostics: one GPU solve of a BASELINE config (python scripts/solve_cfg.py CID [method] [max_iter])."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1912_04385_b200 import gen  # noqa: E402
from paper_1912_04385_b200.api import gpu  # noqa: E402

cid = int(sys.argv[1])
method = sys.argv[2] if len(sys.argv) > 2 else "cptr3-amg"
max_iter = int(sys.argv[3]) if len(sys.argv) > 3 else 500
api = gpu()
a, b, _ = gen.generate(cid)
t0 = time.time()
s = api.system(a).setup(method, b)
t1 = time.time()
r = s.solve(1e-8, max_iter)
t2 = time.time()
print(f"config {cid} {method}: setup {t1 - t0:.2f}s solve {t2 - t1:.2f}s iterations {r.iterations} "
      f"converged {r.converged} true_resid {r.final_true_residual:.3e}")
