"""Setup/solve timing probe (diagnostics): python scripts/probe.py CONFIG [method] [max_iter]
Run with MPREC_TRACE=1 for per-phase setup timings."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import ctypes as C  # noqa: E402

from paper_1912_04385_b200 import gen  # noqa: E402
from paper_1912_04385_b200.api import gpu  # noqa: E402

KC = ["spmv", "spmv_col", "ilu_fwd", "ilu_bwd", "gs", "csr", "coarse", "mgs", "blas1"]
cid = int(sys.argv[1])
method = sys.argv[2] if len(sys.argv) > 2 else gen.CONFIG_METHODS[cid][-1]
max_iter = int(sys.argv[3]) if len(sys.argv) > 3 else 500
t0 = time.time()
a, b, xs = gen.generate(cid)
print(f"gen {time.time()-t0:.2f}s nnzb={a.nnzb}", flush=True)
api = gpu()
t0 = time.time()
s = api.system(a)
print(f"create {time.time()-t0:.2f}s", flush=True)
t0 = time.time()
s.setup(method, b)
print(f"setup {time.time()-t0:.2f}s", flush=True)
for st in range(s.n_stages() - 1):
    h = s.stage_amg(st)
    print("  stage", st, [h.level_info(l) for l in range(h.n_levels)], flush=True)
api.call("profile", s.h, 1)
t0 = time.time()
r = s.solve(1e-8, max_iter)
el = time.time() - t0
print(f"solve {el:.2f}s its={r.iterations} total={r.total_iterations} att={r.attempts} conv={r.converged} "
      f"true={r.final_true_residual:.2e} it/s={r.total_iterations/el:.1f}", flush=True)
tot = 0.0
for k, n in enumerate(KC):
    t, L, by = C.c_double(), C.c_int64(), C.c_double()
    api.call("kernel_stats", s.h, k, C.byref(t), C.byref(L), C.byref(by))
    tot += t.value
    gbs = by.value / t.value / 1e6 if t.value else 0
    print(f"  {n:9s} {t.value:10.1f} ms {L.value:8d} launches {gbs:8.1f} GB/s", flush=True)
print(f"  total kernel ms {tot:.1f}")
