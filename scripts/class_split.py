"""Diagnostics: per-kernel-class time split of one GPU solve (CUDA events per launch).

    python scripts/class_split.py CID [max_iter] [method] [reps]
"""
import ctypes as C
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1912_04385_b200 import gen  # noqa: E402
from paper_1912_04385_b200.api import gpu  # noqa: E402

KCLASS = ["spmv", "spmv_col", "ilu_fwd", "ilu_bwd", "gs", "csr", "coarse", "mgs", "blas1"]
cid = int(sys.argv[1])
max_iter = int(sys.argv[2]) if len(sys.argv) > 2 else 100
method = sys.argv[3] if len(sys.argv) > 3 else gen.CONFIG_METHODS[cid][-1]
reps = int(sys.argv[4]) if len(sys.argv) > 4 else 1
api = gpu()
a, b, _ = gen.generate(cid)
t0 = time.time()
s = api.system(a).setup(method, b)
print(f"c{cid} {method}: setup {time.time() - t0:.2f}s", flush=True)
s.solve(1e-8, 3)  # warm-up
for rep in range(reps):
    api.call("reset_stats", s.h)
    api.call("profile", s.h, 1)
    t0 = time.time()
    r = s.solve(1e-8, max_iter)
    wall = time.time() - t0
    api.call("profile", s.h, 0)
    tot = 0.0
    rows = []
    for k, name in enumerate(KCLASS):
        t, n, by = C.c_double(), C.c_int64(), C.c_double()
        api.call("kernel_stats", s.h, k, C.byref(t), C.byref(n), C.byref(by))
        tot += t.value
        rows.append((name, t.value, n.value, by.value))
    it = r.total_iterations
    print(f"solve: {it} iterations in {wall:.3f}s wall ({1e3 * wall / max(it, 1):.2f} ms/it), "
          f"kernel sum {tot:.1f} ms, last rel {r.residual_history[-1]:.8e}", flush=True)
    for name, ms, n, by in rows:
        if n:
            print(f"  {name:9s} {ms:9.2f} ms {100 * ms / max(tot, 1e-9):5.1f}%  {n:7d} launches  "
                  f"{by / max(ms, 1e-9) / 1e6:8.1f} GB/s  {ms / max(it, 1):7.3f} ms/it", flush=True)
