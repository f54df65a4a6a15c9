"""Diagnostics: level-synchronous GS programs (gs_ls.cu) vs the current sweep
kernel, per AMG level.  python scripts/gs_ls_exp.py CID [stage] [K,K,...]"""
import ctypes as C
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1912_04385_b200 import gen  # noqa: E402
from paper_1912_04385_b200.api import gpu  # noqa: E402

cid = int(sys.argv[1])
stage = int(sys.argv[2]) if len(sys.argv) > 2 else 0
Ks = [int(k) for k in sys.argv[3].split(",")] if len(sys.argv) > 3 else [148, 74, 32, 16, 8, 4, 2, 1]
only = int(sys.argv[4]) if len(sys.argv) > 4 else -1  # a single level
api = gpu()
a, b, _ = gen.generate(cid)
t0 = time.time()
s = api.system(a).setup("cptr3-amg", b)
print(f"setup {time.time() - t0:.1f}s", flush=True)
f = api.lib.mprec_gpu_debug_gs_ls
f.argtypes = [C.c_void_p, C.c_int, C.c_int, C.c_int, C.c_int, C.c_void_p]
h = s.stage_amg(stage)
tot_cur = tot_best = 0.0
for l in range(h.n_levels - 1):
    if only >= 0 and l != only:
        continue
    n, nnz, _ = h.level_info(l)
    best = None
    cur = None
    for K in Ks:
        if n < 64 * K:
            continue
        out = (C.c_double * 10)()
        t0 = time.time()
        api.check(f(s.h, stage, l, K, 4, out))
        bt = time.time() - t0
        if out[9] == 0:
            print(f"level {l:2d} n={n:8d} K={K:3d}: not eligible", flush=True)
            continue
        cur = out[2] + out[3]
        ls = out[0] + out[1]
        print(f"level {l:2d} n={n:8d} nnz={nnz:9d} K={K:3d} W={int(out[6])} hmax={int(out[7])} steps={int(out[8])}: "
              f"ls fwd {out[0]:.3f} bwd {out[1]:.3f} ms | cur fwd {out[2]:.3f} bwd {out[3]:.3f} ms | "
              f"err {out[4]:.1e} {out[5]:.1e} | build+run {bt:.1f}s", flush=True)
        if best is None or ls < best:
            best = ls
    if cur is not None:
        tot_cur += cur
        tot_best += min(best, cur)
print(f"sum fwd+bwd: current {tot_cur:.2f} ms, with best ls {tot_best:.2f} ms")
