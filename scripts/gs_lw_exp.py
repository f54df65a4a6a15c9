"""Diagnostics: level-synchronous sweep programs (gs_ls.cu) with given group
counts / warps per group / dependency class, per AMG level, against the level's
current kernel.  python scripts/gs_lw_exp.py CID STAGE "NW[/ND]:K,K,..;NW:K,.." [LEVELS]
MPREC_LS_STATS=2 prints per-group timelines, MPREC_LS_TRACE=1 the program statistics."""
import ctypes as C
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1912_04385_b200 import gen  # noqa: E402
from paper_1912_04385_b200.api import gpu  # noqa: E402

cid, stage = int(sys.argv[1]), int(sys.argv[2])
combos = []
for part in sys.argv[3].split(";"):
    nw, ks = part.split(":")
    nd = 0
    if "/" in nw:
        nw, nd = nw.split("/")
    combos += [(int(nw), int(k), int(nd)) for k in ks.split(",")]
levels = [int(x) for x in sys.argv[4].split(",")] if len(sys.argv) > 4 else None
api = gpu()
a, b, _ = gen.generate(cid)
t0 = time.time()
s = api.system(a).setup("cptr3-amg", b)
print(f"setup {time.time() - t0:.1f}s", flush=True)
f = api.lib.mprec_gpu_debug_gs_ls
f.argtypes = [C.c_void_p, C.c_int, C.c_int, C.c_int, C.c_int, C.c_void_p]
h = s.stage_amg(stage)
fb = api.lib.mprec_gpu_debug_gs
fb.argtypes = [C.c_void_p, C.c_int, C.c_int, C.c_int] + [C.c_void_p] * 4
best_sum = cur_sum = 0.0
for l in range(h.n_levels - 1):
    if levels is not None and l not in levels:
        continue
    n, nnz, _ = h.level_info(l)
    best = cur = None
    mf, mb, nf, nbk = C.c_double(), C.c_double(), C.c_int(), C.c_int()
    api.check(fb(s.h, stage, l, 2, C.byref(mf), C.byref(mb), C.byref(nf), C.byref(nbk)))
    print(f"level {l:2d} n={n} nnz={nnz} DAG depth {nf.value} ({n / max(nf.value, 1):.0f} rows/level)", flush=True)
    for nw, K, nd in combos:
        if n < 64 * K:
            continue
        os.environ["MPREC_GS_LS_NW"] = str(nw)
        os.environ["MPREC_GS_LS_ND"] = str(nd)
        out = (C.c_double * 10)()
        api.check(f(s.h, stage, l, K, 4, out))
        if out[9] == 0:
            print(f"level {l:2d} n={n:8d} nw={nw} nd={nd} K={K:3d}: not eligible", flush=True)
            continue
        cur = out[2] + out[3]
        ls = out[0] + out[1]
        print(f"level {l:2d} n={n:8d} nw={nw} nd={nd} K={K:3d} W={int(out[6])} hmax={int(out[7])} steps={int(out[8]) % 1000000}: "
              f"fwd {out[0]:.3f} bwd {out[1]:.3f} ms | cur fwd {out[2]:.3f} bwd {out[3]:.3f} | err {out[4]:.1e} {out[5]:.1e}",
              flush=True)
        if out[4] < 1e-10 and out[5] < 1e-10 and (best is None or ls < best[0]):
            best = (ls, nw, nd, K)
    if cur is not None:
        cur_sum += cur
        best_sum += min(best[0], cur) if best else cur
        print(f"level {l:2d}: best {best}", flush=True)
print(f"sum fwd+bwd: current {cur_sum:.2f} ms, best variant {best_sum:.2f} ms")
