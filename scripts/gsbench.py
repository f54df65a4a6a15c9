"""Diagnostics: GS sweep time per AMG level.  python scripts/gsbench.py CID [stage]"""
import ctypes as C
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1912_04385_b200 import gen  # noqa: E402
from paper_1912_04385_b200.api import gpu  # noqa: E402

cid = int(sys.argv[1])
stage = int(sys.argv[2]) if len(sys.argv) > 2 else 0
api = gpu()
a, b, _ = gen.generate(cid)
s = api.system(a).setup("cptr3-amg", b)
f = api.lib.mprec_gpu_debug_gs
f.argtypes = [C.c_void_p, C.c_int, C.c_int, C.c_int] + [C.c_void_p] * 4
h = s.stage_amg(stage)
tot = 0.0
for l in range(h.n_levels - 1):
    mf, mb, nf, nbk = C.c_double(), C.c_double(), C.c_int(), C.c_int()
    api.check(f(s.h, stage, l, 3, C.byref(mf), C.byref(mb), C.byref(nf), C.byref(nbk)))
    n, nnz, _ = h.level_info(l)
    tot += mf.value + mb.value
    print(f"level {l:2d} n={n:8d} nnz={nnz:9d} fwd {mf.value:7.3f} ms ({nf.value} lev, {1e3*mf.value/max(nf.value,1):.2f} us/lev)"
          f"  bwd {mb.value:7.3f} ms ({nbk.value} lev)", flush=True)
print(f"sum fwd+bwd over levels: {tot:.2f} ms (x2 per V-cycle)")
