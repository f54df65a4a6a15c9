"""Diagnostics: sweep the segment-chain GS launch parameters on one system.
python scripts/segsweep.py CID stage levels..."""
import ctypes as C
import itertools
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
os.environ["MPREC_GS_MODE"] = "seg"
from paper_1912_04385_b200 import gen  # noqa: E402
from paper_1912_04385_b200.api import gpu  # noqa: E402

cid, stage = int(sys.argv[1]), int(sys.argv[2])
levels = [int(x) for x in sys.argv[3:]] or [0, 1, 2]
api = gpu()
a, b, _ = gen.generate(cid)
s = api.system(a).setup("cptr3-amg", b)
f = api.lib.mprec_gpu_debug_gs
f.argtypes = [C.c_void_p, C.c_int, C.c_int, C.c_int] + [C.c_void_p] * 4
for wp, slp in itertools.product([int(x) for x in os.environ.get("SW_WARPS", "8 16").split()], [int(x) for x in os.environ.get("SW_SLP", "0 50 200").split()]):
    os.environ["MPREC_GS_SEG_WARPS"] = str(wp)
    os.environ["MPREC_GS_SEG_SLEEP"] = str(slp)
    blk = wp
    win = 0
    out = []
    for l in levels:
        mf, mb, nf, nbk = C.c_double(), C.c_double(), C.c_int(), C.c_int()
        api.check(f(s.h, stage, l, 3, C.byref(mf), C.byref(mb), C.byref(nf), C.byref(nbk)))
        out.append(f"L{l} {mf.value:6.3f}/{mb.value:6.3f}")
    print(f"warps {wp:2d} sleep {slp:3d}: " + "  ".join(out), flush=True)
