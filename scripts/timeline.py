"""Diagnostics: per-row completion timeline of one forward ILU sweep."""
import ctypes as C
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1912_04385_b200 import gen  # noqa: E402
from paper_1912_04385_b200.api import gpu  # noqa: E402

cid = int(sys.argv[1])
api = gpu()
a, b, _ = gen.generate(cid)
s = api.system(a).setup("ilu0", b)
f = api.lib.mprec_gpu_debug_ilu_timeline
f.argtypes = [C.c_void_p, C.c_int, C.c_void_p, C.c_void_p, C.c_void_p]
nc = a.n_cells
for blocks in [int(x) for x in sys.argv[2:]] or [0]:
    ts = np.zeros(2 * nc, np.int64)
    order = np.zeros(nc, np.int32)
    nlev = C.c_int()
    api.check(f(s.h, blocks, ts.ctypes.data, order.ctypes.data, C.byref(nlev)))
    t = ts[0::2]
    t = (t - t.min()) / 1e3  # us
    print(f"blocks={blocks} nlev={nlev.value} span={t.max():.1f} us  per-level={t.max()/nlev.value:.2f} us")
    q = np.quantile(t, [0.01, 0.1, 0.5, 0.9, 0.99])
    print("  completion quantiles (us):", np.round(q, 1))
    print("  first slots:", np.round(t[:12], 2))
    who = ts[1::2]
    print("  distinct SMs:", len(set((who // 1000000).tolist())), " distinct warps:", len(set(who.tolist())))
    dt = np.diff(np.sort(t))
    print("  max gap between consecutive completions (us):", round(float(dt.max()), 1))
