"""Diagnostics: per-band timeline of one forward band GS sweep."""
import ctypes as C
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1912_04385_b200 import gen  # noqa: E402
from paper_1912_04385_b200.api import gpu  # noqa: E402

cid, level = int(sys.argv[1]), int(sys.argv[2]) if len(sys.argv) > 2 else 0
api = gpu()
a, b, _ = gen.generate(cid)
s = api.system(a).setup("cptr3-amg", b)
f = api.lib.mprec_gpu_debug_band_timeline
f.argtypes = [C.c_void_p, C.c_int, C.c_int, C.c_void_p, C.c_void_p]
ts = np.zeros(3 * 4096 + 2 * 400000, np.int64)
nb = C.c_int()
api.check(f(s.h, 0, level, ts.ctypes.data, C.byref(nb)))
t = ts[:3 * nb.value].reshape(-1, 3)
t0 = t[:, 0].min()
st, en = (t[:, 0] - t0) / 1e3, (t[:, 1] - t0) / 1e3
for i in list(range(0, min(8, len(st)))) + list(range(len(st) - 3, len(st))):
    print(f"band {i:4d} start {st[i]:9.1f} us end {en[i]:9.1f} us dur {en[i]-st[i]:8.1f} chunks {t[i,2]}")
print("span", en.max(), "us; mean dur", (en - st).mean(), "us")
# band-0 per-chunk detail
n0 = int(t[0, 2])
d = ts[3 * nb.value: 3 * nb.value + 2 * n0].reshape(-1, 2)
prod, cons = (d[:, 0] - t0) / 1e3, (d[:, 1] - t0) / 1e3
print("band0 producer iteration dt (us): median", np.median(np.diff(prod)), " consumer chunk dt median", np.median(np.diff(cons)))
print("band0 first producer/consumer times:", np.round(prod[:6], 2), np.round(cons[:6], 2))
print("consumer lag behind producer (us) median:", np.median(cons - prod))
