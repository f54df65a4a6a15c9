"""Diagnostics: per-segment timeline of the band-segment GS sweep (level 0 grid lines).
MPREC_GS_MODE=seg python scripts/segtl.py CID [stage] [level] [nx]"""
import ctypes as C
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1912_04385_b200 import gen  # noqa: E402
from paper_1912_04385_b200.api import gpu  # noqa: E402

cid = int(sys.argv[1])
stage = int(sys.argv[2]) if len(sys.argv) > 2 else 0
level = int(sys.argv[3]) if len(sys.argv) > 3 else 0
per_line = int(sys.argv[4]) if len(sys.argv) > 4 else 63
api = gpu()
a, b, _ = gen.generate(cid)
s = api.system(a).setup("cptr3-amg", b)
n = s.stage_amg(stage).level_info(level)[0]
buf = np.zeros(4 * n, dtype=np.int64)
f = api.lib.mprec_gpu_debug_seg_timeline
f.argtypes = [C.c_void_p, C.c_int, C.c_int, C.c_void_p, C.c_void_p]
ns = C.c_int()
api.check(f(s.h, stage, level, buf.ctypes.data, C.byref(ns)))
nseg = ns.value
tl = buf[: 4 * nseg].reshape(-1, 4)
t0 = tl[:, 0].min()
claim, first, end = (tl[:, 0] - t0) / 1e3, (tl[:, 1] - t0) / 1e3, (tl[:, 2] - t0) / 1e3
rounds = tl[:, 3]
band = np.zeros(nseg, dtype=np.int64)
pct = lambda x: "p10 %.2f p50 %.2f p90 %.2f" % tuple(np.percentile(x, [10, 50, 90]))
print(f"n={n} nseg={nseg} total {end.max():.1f} us")
print("rounds per segment:", pct(rounds) if False else np.percentile(rounds, [10, 50, 90]))


print("claim->first us:", pct(first - claim))
print("first->end us:", pct(end - first))
print("claim->end us:", pct(end - claim))
for k in [0, 1, 2, per_line, per_line + 1, 2 * per_line, 3 * per_line, 4 * per_line, 5 * per_line, 8 * per_line, 9 * per_line]:
    if k < nseg:
        print(f"seg {k:6d} band {band[k]:4d}: claim {claim[k]:8.2f} first {first[k]:8.2f} end {end[k]:8.2f}")
y0 = np.arange(0, nseg, per_line)
d = np.diff(first[y0])
print("first-row step between consecutive lines (s=0): p10 %.2f p50 %.2f p90 %.2f us" % tuple(np.percentile(d, [10, 50, 90])))
last = np.arange(per_line - 1, nseg, per_line)
print("end of last segment per line: per line %.3f us" % ((end[last[-1]] - end[last[0]]) / (len(last) - 1)))

B = int(os.environ.get("MPREC_GS_SEG_B", "8192"))
nxl = int(os.environ.get("NX", "2000"))
# per grid line y (segment s=0 of line y starts at row y*nx): band-relative line index
lines = np.arange(1, len(y0))
rows0 = lines * nxl
band_of = np.searchsorted(np.cumsum([0]), 0)
step = first[y0[1:]] - first[y0[:-1]]
# a line whose first row shares the band with the previous line's first row -> in-band hop
inband = (rows0 // B) == ((rows0 - nxl) // B)
print("line step in-band:   p50 %.2f mean %.2f us (%d lines)" % (np.median(step[inband]), step[inband].mean(), inband.sum()))
print("line step crossing:  p50 %.2f mean %.2f us (%d lines)" % (np.median(step[~inband]), step[~inband].mean(), (~inband).sum()))
ch = end - first
print("segment first->end us: p50 %.2f" % np.median(ch))
