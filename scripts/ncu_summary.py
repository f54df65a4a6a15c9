"""Summarise an ncu launch-list CSV (--metrics gpu__time_duration.sum) by kernel."""
import collections
import csv
import json
import re
import sys

rows = list(csv.reader(open(sys.argv[1])))
hdr_i = [i for i, r in enumerate(rows) if r and r[0] == "ID"][0]
hdr, data = rows[hdr_i], rows[hdr_i + 1:]
ki, mi, ui = hdr.index("Kernel Name"), hdr.index("Metric Value"), hdr.index("Metric Unit")
scale = {"nsecond": 1e-3, "ns": 1e-3, "usecond": 1.0, "us": 1.0, "msecond": 1e3, "ms": 1e3, "second": 1e6, "s": 1e6}
agg = collections.defaultdict(lambda: [0, 0.0])
for r in data:
    if len(r) <= mi:
        continue
    name = r[ki]
    m = re.search(r"(k_\w+)(<[^>]*>)?", name)
    short = (m.group(1) + (m.group(2) or "")) if m else name[:40]
    agg[short][0] += 1
    agg[short][1] += float(r[mi].replace(",", "")) * scale[r[ui]]
tot = sum(a[1] for a in agg.values())
out = {"total_us": tot, "launches": sum(a[0] for a in agg.values()), "kernels": {}}
print(f"total {tot/1e3:.2f} ms over {out['launches']} launches (cold-cache, serialised)")
for k, (n, t) in sorted(agg.items(), key=lambda x: -x[1][1]):
    out["kernels"][k] = {"launches": n, "us": t, "share": t / tot}
    print(f"{k:24s} {n:6d} launches {t/1e3:10.3f} ms  share {100*t/tot:5.1f}%  avg {t/n:9.1f} us")
if len(sys.argv) > 2:
    json.dump(out, open(sys.argv[2], "w"), indent=1)
