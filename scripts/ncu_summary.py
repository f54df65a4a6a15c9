"""Summarise an ncu launch-list CSV by kernel: launches, time (gpu__time_duration.sum)
and, when captured, DRAM bytes (dram__bytes_read.sum + dram__bytes_write.sum).

    python scripts/ncu_summary.py LAUNCHES.csv [OUT.json]
"""
import collections
import csv
import json
import re
import sys

rows = list(csv.reader(open(sys.argv[1])))
hdr_i = [i for i, r in enumerate(rows) if r and r[0] == "ID"][0]
hdr, data = rows[hdr_i], rows[hdr_i + 1:]
ki, ni, mi, ui = hdr.index("Kernel Name"), hdr.index("Metric Name"), hdr.index("Metric Value"), hdr.index("Metric Unit")
ii = hdr.index("ID")
tscale = {"nsecond": 1e-3, "ns": 1e-3, "usecond": 1.0, "us": 1.0, "msecond": 1e3, "ms": 1e3, "second": 1e6, "s": 1e6}
bscale = {"byte": 1.0, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "KB": 1e3, "MB": 1e6, "GB": 1e9}
per_launch = collections.defaultdict(dict)
names = {}
for r in data:
    if len(r) <= mi:
        continue
    m = re.search(r"(k_\w+)(<[^>]*>)?", r[ki])
    names[r[ii]] = (m.group(1) + (m.group(2) or "")) if m else r[ki][:40]
    v = float(r[mi].replace(",", ""))
    if r[ni] == "gpu__time_duration.sum":
        per_launch[r[ii]]["us"] = v * tscale[r[ui]]
    elif r[ni].startswith("dram__bytes"):
        per_launch[r[ii]]["bytes"] = per_launch[r[ii]].get("bytes", 0.0) + v * bscale.get(r[ui], 1.0)
agg = collections.defaultdict(lambda: [0, 0.0, 0.0])
for lid, d in per_launch.items():
    a = agg[names[lid]]
    a[0] += 1
    a[1] += d.get("us", 0.0)
    a[2] += d.get("bytes", 0.0)
tot = sum(a[1] for a in agg.values())
out = {"total_us": tot, "launches": sum(a[0] for a in agg.values()), "kernels": {}}
print(f"total {tot/1e3:.2f} ms over {out['launches']} launches (cold-cache, serialised)")
for k, (n, t, b) in sorted(agg.items(), key=lambda x: -x[1][1]):
    out["kernels"][k] = {"launches": n, "us": t, "share": t / tot, "dram_bytes": b,
                         "dram_GBps": (b / (t * 1e3)) if t else None}
    print(f"{k:26s} {n:6d} launches {t/1e3:10.3f} ms  share {100*t/tot:5.1f}%  avg {t/n:9.1f} us"
          f"  DRAM {b/1e9:8.3f} GB ({(b / (t * 1e3)) if t else 0:7.1f} GB/s)")
if len(sys.argv) > 2:
    json.dump(out, open(sys.argv[2], "w"), indent=1)
