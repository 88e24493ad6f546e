"""Per-kernel mean duration from an `ncu --metrics gpu__time_duration.sum --csv`
launch list: python tools/launch_times.py list.csv"""
import collections
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
start = next(i for i, r in enumerate(rows) if r and r[0] == "ID")
h = rows[start]
ik, iv, iu = h.index("Kernel Name"), h.index("Metric Value"), h.index("Metric Unit")
c = collections.defaultdict(list)
for r in rows[start + 1:]:
    if len(r) <= iv:
        continue
    v = float(r[iv].replace(",", ""))
    v *= {"nsecond": 1e-3, "ns": 1e-3, "usecond": 1.0, "us": 1.0, "msecond": 1e3, "ms": 1e3}.get(r[iu], 1.0)
    c[r[ik].split("(")[0][-60:]].append(v)
for k, v in sorted(c.items(), key=lambda kv: -sum(kv[1])):
    print(f"{k:60s} n={len(v):3d} mean_us={sum(v) / len(v):9.1f}")
