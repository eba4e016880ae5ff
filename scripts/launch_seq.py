"""Print the launch sequence (stream, kernel, grid, us) of a one-step ncu CSV."""
import collections
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
thr = float(sys.argv[2]) if len(sys.argv) > 2 else 100.0
hi = next(i for i, r in enumerate(rows) if r and r[0] == "ID")
h = rows[hi]
ki, mi, vi, si = h.index("Kernel Name"), h.index("Metric Name"), h.index("Metric Value"), h.index("Stream")
per = collections.OrderedDict()
for r in rows[hi + 1:]:
    if len(r) <= vi:
        continue
    d = per.setdefault(int(r[0]), {"name": r[ki].split("(")[0].split("::")[-1], "st": r[si]})
    d[r[mi]] = float(r[vi].replace(",", ""))
bys = collections.defaultdict(float)
for i, d in per.items():
    us = d["gpu__time_duration.sum"] / 1e3
    bys[d["st"]] += us
    if us > thr:
        print(i, d["st"], d["name"][:28], int(d.get("launch__grid_size", 0)), f"{us:.0f}us")
print("per-stream serialised ms:", {k: round(v / 1e3, 2) for k, v in bys.items()})
