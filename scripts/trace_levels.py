"""Per-level summary of an SBX_SWEEP_TRACE timeline (diagnostic).

  python scripts/trace_levels.py <trace file> [run index]

Columns: level, items, first ticket (t0), first wait done (t1), last done
(t2), all relative to the run's first ticket, in microseconds; 'span' is
last done minus the previous level's last done (the level's share of the
critical path) and 'work' the mean compute+publish time (t2 - t1)."""
import sys

runs, cur = [], None
for line in open(sys.argv[1]):
    if line.startswith("#"):
        cur = {"hdr": line.strip(), "rows": []}
        runs.append(cur)
        continue
    f = line.split()
    cur["rows"].append(tuple(int(x) for x in f))
run = runs[int(sys.argv[2]) if len(sys.argv) > 2 else -1]
rows = run["rows"]
base = min(r[6] for r in rows)
lv = {}
for r in rows:
    lv.setdefault(r[1], []).append(r)
print(run["hdr"])
print(f"{'lvl':>3} {'items':>6} {'t0':>8} {'t1min':>8} {'t1max':>8} {'t2max':>8} {'span':>7} {'work':>6}")
prev = 0.0
order = sorted(lv, key=lambda l: max(r[8] for r in lv[l]))
for l in order:
    rs = lv[l]
    t0 = (min(r[6] for r in rs) - base) / 1e3
    t1a = (min(r[7] for r in rs) - base) / 1e3
    t1b = (max(r[7] for r in rs) - base) / 1e3
    t2 = (max(r[8] for r in rs) - base) / 1e3
    work = sum(r[8] - r[7] for r in rs) / len(rs) / 1e3
    print(f"{l:3d} {len(rs):6d} {t0:8.2f} {t1a:8.2f} {t1b:8.2f} {t2:8.2f} {t2 - prev:7.2f} {work:6.2f}")
    prev = t2
