"""Top source lines by warp-stall samples with their dominant stall reasons
(one kernel launch of an ncu report).

  python scripts/ncu_stalls.py <rep> <kernel-regex> [launch-skip] [top]"""
import csv
import io
import subprocess
import sys

rep, kern = sys.argv[1], sys.argv[2]
skip = sys.argv[3] if len(sys.argv) > 3 else "0"
top = int(sys.argv[4]) if len(sys.argv) > 4 else 25
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass",
                      "--kernel-name", f"regex:{kern}", "--launch-skip", skip, "--launch-count", "1"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
hdr = None
fname = "?"
agg = []
for r in rows:
    if r and r[0] == "File Path":
        fname = r[1].split("/")[-1]
    elif r and r[0] == "Line No":
        hdr = r
    elif hdr and len(r) == len(hdr) and r[0].isdigit() and r[4].isdigit():
        d = dict(zip(hdr, r))
        try:
            s = int(d["Warp Stall Sampling (All Samples)"])
        except ValueError:
            continue
        if s == 0:
            continue
        reasons = sorted(((int(d[k]), k[6:]) for k in hdr if k.startswith("stall_") and "Not Issued" not in k
                          and d[k].isdigit()), reverse=True)[:3]
        agg.append((s, fname, int(r[0]), r[1].strip(), reasons))
    elif hdr and len(r) == len(hdr) and not r[0].isdigit():
        pass
tot = sum(a[0] for a in agg) or 1
print(f"total samples {tot}")
for s, f, ln, src, rs in sorted(agg, reverse=True)[:top]:
    why = " ".join(f"{k}:{100 * v // s}%" for v, k in rs if v)
    print(f"{100 * s / tot:5.1f}%  {f}:{ln:<5d} {src[:70]:70s} {why}")
