"""Top source lines by warp-stall samples for one kernel launch of an ncu report.

  python scripts/ncu_lines.py <rep> <kernel-regex> <launch-skip> [top]"""
import csv
import io
import subprocess
import sys

rep, kern, skip = sys.argv[1], sys.argv[2], sys.argv[3]
top = int(sys.argv[4]) if len(sys.argv) > 4 else 25
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass",
                      "--kernel-name", f"regex:{kern}", "--launch-skip", skip, "--launch-count", "1"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
lines = []
fname = "?"
for r in rows:
    if r and r[0] == "File Path":
        fname = r[1].split("/")[-1]
    if len(r) > 4 and r[0].isdigit() and r[4].isdigit():
        lines.append((int(r[4]), fname, int(r[0]), r[1].strip()))
tot = sum(x[0] for x in lines) or 1
print(f"total samples {tot}")
for s, f, ln, src in sorted(lines, reverse=True)[:top]:
    print(f"{100 * s / tot:5.1f}%  {f}:{ln:<5d} {src[:90]}")
