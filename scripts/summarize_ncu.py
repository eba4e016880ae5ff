"""Summarise ncu artefacts into profiles/ (markdown).

  python scripts/summarize_ncu.py launches <launches.csv> > profiles/x.md
  python scripts/summarize_ncu.py report <prof.ncu-rep> > profiles/y.md
"""
import collections
import csv
import io
import subprocess
import sys


def launches(path, what="the whole bench.py process (setup + warm-up + timed + e2e + roofline steps)"):
    rows = list(csv.reader(open(path)))
    hi = next(i for i, r in enumerate(rows) if r and r[0] == "ID")
    h = rows[hi]
    data = rows[hi + 1:]
    ki, vi = h.index("Kernel Name"), h.index("Metric Value")
    agg = collections.defaultdict(lambda: [0, 0.0])
    tot = 0.0
    for r in data:
        if len(r) <= vi:
            continue
        us = float(r[vi].replace(",", "")) / 1000.0
        name = r[ki].split("(")[0].replace("sbx::<unnamed>::", "")
        agg[name][0] += 1
        agg[name][1] += us
        tot += us
    print(f"# ncu launch list summary: `{path}`\n")
    print(f"`ncu --metrics gpu__time_duration.sum --clock-control none` over {what}; cold-cache "
          "serialised launches, so compare shares, not absolutes.\n")
    print(f"Total kernel time {tot / 1e3:.2f} ms over {len(data)} launches.\n")
    print("| kernel | launches | total ms | share | mean us |")
    print("|---|---:|---:|---:|---:|")
    for k, (c, t) in sorted(agg.items(), key=lambda x: -x[1][1]):
        print(f"| {k} | {c} | {t / 1e3:.3f} | {100 * t / tot:.1f}% | {t / c:.1f} |")


def steplist(path):
    """Per-kernel summary of a one-step capture with grid sizes (SM share)."""
    rows = list(csv.reader(open(path)))
    hi = next(i for i, r in enumerate(rows) if r and r[0] == "ID")
    h = rows[hi]
    ki, mi, vi = h.index("Kernel Name"), h.index("Metric Name"), h.index("Metric Value")
    per = collections.defaultdict(dict)
    for r in rows[hi + 1:]:
        if len(r) <= vi:
            continue
        per[int(r[0])]["name"] = r[ki].split("(")[0].replace("sbx::<unnamed>::", "")
        per[int(r[0])][r[mi]] = float(r[vi].replace(",", ""))
    agg = collections.defaultdict(lambda: [0, 0.0, 0.0, 0.0])
    tot = 0.0
    for d in per.values():
        us = d.get("gpu__time_duration.sum", 0.0) / 1000.0
        g = d.get("launch__grid_size", 0.0)
        a = agg[d["name"]]
        a[0] += 1
        a[1] += us
        a[2] += g
        a[3] += us * min(1.0, g / 148.0)
        tot += us
    print(f"# one-step launch list: `{path}`\n")
    print(f"Serialised kernel time {tot / 1e3:.2f} ms over {len(per)} launches "
          "(ncu replays kernels one at a time, cold caches).\n")
    print("| kernel | launches | total ms | share | mean us | mean grid | SM-weighted ms |")
    print("|---|---:|---:|---:|---:|---:|---:|")
    for k, (c, t, g, w) in sorted(agg.items(), key=lambda x: -x[1][1]):
        print(f"| {k} | {c} | {t / 1e3:.3f} | {100 * t / tot:.1f}% | {t / c:.1f} | {g / c:.0f} | {w / 1e3:.3f} |")


WANT = [
    "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
    "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
    "sm__throughput.avg.pct_of_peak_sustained_elapsed",
    "sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active",
    "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread",
    "launch__grid_size", "launch__block_size", "launch__shared_mem_per_block_dynamic",
    "smsp__cycles_active.avg", "l1tex__t_bytes.sum", "lts__t_bytes.sum",
    "sm__pipe_tensor_subpipe_dmma_cycles_active.avg.pct_of_peak_sustained_active",
    "smsp__issue_active.avg.pct_of_peak_sustained_active",
]


def report(path):
    raw = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True,
                         text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    h, units = rows[0], rows[1]
    print(f"# ncu --set full summary: `{path}`\n")
    for v in rows[2:]:
        name = v[h.index("Kernel Name")] if "Kernel Name" in h else "?"
        print(f"## {name[:120]}\n")
        print("| metric | value | unit |")
        print("|---|---:|---|")
        for w in WANT:
            if w in h:
                i = h.index(w)
                print(f"| {w} | {v[i]} | {units[i]} |")
        print()
    out = subprocess.run(["ncu", "-i", path, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                         capture_output=True, text=True).stdout
    lines, fname = [], "?"
    for r in csv.reader(io.StringIO(out)):
        if r and r[0] == "File Path":
            fname = r[1].split("/")[-1]
        if len(r) > 4 and r[0].isdigit() and r[4].isdigit():
            lines.append((int(r[4]), fname, int(r[0]), r[1].strip()))
    tot = sum(x[0] for x in lines) or 1
    print("### top source lines by warp-stall samples\n")
    print("| share | line | source |")
    print("|---:|---|---|")
    for smp, f, ln, src_ in sorted(lines, reverse=True)[:15]:
        print(f"| {100 * smp / tot:.1f}% | {f}:{ln} | `{src_[:90]}` |")


if __name__ == "__main__":
    {"launches": launches, "report": report, "steplist": steplist}[sys.argv[1]](*sys.argv[2:])
