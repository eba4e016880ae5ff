"""Kernel timeline of cfg2 refined-wall steps through torch.profiler (CUPTI
activity records of every kernel in the process, the library's included).
Writes gpurun_out/timeline.json (chrome trace) and prints, for the slowest
step, the kernels per stream with their start / duration.  Diagnostic."""
import json
import sys
import time
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch  # noqa: E402
import paper_2108_07205_b200 as sb  # noqa: E402
from paper_2108_07205_b200.configs import CONFIGS  # noqa: E402


def main():
    steps = int(sys.argv[1]) if len(sys.argv) > 1 else 30
    c = CONFIGS["cfg2"]
    torch.cuda.init()
    sb.init(0)
    g0 = sb.panelize(sb.star(c.prongs, c.amplitude, c.a), c.n_panels, c.q)
    h = sb.hbs_invert(sb.hbs_compress(g0, opts=sb.HbsOptions(eps=c.eps, leaf_nodes=c.leaf)))
    panels = c.refine_panels(g0.nodes())
    lib = sb.api.lib()

    def step():
        g1, plan = sb.refine(g0, panels, c.m)
        upd = sb.compress_update(g0, g1, plan, c.eps, seed=c.seed)
        sb.els_build(h, g0, g1, plan, upd)
        lib.sbx_sync()

    for _ in range(5):
        step()
    marks = []
    with torch.profiler.profile(activities=[torch.profiler.ProfilerActivity.CUDA, torch.profiler.ProfilerActivity.CPU]) as prof:
        for _ in range(steps):
            t0 = time.perf_counter()
            step()
            marks.append((t0, time.perf_counter()))
    prof.export_chrome_trace("gpurun_out/timeline.json")
    allev = json.load(open("gpurun_out/timeline.json"))["traceEvents"]
    ev = [e for e in allev if e.get("cat") == "kernel" and "dur" in e]
    rt = sorted((e for e in allev if e.get("cat") == "cuda_runtime" and "dur" in e), key=lambda e: -e["dur"])
    print("longest CUDA runtime calls:")
    for e in rt[:25]:
        print(f"  {1e-3 * e['dur']:9.3f} ms  tid {e.get('tid')}  {e['name']}")
    from collections import defaultdict
    tot = defaultdict(lambda: [0.0, 0])
    for e in rt:
        tot[e["name"]][0] += e["dur"] * 1e-3
        tot[e["name"]][1] += 1
    print("runtime call totals (ms, count):")
    for k, v in sorted(tot.items(), key=lambda kv: -kv[1][0])[:15]:
        print(f"  {v[0]:9.2f} ms {v[1]:7d}  {k}")
    ev.sort(key=lambda e: e["ts"])
    walls = [1e3 * (b - a) for a, b in marks]
    print("step wall ms:", " ".join(f"{w:.1f}" for w in walls))
    # the slowest step: every runtime call / kernel longer than 1 ms in it
    # (trace timestamps are microseconds on the profiler's clock; the steps
    # are located by the gaps between them, so take the longest busy window)
    cpu = [e for e in allev if e.get("ph") == "X" and "dur" in e and e["dur"] > 1000.0]
    cpu.sort(key=lambda e: e["ts"])
    print("events > 1 ms (all steps):")
    for e in cpu[:80]:
        print(f"  ts {e['ts']:.0f} dur {1e-3 * e['dur']:8.3f} ms  cat {e.get('cat')}  tid {e.get('tid')}  {e['name'][:60]}")
    # split kernels into steps by gaps > 0.3 ms with no kernel running (host sync)
    groups, cur, end = [], [], -1.0
    for e in ev:
        if cur and e["ts"] > end + 300.0:
            groups.append(cur)
            cur = []
        cur.append(e)
        end = max(end, e["ts"] + e["dur"])
    groups.append(cur)
    spans = [(g[0]["ts"], max(x["ts"] + x["dur"] for x in g), g) for g in groups]
    long = sorted(spans, key=lambda s: s[0] - s[1])[:3]
    for a, b, g in long:
        print(f"\n=== busy span {1e-3 * (b - a):.2f} ms, {len(g)} kernels")
        t0 = a
        for e in g:
            if e["dur"] > 200.0 or (e["ts"] - t0) > 1e9:
                print(f"  +{1e-3 * (e['ts'] - t0):8.3f} ms  dur {1e-3 * e['dur']:8.3f}  stream {e['args'].get('stream')}  {e['name'][:70]}")


if __name__ == "__main__":
    main()
