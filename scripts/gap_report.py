"""GPU idle gaps inside cfg2 refined-wall steps: merges the activity intervals
of all streams (CUPTI via torch.profiler) and lists every gap above a
threshold with the kernel before / after it.  Diagnostic."""
import json
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch  # noqa: E402
import paper_2108_07205_b200 as sb  # noqa: E402
from paper_2108_07205_b200.configs import CONFIGS  # noqa: E402

thr = float(sys.argv[1]) if len(sys.argv) > 1 else 40.0
c = CONFIGS["cfg2"]
torch.cuda.init()
sb.init(0)
g0 = sb.panelize(sb.star(c.prongs, c.amplitude, c.a), c.n_panels, c.q)
h = sb.hbs_invert(sb.hbs_compress(g0, opts=sb.HbsOptions(eps=c.eps, leaf_nodes=c.leaf)))
panels = c.refine_panels(g0.nodes())
lib = sb.api.lib()
g1, plan = sb.refine(g0, panels, c.m)
G = torch.from_numpy(__import__("numpy").stack(
    [sb.gather_kept_added(plan, sb.boundary_data(g1, s)) for s in c.sources()], 1)).cuda()
stream = torch.cuda.ExternalStream(lib.sbx_stream())


def step():
    with torch.profiler.record_function("STEP"):
        g1, plan = sb.refine(g0, panels, c.m)
        upd = sb.compress_update(g0, g1, plan, c.eps, seed=c.seed)
        els = sb.els_build(h, g0, g1, plan, upd)
        with torch.cuda.stream(stream):
            sb.els_solve(els, G)
        lib.sbx_sync()


for _ in range(5):
    step()
with torch.profiler.profile(activities=[torch.profiler.ProfilerActivity.CUDA, torch.profiler.ProfilerActivity.CPU]) as prof:
    for _ in range(3):
        step()
prof.export_chrome_trace("gpurun_out/gap_timeline.json")
allev = json.load(open("gpurun_out/gap_timeline.json"))["traceEvents"]
marks = sorted((e for e in allev if e.get("name") == "STEP" and e.get("ph") == "X" and e.get("cat") == "user_annotation"), key=lambda e: e["ts"])
m = marks[-1]
a, b = m["ts"], m["ts"] + m["dur"]
gpu = sorted((e for e in allev if e.get("cat") in ("kernel", "gpu_memcpy", "gpu_memset") and "dur" in e
              and a <= e["ts"] <= b), key=lambda e: e["ts"])
print(f"step host span {1e-3 * m['dur']:.3f} ms, {len(gpu)} GPU activities")
end, last, idle = a, None, 0.0
for e in gpu:
    if e["ts"] > end + thr:
        gap = e["ts"] - end
        idle += gap
        print(f"  gap {gap:7.1f} us at +{1e-3 * (end - a):7.3f} ms   after [{(last or {}).get('name', 'start')[:48]}]  before [{e['name'][:48]}]")
    if e["ts"] + e["dur"] > end:
        end, last = e["ts"] + e["dur"], e
tot_idle = 0.0
end = a
for e in gpu:
    if e["ts"] > end:
        tot_idle += e["ts"] - end
    end = max(end, e["ts"] + e["dur"])
print(f"idle in gaps > {thr:.0f} us: {idle:.1f} us; all idle: {tot_idle:.1f} us of {end - a:.1f} us")
