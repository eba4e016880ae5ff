"""GPU activity timeline (kernels, memcpys, memsets) of the els_build tail of
cfg2 refined-wall steps (torch.profiler / CUPTI).  Diagnostic."""
import json
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch  # noqa: E402
import paper_2108_07205_b200 as sb  # noqa: E402
from paper_2108_07205_b200.configs import CONFIGS  # noqa: E402

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
    lib.sbx_sync()
    torch.cuda.synchronize()
    with torch.profiler.record_function("ELS_BUILD"):
        sb.els_build(h, g0, g1, plan, upd)
        lib.sbx_sync()


for _ in range(5):
    step()
with torch.profiler.profile(activities=[torch.profiler.ProfilerActivity.CUDA, torch.profiler.ProfilerActivity.CPU]) as prof:
    for _ in range(4):
        step()
prof.export_chrome_trace("gpurun_out/els_timeline.json")
allev = json.load(open("gpurun_out/els_timeline.json"))["traceEvents"]
marks = [e for e in allev if e.get("name") == "ELS_BUILD" and e.get("ph") == "X" and e.get("cat") in ("user_annotation", "cpu_op")]
marks.sort(key=lambda e: e["ts"])
m = marks[-1]
a, b = m["ts"], m["ts"] + m["dur"]
print(f"els_build host span {1e-3 * m['dur']:.3f} ms")
gpu = [e for e in allev if e.get("cat") in ("kernel", "gpu_memcpy", "gpu_memset") and "dur" in e and a <= e["ts"] <= b + 50]
gpu.sort(key=lambda e: e["ts"])
busy = 0.0
for e in gpu:
    busy += e["dur"]
    print(f"  +{e['ts'] - a:9.1f} us  dur {e['dur']:8.1f}  {e.get('cat'):10s} {e['name'][:80]}")
print(f"gpu busy {busy:.1f} us of {gpu[-1]['ts'] + gpu[-1]['dur'] - a:.1f} us")
rt = [e for e in allev if e.get("cat") == "cuda_runtime" and "dur" in e and a <= e["ts"] <= b and e["dur"] > 15]
rt.sort(key=lambda e: e["ts"])
print("runtime calls > 15 us:")
for e in rt:
    print(f"  +{e['ts'] - a:9.1f} us  dur {e['dur']:8.1f}  {e['name']}")
print("all runtime calls in the first 200 us:")
rt = [e for e in allev if e.get("cat") in ("cuda_runtime", "cuda_driver") and "dur" in e and a <= e["ts"] <= a + 200]
rt.sort(key=lambda e: e["ts"])
for e in rt:
    print(f"  +{e['ts'] - a:9.1f} us  dur {e['dur']:8.1f}  {e['name']}")
