"""Per-step wall-time distribution of the cfg2 refined-wall step (device
synchronised after each step).  Diagnostic for bench variance."""
import sys
import time
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import paper_2108_07205_b200 as sb  # noqa: E402
from paper_2108_07205_b200.configs import CONFIGS  # noqa: E402


def main():
    steps = int(sys.argv[1]) if len(sys.argv) > 1 else 40
    c = CONFIGS["cfg2"]
    sb.init(0)
    curve = sb.star(c.prongs, c.amplitude, c.a)
    g0 = sb.panelize(curve, c.n_panels, c.q)
    h = sb.hbs_invert(sb.hbs_compress(g0, opts=sb.HbsOptions(eps=c.eps, leaf_nodes=c.leaf)))
    panels = c.refine_panels(g0.nodes())
    lib = sb.api.lib()
    import gc
    import os
    if os.environ.get("GC_MODE") == "freeze":
        gc.collect()
        gc.freeze()
    elif os.environ.get("GC_MODE") == "off":
        gc.disable()
    ts = []
    import ctypes
    lib.sbx_kernel_timing(1)
    names = [b"id_factor"]
    def ktime(name):
        ms = ctypes.c_double(0.0)
        cnt = ctypes.c_int64(0)
        lib.sbx_kernel_time(name, 1, ctypes.byref(ms), ctypes.byref(cnt))
        return ms.value, cnt.value
    for i in range(steps + 5):
        lib.sbx_sync()
        print(f"--- step {i}", file=sys.stderr, flush=True)
        t0 = time.perf_counter()
        g1, plan = sb.refine(g0, panels, c.m)
        upd = sb.compress_update(g0, g1, plan, c.eps, seed=c.seed)
        els = sb.els_build(h, g0, g1, plan, upd)
        lib.sbx_sync()
        if i >= 5:
            ts.append(1e3 * (time.perf_counter() - t0))
            idm, idc = ktime(b"id_factor")
            print(f"--- step {i} took {ts[-1]:.1f} ms, id_factor {idm:.2f} ms in {idc} batches", file=sys.stderr, flush=True)
        else:
            ktime(b"id_factor")
    ts = np.array(ts)
    print(f"steps {steps}: min {ts.min():.2f} p25 {np.percentile(ts, 25):.2f} median {np.median(ts):.2f} "
          f"p75 {np.percentile(ts, 75):.2f} max {ts.max():.2f} ms")
    print(" ".join(f"{t:.1f}" for t in ts))


if __name__ == "__main__":
    main()
