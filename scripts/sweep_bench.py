"""Device-resident HBS sweep timing (CUDA events on the library stream)."""
import argparse
import sys
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import paper_2108_07205_b200 as sb  # noqa: E402
from paper_2108_07205_b200.configs import CONFIGS  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--cfg", default="cfg3")
    ap.add_argument("--nrhs", default="1,32,256")
    ap.add_argument("--reps", type=int, default=10)
    a = ap.parse_args()
    c = CONFIGS[a.cfg]
    sb.init(0)
    curve = sb.star(c.prongs, c.amplitude, c.a) if c.kind == "star" else sb.ellipse(c.a, c.b)
    g = sb.panelize(curve, c.n_panels, c.q)
    h = sb.hbs_invert(sb.hbs_compress(g, opts=sb.HbsOptions(eps=c.eps)))
    info = h.info()
    n = info["n"]
    fb = info["factor_doubles"] * 8
    stream = torch.cuda.ExternalStream(sb.api.lib().sbx_stream())
    for nrhs in [int(x) for x in a.nrhs.split(",")]:
        b = torch.empty((n, nrhs), dtype=torch.float64, device="cuda").uniform_(-1, 1)
        torch.cuda.synchronize()
        with torch.cuda.stream(stream):
            for _ in range(3):
                x = sb.hbs_solve(h, b)
            sb.api.kernel_timing(True)
            sb.api.kernel_time("sweep_flow_dmma")
            sb.api.kernel_time("sweep_flow_gemv")
            e0 = torch.cuda.Event(enable_timing=True)
            e1 = torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            for _ in range(a.reps):
                x = sb.hbs_solve(h, b)
            e1.record(stream)
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / a.reps
        kname = "sweep_flow_gemv" if nrhs == 1 else "sweep_flow_dmma"
        kms, kcnt = sb.api.kernel_time(kname)
        sb.api.kernel_timing(False)
        kms /= max(kcnt, 1)
        flops = 2.0 * nrhs * info["factor_doubles"]
        print(f"nrhs={nrhs:4d}: call {ms*1e3:8.1f} us, kernel {kms*1e3:8.1f} us  factor bytes {fb/1e6:.1f} MB"
              f" -> kernel {fb/kms/1e6:.1f} GB/s (1 pass), {flops/kms/1e9:.2f} TF/s", flush=True)
    i2 = h.info()
    print(f"collapsed top: depth {i2['top_L']}, K {i2['top_K']} ({i2['top_K'] ** 2 * 8 / 1e6:.1f} MB)")


if __name__ == "__main__":
    main()
