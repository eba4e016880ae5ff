"""Per-phase wall times of the refined-wall path on the device (and
optionally the oracle), for one BASELINE config.  Diagnostic only."""
import argparse
import sys
import time
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import paper_2108_07205_b200 as sb  # noqa: E402
from paper_2108_07205_b200.configs import CONFIGS  # noqa: E402


def t():
    sb.api.lib().sbx_sync()
    return time.perf_counter()


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--cfg", default="cfg2")
    ap.add_argument("--reps", type=int, default=3)
    ap.add_argument("--oracle", action="store_true")
    ap.add_argument("--profile-last", action="store_true",
                    help="cudaProfilerStart/Stop around the last step (ncu --profile-from-start off)")
    a = ap.parse_args()
    c = CONFIGS[a.cfg]
    sb.init(0)
    curve = sb.ellipse(c.a, c.b) if c.kind == "ellipse" else sb.star(c.prongs, c.amplitude, c.a)
    t0 = t()
    g0 = sb.panelize(curve, c.n_panels, c.q)
    t1 = t()
    h = sb.hbs_compress(g0, opts=sb.HbsOptions(eps=c.eps, leaf_nodes=c.leaf))
    t2 = t()
    sb.hbs_invert(h)
    t3 = t()
    info = h.info()
    print(f"[{a.cfg}] panelize {t1-t0:.3f}s compress {t2-t1:.3f}s invert {t3-t2:.3f}s "
          f"n={info['n']} nodes={info['nodes']} max_k={info['max_k']} "
          f"solve_factor_MB={info['factor_doubles']*8/1e6:.1f}", flush=True)
    if c.n_refine == 0:
        for nrhs in (1, 32, 256):
            b = np.random.default_rng(0).uniform(-1, 1, (info["n"], nrhs))
            sb.hbs_solve(h, b)
            t4 = t()
            for _ in range(a.reps):
                sb.hbs_solve(h, b)
            t5 = t()
            print(f"  hbs_solve nrhs={nrhs}: {(t5-t4)/a.reps*1e3:.3f} ms (host in/out)")
        return
    panels = c.refine_panels(g0.nodes())
    srcs = c.sources()
    for rep in range(a.reps):
        if a.profile_last and rep == a.reps - 1:
            import torch
            torch.cuda.init()
            torch.cuda.profiler.start()
        s0 = t()
        g1, plan = sb.refine(g0, panels, c.m)
        s1 = t()
        upd = sb.compress_update(g0, g1, plan, c.eps, seed=c.seed)
        s2 = t()
        els = sb.els_build(h, g0, g1, plan, upd)
        s3 = t()
        G = np.stack([sb.gather_kept_added(plan, sb.boundary_data(g1, s)) for s in srcs], 1)
        s4 = t()
        tau = sb.els_solve(els, G)
        s5 = t()
        if a.profile_last and rep == a.reps - 1:
            torch.cuda.profiler.stop()
        ui = upd.info()
        print(f"  step {rep}: refine {s1-s0:.4f} update {s2-s1:.4f} els_build {s3-s2:.4f} "
              f"rhs {s4-s3:.4f} solve {s5-s4:.4f}  total {s5-s0-(s4-s3):.4f}s  k={ui['k']} k1={ui['k1']} "
              f"(kc {ui['kc']} kp {ui['kp']} pk {ui['pk']}) n_ext={ui['n_ext']} app_hbs={els.info()['app_hbs']}",
              flush=True)
    if a.oracle:
        from oracle import pyoracle as po
        kind = po.ELLIPSE if c.kind == "ellipse" else po.STAR
        o0 = (po.Geom.create(kind, c.n_panels, scale=c.a, aspect=c.b / c.a) if c.kind == "ellipse"
              else po.Geom.create(kind, c.n_panels, prongs=c.prongs, amplitude=c.amplitude, scale=c.a))
        a0 = po.Assembler.create(o0)
        q0 = time.perf_counter()
        oh = po.Hbs.compress(a0, c.eps).invert()
        q1 = time.perf_counter()
        o1, op = o0.refine(panels, c.m)
        a1 = po.Assembler.create(o1)
        ou = po.Update.compress(a0, a1, op, c.eps, c.seed)
        q2 = time.perf_counter()
        oe = po.Els.build(oh, a0, a1, op, ou)
        q3 = time.perf_counter()
        OG = np.stack([po.gather_kept_added(op.maps(), o1.boundary_data(s)) for s in srcs], 1)
        otau = oe.solve(OG)
        q4 = time.perf_counter()
        print(f"  oracle: static {q1-q0:.2f}s update {q2-q1:.2f}s els_build {q3-q2:.2f}s solve {q4-q3:.2f}s "
              f"k={ou.info()['k']}; rel diff vs device {np.linalg.norm(tau-otau)/np.linalg.norm(otau):.2e}")


if __name__ == "__main__":
    main()
