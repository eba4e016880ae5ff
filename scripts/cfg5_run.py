"""cfg5 (configs[4]) end to end on one GPU: static HBS of the multiply
connected wall (Mixed formulation, 524288 unknowns), then refined-wall steps
(8 obstacle regions, m = 16) with 128 right-hand sides; checks the computed
velocity against the generating Stokeslet field at fluid targets through the
oracle's evaluate_solution (diagnostic, not a bench line)."""
import argparse
import sys
import time
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import paper_2108_07205_b200 as sb  # noqa: E402
from paper_2108_07205_b200.configs import CONFIGS  # noqa: E402


def stokeslet_field(src, tg, mu=1.0):
    """Analytic velocity of point forces (x, y, fx, fy) at targets (kernels.cpp:13-31)."""
    out = np.zeros((len(tg), 2))
    for x, y, fx, fy in src:
        r = tg - np.array([x, y])
        r2 = np.sum(r * r, 1)
        lg = -0.5 * np.log(r2)
        rf = r[:, 0] * fx + r[:, 1] * fy
        out[:, 0] += (lg * fx + r[:, 0] * rf / r2) / (4 * np.pi * mu)
        out[:, 1] += (lg * fy + r[:, 1] * rf / r2) / (4 * np.pi * mu)
    return out


def t():
    sb.api.lib().sbx_sync()
    return time.perf_counter()


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--steps", type=int, default=2)
    ap.add_argument("--check-rhs", type=int, default=2)
    ap.add_argument("--wall-panels", type=int, default=0, help="override the wall panel count")
    ap.add_argument("--hole-panels", type=int, default=0, help="override the panels per hole")
    ap.add_argument("--ppr", type=int, default=0, help="override the refined panels per region")
    ap.add_argument("--m", type=int, default=0, help="override the split factor")
    ap.add_argument("--arclength", action="store_true", help="BASELINE's equal arc-length split 9216 + 16 x 448")
    a = ap.parse_args()
    import dataclasses
    c = CONFIGS["cfg5"]
    if a.arclength:
        c = dataclasses.replace(c, wall_panels=9216, hole_panels=448)
    over = {k: v for k, v in (("wall_panels", a.wall_panels), ("hole_panels", a.hole_panels),
                              ("panels_per_region", a.ppr), ("m", a.m)) if v}
    if over:
        c = dataclasses.replace(c, **over)
    sb.init(0)
    t0 = t()
    wall = sb.panelize(sb.ellipse(c.a, c.b), c.wall_panels, c.q)
    base, _ = sb.add_holes(wall, [(sb.circle(c.hole_radius, tuple(p)), c.hole_panels, c.q)
                                  for p in c.hole_centers()])
    t1 = t()
    h = sb.hbs_invert(sb.hbs_compress(base, sb.MIXED, opts=sb.HbsOptions(eps=c.eps, leaf_nodes=c.leaf)))
    t2 = t()
    info = h.info()
    print(f"[cfg5] geometry {t1 - t0:.2f}s  static HBS compress+invert {t2 - t1:.2f}s  n={info['n']} "
          f"nodes={info['nodes']} max_k={info['max_k']} factor_MB={info['factor_doubles'] * 8 / 1e6:.0f}",
          flush=True)
    panels = c.refine_panels(base.nodes())
    srcs = c.sources()
    if a.check_rhs:  # the static inverse alone on the base mesh
        tg = c.targets(20)
        for j in range(a.check_rhs):
            tau0 = sb.hbs_solve(h, sb.boundary_data(base, srcs[j]))
            vel, _, _ = sb.evaluate_solution(base, sb.MIXED, tau0, tg)
            ex = stokeslet_field(srcs[j], tg)
            err = np.max(np.linalg.norm(vel - ex, axis=1) / np.linalg.norm(ex, axis=1))
            print(f"  static rhs {j}: max relative velocity error {err:.2e}", flush=True)
    for step in range(a.steps):
        s0 = t()
        g1, plan = sb.refine(base, panels, c.m)
        s1 = t()
        upd = sb.compress_update(base, g1, plan, c.eps, formulation=sb.MIXED)
        s2 = t()
        els = sb.els_build(h, base, g1, plan, upd, formulation=sb.MIXED)
        s3 = t()
        G = np.stack([sb.gather_kept_added(plan, sb.boundary_data(g1, s)) for s in srcs], 1)
        s4 = t()
        tau = sb.els_solve(els, G)
        s5 = t()
        ui = upd.info()
        print(f"  step {step}: refine {s1 - s0:.3f} update {s2 - s1:.3f} els_build {s3 - s2:.3f} "
              f"solve {s5 - s4:.3f}  total {s5 - s0 - (s4 - s3):.3f}s  k={ui['k']} n_ext={ui['n_ext']} "
              f"app_hbs={els.info()['app_hbs']}", flush=True)
    if a.check_rhs:
        tg = c.targets(20)
        for j in range(a.check_rhs):
            dens = sb.density_on_refined(els, tau[:, j])
            vel, _, near = sb.evaluate_solution(g1, sb.MIXED, dens, tg)
            ex = stokeslet_field(srcs[j], tg)
            err = np.max(np.linalg.norm(vel - ex, axis=1) / np.linalg.norm(ex, axis=1))
            print(f"  rhs {j}: max relative velocity error at {len(tg)} fluid targets {err:.2e} "
                  f"(near-boundary targets: {int(near.sum())})", flush=True)


if __name__ == "__main__":
    main()
