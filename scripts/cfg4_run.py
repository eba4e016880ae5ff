"""cfg4 (configs[3]) on one GPU: 200-step transient on the wavy channel
(scenario.cpp:844-915 snapshot loop without its cache).  Per step: pick the
base panels within 5 gaps of the descending disk, refine them with
m = ceil(max length / gap) (m = 1 keeps the base mesh: identity plan, k = 0,
plain hbs_solve), compress_update, els_build, els_solve; the velocity at
fluid targets is checked against the generating Stokeslet field with the
device evaluate_solution.  Prints per-step phase times and a summary line."""
import argparse
import json
import sys
import time
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import paper_2108_07205_b200 as sb  # noqa: E402
from paper_2108_07205_b200.configs import CONFIGS  # noqa: E402


def stokeslet_field(src, tg, mu=1.0):
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
    ap.add_argument("--steps", type=int, default=200)
    ap.add_argument("--every", type=int, default=20, help="print every n-th step")
    a = ap.parse_args()
    c = CONFIGS["cfg4"]
    sb.init(0)
    scale, cc, ss = c.fourier()
    curve = sb.CurveParams(kind=sb.FOURIER, center=(4.0, 0.0), scale=scale, cos_coef=cc, sin_coef=ss)
    t0 = t()
    base = sb.panelize(curve, c.n_panels, c.q)
    h = sb.hbs_invert(sb.hbs_compress(base, opts=sb.HbsOptions(eps=c.eps, leaf_nodes=c.leaf)))
    t1 = t()
    nd = base.nodes()
    src = c.sources()
    tg = c.targets()
    exact = stokeslet_field(src, tg)
    g_base = sb.boundary_data(base, src)
    # the disk approaches the right end cap along y = 0, where the base panels
    # are longest (equal-parameter panels of a radial curve)
    right = (np.abs(nd["y"]) < 0.05) & (nd["x"] > 4.0)
    x_wall = float(np.min(nd["x"][right]))
    plen = np.zeros(c.n_panels)
    np.add.at(plen, nd["panel_of"], nd["w"])
    print(f"[cfg4] static HBS {t1 - t0:.2f}s  n={h.info()['n']} cap at y=0: x={x_wall:.4f}", flush=True)
    rows, worst = [], 0.0
    for step, gap in enumerate(c.gaps()[: a.steps]):
        cx = x_wall - c.disk_radius - gap
        d = np.hypot(nd["x"] - cx, nd["y"]) - c.disk_radius
        near = np.unique(nd["panel_of"][d < 5 * gap])
        m = int(np.ceil(np.max(plen[near]) / gap)) if len(near) else 1
        s0 = t()
        if m <= 1 or len(near) == 0:  # identity plan: plain solve on the base mesh
            tau = sb.hbs_solve(h, g_base)
            dens, geom, k = tau, base, 0
            s1 = s2 = s3 = t()
        else:
            g1, plan = sb.refine(base, near, m)
            s1 = t()
            upd = sb.compress_update(base, g1, plan, c.eps)
            s2 = t()
            els = sb.els_build(h, base, g1, plan, upd)
            s3 = t()
            tau_n = sb.els_solve(els, sb.gather_kept_added(plan, sb.boundary_data(g1, src)))
            dens, geom, k = sb.density_on_refined(els, tau_n), g1, upd.info()["k"]
        s4 = t()
        vel, _, _ = sb.evaluate_solution(geom, sb.INTERIOR_DIRICHLET, dens, tg)
        err = float(np.max(np.linalg.norm(vel - exact, axis=1) / np.linalg.norm(exact, axis=1)))
        worst = max(worst, err)
        rows.append({"step": step, "gap": gap, "panels": int(len(near)), "m": m, "k": int(k),
                     "refine": s1 - s0, "update": s2 - s1, "els_build": s3 - s2, "solve": s4 - s3,
                     "total": s4 - s0, "err": err})
        if step % a.every == 0 or step == a.steps - 1:
            r = rows[-1]
            print(f"  step {step:3d} gap {gap:.4f} panels {r['panels']:3d} m {m:3d} k {k:4d}  "
                  f"refine {r['refine']*1e3:6.2f} update {r['update']*1e3:7.2f} els {r['els_build']*1e3:6.2f} "
                  f"solve {r['solve']*1e3:6.2f} ms  err {err:.1e}", flush=True)
    tot = sum(r["total"] for r in rows)
    print(json.dumps({"cfg": "cfg4", "steps": len(rows), "total_s": round(tot, 3),
                      "mean_step_ms": round(1e3 * tot / len(rows), 3),
                      "max_rel_velocity_error": worst, "static_hbs_s": round(t1 - t0, 3)}))


if __name__ == "__main__":
    main()
