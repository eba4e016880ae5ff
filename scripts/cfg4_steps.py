"""cfg4: per-step velocity error of a few schedule points (diagnostic)."""
import sys
from pathlib import Path
import numpy as np
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import bench
import paper_2108_07205_b200 as sb
from paper_2108_07205_b200.configs import CONFIGS
cfg = CONFIGS["cfg4"]
sb.init(0)
base = sb.panelize(cfg.curve(sb), cfg.n_panels, cfg.q)
h = sb.hbs_invert(sb.hbs_compress(base, opts=sb.HbsOptions(eps=cfg.eps, leaf_nodes=cfg.leaf)))
nd = base.nodes()
plen = np.zeros(cfg.n_panels)
np.add.at(plen, nd["panel_of"], nd["w"])
src, tg = cfg.sources(), cfg.targets()
gaps = cfg.gaps()
exact = bench.stokeslet_field(src, tg)
g_base = sb.boundary_data(base, src)
steps = [int(x) for x in sys.argv[1:]] or bench.transient_schedule(cfg, 5)
for i in steps:
    near, m = cfg.step_plan(nd, plen, gaps[i])
    if m <= 1:
        tau = sb.hbs_solve(h, g_base)
        vel, _, _ = sb.evaluate_solution(base, sb.INTERIOR_DIRICHLET, tau, tg)
        k = 0
    else:
        g1, plan = sb.refine(base, near, m)
        upd = sb.compress_update(base, g1, plan, cfg.eps)
        els = sb.els_build(h, base, g1, plan, upd)
        gn = sb.gather_kept_added(plan, sb.boundary_data(g1, src))
        tau = sb.els_solve(els, gn)
        vel, _, _ = sb.evaluate_solution(g1, sb.INTERIOR_DIRICHLET, sb.density_on_refined(els, tau), tg)
        k = upd.k
    err = float(np.max(np.linalg.norm(vel - exact, axis=1) / np.linalg.norm(exact, axis=1)))
    print(f"step {i}: gap {gaps[i]:.4f} m {m} panels {len(near)} k {k} err {err:.3e}", flush=True)
