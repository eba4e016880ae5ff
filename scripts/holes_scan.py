"""Diagnostic: static Mixed-formulation HBS on scaled-down cfg5 geometries."""
import sys
from pathlib import Path
import numpy as np
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import paper_2108_07205_b200 as sb  # noqa: E402
from paper_2108_07205_b200.configs import CONFIGS  # noqa: E402

c = CONFIGS["cfg5"]
sb.init(0)
for W, H in [(int(a), int(b)) for a, b in (x.split(":") for x in sys.argv[1:])]:
    wall = sb.panelize(sb.ellipse(c.a, c.b), W, c.q)
    base, _ = sb.add_holes(wall, [(sb.circle(c.hole_radius, tuple(p)), H, c.q) for p in c.hole_centers()])
    h = sb.hbs_compress(base, sb.MIXED, opts=sb.HbsOptions(eps=c.eps))
    info = h.info()
    try:
        sb.hbs_invert(h)
        b = np.random.default_rng(0).standard_normal(info["n"])
        x = sb.hbs_solve(h, b)
        r = np.linalg.norm(sb.hbs_apply(h, x) - b) / np.linalg.norm(b)
        print(W, H, info["n"], "ok", f"{r:.2e}", info["max_k"], flush=True)
    except Exception as e:  # noqa: BLE001
        print(W, H, info["n"], "FAIL", e, info["max_k"], info["max_depth"], flush=True)
