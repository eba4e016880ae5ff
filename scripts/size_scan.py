"""Diagnostic: static interior HBS at growing sizes (overflow hunt)."""
import sys
from pathlib import Path
import numpy as np
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import paper_2108_07205_b200 as sb  # noqa: E402

sb.init(0)
for spec in sys.argv[1:]:
    kind, P = spec.split(":")
    P = int(P)
    curve = sb.star(5, 0.3) if kind == "star" else sb.ellipse(8.0, 4.0)
    g = sb.panelize(curve, P, 16)
    h = sb.hbs_compress(g, opts=sb.HbsOptions(eps=1e-10))
    info = h.info()
    try:
        sb.hbs_invert(h)
        b = np.random.default_rng(0).standard_normal(info["n"])
        x = sb.hbs_solve(h, b)
        r = np.linalg.norm(sb.hbs_apply(h, x) - b) / np.linalg.norm(b)
        print(spec, info["n"], "ok", f"{r:.2e}", info["max_k"], info["max_depth"], flush=True)
    except Exception as e:  # noqa: BLE001
        print(spec, info["n"], "FAIL", e, info["max_k"], info["max_depth"], flush=True)
