"""Diagnostic: accuracy of the compressed Mixed HBS (apply vs exact rows)."""
import sys
from pathlib import Path
import numpy as np
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import paper_2108_07205_b200 as sb  # noqa: E402
from paper_2108_07205_b200.configs import CONFIGS  # noqa: E402
c = CONFIGS["cfg5"]
sb.init(0)
for spec in sys.argv[1:]:
    W, H = [int(x) for x in spec.split(":")]
    wall = sb.panelize(sb.ellipse(c.a, c.b), W, c.q)
    base, _ = sb.add_holes(wall, [(sb.circle(c.hole_radius, tuple(p)), H, c.q) for p in c.hole_centers()])
    h = sb.hbs_compress(base, sb.MIXED, opts=sb.HbsOptions(eps=c.eps))
    n = 2 * base.n_nodes()
    x = np.random.default_rng(1).standard_normal(n)
    y = sb.hbs_apply(h, x)
    rng = np.random.default_rng(2)
    rows = np.sort(rng.choice(n, 64, replace=False))
    ex = np.zeros(64)
    for c0 in range(0, n, 65536):
        cols = np.arange(c0, min(n, c0 + 65536))
        ex += sb.submatrix(base, rows, cols, sb.MIXED) @ x[cols]
    print(spec, n, "apply rel err on 64 rows", np.linalg.norm(y[rows] - ex) / np.linalg.norm(ex), flush=True)
