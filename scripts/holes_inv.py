"""Diagnostic: telescoping inverse of one subtree in numpy from the device-compressed factors."""
import sys
from pathlib import Path
import numpy as np
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
sys.path.insert(0, str(Path(__file__).resolve().parents[1] / "tests"))
import paper_2108_07205_b200 as sb  # noqa: E402
from paper_2108_07205_b200.configs import CONFIGS  # noqa: E402
from hbs1_np import read_hbs1  # noqa: E402
c = CONFIGS["cfg5"]
sb.init(0)
W, H = [int(x) for x in sys.argv[1].split(":")]
root = int(sys.argv[2])
wall = sb.panelize(sb.ellipse(c.a, c.b), W, c.q)
base, _ = sb.add_holes(wall, [(sb.circle(c.hole_radius, tuple(p)), H, c.q) for p in c.hole_centers()])
h = sb.hbs_compress(base, sb.MIXED, opts=sb.HbsOptions(eps=c.eps))
sb.hbs_save(h, "/tmp/hc.hbs1")
op = read_hbs1("/tmp/hc.hbs1")
nodes = op["nodes"]
dhat = {}
worst = []


def rc(m):
    s = np.linalg.svd(m, compute_uv=False)
    return s[-1] / s[0] if s[0] > 0 else 0.0


def inv(i):
    nd = nodes[i]
    if nd.left < 0:
        x = nd.d
    else:
        inv(nd.left)
        inv(nd.right)
        L, R = nodes[nd.left], nodes[nd.right]
        x = np.block([[dhat[nd.left], L.b_sib], [R.b_sib, dhat[nd.right]]])
    r1 = rc(x)
    xi = np.linalg.inv(x)
    tu = nd.v.T @ xi @ nd.u
    r2 = rc(tu)
    dhat[i] = np.linalg.inv(tu)
    if nd.depth <= 4 or r1 < 1e-10 or r2 < 1e-10:
        print(i, nd.depth, (nd.begin, nd.end), "c", x.shape[0], "k", nd.k, "rcond x %.2e" % r1,
              "rcond tu %.2e" % r2, flush=True)


inv(root)
