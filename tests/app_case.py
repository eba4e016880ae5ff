"""Subprocess body of test_gpu_parity.test_fused_app_build_bitwise: one
refined-wall solve whose added block is large enough for its own HBS
(2 N_p > 2048 scalars, els.hpp:40); the A_pp build mode is read once per
process (SBX_APP_UNFUSED), so each mode runs in its own interpreter.
argv: output .npy."""
import sys

import numpy as np

import paper_2108_07205_b200 as sb
from oracle import pyoracle as po


def main():
    sb.init(0)
    eps = 1e-10
    g0 = sb.panelize(sb.star(5, 0.3), 64, 16)
    h = sb.hbs_invert(sb.hbs_compress(g0, opts=sb.HbsOptions(eps=eps)))
    g1, plan = sb.refine(g0, [10, 11, 12, 13, 14, 15, 16, 17], 16)
    upd = sb.compress_update(g0, g1, plan, eps)
    els = sb.els_build(h, g0, g1, plan, upd)
    assert els.info()["app_hbs"] == 1
    src = po.ring_sources(4, (0.0, 0.0), 3.0)
    tau = sb.els_solve(els, sb.gather_kept_added(plan, sb.boundary_data(g1, src)))
    np.save(sys.argv[1], tau)


if __name__ == "__main__":
    main()
