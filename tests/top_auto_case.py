"""Subprocess body of test_gpu_parity.test_collapsed_top_auto: a device
compressed cfg2-size wall (tree depth 8), solved with the default top
choice; argv: output .npy; prints the chosen depth."""
import sys

import numpy as np

import paper_2108_07205_b200 as sb


def main():
    sb.init(0)
    g = sb.panelize(sb.star(5, 0.3), 1024, 16)
    h = sb.hbs_invert(sb.hbs_compress(g, opts=sb.HbsOptions(eps=1e-10)))
    b = np.random.default_rng(2).uniform(-1, 1, (h.info()["n"], 3))
    x = sb.hbs_solve(h, b)
    np.save(sys.argv[1], np.concatenate([x, sb.hbs_solve(h, b, transpose=True)], 1))
    print("top", h.info()["top_L"])


if __name__ == "__main__":
    main()
