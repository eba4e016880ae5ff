"""Subprocess body of test_gpu_parity.test_collapsed_top_matches_oracle: the
collapse depth is read once per process (SBX_SWEEP_TOP), so each depth runs
in its own interpreter.  argv: hbs1 path, rhs .npy, oracle solve .npy,
oracle transposed solve .npy."""
import sys

import numpy as np

import paper_2108_07205_b200 as sb


def rel(a, b):
    return float(np.linalg.norm(a - b) / np.linalg.norm(b))


def main():
    path, bp, xp, xtp = sys.argv[1:5]
    sb.init(0)
    d = sb.hbs_load(path)
    b, x, xt = np.load(bp), np.load(xp), np.load(xtp)
    for nrhs in (1, 3, 64, 130):
        e = rel(sb.hbs_solve(d, b[:, :nrhs]), x[:, :nrhs])
        et = rel(sb.hbs_solve(d, b[:, :nrhs], transpose=True), xt[:, :nrhs])
        print(f"nrhs {nrhs}: {e:.2e} {et:.2e}")
        assert e < 1e-12 and et < 1e-12, (nrhs, e, et)
    print("top", d.info().get("top_L", "?"))


if __name__ == "__main__":
    main()
