"""Subprocess body of test_gpu_fullsize.test_cfg3_tier1_collapsed_top: the
collapse depth is read once per process (SBX_SWEEP_TOP), so the forced depth
runs in its own interpreter.  argv: directory holding h.hbs1 (oracle
factors, 131072 unknowns), b.npy (n x 256) and x.npy (oracle solve)."""
import sys
from pathlib import Path

import numpy as np

import paper_2108_07205_b200 as sb


def rel(a, b):
    return float(np.linalg.norm(a - b) / np.linalg.norm(b))


def main():
    d = Path(sys.argv[1])
    sb.init(0)
    import torch
    h = sb.hbs_load(d / "h.hbs1")
    b, x = np.load(d / "b.npy"), np.load(d / "x.npy")
    for nrhs in (1, 32, 256):
        xd = sb.hbs_solve(h, torch.from_numpy(np.ascontiguousarray(b[:, :nrhs])).cuda()).cpu().numpy()
        e = rel(xd, x[:, :nrhs])
        print(f"nrhs {nrhs}: {e:.2e}", flush=True)
        assert e < 1e-12, (nrhs, e)
    print("top", h.info()["top_L"])


if __name__ == "__main__":
    main()
