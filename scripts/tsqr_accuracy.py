"""Diagnostic: ID error of the crowded-batch TSQR engine (engine 1) on tall
W^T with a decaying spectrum; run once per kernel (SBX_TSQR_WARP=1 selects
the warp-layout kernel) and compare."""
import sys
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import paper_2108_07205_b200 as sb  # noqa: E402


def spectrum_matrix(m, n, sv, rng):
    u = np.linalg.qr(rng.standard_normal((m, len(sv))))[0]
    v = np.linalg.qr(rng.standard_normal((n, len(sv))))[0]
    return (u * sv) @ v.T


sb.init(0)
for (m, n) in [(128, 700), (114, 855), (64, 3000), (127, 511), (96, 400), (120, 1200)]:
    errs, ks = [], []
    for seed in range(6):
        rng = np.random.default_rng(seed * 1000 + m)
        r = min(m, n)
        w = spectrum_matrix(m, n, 10.0 ** (-16 * np.arange(r) / r), rng)
        k, J, P = sb.row_id(w, 1e-10, engine=1)
        errs.append(np.linalg.norm(w - P @ w[J[:k]], 2) / np.linalg.norm(w, 2))
        ks.append(k)
    print(f"{m}x{n}: k {ks}  err max {max(errs):.2e} mean {np.mean(errs):.2e}")
