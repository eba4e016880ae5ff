"""Bisect helper: device row ID engines vs the oracle on one matrix."""
import sys
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import paper_2108_07205_b200 as sb  # noqa: E402
from oracle import pyoracle as po  # noqa: E402

sb.init(0)
for (m, n) in [(128, 700), (300, 5000), (2500, 300)]:
    rng = np.random.default_rng(m * 7 + n)
    r = min(m, n)
    u = np.linalg.qr(rng.standard_normal((m, r)))[0]
    v = np.linalg.qr(rng.standard_normal((n, r)))[0]
    w = (u * 10.0 ** (-14 * np.arange(r) / r)) @ v.T
    ko, Jo, Po = po.row_id(w, 1e-10)
    for e in (1, 2):
        k, J, P = sb.row_id(w, 1e-10, engine=e)
        first = next((i for i in range(min(k, ko)) if J[i] != Jo[i]), None)
        err = np.linalg.norm(w - P @ w[J[:k]], 2) / np.linalg.norm(w, 2)
        print(m, n, "engine", e, "k", k, "oracle", ko, "first pivot diff", first, "err", err, flush=True)
