"""Diagnostic: ID error and rank of each CPQR engine on tall W^T with a
decaying spectrum (the shapes the per-step batches route to them)."""
import sys
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import paper_2108_07205_b200 as sb  # noqa: E402
from oracle import pyoracle as po  # noqa: E402


def spectrum_matrix(m, n, sv, rng):
    u = np.linalg.qr(rng.standard_normal((m, len(sv))))[0]
    v = np.linalg.qr(rng.standard_normal((n, len(sv))))[0]
    return (u * sv) @ v.T


sb.init(0)
for (m, n) in [(136, 600), (140, 800), (132, 520), (144, 770), (120, 700)]:
    line = f"{m}x{n}:"
    for eng in (1, 3, 4, 5):
        errs, ks, dj = [], [], []
        for seed in range(4):
            rng = np.random.default_rng(seed * 1000 + m)
            r = min(m, n)
            w = spectrum_matrix(m, n, 10.0 ** (-16 * np.arange(r) / r), rng)
            try:
                k, J, P = sb.row_id(w, 1e-10, engine=eng)
            except Exception as ex:  # engine not applicable
                errs.append(np.nan)
                continue
            ko, Jo, Po = po.row_id(w, 1e-10)
            errs.append(np.linalg.norm(w - P @ w[J[:k]], 2) / np.linalg.norm(w, 2))
            ks.append(k - ko)
            dj.append(int(np.argmax(J[:min(k, ko)] != Jo[:min(k, ko)])) if not np.array_equal(J[:min(k, ko)], Jo[:min(k, ko)]) else -1)
        line += f"  e{eng} err {np.nanmax(errs):.1e} dk {ks} firstdiff {dj}"
    print(line, flush=True)
