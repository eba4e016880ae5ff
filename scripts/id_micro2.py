"""Diagnostic: one-CTA CPQR kernel time (CUDA events) on merge / HBS-round shapes."""
import sys
from pathlib import Path
import numpy as np
import torch
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import paper_2108_07205_b200 as sb  # noqa: E402

sb.init(0)
rng = np.random.default_rng(0)
for m, n, r in [(80, 257, 60), (140, 513, 70), (128, 900, 60), (128, 600, 100), (250, 300, 120)]:
    u = np.linalg.qr(rng.standard_normal((m, r)))[0]
    v = np.linalg.qr(rng.standard_normal((n, r)))[0]
    w = (u * 10.0 ** (-14 * np.arange(r) / r)) @ v.T
    sb.row_id(w, 1e-15, engine=1)
    t0 = torch.cuda.Event(enable_timing=True); t1 = torch.cuda.Event(enable_timing=True)
    import time
    ts = []
    for _ in range(5):
        a = time.perf_counter(); sb.row_id(w, 1e-15, engine=1); ts.append(time.perf_counter() - a)
    print(f"W {m}x{n} (rank {r}): {1e3*min(ts):.3f} ms (incl. host copies)", flush=True)
