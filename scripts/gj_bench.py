"""Kernel time of the dense inverse (CUDA events, sbx_kernel_time) per size."""
import sys
from pathlib import Path
import numpy as np
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import paper_2108_07205_b200 as sb
sb.init(0)
sb.api.kernel_timing(True)
for n in (96, 128, 146, 160):
    a = np.eye(n) + np.random.default_rng(n).standard_normal((n, n)) * 0.1
    for _ in range(3):
        sb.dense_inverse(a)
    for name in ("gj_inverse_dmma", "gj_inverse"):
        sb.api.kernel_time(name, True)
    for _ in range(10):
        inv, rc = sb.dense_inverse(a)
    for name in ("gj_inverse_dmma", "gj_inverse"):
        ms, cnt = sb.api.kernel_time(name, True)
        if cnt:
            print(f"n={n} {name}: {1e3 * ms / cnt:.1f} us per launch ({cnt}), resid {np.linalg.norm(inv @ a - np.eye(n)):.2e} rc {rc:.3e}")
