"""Row-ID engine micro-benchmark on representative W shapes (diagnostic).

  python scripts/id_micro.py [engine ...]
Shapes (W rows = candidates, cols = functionals): final-ID far group
(31000 x 56), an HBS sample round box (128 x 900), a far-ID leaf (256 x 513),
a near-ID chunk (256 x 8192)."""
import sys
import time
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import paper_2108_07205_b200 as sb  # noqa: E402

SHAPES = [(31000, 56, 56), (128, 900, 60), (256, 513, 70), (256, 8192, 30)]


def mat(m, n, r, rng):
    u = np.linalg.qr(rng.standard_normal((m, r)))[0]
    v = np.linalg.qr(rng.standard_normal((n, r)))[0]
    return (u * 10.0 ** (-12 * np.arange(r) / r)) @ v.T


def main():
    engines = [int(e) for e in sys.argv[1:]] or [1, 3]
    sb.init(0)
    rng = np.random.default_rng(0)
    for m, n, r in SHAPES:
        w = mat(m, n, r, rng)
        for e in engines:
            sb.row_id(w, 1e-10, engine=e)
            t0 = time.perf_counter()
            k, J, P = sb.row_id(w, 1e-10, engine=e)
            t1 = time.perf_counter()
            print(f"W {m}x{n} engine {e}: k={k} {1e3 * (t1 - t0):.2f} ms (with host copies)", flush=True)


if __name__ == "__main__":
    main()
