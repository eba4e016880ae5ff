"""Kernel time of the Woodbury operator's R X product (146 x 40960 x 146)."""
import sys
from pathlib import Path
import numpy as np
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import paper_2108_07205_b200 as sb
sb.init(0)
sb.api.kernel_timing(True)
rng = np.random.default_rng(0)
for (m, k, n) in ((146, 40960, 146), (160, 40960, 160), (100, 40960, 100), (146, 40960, 64)):
    a = rng.standard_normal((m, k)); b = rng.standard_normal((k, n))
    for _ in range(3):
        sb.matmul(a, b)
    sb.api.kernel_time("thin_gemm", True)
    for _ in range(10):
        c = sb.matmul(a, b)
    ms, cnt = sb.api.kernel_time("thin_gemm", True)
    if cnt:
        print(f"{m}x{k}x{n} thin_gemm: {1e3*ms/cnt:.1f} us, {2*m*k*n/(ms/cnt*1e-3)/1e12:.2f} TF/s (incl. reduce)")
