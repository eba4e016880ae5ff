"""cfg3 1-RHS hbs_solve: kernel time vs whole-call time (device tensors), with
and without the kernel timer's events."""
import sys, time
from pathlib import Path
import numpy as np
import torch
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import paper_2108_07205_b200 as sb
from paper_2108_07205_b200.configs import CONFIGS
sb.init(0)
c = CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "cfg3"]
g = sb.panelize(sb.star(c.prongs, c.amplitude, c.a), c.n_panels, c.q)
h = sb.hbs_invert(sb.hbs_compress(g, opts=sb.HbsOptions(eps=c.eps, leaf_nodes=c.leaf)))
n = h.info()["n"]
stream = torch.cuda.ExternalStream(sb.api.lib().sbx_stream())
b = torch.empty((n, 1), dtype=torch.float64, device="cuda").uniform_(-1, 1)
ref = sb.hbs_solve(h, b.cpu().numpy())
with torch.cuda.stream(stream):
    x = sb.hbs_solve(h, b)
torch.cuda.synchronize()
print("device vs host-path result:", float(np.linalg.norm(x.cpu().numpy() - ref) / np.linalg.norm(ref)))
for timing in (False, True):
    with torch.cuda.stream(stream):
        for _ in range(5):
            sb.hbs_solve(h, b)
        sb.api.kernel_timing(timing)
        sb.api.kernel_time("sweep_flow_gemv")
        e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        for _ in range(50):
            sb.hbs_solve(h, b)
        e1.record(stream)
    torch.cuda.synchronize()
    kms, cnt = sb.api.kernel_time("sweep_flow_gemv")
    sb.api.kernel_timing(False)
    print(f"kernel timing {timing}: call {e0.elapsed_time(e1)/50*1e3:.1f} us, kernel {1e3*kms/max(cnt,1):.1f} us ({cnt})")
