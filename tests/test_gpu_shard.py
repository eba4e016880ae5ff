"""Device subtree-partitioned solve (sbx_hbs_solve_shard_up/down) against the
unpartitioned device hbs_solve.  One GPU here: the G ranks run one after the
other in this process and the all-gather is a host-side stack; the real
exchange over NCCL is the same ShardedHbsSolver.solve call exercised over
gloo in test_parallel_gloo.py."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def setup():
    import torch

    import paper_2108_07205_b200 as sb
    from paper_2108_07205_b200.parallel import DeviceExecutor
    sb.init(0)
    g = sb.panelize(sb.star(5, 0.3), 64, 16)  # 1024 nodes, 16 leaves, depth 4
    h = sb.hbs_invert(sb.hbs_compress(g, opts=sb.HbsOptions(eps=1e-10)))
    return sb, torch, DeviceExecutor, h


@pytest.mark.parametrize("G", [1, 2, 4, 8])
@pytest.mark.parametrize("nrhs", [1, 5, 64])
def test_shard_solve_matches_full(setup, G, nrhs):
    sb, torch, DeviceExecutor, h = setup
    n = h.info()["n"]
    b = torch.empty((n, nrhs), dtype=torch.float64, device="cuda").uniform_(-1, 1)
    ref = sb.hbs_solve(h, b)
    exes = [DeviceExecutor(h, G, p) for p in range(G)]
    rows = [(e.row0, e.row1) for e in exes]
    assert rows[0][0] == 0 and rows[-1][1] == n
    assert all(rows[p][1] == rows[p + 1][0] for p in range(G - 1))
    hats = [exes[p].up(b[rows[p][0]:rows[p][1]]) for p in range(G)]
    kmax = exes[0].kmax
    gathered = (torch.stack(hats) if kmax > 0
                else torch.zeros((G, 0, nrhs), dtype=torch.float64, device="cuda"))
    x = torch.empty_like(b)
    for p in range(G):
        x[rows[p][0]:rows[p][1]] = exes[p].down(gathered, nrhs)
    torch.cuda.synchronize()
    err = (torch.linalg.norm(x - ref) / torch.linalg.norm(ref)).item()
    assert err <= 1e-13, err


def test_shard_rejects_bad_rank_count(setup):
    sb, torch, DeviceExecutor, h = setup
    with pytest.raises(ValueError):
        DeviceExecutor(h, 3, 0)
    with pytest.raises(ValueError):
        DeviceExecutor(h, 64, 0)  # deeper than the tree
