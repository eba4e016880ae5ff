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
    return sb, torch, DeviceExecutor, h, g


@pytest.mark.parametrize("G", [1, 2, 4, 8])
@pytest.mark.parametrize("nrhs", [1, 5, 64])
def test_shard_solve_matches_full(setup, G, nrhs):
    sb, torch, DeviceExecutor, h, _ = setup
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
    sb, torch, DeviceExecutor, h, _ = setup
    with pytest.raises(ValueError):
        DeviceExecutor(h, 3, 0)
    with pytest.raises(ValueError):
        DeviceExecutor(h, 64, 0)  # deeper than the tree


@pytest.mark.parametrize("n_refine", [2, 8])
def test_sharded_woodbury_device_matches_els(setup, n_refine):
    """ShardedWoodbury (parallel.py) on the device pieces — the partitioned
    HBS solve, sbx_app_solve for the added block, the update factors — on a
    one-rank NCCL group; equals the device els_solve_raw.  The multi-rank
    exchange is covered over gloo (test_parallel_gloo.py).  8 refined panels
    at m = 16 put the added block on its own HBS (2 N_p > 2048)."""
    import os
    import socket

    import torch.distributed as dist

    from paper_2108_07205_b200.parallel import ShardedHbsSolver, ShardedWoodbury
    sb, torch, DeviceExecutor, h, g = setup
    if not dist.is_initialized():
        s = socket.socket()
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
        s.close()
        os.environ["MASTER_ADDR"] = "127.0.0.1"
        os.environ["MASTER_PORT"] = str(port)
        dist.init_process_group("nccl", rank=0, world_size=1, device_id=torch.device("cuda", 0))
    panels = list(range(10, 10 + n_refine))
    g1, plan = sb.refine(g, panels, 16 if n_refine == 8 else 4)
    upd = sb.compress_update(g, g1, plan, 1e-10)
    els = sb.els_build(h, g, g1, plan, upd)
    app = sb.app_build(g1, plan, 1e-10)
    assert app.info()["hbs"] == (1 if n_refine == 8 else 0)
    L, R = upd.factors()
    m = plan.maps()

    def scal(v):
        return np.stack([2 * v, 2 * v + 1], 1).reshape(-1)

    old_of_ext = np.concatenate([scal(m["kept_old"]), scal(m["cut_old"])])
    n_k, n_c, n_p = 2 * len(m["kept_old"]), 2 * len(m["cut_old"]), 2 * len(m["added_new"])
    gx = torch.empty((n_k + n_c + n_p, 4), dtype=torch.float64, device="cuda").uniform_(-1, 1)
    gx[n_k:n_k + n_c] = 0.0
    wb = ShardedWoodbury(ShardedHbsSolver(DeviceExecutor(h, 1, 0)), torch.from_numpy(L).cuda(),
                         torch.from_numpy(R).cuda(), old_of_ext, n_k, n_c, n_p, app_solve=app.solve)
    y, y_p = wb.solve(wb.local_rows(gx), gx[n_k + n_c:])
    out = torch.zeros_like(gx)
    out[wb.own] = y[wb.pos]
    out[n_k + n_c:] = y_p
    ref = sb.els_solve_raw(els, gx)
    err = (torch.linalg.norm(out - ref) / torch.linalg.norm(ref)).item()
    if n_refine == 8 and dist.is_initialized():  # the last parametrisation tears the group down
        dist.destroy_process_group()
    assert err <= 1e-10, err


@pytest.mark.parametrize("n_refine,m", [(2, 4), (8, 16)])
def test_app_block_solver(setup, n_refine, m):
    """sbx_app_build / sbx_app_solve (the added block of els_build,
    els.cpp:107-118): dense LU below 2048 scalars, its own HBS above; the
    plain and transposed solves against a dense solve of A_pp."""
    sb, torch, DeviceExecutor, h, g = setup
    g1, plan = sb.refine(g, list(range(20, 20 + n_refine)), m)
    app = sb.app_build(g1, plan, 1e-10)
    added = plan.maps()["added_new"]
    s = np.stack([2 * added, 2 * added + 1], 1).reshape(-1)
    A = sb.submatrix(g1, s, s)
    assert app.info() == {"n_p": len(s), "hbs": 1 if len(s) > 2048 else 0}
    v = np.random.default_rng(n_refine).uniform(-1, 1, (len(s), 3))
    tol = 1e-11 if len(s) <= 2048 else 1e-8
    for tr in (False, True):
        ref = np.linalg.solve(A.T if tr else A, v)
        got = app.solve(v, transpose=tr)
        assert np.linalg.norm(got - ref) <= tol * np.linalg.norm(ref), tr
    vt = torch.from_numpy(v).cuda()
    assert np.allclose(app.solve(vt).cpu().numpy(), app.solve(v), rtol=0, atol=1e-13 * np.abs(v).max() * 1e3)
