"""Device subtree-partitioned solve and Woodbury through the native C-ABI
path (sbx_hbs_solve_sharded, sbx_els_shard_*; multigpu.cpp) against the
unpartitioned device solves.  One GPU here, so the G ranks are a loopback
group (sbx_comm_create_loopback): one host thread and one stream per rank,
each with its own copy of the HBS operator (as on separate GPUs), exchanging
through the same Collective interface the NCCL communicator implements.  The
NCCL communicator itself runs with world size 1; the exchange protocol at
world sizes 2 and 4 is also covered over gloo (test_parallel_gloo.py)."""
import threading

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def setup(tmp_path_factory):
    import torch

    import paper_2108_07205_b200 as sb
    sb.init(0)
    g = sb.panelize(sb.star(5, 0.3), 64, 16)  # 1024 nodes, 16 leaves, depth 4
    h = sb.hbs_invert(sb.hbs_compress(g, opts=sb.HbsOptions(eps=1e-10)))
    path = tmp_path_factory.mktemp("shard") / "h.hbs1"
    sb.hbs_save(h, path)
    return sb, torch, h, g, path


def _ranks(G, fn):
    """Run fn(p) for p < G in G threads (loopback ranks); re-raise the first error."""
    errs, out = [], [None] * G

    def run(p):
        try:
            out[p] = fn(p)
        except BaseException as e:  # noqa: BLE001
            errs.append(e)

    th = [threading.Thread(target=run, args=(p,)) for p in range(G)]
    for t in th:
        t.start()
    for t in th:
        t.join(timeout=600)
    assert not any(t.is_alive() for t in th), "loopback ranks did not finish"
    if errs:
        raise errs[0]
    return out


@pytest.mark.parametrize("G", [1, 2, 4, 8])
@pytest.mark.parametrize("nrhs", [1, 5, 64])
def test_native_sharded_solve_matches_full(setup, G, nrhs):
    from paper_2108_07205_b200.parallel import Comm, NativeShardedSolver
    sb, torch, h, _, path = setup
    n = h.info()["n"]
    b = torch.empty((n, nrhs), dtype=torch.float64, device="cuda").uniform_(-1, 1)
    ref = sb.hbs_solve(h, b)
    comms = Comm.loopback(G)
    ops = [sb.hbs_load(path) for _ in range(G)]  # one operator per rank, as on G GPUs
    streams = [torch.cuda.Stream() for _ in range(G)]

    def rank(p):
        solver = NativeShardedSolver(ops[p], comms[p])
        r0, r1 = solver.rows
        with torch.cuda.stream(streams[p]):
            x = solver.solve(b[r0:r1])
            streams[p].synchronize()
        return r0, r1, x

    res = _ranks(G, rank)
    assert res[0][0] == 0 and res[-1][1] == n
    assert all(res[p][1] == res[p + 1][0] for p in range(G - 1))
    x = torch.cat([r[2] for r in res])
    err = (torch.linalg.norm(x - ref) / torch.linalg.norm(ref)).item()
    assert err <= 1e-13, err
    # host buffers through the same call
    xh = _ranks(G, lambda p: NativeShardedSolver(ops[p], comms[p]).solve(
        b[res[p][0]:res[p][1]].cpu().numpy()))
    assert np.linalg.norm(np.vstack(xh) - ref.cpu().numpy()) <= 1e-13 * np.linalg.norm(ref.cpu().numpy())


def test_nccl_communicator_world_one(setup):
    """The NCCL communicator set of the C-ABI (world size 1 on one GPU)."""
    from paper_2108_07205_b200.parallel import Comm, NativeShardedSolver
    sb, torch, h, _, _ = setup
    c = Comm.create(Comm.unique_id(), 1, 0)
    assert c.info() == (1, 0)
    b = torch.empty((h.n, 3), dtype=torch.float64, device="cuda").uniform_(-1, 1)
    x = NativeShardedSolver(h, c).solve(b)
    assert torch.equal(x, sb.hbs_solve(h, b))


def test_shard_rejects_bad_rank_count(setup):
    from paper_2108_07205_b200.parallel import Comm, NativeShardedSolver
    sb, torch, h, _, _ = setup
    with pytest.raises(ValueError):
        NativeShardedSolver(h, Comm.loopback(3)[0])
    with pytest.raises(ValueError):
        NativeShardedSolver(h, Comm.loopback(64)[0])  # deeper than the tree


@pytest.mark.parametrize("G", [1, 2, 4])
@pytest.mark.parametrize("n_refine", [2, 8])
def test_native_sharded_woodbury_matches_els(setup, G, n_refine):
    """sbx_els_shard_build / solve (X rows and R columns by subtree, A_pp on
    rank 0, all-reduce of R X and R y, W^{-1} on every rank) against the
    unpartitioned els_solve_raw.  8 refined panels at m = 16 put the added
    block on its own HBS (2 N_p > 2048)."""
    from paper_2108_07205_b200.parallel import Comm, NativeShardedWoodbury
    sb, torch, h, g, path = setup
    panels = list(range(10, 10 + n_refine))
    g1, plan = sb.refine(g, panels, 16 if n_refine == 8 else 4)
    upd = sb.compress_update(g, g1, plan, 1e-10)
    els = sb.els_build(h, g, g1, plan, upd)
    info = els.info()
    n_k, n_c, n_p = info["n_k"], info["n_c"], info["n_p"]
    gx = torch.empty((n_k + n_c + n_p, 4), dtype=torch.float64, device="cuda").uniform_(-1, 1)
    gx[n_k:n_k + n_c] = 0.0
    ref = sb.els_solve_raw(els, gx)
    comms = Comm.loopback(G)
    ops = [sb.hbs_load(path) for _ in range(G)]
    streams = [torch.cuda.Stream() for _ in range(G)]

    def rank(p):
        with torch.cuda.stream(streams[p]):
            wb = NativeShardedWoodbury(ops[p], comms[p], g, g1, plan, upd, stream=streams[p].cuda_stream)
            y, y_p = wb.solve(wb.local_rows(gx), gx[n_k + n_c:] if p == 0 else None)
            streams[p].synchronize()
        return wb.ext_rows, y, y_p, wb.k

    res = _ranks(G, rank)
    out = torch.zeros_like(gx)
    for p, (rows, y, y_p, k) in enumerate(res):
        assert k == upd.k
        out[torch.as_tensor(rows, device="cuda")] = y
        if p == 0 and n_p:
            out[n_k + n_c:] = y_p
    covered = np.sort(np.concatenate([r[0] for r in res]))
    assert np.array_equal(covered, np.arange(n_k + n_c))
    err = (torch.linalg.norm(out - ref) / torch.linalg.norm(ref)).item()
    assert err <= 1e-10, err


@pytest.mark.parametrize("n_refine,m", [(2, 4), (8, 16)])
def test_app_block_solver(setup, n_refine, m):
    """sbx_app_build / sbx_app_solve (the added block of els_build,
    els.cpp:107-118): dense LU below 2048 scalars, its own HBS above; the
    plain and transposed solves against a dense solve of A_pp."""
    sb, torch, h, g, _ = setup
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


@pytest.mark.parametrize("G", [2, 4])
@pytest.mark.parametrize("panels", [64, 256])
def test_sharded_compression_and_storage(setup, po, G, panels):
    """sbx_hbs_compress_sharded (one-time compression and
    factor storage by subtree): each loopback rank compresses and inverts only
    its subtree plus the top levels (skeleton lists, the subtree roots'
    couplings and dhat blocks exchanged through the communicator), stores a
    fraction of the factors, and the sharded solve over those factors matches
    the unsharded operator's solve and the dense system."""
    from paper_2108_07205_b200.parallel import Comm, NativeShardedSolver, compress_sharded
    sb, torch, _, _, _ = setup
    g = sb.panelize(sb.star(5, 0.3), panels, 16)
    full = sb.hbs_invert(sb.hbs_compress(g, opts=sb.HbsOptions(eps=1e-10)))
    n = full.n
    b = torch.empty((n, 3), dtype=torch.float64, device="cuda").uniform_(-1, 1)
    ref = sb.hbs_solve(full, b)
    comms = Comm.loopback(G)
    streams = [torch.cuda.Stream() for _ in range(G)]

    def rank(p):
        with torch.cuda.stream(streams[p]):
            h = compress_sharded(g, comms[p], opts=sb.HbsOptions(eps=1e-10))
            sb.hbs_invert(h)
            solver = NativeShardedSolver(h, comms[p])
            r0, r1 = solver.rows
            x = solver.solve(b[r0:r1])
            streams[p].synchronize()
        return r0, r1, x, h.info()

    res = _ranks(G, rank)
    x = torch.cat([r[2] for r in res])
    err = (torch.linalg.norm(x - ref) / torch.linalg.norm(ref)).item()
    assert err <= 1e-9, err
    full_arena = full.info()["arena_doubles"]
    for r0, r1, _, info in res:
        assert info["sharded"] == 1
        assert info["arena_doubles"] < 0.75 * full_arena, (info["arena_doubles"], full_arena)
    # the dense system (oracle assembler) is solved
    if panels == 64:
        A = po.Assembler.create(po.Geom.create(po.STAR, panels, prongs=5, amplitude=0.3)).full_matrix()
        xb = x.cpu().numpy()
        assert np.linalg.norm(A @ xb - b.cpu().numpy()) <= 1e-8 * np.linalg.norm(b.cpu().numpy())
    # a sharded operator refuses the unsharded paths
    h0 = res[0][3]
    assert h0["has_inverse"] == 1
