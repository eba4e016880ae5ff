"""N > 1 path on CPU: the subtree-partitioned HBS solve of
paper_2108_07205_b200/parallel.py (exchange protocol) over gloo with
world_size 2 and 4, each rank computing its subtree with the host executor
of tests/hbs1_np.py on the oracle's HBS1 factors; the gathered solution must
equal the oracle's unpartitioned hbs_solve (hbs.cpp:589-625)."""
import os
import socket
import sys
from pathlib import Path

import numpy as np
import pytest

ROOT = Path(__file__).resolve().parents[1]


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, hbs_path, b_path, out_dir):
    sys.path.insert(0, str(ROOT))
    sys.path.insert(0, str(ROOT / "tests"))
    import torch
    import torch.distributed as dist

    from hbs1_np import HostShardExecutor, read_hbs1
    from paper_2108_07205_b200.parallel import ShardedHbsSolver

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        op = read_hbs1(hbs_path)
        b = np.load(b_path)

        class TorchHost(HostShardExecutor):  # gloo exchanges torch CPU tensors
            def up(self, b_local):
                return torch.from_numpy(super().up(b_local.numpy()))

            def down(self, hats, nrhs):
                return torch.from_numpy(super().down(hats.numpy(), nrhs))

        ex = TorchHost(op, world, rank)
        solver = ShardedHbsSolver(ex)
        r0, r1 = solver.rows
        x = solver.solve(torch.from_numpy(np.ascontiguousarray(b[r0:r1])))
        np.save(Path(out_dir) / f"x{rank}.npy", x.numpy())
        np.save(Path(out_dir) / f"r{rank}.npy", np.array([r0, r1]))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 4])
def test_subtree_partitioned_solve_matches_oracle(po, tmp_path, world):
    import torch.multiprocessing as mp
    g = po.Geom.create(po.STAR, 24, prongs=5, amplitude=0.3)  # 384 nodes, depth 3
    h = po.Hbs.compress(po.Assembler.create(g), 1e-10).invert()
    h.save(tmp_path / "h.hbs1")
    n = 2 * g.n_nodes
    b = np.random.default_rng(3).uniform(-1, 1, (n, 3))
    np.save(tmp_path / "b.npy", b)
    mp.start_processes(_worker, args=(world, _free_port(), str(tmp_path / "h.hbs1"), str(tmp_path / "b.npy"),
                                      str(tmp_path)), nprocs=world, join=True, start_method="spawn")
    x = np.zeros_like(b)
    covered = np.zeros(n, dtype=int)
    for r in range(world):
        r0, r1 = np.load(tmp_path / f"r{r}.npy")
        x[r0:r1] = np.load(tmp_path / f"x{r}.npy")
        covered[r0:r1] += 1
    assert np.all(covered == 1)  # the subtrees tile the rows exactly once
    ref = h.solve(b)
    assert np.linalg.norm(x - ref) <= 1e-12 * np.linalg.norm(ref)


def _scalars(nodes):
    return np.stack([2 * np.asarray(nodes), 2 * np.asarray(nodes) + 1], 1).reshape(-1)


def _wb_worker(rank, world, port, case_dir):
    sys.path.insert(0, str(ROOT))
    sys.path.insert(0, str(ROOT / "tests"))
    import torch
    import torch.distributed as dist

    from hbs1_np import HostShardExecutor, read_hbs1
    from paper_2108_07205_b200.parallel import ShardedHbsSolver, ShardedWoodbury

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        d = np.load(Path(case_dir) / "case.npz")
        op = read_hbs1(str(Path(case_dir) / "h.hbs1"))

        class TorchHost(HostShardExecutor):
            def up(self, b_local):
                return torch.from_numpy(super().up(b_local.numpy()))

            def down(self, hats, nrhs):
                return torch.from_numpy(super().down(hats.numpy(), nrhs))

        app = d["app"]

        def app_solve(v):  # the dense branch of els_build (2 N_p <= 2048), rank 0 only
            return torch.from_numpy(np.linalg.solve(app, v.numpy()))

        n_k, n_c, n_p = (int(x) for x in d["sizes"])
        hbs = ShardedHbsSolver(TorchHost(op, world, rank))
        wb = ShardedWoodbury(hbs, torch.from_numpy(d["L"]), torch.from_numpy(d["R"]), d["old_of_ext"],
                             n_k, n_c, n_p, app_solve=app_solve if rank == 0 else None)
        g = torch.from_numpy(d["g"])
        y, y_p = wb.solve(wb.local_rows(g), g[n_k + n_c:] if rank == 0 else None)
        np.save(Path(case_dir) / f"y{rank}.npy", y.numpy())
        np.save(Path(case_dir) / f"own{rank}.npy", np.stack([wb.own.numpy(), wb.pos.numpy()]))
        if rank == 0:
            np.save(Path(case_dir) / "yp.npy", y_p.numpy())
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 4])
def test_sharded_woodbury_matches_oracle(po, tmp_path, world):
    """ShardedWoodbury (parallel.py): X and R follow the subtree row
    ownership, A_pp on rank 0, all-reduce of R X and R y; the assembled
    extended solution equals the oracle's els_solve_raw (els.cpp:147-179)."""
    import torch.multiprocessing as mp
    eps = 1e-10
    o0 = po.Geom.create(po.STAR, 24, prongs=5, amplitude=0.3)
    o1, plan = o0.refine([3, 17], 4)
    a0, a1 = po.Assembler.create(o0), po.Assembler.create(o1)
    h = po.Hbs.compress(a0, eps).invert()
    h.save(tmp_path / "h.hbs1")
    upd = po.Update.compress(a0, a1, plan, eps)
    els = po.Els.build(h, a0, a1, plan, upd)
    f = upd.factors()
    m = plan.maps()
    old_of_ext = np.concatenate([_scalars(m["kept_old"]), _scalars(m["cut_old"])])
    added = _scalars(m["added_new"])
    n_k, n_c, n_p = 2 * len(m["kept_old"]), 2 * len(m["cut_old"]), len(added)
    g = np.random.default_rng(11).uniform(-1, 1, (n_k + n_c + n_p, 3))
    g[n_k:n_k + n_c] = 0.0  # g_ext = (g_k, 0, g_p)  (els.cpp:167-169)
    np.savez(tmp_path / "case.npz", L=f["L"], R=f["R"], old_of_ext=old_of_ext, app=a1.submatrix(added, added),
             sizes=np.array([n_k, n_c, n_p]), g=g)
    mp.start_processes(_wb_worker, args=(world, _free_port(), str(tmp_path)), nprocs=world, join=True,
                       start_method="spawn")
    y = np.zeros_like(g)
    covered = np.zeros(n_k + n_c, dtype=int)
    for r in range(world):
        own, pos = np.load(tmp_path / f"own{r}.npy")
        y[own] = np.load(tmp_path / f"y{r}.npy")[pos]
        covered[own] += 1
    assert np.all(covered == 1)
    y[n_k + n_c:] = np.load(tmp_path / "yp.npy")
    ref = els.solve_raw(g)
    assert np.linalg.norm(y - ref) <= 1e-10 * np.linalg.norm(ref)


def _col_worker(rank, world, port, hbs_path, b_path, out_dir):
    sys.path.insert(0, str(ROOT))
    sys.path.insert(0, str(ROOT / "tests"))
    import torch.distributed as dist

    from hbs1_np import read_hbs1, HostShardExecutor
    from paper_2108_07205_b200.parallel import solve_columns

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        op = read_hbs1(hbs_path)
        b = np.load(b_path)
        full = HostShardExecutor(op, 1, 0)  # one "rank" owning the whole tree: the plain host solve

        def host_solve(_h, blk):
            return full.down(full.up(blk)[None], blk.shape[1])

        (c0, c1), x = solve_columns(op, b, solve=host_solve)
        np.save(Path(out_dir) / f"c{rank}.npy", np.array([c0, c1]))
        np.save(Path(out_dir) / f"x{rank}.npy", x)
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_column_sharded_solve_matches_oracle(po, tmp_path, world):
    """Batched right-hand sides split by column across ranks (no exchange,
    parallel.solve_columns): the assembled columns equal the oracle's
    unpartitioned hbs_solve."""
    import torch.multiprocessing as mp
    o = po.Geom.create(po.STAR, 16, prongs=5, amplitude=0.3)
    h = po.Hbs.compress(po.Assembler.create(o), 1e-10).invert()
    h.save(tmp_path / "h.hbs1")
    b = np.random.default_rng(2).standard_normal((h.info()["n"], 7))
    np.save(tmp_path / "b.npy", b)
    mp.start_processes(_col_worker, args=(world, _free_port(), str(tmp_path / "h.hbs1"), str(tmp_path / "b.npy"),
                                          str(tmp_path)), nprocs=world, join=True, start_method="spawn")
    x = np.zeros_like(b)
    seen = np.zeros(b.shape[1], dtype=int)
    for r in range(world):
        c0, c1 = np.load(tmp_path / f"c{r}.npy")
        x[:, c0:c1] = np.load(tmp_path / f"x{r}.npy")
        seen[c0:c1] += 1
    assert np.all(seen == 1)
    ref = h.solve(b)
    assert np.linalg.norm(x - ref) <= 1e-12 * np.linalg.norm(ref)
