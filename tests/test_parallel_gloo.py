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
