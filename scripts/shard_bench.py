"""cfg3 HBS-apply microbenchmark split by leaf subtrees across GPUs
(SURVEY.md §8e).  Launch one process per GPU:

  python -m torch.distributed.run --nnodes=1 --nproc-per-node N \
      --master-addr 127.0.0.1 --master-port 29511 scripts/shard_bench.py --nrhs 1,32,256

Each rank builds the static HBS inverse of cfg3 (the same operator on every
rank), then times `NativeShardedSolver.solve` (sbx_hbs_solve_sharded: local up-sweep, NCCL all-gather
of the subtree-root hats, top levels + local down-sweep) with CUDA events on
its stream; rank 0 prints the max over ranks and checks the gathered
solution against a single-GPU hbs_solve.
"""
import argparse
import json
import os
import sys
from pathlib import Path

import torch
import torch.distributed as dist

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import paper_2108_07205_b200 as sb  # noqa: E402
from paper_2108_07205_b200.configs import CONFIGS  # noqa: E402
from paper_2108_07205_b200.parallel import Comm, NativeShardedSolver  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--cfg", default="cfg3")
    ap.add_argument("--nrhs", default="1,32,256")
    ap.add_argument("--reps", type=int, default=10)
    a = ap.parse_args()
    rank = int(os.environ.get("RANK", 0))
    world = int(os.environ.get("WORLD_SIZE", 1))
    local = int(os.environ.get("LOCAL_RANK", 0))
    torch.cuda.set_device(local)
    dist.init_process_group("nccl" if world > 1 else "gloo", rank=rank, world_size=world,
                            device_id=torch.device("cuda", local) if world > 1 else None)
    sb.init(local)
    c = CONFIGS[a.cfg]
    g = sb.panelize(sb.star(c.prongs, c.amplitude, c.a), c.n_panels, c.q)
    h = sb.hbs_invert(sb.hbs_compress(g, opts=sb.HbsOptions(eps=c.eps, leaf_nodes=c.leaf)))
    n = h.info()["n"]
    solver = NativeShardedSolver(h, Comm.from_process_group())
    r0, r1 = solver.rows
    out = []
    for nrhs in [int(x) for x in a.nrhs.split(",")]:
        gen = torch.Generator(device="cuda").manual_seed(7)
        b = torch.empty((n, nrhs), dtype=torch.float64, device="cuda").uniform_(-1, 1, generator=gen)
        bl = b[r0:r1].contiguous()
        for _ in range(3):
            x = solver.solve(bl)
        dist.barrier()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(a.reps):
            x = solver.solve(bl)
        e1.record()
        torch.cuda.synchronize()
        ms = torch.tensor([e0.elapsed_time(e1) / a.reps], device="cuda")
        if world > 1:
            dist.all_reduce(ms, op=dist.ReduceOp.MAX)
        ref = sb.hbs_solve(h, b)[r0:r1]
        err = torch.tensor([(torch.linalg.norm(x - ref) / torch.linalg.norm(ref)).item()], device="cuda")
        if world > 1:
            dist.all_reduce(err, op=dist.ReduceOp.MAX)
        fb = h.info()["factor_doubles"] * 8
        out.append({"nrhs": nrhs, "ms": round(ms.item(), 4), "rel_err_vs_1gpu": err.item(),
                    "factor_GBps_per_pass": round(fb / (ms.item() * 1e-3) / 1e9, 1)})
    if rank == 0:
        print(json.dumps({"bench": "sharded hbs_solve", "cfg": a.cfg, "n": n, "gpus": world,
                          "results": out}))
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
