"""Multi-GPU HBS solve partitioned by leaf subtrees.

One process per GPU.  For G = 2^g ranks, rank p owns the subtree rooted at
the p-th BFS node of depth g of the HBS tree (hbs.cpp:379-383 halving makes
it a contiguous range of old-mesh rows).  One solve:

  1. local up-sweep of the owned subtree          (sbx_hbs_solve_shard_up)
  2. all-gather of the G subtree-root hat vectors  (NCCL over NVLink; the
     only data exchanged: G x kmax x nrhs doubles)
  3. top g levels, redundantly on every rank, and the local down-sweep
                                                   (sbx_hbs_solve_shard_down)

The sweeps run on the caller's current CUDA stream and the collective is
issued on that same stream through torch.distributed, so the exchange is
ordered with the sweeps without host synchronisation.
Batched right-hand sides can instead be split by column with no exchange at
all (`solve_columns`).

The executor abstraction separates the exchange protocol (this module) from
the per-rank compute: `DeviceExecutor` drives libsbx; tests drive the same
protocol with a host executor over gloo.
"""
from __future__ import annotations

import ctypes as C

from . import _sbx
from ._sbx import check, lib

VP = C.c_void_p


class DeviceExecutor:
    """Per-rank compute of the partitioned solve on this process's GPU."""

    def __init__(self, h, G: int, p: int):
        import torch
        self.torch = torch
        self.h, self.G, self.p = h, G, p
        r0, r1, km = C.c_int64(), C.c_int64(), C.c_int64()
        check(lib().sbx_hbs_shard_info(h.ptr, G, p, C.byref(r0), C.byref(r1), C.byref(km)))
        self.row0, self.row1, self.kmax = r0.value, r1.value, km.value

    def _stream(self):
        from .api import torch_stream_handle
        return VP(torch_stream_handle())

    def up(self, b_local):
        """b_local: CUDA float64 (rows x nrhs) -> packed hat (kmax x nrhs, row-major)."""
        torch = self.torch
        nrhs = b_local.shape[1]
        bcm = b_local.t().contiguous()  # column-major storage
        hat = torch.zeros((max(self.kmax, 1), nrhs), dtype=torch.float64, device=b_local.device)
        check(lib().sbx_hbs_solve_shard_up(self.h.ptr, self.G, self.p, VP(bcm.data_ptr()), bcm.shape[1],
                                           nrhs, VP(hat.data_ptr()), _sbx.SBX_DEVICE_PTRS, self._stream()))
        return hat[: self.kmax]

    def down(self, hats, nrhs):
        """hats: (G, kmax, nrhs) gathered blocks -> x_local (rows x nrhs)."""
        torch = self.torch
        rows = self.row1 - self.row0
        out = torch.empty((nrhs, rows), dtype=torch.float64, device=hats.device)  # column-major
        h = hats.contiguous()
        check(lib().sbx_hbs_solve_shard_down(self.h.ptr, self.G, self.p, VP(h.data_ptr()), nrhs,
                                             VP(out.data_ptr()), rows, _sbx.SBX_DEVICE_PTRS, self._stream()))
        return out.t()


class ShardedHbsSolver:
    """x = A_oo^{-1} b with the HBS tree split across the ranks of `group`."""

    def __init__(self, executor, group=None):
        import torch.distributed as dist
        self.dist = dist
        self.group = group
        self.ex = executor
        self.G = dist.get_world_size(group)
        self.p = dist.get_rank(group)
        if self.G & (self.G - 1):
            raise ValueError("sharded solve needs a power-of-two rank count")

    @property
    def rows(self):
        return self.ex.row0, self.ex.row1

    def solve(self, b_local):
        """b_local: this rank's rows [row0, row1) of b (rows x nrhs)."""
        import torch
        nrhs = b_local.shape[1]
        hat = self.ex.up(b_local)
        kmax = self.ex.kmax
        flat = torch.empty((self.G * kmax, nrhs), dtype=hat.dtype, device=hat.device)
        if kmax > 0:
            self.dist.all_gather_into_tensor(flat, hat.contiguous(), group=self.group)
        return self.ex.down(flat.view(self.G, kmax, nrhs), nrhs)


def solve_columns(h, b, group=None):
    """Batched RHS split by column across ranks (no exchange): rank p solves
    its contiguous block of columns of b with the full local operator."""
    import torch.distributed as dist
    from .api import hbs_solve
    G, p = dist.get_world_size(group), dist.get_rank(group)
    n = b.shape[1]
    c0, c1 = n * p // G, n * (p + 1) // G
    return (c0, c1), hbs_solve(h, b[:, c0:c1])
