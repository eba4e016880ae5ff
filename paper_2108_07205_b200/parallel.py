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

The Woodbury part of the extended system (`ShardedWoodbury`, els.cpp:80-179)
shards the same way: the rows of X = Atilde^{-1} L and the columns of R
follow the old-mesh row ownership, the added-unknown block (A_pp, and the
rows of X and y it produces) lives on rank 0, and the two u-row products
R X (u x u) and R y (u x nrhs) are the only exchanges (all-reduce sums);
W^{-1} is formed redundantly on every rank.

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


class ShardedWoodbury:
    """Woodbury build and solve of the extended system split across ranks
    (reference els_build / els_solve_raw, els.cpp:80-179).

    hbs:        ShardedHbsSolver of A_oo (rank p owns old-mesh rows [row0, row1))
    L, R:       the update factors (n_ext x u, u x n_ext; replicated torch tensors)
    old_of_ext: old-mesh scalar row of each ext row < n_k + n_c (kept, cut)
    app_solve:  rank 0 only: v -> A_pp^{-1} v on n_p x m blocks

    Build: X_old = A_oo^{-1} L_old by the sharded solve (u columns), rank 0
    adds X_p = A_pp^{-1} L_p; W = I + sum_p R_p X_p (all-reduce), W^{-1} on
    every rank; rcond(W) >= sqrt(eps) is checked with the exact 1-norm
    condition (the reference's Hager estimate bounds it from above).
    Solve: y = Atilde^{-1} g on the owned rows, t = sum_p R_p y_p
    (all-reduce), y -= X W^{-1} t.  Inputs and outputs are each rank's own
    rows in old-mesh order (`local_rows`), plus the added block on rank 0.
    """

    def __init__(self, hbs, L, R, old_of_ext, n_k, n_c, n_p, app_solve=None, group=None):
        import numpy as np
        import torch
        import torch.distributed as dist
        self.dist, self.group, self.hbs = dist, group, hbs
        self.rank = dist.get_rank(group)
        self.n_k, self.n_c, self.n_p = n_k, n_c, n_p
        nkc = n_k + n_c
        r0, r1 = hbs.rows
        old = np.asarray(old_of_ext, dtype=np.int64)
        own = np.nonzero((old >= r0) & (old < r1))[0]
        if len(own) != r1 - r0:
            raise ValueError("sharded woodbury: ext rows do not cover the owned old-mesh rows")
        dev = L.device
        self.own = torch.as_tensor(own, device=dev)
        self.pos = torch.as_tensor(old[own] - r0, device=dev)
        u = L.shape[1]
        self.u = u
        Lloc = torch.zeros((r1 - r0, u), dtype=L.dtype, device=dev)
        Lloc[self.pos] = L[self.own]
        self.X = hbs.solve(Lloc) if u else Lloc  # owned rows of X, old-mesh order
        self.R_loc = torch.zeros((u, r1 - r0), dtype=R.dtype, device=dev)
        self.R_loc[:, self.pos] = R[:, self.own]
        Wp = self.R_loc @ self.X
        self.app_solve = app_solve if self.rank == 0 else None
        self.X_p = self.R_p = None
        if self.rank == 0 and n_p:
            if app_solve is None:
                raise ValueError("sharded woodbury: rank 0 needs the A_pp solver")
            self.R_p = R[:, nkc:nkc + n_p]
            self.X_p = app_solve(L[nkc:nkc + n_p])
            Wp = Wp + self.R_p @ self.X_p
        if u:
            dist.all_reduce(Wp, group=group)
        W = torch.eye(u, dtype=Wp.dtype, device=dev) + Wp
        self.W = W
        self.Winv = torch.linalg.inv(W) if u else W
        if u:
            rc = 1.0 / (torch.linalg.matrix_norm(W, 1) * torch.linalg.matrix_norm(self.Winv, 1)).item()
            if not rc >= float(np.sqrt(np.finfo(np.float64).eps)):
                raise ValueError("woodbury operator numerically singular; consider the optimal-basis "
                                 "compression mode at woodbury solve")

    def local_rows(self, g_ext):
        """This rank's owned rows (old-mesh order) of an ext-ordered block."""
        out = g_ext.new_zeros((len(self.pos), g_ext.shape[1]))
        out[self.pos] = g_ext[self.own]
        return out

    def solve(self, g_local, g_p=None):
        """g_local: owned rows of g_ext (old-mesh order, rows x m); g_p: the
        added rows (rank 0).  Returns (y_local, y_p or None)."""
        y = self.hbs.solve(g_local)
        t = self.R_loc @ y
        y_p = None
        if self.rank == 0 and self.n_p:
            y_p = self.app_solve(g_p)
            t = t + self.R_p @ y_p
        if self.u:
            self.dist.all_reduce(t, group=self.group)
            z = self.Winv @ t
            y = y - self.X @ z
            if y_p is not None:
                y_p = y_p - self.X_p @ z
        return y, y_p

