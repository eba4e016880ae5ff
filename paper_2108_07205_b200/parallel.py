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

The device path is native: `Comm` (an NCCL communicator set owned by the
C-ABI, sbx_comm_*), `NativeShardedSolver` (sbx_hbs_solve_sharded) and
`NativeShardedWoodbury` (sbx_els_shard_*) run the sweeps, the GEMMs, W^{-1}
and the NCCL collectives inside libsbx on the caller's stream -- no torch
arithmetic.  `Comm.loopback(G)` gives G in-process members (one host thread
each) so the same C++ protocol runs on one GPU.

`ShardedHbsSolver` / `ShardedWoodbury` below restate the same exchange
protocol over torch.distributed with a pluggable per-rank executor; the CPU
tests drive them over gloo with host executors on the oracle's factors
(tests/test_parallel_gloo.py), which checks the protocol itself on world
sizes 2 and 4 where no multi-GPU box is available.
"""
from __future__ import annotations

import ctypes as C

from . import _sbx
from ._sbx import check, lib

VP = C.c_void_p


def _stream():
    from .api import torch_stream_handle
    try:
        return VP(torch_stream_handle())
    except Exception:  # no torch CUDA context: the library stream
        return VP()


class Comm:
    """A communicator set of the C-ABI (sbx_comm): NCCL for one process per
    GPU, or a loopback member for in-process emulation."""

    def __init__(self, ptr):
        self.ptr = ptr if isinstance(ptr, VP) else VP(ptr)

    @staticmethod
    def unique_id() -> bytes:
        buf = (C.c_uint8 * 128)()
        check(lib().sbx_comm_unique_id(buf))
        return bytes(buf)

    @classmethod
    def create(cls, unique_id: bytes, world: int, rank: int) -> "Comm":
        buf = (C.c_uint8 * 128).from_buffer_copy(unique_id)
        out = VP()
        check(lib().sbx_comm_create(buf, world, rank, C.byref(out)))
        return cls(out)

    @classmethod
    def from_process_group(cls, group=None) -> "Comm":
        """NCCL communicator over the ranks of a torch.distributed group: rank 0
        makes the unique id, the group broadcasts it (the only use of torch)."""
        import torch.distributed as dist
        world, rank = dist.get_world_size(group), dist.get_rank(group)
        obj = [cls.unique_id() if rank == 0 else None]
        dist.broadcast_object_list(obj, src=dist.get_global_rank(group, 0) if group else 0, group=group)
        return cls.create(obj[0], world, rank)

    @classmethod
    def loopback(cls, world: int):
        arr = (VP * world)()
        check(lib().sbx_comm_create_loopback(world, arr))
        return [cls(VP(arr[i])) for i in range(world)]

    def info(self):
        w, r = C.c_int(), C.c_int()
        check(lib().sbx_comm_info(self.ptr, C.byref(w), C.byref(r)))
        return w.value, r.value

    def __del__(self):
        try:
            if self.ptr and self.ptr.value and _sbx._lib is not None:
                _sbx._lib.sbx_comm_destroy(self.ptr)
                self.ptr = VP()
        except Exception:
            pass


def compress_sharded(d, comm: Comm, formulation=0, opts=None, mu: float = 1.0):
    """hbs_compress over the subtree partition of `comm` (sbx_hbs_compress_sharded):
    this rank's subtree and the top levels only; invert with api.hbs_invert,
    solve with NativeShardedSolver on the same communicator (which must
    outlive the operator)."""
    from .api import HbsOperator, HbsOptions
    o = (opts or HbsOptions()).to_c()
    out = VP()
    check(lib().sbx_hbs_compress_sharded(d.ptr, formulation, mu, C.byref(o), comm.ptr, C.byref(out)))
    h = HbsOperator(out)
    h._comm = comm  # keep the communicator alive as long as the operator
    return h


def _cm_call(x, rows):
    """Column-major device (or host) view of a rows x m block: (keepalive, ptr, ld, m, device?)."""
    if hasattr(x, "is_cuda") and x.is_cuda:
        import torch
        x2 = x.reshape(-1, 1) if x.dim() == 1 else x
        if x2.shape[0] != rows or x2.dtype != torch.float64:
            raise ValueError("sharded call: expected float64 with the owned row count")
        cm = x2.t().contiguous()
        return cm, VP(cm.data_ptr()), rows, x2.shape[1], True
    import numpy as np
    a = np.asfortranarray(np.asarray(x, dtype=np.float64).reshape(rows, -1))
    return a, VP(a.ctypes.data), rows, a.shape[1], False


def _cm_out(like, rows, m, dev):
    if dev:
        import torch
        return torch.empty((m, rows), dtype=torch.float64, device=like.device)
    import numpy as np
    return np.zeros((rows, m), order="F")


def _cm_result(out, dev):
    return out.t() if dev else out


class NativeShardedSolver:
    """x_local = A_oo^{-1} b on this rank's subtree rows (sbx_hbs_solve_sharded):
    local up-sweep, NCCL all-gather of the subtree-root hats, top levels,
    local down-sweep -- all inside libsbx on the caller's stream."""

    def __init__(self, h, comm: Comm):
        self.h, self.comm = h, comm
        self.G, self.p = comm.info()
        r0, r1, km = C.c_int64(), C.c_int64(), C.c_int64()
        check(lib().sbx_hbs_shard_info(h.ptr, self.G, self.p, C.byref(r0), C.byref(r1), C.byref(km)))
        self.row0, self.row1, self.kmax = r0.value, r1.value, km.value

    @property
    def rows(self):
        return self.row0, self.row1

    def solve(self, b_local):
        n = self.row1 - self.row0
        keep, ptr, ld, m, dev = _cm_call(b_local, n)
        out = _cm_out(keep, n, m, dev)
        optr = VP(out.data_ptr()) if dev else VP(out.ctypes.data)
        check(lib().sbx_hbs_solve_sharded(self.h.ptr, self.comm.ptr, ptr, ld, m, optr, n,
                                          _sbx.SBX_DEVICE_PTRS if dev else 0, _stream() if dev else VP()))
        return _cm_result(out, dev)


class NativeShardedWoodbury:
    """ELS / Woodbury on the subtree ownership inside libsbx (sbx_els_shard_*):
    X rows and R columns by subtree, A_pp on rank 0, all-reduce of R X and
    R y over NCCL, W^{-1} on every rank."""

    def __init__(self, a_oo, comm: Comm, d_old, d_new, plan, update, formulation=0, mu=1.0, stream=None):
        import numpy as np
        self.comm, self._keep = comm, (a_oo, d_old, d_new, plan, update)
        out = VP()
        check(lib().sbx_els_shard_build(a_oo.ptr, comm.ptr, d_old.ptr, d_new.ptr, plan.ptr, update.ptr,
                                        formulation, mu, VP(stream) if stream else VP(), C.byref(out)))
        self.ptr = out
        info = np.zeros(7, dtype=np.int64)
        check(lib().sbx_els_shard_info(self.ptr, info.ctypes.data_as(_sbx.I64P)))
        self.row0, self.row1, self.n_p_local, self.k, self.n_ext, self.G, self.p = (int(v) for v in info)
        self.ext_rows = np.zeros(self.row1 - self.row0, dtype=np.int64)
        check(lib().sbx_els_shard_rows(self.ptr, self.ext_rows.ctypes.data_as(_sbx.I64P)))

    def local_rows(self, g_ext):
        """This rank's owned rows (old-mesh order) of an ext-ordered block."""
        return g_ext[self.ext_rows] if not hasattr(g_ext, "is_cuda") else g_ext[
            __import__("torch").as_tensor(self.ext_rows, device=g_ext.device)]

    def solve(self, g_local, g_p=None):
        """(y_local, y_p): owned rows of ELS^{-1} g, and the added rows on rank 0."""
        n = self.row1 - self.row0
        keep, ptr, ld, m, dev = _cm_call(g_local, n)
        out = _cm_out(keep, n, m, dev)
        optr = VP(out.data_ptr()) if dev else VP(out.ctypes.data)
        pk = pptr = pout = poptr = None
        ldp = 1
        if self.n_p_local:
            pk, pptr, ldp, _, _ = _cm_call(g_p, self.n_p_local)
            pout = _cm_out(keep, self.n_p_local, m, dev)
            poptr = VP(pout.data_ptr()) if dev else VP(pout.ctypes.data)
        check(lib().sbx_els_shard_solve(self.ptr, ptr, ld, pptr or VP(), ldp, m, optr, n, poptr or VP(), ldp,
                                        _sbx.SBX_DEVICE_PTRS if dev else 0, _stream() if dev else VP()))
        return _cm_result(out, dev), (_cm_result(pout, dev) if pout is not None else None)

    def __del__(self):
        try:
            if self.ptr and self.ptr.value and _sbx._lib is not None:
                _sbx._lib.sbx_els_shard_destroy(self.ptr)
                self.ptr = VP()
        except Exception:
            pass


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


def column_range(ncols: int, world: int, rank: int):
    """Rank `rank`'s contiguous block of `ncols` right-hand sides."""
    return ncols * rank // world, ncols * (rank + 1) // world


def solve_columns(h, b, group=None, solve=None):
    """Batched RHS split by column across ranks (no
    exchange): rank p solves its contiguous block of columns of b with the
    full local operator (`solve(h, block)`, default api.hbs_solve).  Returns
    ((c0, c1), x block)."""
    import torch.distributed as dist
    from .api import hbs_solve
    G, p = dist.get_world_size(group), dist.get_rank(group)
    c0, c1 = column_range(b.shape[1], G, p)
    return (c0, c1), (solve or hbs_solve)(h, b[:, c0:c1])


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

