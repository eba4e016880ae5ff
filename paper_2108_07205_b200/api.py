"""Host-side mirror of the reference solver API (proj/include/stokesbie/*.hpp)
over the sbx C-ABI.  Names, argument meaning and error behaviour follow the
reference so that code written against it ports line by line:

  reference (C++)                          here
  ---------------------------------------  ------------------------------------
  panelize(ParametricCurve(cp), n, q)      panelize(CurveParams(...), n, q)
  refine(d, panel_ids, m)                  refine(d, panel_ids, m) -> (d1, plan)
  coarsen(d, plan)                         coarsen(d, plan)
  add_holes(d, holes)                      add_holes(d, holes) -> (d1, plan)
  hbs_compress(make_hbs_source(a), opts)   hbs_compress(d, formulation, opts)
  hbs_invert(op)                           hbs_invert(op)
  hbs_solve / hbs_apply                    hbs_solve / hbs_apply
  hbs_save / hbs_load                      hbs_save / hbs_load (HBS1, bit compatible)
  compress_update(blocks, proxy, eps, ..)  compress_update(d0, d1, plan, eps, ...)
  els_build(a_oo, blocks, plan, update)    els_build(a_oo, d0, d1, plan, update)
  els_solve / els_solve_raw                els_solve / els_solve_raw
  density_on_refined                       density_on_refined
  boundary_data(d, sources, mu)            boundary_data(d, sources, mu)

Exceptions: ValueError (std::invalid_argument), GeometryError,
SingularMatrixError (message carries `where`), ProxyViolationError.
Arrays are numpy float64 (host) or torch CUDA float64 tensors (device, no
host round trip).
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, field
from typing import Sequence

import numpy as np

from . import _sbx
from ._sbx import F64P, I64P, VP, check, lib

CIRCLE, ELLIPSE, STAR, FOURIER, CHANNEL = 0, 1, 2, 3, 4
INTERIOR_DIRICHLET, EXTERIOR_COMBINED, MIXED = 0, 1, 2

_initialized = False


def init(device: int = 0):
    global _initialized
    check(lib().sbx_init(device))
    _initialized = True


def _ensure():
    if not _initialized:
        init(0)


@dataclass
class CurveParams:
    """geometry.hpp:14-26."""
    kind: int = CIRCLE
    center: tuple = (0.0, 0.0)
    scale: float = 1.0
    flip_normal: bool = False
    n_prongs: int = 0
    amplitude: float = 0.0
    aspect: float = 1.0
    cos_coef: Sequence[float] = field(default_factory=list)
    sin_coef: Sequence[float] = field(default_factory=list)

    def to_c(self) -> _sbx.sbx_curve:
        c = _sbx.sbx_curve()
        c.kind = self.kind
        c.center_x, c.center_y = float(self.center[0]), float(self.center[1])
        c.scale = self.scale
        c.flip_normal = int(self.flip_normal)
        c.n_prongs = self.n_prongs
        c.amplitude = self.amplitude
        c.aspect = self.aspect
        c.n_cos, c.n_sin = len(self.cos_coef), len(self.sin_coef)
        for i, v in enumerate(self.cos_coef):
            c.cos_coef[i] = v
        for i, v in enumerate(self.sin_coef):
            c.sin_coef[i] = v
        return c


def ellipse(a: float, b: float, center=(0.0, 0.0)) -> CurveParams:
    return CurveParams(kind=ELLIPSE, center=center, scale=a, aspect=b / a)


def star(n_prongs: int, amplitude: float, scale=1.0, center=(0.0, 0.0)) -> CurveParams:
    return CurveParams(kind=STAR, center=center, scale=scale, n_prongs=n_prongs, amplitude=amplitude)


def channel(length: float = 8.0, half_width: float = 1.0, amplitude: float = 0.2, periods: int = 2,
            cap_speed: float = 3.0, fractions=(45 / 128, 21 / 128), center=(0.0, 0.0)) -> CurveParams:
    """The closed wavy channel of BASELINE configs[3] (sbx.h SBX_CHANNEL):
    walls y = -/+ h (1 + a sin(2 pi periods x / length)), x in [0, length],
    closed by degree-9 polynomial caps that continue the walls with matching
    derivatives up to the fourth (position, tangent, curvature and its first
    two derivatives are continuous).  cap_speed scales the caps' parameter
    speed against the walls' (their bulge); fractions (bottom / top wall,
    right cap) of the parameter circle are multiples of 1/128, so any panel
    count divisible by 128 puts the four joins on panel ends."""
    from math import factorial
    lam_len = length / half_width
    k = 2 * np.pi * periods / lam_len

    def wall(top, x, d):  # d-th x-derivative of (X, Y) on the scaled top / bottom wall
        X = x if d == 0 else (1.0 if d == 1 else 0.0)
        ph = (np.sin, np.cos, lambda z: -np.sin(z), lambda z: -np.cos(z))[d % 4]
        Y = (1.0 + amplitude * np.sin(k * x)) if d == 0 else amplitude * k ** d * ph(k * x)
        return np.array([X, Y if top else -Y])

    def cap(P0, P1):  # degree-9 polynomial with 5 derivative conditions at u = 0 and u = 1
        A, b = [], []
        for u, P in ((0.0, P0), (1.0, P1)):
            for d in range(5):
                A.append([factorial(j) / factorial(j - d) * u ** (j - d) if j >= d else 0.0 for j in range(10)])
                b.append(P[d])
        return np.linalg.solve(np.array(A), np.array(b))  # (10, 2)

    lam = cap_speed
    right = cap([wall(False, lam_len, d) * lam ** d for d in range(5)],
                [wall(True, lam_len, d) * (-lam) ** d for d in range(5)])
    left = cap([wall(True, 0.0, d) * (-lam) ** d for d in range(5)],
               [wall(False, 0.0, d) * lam ** d for d in range(5)])
    coef = np.concatenate([right[:, 0], right[:, 1], left[:, 0], left[:, 1]])
    return CurveParams(kind=CHANNEL, center=center, scale=half_width, n_prongs=int(periods),
                       amplitude=amplitude, aspect=lam_len, cos_coef=[float(c) for c in coef],
                       sin_coef=[float(fractions[0]), float(fractions[1])])


def circle(radius=1.0, center=(0.0, 0.0)) -> CurveParams:
    return CurveParams(kind=CIRCLE, center=center, scale=radius)


class _Handle:
    _destroy = None

    def __init__(self, ptr):
        self._ptr = VP(ptr) if not isinstance(ptr, VP) else ptr

    @property
    def ptr(self):
        return self._ptr

    def __del__(self):
        try:
            if self._ptr and self._ptr.value and self._destroy and _sbx._lib is not None:
                getattr(_sbx._lib, self._destroy)(self._ptr)
                self._ptr = VP()
        except Exception:  # interpreter shutdown
            pass


class Discretization(_Handle):
    """geometry.hpp:60-101 (SoA node arrays, interleaved unknowns)."""
    _destroy = "sbx_geom_destroy"

    def info(self):
        a, b, c = C.c_int64(), C.c_int64(), C.c_int64()
        check(lib().sbx_geom_info(self.ptr, C.byref(a), C.byref(b), C.byref(c)))
        return a.value, b.value, c.value

    def n_nodes(self):
        return self.info()[0]

    def n_unknowns(self):
        return 2 * self.n_nodes()

    def n_panels(self):
        return self.info()[1]

    def nodes(self) -> dict:
        n = self.n_nodes()
        out = np.zeros(9 * n)
        pan = np.zeros(n, dtype=np.int64)
        check(lib().sbx_geom_nodes(self.ptr, out.ctypes.data_as(F64P), pan.ctypes.data_as(I64P)))
        o = out.reshape(9, n)
        keys = ("x", "y", "nx", "ny", "tx", "ty", "w", "curvature", "param")
        d = {k: o[i].copy() for i, k in enumerate(keys)}
        d["panel_of"] = pan
        return d

    def panels_near_point(self, point, radius) -> np.ndarray:
        cap = self.n_panels()
        out = np.zeros(cap, dtype=np.int64)
        cnt = C.c_int64()
        check(lib().sbx_panels_near_point(self.ptr, float(point[0]), float(point[1]), float(radius),
                                          out.ctypes.data_as(I64P), cap, C.byref(cnt)))
        return out[: cnt.value]


class RefinementPlan(_Handle):
    """geometry.hpp:105-116."""
    _destroy = "sbx_plan_destroy"

    def sizes(self):
        a, b, c = C.c_int64(), C.c_int64(), C.c_int64()
        check(lib().sbx_plan_sizes(self.ptr, C.byref(a), C.byref(b), C.byref(c)))
        return a.value, b.value, c.value

    def n_k(self):
        return self.sizes()[0]

    def n_c(self):
        return self.sizes()[1]

    def n_p(self):
        return self.sizes()[2]

    def maps(self) -> dict:
        nk, nc, npp = self.sizes()
        ko, kn = np.zeros(nk, np.int64), np.zeros(nk, np.int64)
        co, an = np.zeros(nc, np.int64), np.zeros(npp, np.int64)
        check(lib().sbx_plan_maps(self.ptr, ko.ctypes.data_as(I64P), kn.ctypes.data_as(I64P),
                                  co.ctypes.data_as(I64P), an.ctypes.data_as(I64P)))
        return {"kept_old": ko, "kept_new": kn, "cut_old": co, "added_new": an}


def panelize(curve: CurveParams, n_panels: int, q: int = 16) -> Discretization:
    _ensure()
    out = VP()
    c = curve.to_c()
    check(lib().sbx_geom_create(C.byref(c), n_panels, q, C.byref(out)))
    return Discretization(out)


def refine(d: Discretization, panel_ids, m: int):
    ids = np.ascontiguousarray(np.asarray(panel_ids, dtype=np.int64))
    g, p = VP(), VP()
    check(lib().sbx_refine(d.ptr, ids.ctypes.data_as(I64P), len(ids), m, C.byref(g), C.byref(p)))
    return Discretization(g), RefinementPlan(p)


def coarsen(d: Discretization, plan: RefinementPlan) -> Discretization:
    g = VP()
    check(lib().sbx_coarsen(d.ptr, plan.ptr, C.byref(g)))
    return Discretization(g)


def add_holes(d: Discretization, holes):
    """holes: iterable of (CurveParams, n_panels, q)."""
    holes = list(holes)
    arr = (_sbx.sbx_curve * len(holes))(*[h[0].to_c() for h in holes])
    npn = (C.c_int32 * len(holes))(*[h[1] for h in holes])
    qs = (C.c_int32 * len(holes))(*[h[2] for h in holes])
    g, p = VP(), VP()
    check(lib().sbx_geom_add_holes(d.ptr, len(holes), arr, npn, qs, C.byref(g), C.byref(p)))
    return Discretization(g), RefinementPlan(p)


def evaluate_solution(d: Discretization, formulation, tau, targets, mu: float = 1.0, with_pressure=False):
    """nystrom.cpp:408-448 on the device.  tau: 2N (or 2N x nrhs) density;
    returns velocity (T x 2 [x nrhs]), pressure (T [x nrhs]) or None, and the
    near-boundary flags (T)."""
    t = np.asfortranarray(np.asarray(tau, dtype=np.float64))
    vec = t.ndim == 1
    t2 = t.reshape(-1, 1, order="F") if vec else t
    tg = np.ascontiguousarray(np.asarray(targets, dtype=np.float64).reshape(-1, 2))
    nt, nr = len(tg), t2.shape[1]
    vel = np.zeros((nr, nt, 2))
    pre = np.zeros((nr, nt)) if with_pressure else None
    near = np.zeros(nt, dtype=np.uint8)
    check(lib().sbx_evaluate_solution(d.ptr, formulation, mu, t2.ctypes.data_as(F64P), t2.shape[0], nr,
                                      tg.ctypes.data_as(F64P), nt, int(with_pressure),
                                      vel.ctypes.data_as(F64P),
                                      pre.ctypes.data_as(F64P) if with_pressure else None,
                                      near.ctypes.data_as(C.POINTER(C.c_uint8))))
    v = vel[0] if vec else np.moveaxis(vel, 0, -1)
    p = (pre[0] if vec else pre.T) if with_pressure else None
    return v, p, near.astype(bool)


def boundary_data(d: Discretization, sources, mu: float = 1.0) -> np.ndarray:
    """nystrom.cpp:383-392; sources rows (x, y, fx, fy)."""
    s = np.ascontiguousarray(np.asarray(sources, dtype=np.float64).reshape(-1, 4))
    out = np.zeros(d.n_unknowns())
    check(lib().sbx_boundary_data(d.ptr, len(s), s.ctypes.data_as(F64P), mu, out.ctypes.data_as(F64P)))
    return out


def submatrix(d: Discretization, rows, cols, formulation=INTERIOR_DIRICHLET, mu=1.0) -> np.ndarray:
    """BieAssembler::submatrix (nystrom.cpp:200-217), evaluated on the device."""
    r = np.ascontiguousarray(np.asarray(rows, dtype=np.int64))
    c = np.ascontiguousarray(np.asarray(cols, dtype=np.int64))
    out = np.zeros((len(r), len(c)), order="F")
    check(lib().sbx_submatrix(d.ptr, formulation, mu, r.ctypes.data_as(I64P), len(r),
                              c.ctypes.data_as(I64P), len(c), out.ctypes.data_as(F64P)))
    return out


@dataclass
class HbsOptions:
    """hbs.hpp:39-46."""
    eps: float = 1e-10
    leaf_nodes: int = 64
    n_proxy: int = 64
    bas_factor: float = 1.5
    div_factor: float = 3.0

    def to_c(self):
        o = _sbx.sbx_hbs_options()
        o.eps, o.leaf_nodes, o.n_proxy = self.eps, self.leaf_nodes, self.n_proxy
        o.bas_factor, o.div_factor = self.bas_factor, self.div_factor
        return o


class HbsOperator(_Handle):
    """hbs.hpp:64-74; factors live in a device arena."""
    _destroy = "sbx_hbs_destroy"

    def info(self) -> dict:
        out = np.zeros(14, dtype=np.int64)
        check(lib().sbx_hbs_info(self.ptr, out.ctypes.data_as(I64P)))
        keys = ("n", "nodes", "total_skeleton", "max_block_drawn", "has_inverse",
                "factor_doubles", "max_depth", "max_k", "apply_factor_doubles", "leaf_nodes",
                "top_L", "top_K", "arena_doubles", "sharded")
        return dict(zip(keys, (int(v) for v in out)))

    @property
    def n(self):
        return self.info()["n"]

    def node_ranks(self) -> np.ndarray:
        n = self.info()["nodes"]
        out = np.zeros(n, dtype=np.int64)
        check(lib().sbx_hbs_node_ranks(self.ptr, out.ctypes.data_as(I64P), n))
        return out


ENTRIES_FN = C.CFUNCTYPE(None, C.c_void_p, I64P, C.c_int64, I64P, C.c_int64, F64P)


def hbs_compress(d: Discretization, formulation=INTERIOR_DIRICHLET, opts: HbsOptions | None = None,
                 mu: float = 1.0, subset=None, entries=None, with_completion: bool = True) -> HbsOperator:
    """hbs_compress(make_hbs_source(a), opts) (hbs.cpp:349-425).  entries:
    the HbsSource::entries plugin (hbs.hpp:19-31) -- a callable
    (rows, cols) -> (len(rows) x len(cols)) array over scalar indices that
    replaces the kernel entries of every block the compression draws;
    with_completion=False drops the completion functionals (row_null /
    col_null empty)."""
    o = (opts or HbsOptions()).to_c()
    out = VP()
    if entries is not None:
        if subset is not None:
            raise ValueError("hbs_compress: a custom entry oracle covers the whole discretization")
        errs = []

        def cb(_ctx, rows, nr, cols, nc, outp):
            try:
                r = np.ctypeslib.as_array(rows, shape=(nr,)).copy()
                c = np.ctypeslib.as_array(cols, shape=(nc,)).copy()
                blk = np.asarray(entries(r, c), dtype=np.float64).reshape(nr, nc)
                np.ctypeslib.as_array(outp, shape=(nc, nr))[:] = blk.T  # column-major out
            except BaseException as e:  # noqa: BLE001  (re-raised after the C call)
                errs.append(e)

        fn = ENTRIES_FN(cb)
        code = lib().sbx_hbs_compress_custom(d.ptr, formulation, mu, C.cast(fn, VP), None, int(bool(with_completion)),
                                             C.byref(o), C.byref(out))
        if errs:
            raise errs[0]
        check(code)
        return HbsOperator(out)
    if subset is None:
        check(lib().sbx_hbs_compress(d.ptr, formulation, mu, C.byref(o), C.byref(out)))
    else:
        s = np.ascontiguousarray(np.asarray(subset, dtype=np.int64))
        check(lib().sbx_hbs_compress_subset(d.ptr, formulation, mu, s.ctypes.data_as(I64P), len(s),
                                            C.byref(o), C.byref(out)))
    return HbsOperator(out)


def hbs_invert(op: HbsOperator) -> HbsOperator:
    check(lib().sbx_hbs_invert(op.ptr))
    return op


def _is_torch_cuda(x):
    return type(x).__module__.startswith("torch") and getattr(x, "is_cuda", False)


CUDA_STREAM_LEGACY = 1  # cudaStreamLegacy: a null handle means "library stream" in sbx.h


def torch_stream_handle():
    """The caller's current torch stream as an sbx.h stream argument (the
    legacy default stream is passed as cudaStreamLegacy, not as null)."""
    import torch
    s = torch.cuda.current_stream().cuda_stream
    return s if s else CUDA_STREAM_LEGACY


def _sweep(fn, op_ptr, b, n, stream=None, flags=0, row_major_ok=False):
    """Column-major n x nrhs sweep through the C-ABI (host numpy or CUDA torch)."""
    if _is_torch_cuda(b):
        import torch
        vec = b.dim() == 1
        bt = b.reshape(-1, 1) if vec else b
        if bt.dtype != torch.float64 or bt.shape[0] != n:
            raise ValueError("sweep: expected float64 with n rows")
        s = stream if stream is not None else torch_stream_handle()
        if row_major_ok and bt.stride(1) == 1 and bt.stride(0) >= bt.shape[1]:
            # row-major rows (a C-contiguous tensor) are the sweep workspace's
            # own layout: strided copies in and out, no transposes (SBX_ROW_MAJOR)
            out = torch.empty((n, bt.shape[1]), dtype=torch.float64, device=bt.device)
            check(fn(op_ptr, VP(bt.data_ptr()), bt.stride(0), bt.shape[1], VP(out.data_ptr()), bt.shape[1],
                     _sbx.SBX_DEVICE_PTRS | _sbx.SBX_ROW_MAJOR | flags, VP(s)))
            return out.reshape(-1) if vec else out
        bcm = bt.t().contiguous()  # column-major storage = transposed row-major
        out = torch.empty_like(bcm)
        check(fn(op_ptr, VP(bcm.data_ptr()), n, bt.shape[1], VP(out.data_ptr()), n,
                 _sbx.SBX_DEVICE_PTRS | flags, VP(s)))
        res = out.t()
        return res.reshape(-1) if vec else res
    arr = np.asarray(b, dtype=np.float64)
    vec = arr.ndim == 1
    a2 = np.asfortranarray(arr.reshape(-1, 1) if vec else arr)
    if a2.shape[0] != n:
        raise ValueError("sweep: size mismatch")
    out = np.zeros_like(a2, order="F")
    check(fn(op_ptr, VP(a2.ctypes.data), n, a2.shape[1], VP(out.ctypes.data), n, flags, VP()))
    return out[:, 0] if vec else out


def hbs_solve(op: HbsOperator, b, transpose: bool = False):
    """hbs.cpp:589-625; transpose: hbs_solve_t (hbs.cpp:627-664)."""
    return _sweep(lib().sbx_hbs_solve, op.ptr, b, op.n, flags=_sbx.SBX_TRANSPOSE if transpose else 0,
                  row_major_ok=True)


def hbs_apply(op: HbsOperator, v, transpose: bool = False):
    """hbs.cpp:511-544; transpose: hbs_apply_t (hbs.cpp:546-587)."""
    return _sweep(lib().sbx_hbs_apply, op.ptr, v, op.n, flags=_sbx.SBX_TRANSPOSE if transpose else 0,
                  row_major_ok=True)


def hbs_save(op: HbsOperator, path):
    check(lib().sbx_hbs_save_hbs1(op.ptr, str(path).encode()))


def hbs_load(path) -> HbsOperator:
    _ensure()
    out = VP()
    check(lib().sbx_hbs_load_hbs1(str(path).encode(), C.byref(out)))
    return HbsOperator(out)


class LowRankUpdate(_Handle):
    """lowrank.hpp:28-47 (factors on the device)."""
    _destroy = "sbx_update_destroy"

    def info(self) -> dict:
        out = np.zeros(9, dtype=np.int64)
        check(lib().sbx_update_info(self.ptr, out.ctypes.data_as(I64P)))
        keys = ("k", "k1", "kc", "kp", "pk", "n_ext", "nk2", "nc2", "np2")
        return dict(zip(keys, (int(v) for v in out)))

    @property
    def k(self):
        return self.info()["k"]

    def factors(self):
        i = self.info()
        L = np.zeros((i["n_ext"], i["k"]), order="F")
        R = np.zeros((i["k"], i["n_ext"]), order="F")
        if i["k"]:
            check(lib().sbx_update_factor(self.ptr, 0, L.ctypes.data_as(F64P)))
            check(lib().sbx_update_factor(self.ptr, 1, R.ctypes.data_as(F64P)))
        return L, R


TWO_STEP_ID, SVD_OPTIMAL = 0, 1  # CompressionMode (lowrank.hpp:17)


def compress_update(d_old: Discretization, d_new: Discretization, plan: RefinementPlan,
                    eps: float = 1e-10, formulation=INTERIOR_DIRICHLET, mu: float = 1.0,
                    seed: int = 0, mode: int = TWO_STEP_ID) -> LowRankUpdate:
    """compress_update(BlockSource(old, new, plan), make_proxy_geometry(new, plan),
    eps, mode, {seed}) — lowrank.cpp:366-373 (TwoStepId, or the SvdOptimal
    diagnostic mode of lowrank.cpp:329-362)."""
    out = VP()
    if mode == TWO_STEP_ID:
        check(lib().sbx_update_compress(d_old.ptr, d_new.ptr, plan.ptr, formulation, mu, eps,
                                        C.c_uint64(seed), C.byref(out)))
    else:
        check(lib().sbx_update_compress_mode(d_old.ptr, d_new.ptr, plan.ptr, formulation, mu, eps,
                                             C.c_uint64(seed), int(mode), C.byref(out)))
    return LowRankUpdate(out)


def update_from_factors(plan: RefinementPlan, L, R) -> LowRankUpdate:
    L = np.asfortranarray(np.asarray(L, dtype=np.float64))
    R = np.asfortranarray(np.asarray(R, dtype=np.float64))
    out = VP()
    check(lib().sbx_update_from_factors(plan.ptr, L.ctypes.data_as(F64P), R.ctypes.data_as(F64P),
                                        L.shape[0], L.shape[1], C.byref(out)))
    return LowRankUpdate(out)


class UpdateCache(_Handle):
    """run_snapshot_batch's update cache (scenario.cpp:836-899): identical
    (panel ids, m) at the same eps / formulation / mu / seed share one
    compression."""
    _destroy = "sbx_update_cache_destroy"

    def __init__(self):
        _ensure()
        out = VP()
        check(lib().sbx_update_cache_create(C.byref(out)))
        super().__init__(out)

    def compress(self, d_old: Discretization, d_new: Discretization, plan: RefinementPlan, panel_ids, m: int,
                 eps: float = 1e-10, formulation=INTERIOR_DIRICHLET, mu: float = 1.0, seed: int = 0):
        """(update, hit) -- compress_update on a miss, the cached update on a hit."""
        ids = np.ascontiguousarray(np.asarray(panel_ids, dtype=np.int64))
        out, hit = VP(), C.c_int(0)
        check(lib().sbx_update_cache_compress(self.ptr, d_old.ptr, d_new.ptr, plan.ptr, ids.ctypes.data_as(I64P),
                                              len(ids), int(m), formulation, mu, eps, C.c_uint64(seed),
                                              C.byref(out), C.byref(hit)))
        return LowRankUpdate(out), bool(hit.value)

    def stats(self) -> dict:
        e, h, m = C.c_int64(), C.c_int64(), C.c_int64()
        check(lib().sbx_update_cache_stats(self.ptr, C.byref(e), C.byref(h), C.byref(m)))
        return {"entries": e.value, "hits": h.value, "misses": m.value}


def update_dump(u: LowRankUpdate, path_L, path_R):
    """L and R as dump_matrix files (nystrom.cpp:450-461)."""
    check(lib().sbx_update_dump(u.ptr, str(path_L).encode(), str(path_R).encode()))


def update_load(plan: RefinementPlan, path_L, path_R) -> LowRankUpdate:
    """An update from dumped L, R (tier-1 hand-over of external factors)."""
    out = VP()
    check(lib().sbx_update_load(plan.ptr, str(path_L).encode(), str(path_R).encode(), C.byref(out)))
    return LowRankUpdate(out)


def dump_matrix(path, m):
    """nystrom.cpp:450-461 (host; no device work)."""
    a = np.asfortranarray(np.atleast_2d(np.asarray(m, dtype=np.float64)))
    check(lib().sbx_dump_matrix(str(path).encode(), a.ctypes.data_as(F64P), a.shape[0], a.shape[1],
                                max(a.shape[0], 1)))


def load_matrix(path) -> np.ndarray:
    """nystrom.cpp:463-477 (host; no device work)."""
    r, c = C.c_int64(), C.c_int64()
    check(lib().sbx_load_matrix_dims(str(path).encode(), C.byref(r), C.byref(c)))
    out = np.zeros((r.value, c.value), order="F")
    check(lib().sbx_load_matrix(str(path).encode(), out.ctypes.data_as(F64P), max(r.value, 1)))
    return out


class ElsSolver(_Handle):
    """els.hpp:17-37.  Keeps a reference to the HBS handle it solves with."""
    _destroy = "sbx_els_destroy"

    def __init__(self, ptr, a_oo, meshes=()):
        super().__init__(ptr)
        self._a_oo = a_oo
        self._meshes = meshes  # the dense conditioning route reads them

    def info(self) -> dict:
        out = np.zeros(6, dtype=np.int64)
        check(lib().sbx_els_info(self.ptr, out.ctypes.data_as(I64P)))
        return dict(zip(("n_k", "n_c", "n_p", "k", "app_hbs", "app_solve_doubles"), (int(v) for v in out)))

    def n_ext(self):
        i = self.info()
        return i["n_k"] + i["n_c"] + i["n_p"]

    def xw(self):
        i = self.info()
        X = np.zeros((self.n_ext(), i["k"]), order="F")
        W = np.zeros((i["k"], i["k"]), order="F")
        if i["k"]:
            check(lib().sbx_els_xw(self.ptr, X.ctypes.data_as(F64P), W.ctypes.data_as(F64P)))
        return X, W


def els_build(a_oo: HbsOperator, d_old: Discretization, d_new: Discretization,
              plan: RefinementPlan, update: LowRankUpdate, formulation=INTERIOR_DIRICHLET,
              mu: float = 1.0) -> ElsSolver:
    out = VP()
    check(lib().sbx_els_build(a_oo.ptr, d_old.ptr, d_new.ptr, plan.ptr, update.ptr, formulation, mu,
                              C.byref(out)))
    return ElsSolver(out, a_oo, (d_old, d_new))


class AppBlockSolver(_Handle):
    """The added-unknown diagonal block's inverse alone (els.cpp:111-118:
    dense LU up to 2048 scalars, else its own HBS); keeps the refined mesh
    it was built on alive."""
    _destroy = "sbx_app_destroy"

    def __init__(self, ptr, d_new):
        super().__init__(ptr)
        self._d_new = d_new

    def info(self) -> dict:
        out = np.zeros(2, dtype=np.int64)
        check(lib().sbx_app_info(self.ptr, out.ctypes.data_as(I64P)))
        return {"n_p": int(out[0]), "hbs": int(out[1])}

    def solve(self, v, transpose: bool = False):
        return _sweep(lib().sbx_app_solve, self.ptr, v, self.info()["n_p"],
                      flags=_sbx.SBX_TRANSPOSE if transpose else 0)


def app_build(d_new: Discretization, plan: RefinementPlan, eps: float = 1e-10,
              formulation=INTERIOR_DIRICHLET, mu: float = 1.0) -> AppBlockSolver:
    out = VP()
    check(lib().sbx_app_build(d_new.ptr, plan.ptr, formulation, mu, eps, C.byref(out)))
    return AppBlockSolver(out, d_new)


def _els_call(fn, s: ElsSolver, g, rows_in, flags=0):
    if _is_torch_cuda(g):
        import torch
        vec = g.dim() == 1
        gt = g.reshape(-1, 1) if vec else g
        gcm = gt.t().contiguous()
        out = torch.empty_like(gcm)
        check(fn(s.ptr, VP(gcm.data_ptr()), rows_in, gt.shape[1], VP(out.data_ptr()), rows_in,
                 _sbx.SBX_DEVICE_PTRS | flags, VP(torch_stream_handle())))
        res = out.t()
        return res.reshape(-1) if vec else res
    a = np.asarray(g, dtype=np.float64)
    vec = a.ndim == 1
    a2 = np.asfortranarray(a.reshape(-1, 1) if vec else a)
    if a2.shape[0] != rows_in:
        raise ValueError("els_solve: data size mismatch")
    out = np.zeros_like(a2, order="F")
    check(fn(s.ptr, VP(a2.ctypes.data), rows_in, a2.shape[1], VP(out.ctypes.data), rows_in, flags, VP()))
    return out[:, 0] if vec else out


def els_solve(s: ElsSolver, g_n):
    """els.cpp:173-179 (kept, added) data -> (kept, added) density."""
    i = s.info()
    return _els_call(lib().sbx_els_solve, s, g_n, i["n_k"] + i["n_p"])


def els_solve_into(s: ElsSolver, g_n: np.ndarray, tau_n: np.ndarray, stream=None):
    """sbx_els_solve on caller-owned HOST buffers (the drop-in caller path):
    g_n, tau_n are column-major (n_k + n_p) x nrhs float64 arrays (pinned
    memory makes the library's copies asynchronous DMA); returns once tau_n
    holds the density."""
    i = s.info()
    rows = i["n_k"] + i["n_p"]
    for a in (g_n, tau_n):
        if a.dtype != np.float64 or a.ndim != 2 or a.shape[0] != rows or not a.flags.f_contiguous:
            raise ValueError("els_solve_into: expected column-major float64 (n_k + n_p) x nrhs arrays")
    if g_n.shape != tau_n.shape:
        raise ValueError("els_solve_into: shape mismatch")
    check(lib().sbx_els_solve(s.ptr, VP(g_n.ctypes.data), rows, g_n.shape[1], VP(tau_n.ctypes.data), rows, 0,
                              VP(stream) if stream else VP()))
    return tau_n


def els_solve_raw(s: ElsSolver, g_ext, transpose: bool = False):
    """els.cpp:147-152 on extended (kept, cut, added) vectors; transpose:
    els_solve_raw_t (els.cpp:154-163)."""
    return _els_call(lib().sbx_els_solve_raw, s, g_ext, s.n_ext(), _sbx.SBX_TRANSPOSE if transpose else 0)


def els_apply_forward(s: ElsSolver, v, transpose: bool = False) -> np.ndarray:
    """els.cpp:181-186: (Atilde + L R) v on the extended system (n_ext [x nrhs]);
    transpose: els_apply_forward_t (els.cpp:188-193)."""
    a = np.asfortranarray(np.asarray(v, dtype=np.float64))
    vec = a.ndim == 1
    a2 = a.reshape(-1, 1, order="F") if vec else a
    out = np.zeros_like(a2, order="F")
    fn = lib().sbx_els_apply_forward_t if transpose else lib().sbx_els_apply_forward
    check(fn(s.ptr, a2.ctypes.data_as(F64P), a2.shape[0], a2.shape[1], out.ctypes.data_as(F64P), a2.shape[0]))
    return out[:, 0] if vec else out


def els_conditioning(s: ElsSolver, iters: int = 80, dense: bool = False) -> dict:
    """conditioning_report(s, dense) (els.cpp:225-270): exact kappa_w,
    kappa_l, kappa_r (device Jacobi SVD); kappa_ext, kappa_tilde from the
    dense Atilde and Atilde + L R (dense=True) or by seeded power iteration on
    the device operators and solves (linop.cpp:17-43)."""
    out = np.zeros(7)
    check(lib().sbx_els_conditioning_report(s.ptr, int(bool(dense)), int(iters), out.ctypes.data_as(F64P)))
    keys = ("kappa_w", "kappa_l", "kappa_r", "kappa_ext", "kappa_tilde", "bound")
    r = {k: float(v) for k, v in zip(keys, out[:6])}
    r["bound_holds"] = bool(out[6] != 0.0)
    return r


def els_gmres(s: ElsSolver, g_n, precond: bool = True, tol: float = 1e-11, max_iter: int = 600,
              restart: int = 0):
    """GMRES (gmres.cpp:14-126) on the refined system in (kept, added)
    unknowns; precond=True is the paper's PGMRES-Local (left preconditioner
    els_solve, scenario.cpp:694-727).  Returns (tau_n, n_iter, history)."""
    g = np.ascontiguousarray(np.asarray(g_n, dtype=np.float64))
    tau = np.zeros_like(g)
    it = C.c_int64()
    hist = np.zeros(max_iter + 2)
    check(lib().sbx_els_gmres(s.ptr, g.ctypes.data_as(F64P), tau.ctypes.data_as(F64P), int(precond), tol,
                              max_iter, restart, C.byref(it), hist.ctypes.data_as(F64P), len(hist)))
    return tau, it.value, hist[: it.value + 1]


def density_on_refined(s: ElsSolver, tau_n) -> np.ndarray:
    """els.cpp:195-203."""
    t = np.ascontiguousarray(np.asarray(tau_n, dtype=np.float64))
    i = s.info()
    if t.shape[0] != i["n_k"] + i["n_p"]:
        raise ValueError("density_on_refined: size mismatch")
    n_new = (i["n_k"] + i["n_p"]) // 1
    out = np.zeros(_els_new_unknowns(s))
    check(lib().sbx_els_density_on_refined(s.ptr, t.ctypes.data_as(F64P), out.ctypes.data_as(F64P)))
    return out


def _els_new_unknowns(s: ElsSolver) -> int:
    i = s.info()
    return i["n_k"] + i["n_p"]


def row_id(w, eps=1e-10, forced=None, engine=0):
    """Device row ID (idlib.cpp:73-99): returns k, J, P with W ~= P W[J[:k]]."""
    _ensure()
    w = np.asfortranarray(np.asarray(w, dtype=np.float64))
    m, n = w.shape
    k = C.c_int64()
    J = np.zeros(m, dtype=np.int64)
    P = np.zeros(max(1, m * min(m, n)))
    check(lib().sbx_row_id(w.ctypes.data_as(F64P), m, n, eps, -1 if forced is None else forced,
                           engine, C.byref(k), J.ctypes.data_as(I64P), P.ctypes.data_as(F64P)))
    kk = k.value
    return kk, J, P[: m * kk].reshape((m, kk), order="F")


def dense_inverse(a):
    """Explicit inverse and reciprocal condition estimate of a dense matrix on
    the device (els.cpp:111-127: PartialPivLU + rcond()).  Returns inv, rcond."""
    _ensure()
    a = np.asfortranarray(np.asarray(a, dtype=np.float64))
    n = a.shape[0]
    assert a.shape == (n, n)
    inv = np.zeros((n, n), order="F")
    rc = C.c_double(0.0)
    check(lib().sbx_dense_inverse(a.ctypes.data_as(F64P), n, inv.ctypes.data_as(F64P), C.byref(rc)))
    return inv, rc.value


def matmul(a, b):
    """A @ B through the device GEMM dispatcher of the ELS (els.cpp:124, 150)."""
    _ensure()
    a = np.asfortranarray(np.asarray(a, dtype=np.float64))
    b = np.asfortranarray(np.asarray(b, dtype=np.float64))
    m, k = a.shape
    assert b.shape[0] == k
    n = b.shape[1]
    c = np.zeros((m, n), order="F")
    check(lib().sbx_matmul(a.ctypes.data_as(F64P), m, k, b.ctypes.data_as(F64P), n, c.ctypes.data_as(F64P)))
    return c


def kernel_launches(reset: bool = False) -> int:
    return int(lib().sbx_kernel_launches(int(reset)))


def kernel_timing(enable: bool = True):
    """CUDA-event timing of the named hot kernels (sbx_kernel_timing)."""
    check(lib().sbx_kernel_timing(int(enable)))


def kernel_time(name: str, reset: bool = True):
    """(total ms, launches) of a timed kernel since the last reset."""
    ms = C.c_double(0.0)
    cnt = C.c_int64(0)
    check(lib().sbx_kernel_time(name.encode(), int(reset), C.byref(ms), C.byref(cnt)))
    return ms.value, cnt.value


def kernel_flops(name: str, reset: bool = True) -> float:
    """Algorithmic flops attributed to a timed kernel family since the last reset."""
    f = C.c_double(0.0)
    check(lib().sbx_kernel_flops(name.encode(), int(reset), C.byref(f)))
    return f.value


def gather_kept_added(plan: RefinementPlan, g_new):
    """scenario.cpp:253-258."""
    m = plan.maps()
    kn, an = m["kept_new"], m["added_new"]
    ks = np.stack([2 * kn, 2 * kn + 1], 1).ravel()
    as_ = np.stack([2 * an, 2 * an + 1], 1).ravel()
    return np.concatenate([np.asarray(g_new)[ks], np.asarray(g_new)[as_]], axis=0)
