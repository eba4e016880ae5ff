"""ORACLE — TEST INFRASTRUCTURE ONLY.

ctypes front-end to ``oracle/_build/liboracle.so``, the CPU restatement of
the reference stokesbie path (see ``oracle/orc.hpp``).  Imported only by
``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s CPU legs, always as
the checker / baseline, never as the thing measured for the product.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess
from pathlib import Path

import numpy as np

_HERE = Path(__file__).resolve().parent
_LIB_PATH = _HERE / "_build" / "liboracle.so"
_lib = None

I64P = C.POINTER(C.c_int64)
F64P = C.POINTER(C.c_double)
VPP = C.POINTER(C.c_void_p)

CIRCLE, ELLIPSE, STAR, FOURIER, CHANNEL = 0, 1, 2, 3, 4
INTERIOR, EXTERIOR, MIXED = 0, 1, 2
BLOCKS = {"kk": 0, "kc": 1, "ck": 2, "cc": 3, "kp": 4, "pk": 5, "pp": 6}


class OracleError(RuntimeError):
    def __init__(self, code, msg):
        super().__init__(f"[{code}] {msg}")
        self.code = code


def build(force: bool = False) -> Path:
    if force or not _LIB_PATH.exists():
        subprocess.run(["make", "-C", str(_HERE), "-j8"], check=True,
                       stdout=subprocess.DEVNULL)
    return _LIB_PATH


def lib():
    global _lib
    if _lib is None:
        if not _LIB_PATH.exists():
            build()
        _lib = C.CDLL(str(_LIB_PATH))
        _lib.orc_last_error.restype = C.c_char_p
        _lib.orc_panels_near_point.restype = C.c_int64
        _lib.orc_hbs_node_k.restype = C.c_int64
        for name in ("orc_geom_free", "orc_plan_free", "orc_asm_free", "orc_hbs_free",
                     "orc_update_free", "orc_els_free"):
            getattr(_lib, name).restype = None
    return _lib


def _chk(code):
    if code != 0:
        raise OracleError(code, lib().orc_last_error().decode())


def _f(a):
    a = np.ascontiguousarray(a, dtype=np.float64)
    return a, a.ctypes.data_as(F64P)


def _i(a):
    a = np.ascontiguousarray(a, dtype=np.int64)
    return a, a.ctypes.data_as(I64P)


def _fortran(a):
    return np.asfortranarray(np.asarray(a, dtype=np.float64))


class _Handle:
    _free = None

    def __init__(self, ptr):
        self.ptr = ptr

    def __del__(self):
        if self.ptr and self._free and _lib is not None:
            getattr(_lib, self._free)(self.ptr)
            self.ptr = None


class Geom(_Handle):
    _free = "orc_geom_free"

    @staticmethod
    def create(kind, n_panels, q=16, center=(0.0, 0.0), scale=1.0, prongs=0, amplitude=0.0,
               aspect=1.0, cos_coef=(), sin_coef=()):
        p = C.c_void_p()
        if cos_coef or sin_coef:
            cc, cp = _f(np.asarray(cos_coef, dtype=np.float64).reshape(-1))
            ss, sp = _f(np.asarray(sin_coef, dtype=np.float64).reshape(-1))
            _chk(lib().orc_geom_create_curve(kind, C.c_double(center[0]), C.c_double(center[1]),
                                             C.c_double(scale), prongs, C.c_double(amplitude), C.c_double(aspect),
                                             len(cc), cp, len(ss), sp, n_panels, q, C.byref(p)))
            return Geom(p)
        _chk(lib().orc_geom_create(kind, C.c_double(center[0]), C.c_double(center[1]),
                                   C.c_double(scale), prongs, C.c_double(amplitude),
                                   C.c_double(aspect), n_panels, q, C.byref(p)))
        return Geom(p)

    def info(self):
        n, npan, nc = C.c_int64(), C.c_int64(), C.c_int64()
        lib().orc_geom_info(self.ptr, C.byref(n), C.byref(npan), C.byref(nc))
        return n.value, npan.value, nc.value

    @property
    def n_nodes(self):
        return self.info()[0]

    def nodes(self):
        n = self.n_nodes
        out = np.zeros(9 * n)
        pan = np.zeros(n, dtype=np.int64)
        lib().orc_geom_nodes(self.ptr, out.ctypes.data_as(F64P), pan.ctypes.data_as(I64P))
        o = out.reshape(9, n)
        keys = ("x", "y", "nx", "ny", "tx", "ty", "w", "curvature", "param")
        d = {k: o[i].copy() for i, k in enumerate(keys)}
        d["panel_of"] = pan
        return d

    def panels_near_point(self, p, radius):
        cap = self.info()[1]
        out = np.zeros(cap, dtype=np.int64)
        n = lib().orc_panels_near_point(self.ptr, C.c_double(p[0]), C.c_double(p[1]),
                                        C.c_double(radius), out.ctypes.data_as(I64P), cap)
        return out[:n]

    def refine(self, panels, m):
        panels, pp = _i(panels)
        g, pl = C.c_void_p(), C.c_void_p()
        _chk(lib().orc_refine(self.ptr, pp, len(panels), m, C.byref(g), C.byref(pl)))
        return Geom(g), Plan(pl)

    def coarsen(self, plan):
        g = C.c_void_p()
        _chk(lib().orc_coarsen(self.ptr, plan.ptr, C.byref(g)))
        return Geom(g)

    def add_holes(self, holes):
        """holes: list of (cx, cy, radius, n_panels, q)."""
        h, hp = _f(np.asarray(holes, dtype=np.float64).ravel())
        g, pl = C.c_void_p(), C.c_void_p()
        _chk(lib().orc_geom_add_holes(self.ptr, len(holes), hp, C.byref(g), C.byref(pl)))
        return Geom(g), Plan(pl)

    def boundary_data(self, sources, mu=1.0):
        s, sp = _f(np.asarray(sources, dtype=np.float64).reshape(-1, 4))
        out = np.zeros(2 * self.n_nodes)
        _chk(lib().orc_boundary_data(self.ptr, len(s), sp, C.c_double(mu),
                                     out.ctypes.data_as(F64P)))
        return out

    def evaluate_velocity(self, form, tau, targets, mu=1.0):
        t, tp = _f(np.asarray(tau, dtype=np.float64))
        tg, tgp = _f(np.asarray(targets, dtype=np.float64).reshape(-1, 2))
        out = np.zeros((len(tg), 2))
        _chk(lib().orc_evaluate_velocity(self.ptr, form, C.c_double(mu), tp, len(tg), tgp,
                                         out.ctypes.data_as(F64P)))
        return out


class Plan(_Handle):
    _free = "orc_plan_free"

    def sizes(self):
        a, b, c = C.c_int64(), C.c_int64(), C.c_int64()
        lib().orc_plan_sizes(self.ptr, C.byref(a), C.byref(b), C.byref(c))
        return a.value, b.value, c.value

    def maps(self):
        nk, nc, npp = self.sizes()
        ko, kn = np.zeros(nk, np.int64), np.zeros(nk, np.int64)
        co, an = np.zeros(nc, np.int64), np.zeros(npp, np.int64)
        lib().orc_plan_maps(self.ptr, ko.ctypes.data_as(I64P), kn.ctypes.data_as(I64P),
                            co.ctypes.data_as(I64P), an.ctypes.data_as(I64P))
        return {"kept_old": ko, "kept_new": kn, "cut_old": co, "added_new": an}


class Assembler(_Handle):
    _free = "orc_asm_free"

    def __init__(self, ptr, geom):
        super().__init__(ptr)
        self.geom = geom

    @staticmethod
    def create(geom, form=INTERIOR, mu=1.0):
        p = C.c_void_p()
        _chk(lib().orc_asm_create(geom.ptr, form, C.c_double(mu), C.byref(p)))
        return Assembler(p, geom)

    def submatrix(self, rows, cols):
        rows, rp = _i(rows)
        cols, cp = _i(cols)
        out = np.zeros((len(rows), len(cols)), order="F")
        _chk(lib().orc_asm_submatrix(self.ptr, rp, len(rows), cp, len(cols),
                                     out.ctypes.data_as(F64P)))
        return out

    def full_matrix(self):
        n = 2 * self.geom.n_nodes
        idx = np.arange(n)
        return self.submatrix(idx, idx)


class Hbs(_Handle):
    _free = "orc_hbs_free"

    @staticmethod
    def compress(asm, eps=1e-10, leaf=64, subset=None):
        p = C.c_void_p()
        if subset is None:
            _chk(lib().orc_hbs_compress(asm.ptr, None, 0, C.c_double(eps), leaf, C.byref(p)))
        else:
            s, sp = _i(subset)
            _chk(lib().orc_hbs_compress(asm.ptr, sp, len(s), C.c_double(eps), leaf, C.byref(p)))
        return Hbs(p)

    @staticmethod
    def load(path):
        p = C.c_void_p()
        _chk(lib().orc_hbs_load(str(path).encode(), C.byref(p)))
        return Hbs(p)

    def save(self, path):
        _chk(lib().orc_hbs_save(self.ptr, str(path).encode()))

    def invert(self):
        _chk(lib().orc_hbs_invert(self.ptr))
        return self

    def info(self):
        out = np.zeros(8, dtype=np.int64)
        lib().orc_hbs_info(self.ptr, out.ctypes.data_as(I64P))
        keys = ("n", "nodes", "total_skeleton", "max_block_drawn", "has_inverse",
                "factor_doubles", "max_depth", "max_k")
        return dict(zip(keys, (int(v) for v in out)))

    def node_ranks(self):
        n = self.info()["nodes"]
        out = np.zeros(n, dtype=np.int64)
        lib().orc_hbs_node_k(self.ptr, out.ctypes.data_as(I64P), n)
        return out

    def _sweep(self, mode, b):
        b = _fortran(b)
        vec = b.ndim == 1
        if vec:
            b = b.reshape(-1, 1, order="F")
        out = np.zeros_like(b, order="F")
        _chk(lib().orc_hbs_sweep(self.ptr, mode, b.ctypes.data_as(F64P), b.shape[1],
                                 out.ctypes.data_as(F64P)))
        return out[:, 0] if vec else out

    def solve(self, b):
        return self._sweep(0, b)

    def solve_t(self, b):
        return self._sweep(1, b)

    def apply(self, v):
        return self._sweep(2, v)

    def apply_t(self, v):
        return self._sweep(3, v)


def row_id(w, eps=None, forced=None):
    w = _fortran(w)
    m, n = w.shape
    k = C.c_int64()
    J = np.zeros(m, dtype=np.int64)
    P = np.zeros(m * max(1, min(m, n)), dtype=np.float64)
    _chk(lib().orc_row_id(w.ctypes.data_as(F64P), m, n, C.c_double(eps or 0.0),
                          -1 if forced is None else forced, C.byref(k),
                          J.ctypes.data_as(I64P), P.ctypes.data_as(F64P)))
    kk = k.value
    return kk, J, P[: m * kk].reshape((m, kk), order="F")


def randomized_row_id(w, eps, seed):
    w = _fortran(w)
    m, n = w.shape
    k = C.c_int64()
    J = np.zeros(m, dtype=np.int64)
    P = np.zeros(m * max(1, min(m, n)), dtype=np.float64)
    _chk(lib().orc_randomized_row_id(w.ctypes.data_as(F64P), m, n, C.c_double(eps),
                                     C.c_uint64(seed), C.byref(k), J.ctypes.data_as(I64P),
                                     P.ctypes.data_as(F64P)))
    kk = k.value
    return kk, J, P[: m * kk].reshape((m, kk), order="F")


def gaussian_sketch(n, l, seed):
    out = np.zeros(n * l)
    lib().orc_gaussian_sketch(n, l, C.c_uint64(seed), out.ctypes.data_as(F64P))
    return out.reshape((n, l), order="F")


def gauss_rule(n):
    x, w = np.zeros(n), np.zeros(n)
    _chk(lib().orc_gauss_rule(n, x.ctypes.data_as(F64P), w.ctypes.data_as(F64P)))
    return x, w


def log_rule_weights(q, u):
    out = np.zeros(q)
    _chk(lib().orc_log_rule_weights(q, C.c_double(u), out.ctypes.data_as(F64P)))
    return out


def field_velocity(sources, targets, mu=1.0):
    s, sp = _f(np.asarray(sources, dtype=np.float64).reshape(-1, 4))
    t, tp = _f(np.asarray(targets, dtype=np.float64).reshape(-1, 2))
    out = np.zeros((len(t), 2))
    _chk(lib().orc_field_velocity(len(s), sp, C.c_double(mu), len(t), tp,
                                  out.ctypes.data_as(F64P)))
    return out


class Update(_Handle):
    _free = "orc_update_free"

    @staticmethod
    def compress(old_asm, new_asm, plan, eps=1e-10, seed=0):
        p = C.c_void_p()
        _chk(lib().orc_update_compress(old_asm.ptr, new_asm.ptr, plan.ptr, C.c_double(eps),
                                       C.c_uint64(seed), C.byref(p)))
        return Update(p)

    def info(self):
        out = np.zeros(9, dtype=np.int64)
        lib().orc_update_info(self.ptr, out.ctypes.data_as(I64P))
        keys = ("k", "k1", "kc", "kp", "pk", "n_ext", "nk2", "nc2", "np2")
        return dict(zip(keys, (int(v) for v in out)))

    def factors(self):
        i = self.info()
        n, k, k1 = i["n_ext"], i["k"], i["k1"]
        L = np.zeros((n, k), order="F")
        R = np.zeros((k, n), order="F")
        L1 = np.zeros((n, k1), order="F")
        R1 = np.zeros((k1, n), order="F")
        for w, a in enumerate((L, R, L1, R1)):
            lib().orc_update_factor(self.ptr, w, a.ctypes.data_as(F64P))
        sk = np.zeros(k, dtype=np.int64)
        lib().orc_update_skeleton(self.ptr, sk.ctypes.data_as(I64P))
        return {"L": L, "R": R, "L1": L1, "R1": R1, "skeleton": sk}

    def set_factors(self, L, R):
        L, R = _fortran(L), _fortran(R)
        _chk(lib().orc_update_set(self.ptr, L.ctypes.data_as(F64P), R.ctypes.data_as(F64P),
                                  L.shape[0], L.shape[1]))


def dump_matrix(path, m):
    """nystrom.cpp:450-461: u32 rows, u32 cols, row-major doubles."""
    a = _fortran(np.atleast_2d(m))
    _chk(lib().orc_dump_matrix(str(path).encode(), a.ctypes.data_as(F64P), a.shape[0], a.shape[1]))


def load_matrix(path):
    """nystrom.cpp:463-477."""
    r, c = C.c_int64(), C.c_int64()
    _chk(lib().orc_load_matrix_dims(str(path).encode(), C.byref(r), C.byref(c)))
    out = np.zeros((r.value, c.value), order="F")
    _chk(lib().orc_load_matrix(str(path).encode(), out.ctypes.data_as(F64P)))
    return out


def truncated_svd(w, eps):
    """idlib.cpp:134-154 (Eigen BDCSVD there, LAPACK gesdd here): thin SVD,
    k = #{ s_i > eps s_0 }."""
    w = np.asarray(w, dtype=np.float64)
    if w.size == 0:
        return np.zeros((w.shape[0], 0)), np.zeros(0), np.zeros((w.shape[1], 0))
    U, s, Vt = np.linalg.svd(w, full_matrices=False)
    k = int(np.sum(s > eps * s[0])) if s[0] > 0 else 0
    return U[:, :k], s[:k], Vt[:k].T


def svd_optimal(old_asm, new_asm, plan, eps):
    """lowrank.cpp:329-362 (CompressionMode::SvdOptimal) with assemble_stacked
    (lowrank.cpp:240-251): returns dict(L, R, k, k1, kc, kp, pk)."""
    f = {}
    for b in ("kc", "kp", "pk"):
        U, s, V = truncated_svd(block_eval_full(old_asm, new_asm, plan, b), eps)
        f[b] = (U, s[:, None] * V.T)
    nk, nc, npp = plan.sizes()
    nk2, nc2, np2 = 2 * nk, 2 * nc, 2 * npp
    n = nk2 + nc2 + np2
    kpk, kkc, kkp = (f[b][0].shape[1] for b in ("pk", "kc", "kp"))
    k1 = kpk + kkc + kkp
    L1, R1 = np.zeros((n, k1)), np.zeros((k1, n))
    L1[:nk2, kpk:kpk + kkc] = -f["kc"][0]
    L1[:nk2, kpk + kkc:] = f["kp"][0]
    L1[nk2 + nc2:, :kpk] = f["pk"][0]
    R1[:kpk, :nk2] = f["pk"][1]
    R1[kpk:kpk + kkc, nk2:nk2 + nc2] = f["kc"][1]
    R1[kpk + kkc:, nk2 + nc2:] = f["kp"][1]
    if k1 == 0:
        return {"L": np.zeros((n, 0)), "R": np.zeros((0, n)), "k": 0, "k1": 0, "kc": 0, "kp": 0, "pk": 0}
    U, s, V = truncated_svd(L1, eps)
    return {"L": U, "R": (s[:, None] * V.T) @ R1, "k": U.shape[1], "k1": k1, "kc": kkc, "kp": kkp, "pk": kpk}


def block_eval_full(old_asm, new_asm, plan, block):
    nk, nc, npp = plan.sizes()
    size = {"k": 2 * nk, "c": 2 * nc, "p": 2 * npp}
    out = np.zeros((size[block[0]], size[block[1]]), order="F")
    _chk(lib().orc_block_eval_full(old_asm.ptr, new_asm.ptr, plan.ptr, BLOCKS[block],
                                   out.ctypes.data_as(F64P)))
    return out


class Els(_Handle):
    _free = "orc_els_free"

    @staticmethod
    def build(hbs, old_asm, new_asm, plan, upd):
        p = C.c_void_p()
        _chk(lib().orc_els_build(hbs.ptr, old_asm.ptr, new_asm.ptr, plan.ptr, upd.ptr,
                                 C.byref(p)))
        return Els(p)

    def info(self):
        out = np.zeros(5, dtype=np.int64)
        lib().orc_els_info(self.ptr, out.ctypes.data_as(I64P))
        return dict(zip(("n_k", "n_c", "n_p", "k", "app_hbs"), (int(v) for v in out)))

    def _call(self, mode, g):
        g = _fortran(g)
        vec = g.ndim == 1
        if vec:
            g = g.reshape(-1, 1, order="F")
        i = self.info()
        rows = i["n_k"] + i["n_p"] if mode == 0 else i["n_k"] + i["n_c"] + i["n_p"]
        out = np.zeros((rows, g.shape[1]), order="F")
        _chk(lib().orc_els_solve(self.ptr, mode, g.ctypes.data_as(F64P), g.shape[1],
                                 out.ctypes.data_as(F64P)))
        return out[:, 0] if vec else out

    def solve(self, g_n):
        return self._call(0, g_n)

    def solve_raw(self, g_ext):
        return self._call(1, g_ext)

    def solve_raw_t(self, g_ext):
        return self._call(2, g_ext)

    def apply_forward(self, v):
        return self._call(3, v)

    def xw(self):
        i = self.info()
        n = i["n_k"] + i["n_c"] + i["n_p"]
        X = np.zeros((n, i["k"]), order="F")
        W = np.zeros((i["k"], i["k"]), order="F")
        lib().orc_els_xw(self.ptr, X.ctypes.data_as(F64P), W.ctypes.data_as(F64P))
        return X, W


def ring_sources(n, center, radius):
    """nystrom.cpp:372-381 — returns rows (x, y, fx, fy)."""
    out = []
    for s in range(n):
        th = 2 * np.pi * s / n + 0.4
        ph = 2 * np.pi * s / n + 0.7
        out.append((center[0] + radius * np.cos(th), center[1] + radius * np.sin(th),
                    np.cos(ph), np.sin(ph)))
    return np.array(out)


def gather_kept_added(plan_maps, g_new):
    """scenario.cpp:253-258 — (kept, added) gather of refined-mesh scalars."""
    kn = plan_maps["kept_new"]
    an = plan_maps["added_new"]
    ks = np.stack([2 * kn, 2 * kn + 1], 1).ravel()
    as_ = np.stack([2 * an, 2 * an + 1], 1).ravel()
    return np.concatenate([g_new[ks], g_new[as_]], axis=0)
