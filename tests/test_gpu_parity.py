"""Device parity against the CPU oracle (oracle/), through the sbx C-ABI.

Tier 1: identical HBS factors handed over in the reference's HBS1 format ->
device sweeps must match the oracle's sweeps to 1e-12 relative.
Tier 2: independent device compression -> reference test assertions (dense
operator / dense solve / analytic field) and 1e-9 agreement with the
oracle's refined solve.
"""
from pathlib import Path

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def sb():
    import paper_2108_07205_b200 as sb
    sb.init(0)
    return sb


def rel(a, b):
    return float(np.linalg.norm(np.asarray(a) - np.asarray(b)) / np.linalg.norm(np.asarray(b)))


# ---------------------------------------------------------------- geometry / entries
def test_nodes_bitwise_equal_oracle(sb, po):
    g = sb.panelize(sb.star(5, 0.3), 12, 16)
    o = po.Geom.create(po.STAR, 12, prongs=5, amplitude=0.3)
    a, b = g.nodes(), o.nodes()
    for key in ("x", "y", "nx", "ny", "w", "curvature", "param"):
        assert np.array_equal(a[key], b[key]), key
    g1, p1 = sb.refine(g, [5, 2], 3)
    o1, q1 = o.refine([5, 2], 3)
    assert all(np.array_equal(p1.maps()[k], q1.maps()[k]) for k in p1.maps())
    assert np.array_equal(g1.nodes()["x"], o1.nodes()["x"])


def test_entries_bitwise_equal_oracle(sb, po):
    g = sb.panelize(sb.ellipse(2.0, 1.0), 16, 16)
    o = po.Geom.create(po.ELLIPSE, 16, scale=2.0, aspect=0.5)
    a = po.Assembler.create(o)
    rng = np.random.default_rng(0)
    rows = rng.integers(0, 512, 200)
    cols = np.concatenate([rows[:50], rng.integers(0, 512, 150)])
    assert np.array_equal(sb.submatrix(g, rows, cols), a.submatrix(rows, cols))


# ---------------------------------------------------------------- tier 1 sweeps
@pytest.mark.parametrize("nrhs", [1, 3, 64, 130])
def test_tier1_hbs1_sweeps_match_oracle(sb, po, tmp_path, nrhs):
    o = po.Geom.create(po.STAR, 24, prongs=5, amplitude=0.3)
    a = po.Assembler.create(o)
    h = po.Hbs.compress(a, 1e-10).invert()
    h.save(tmp_path / "h.hbs1")
    d = sb.hbs_load(tmp_path / "h.hbs1")
    n = h.info()["n"]
    b = np.random.default_rng(nrhs).standard_normal((n, nrhs))
    assert rel(sb.hbs_solve(d, b), h.solve(b)) < 1e-12
    assert rel(sb.hbs_apply(d, b), h.apply(b)) < 1e-12


def test_hbs1_device_roundtrip_bitwise(sb, po, tmp_path):
    o = po.Geom.create(po.STAR, 10, prongs=3, amplitude=0.35)
    h = po.Hbs.compress(po.Assembler.create(o), 1e-8).invert()
    h.save(tmp_path / "a.hbs1")
    d = sb.hbs_load(tmp_path / "a.hbs1")
    sb.hbs_save(d, tmp_path / "b.hbs1")
    assert (tmp_path / "a.hbs1").read_bytes() == (tmp_path / "b.hbs1").read_bytes()


# ---------------------------------------------------------------- tier 2 compression
def test_device_compress_apply_matches_dense(sb, po):  # test_hbs.cpp:60-90
    g = sb.panelize(sb.circle(1.3, (0.1, -0.2)), 10, 16)
    h = sb.hbs_compress(g, sb.INTERIOR_DIRICHLET, sb.HbsOptions(eps=1e-10), mu=0.8)
    o = po.Geom.create(po.CIRCLE, 10, center=(0.1, -0.2), scale=1.3)
    A = po.Assembler.create(o, po.INTERIOR, 0.8).full_matrix()
    n = A.shape[0]
    assert np.linalg.norm(sb.hbs_apply(h, np.eye(n)) - A) / np.linalg.norm(A) < 1e-9


def test_device_compress_ranks_track_oracle(sb, po):
    g = sb.panelize(sb.star(5, 0.3), 24, 16)
    h = sb.hbs_compress(g)
    o = po.Hbs.compress(po.Assembler.create(po.Geom.create(po.STAR, 24, prongs=5, amplitude=0.3)), 1e-10)
    assert np.max(np.abs(h.node_ranks() - o.node_ranks())) <= 2


def test_device_solve_residual_and_field(sb, po):  # test_hbs.cpp:128-184
    g = sb.panelize(sb.circle(), 20, 16)
    h = sb.hbs_invert(sb.hbs_compress(g))
    o = po.Geom.create(po.CIRCLE, 20)
    A = po.Assembler.create(o).full_matrix()
    b = np.random.default_rng(3).standard_normal(A.shape[0])
    assert np.linalg.norm(A @ sb.hbs_solve(h, b) - b) < 1e-7 * np.linalg.norm(b)
    src = po.ring_sources(5, (0, 0), 3.0)
    tau = sb.hbs_solve(h, sb.boundary_data(g, src))
    tg = np.array([[0.3, 0.1], [0.4, 0.2], [-0.3, 0.4], [0.2, -0.5], [-0.5, -0.1]])
    u = o.evaluate_velocity(po.INTERIOR, tau, tg)
    ref = po.field_velocity(src, tg)
    assert np.max(np.linalg.norm(u - ref, axis=1) / np.linalg.norm(ref, axis=1)) < 1e-8


def test_device_update_matches_dense(sb, po):  # test_lowrank.cpp:64-98
    eps = 1e-10
    g0 = sb.panelize(sb.star(5, 0.3), 10, 16)
    g1, plan = sb.refine(g0, [2, 3], 2)
    u = sb.compress_update(g0, g1, plan, eps)
    L, R = u.factors()
    o0 = po.Geom.create(po.STAR, 10, prongs=5, amplitude=0.3)
    o1, op = o0.refine([2, 3], 2)
    a0, a1 = po.Assembler.create(o0), po.Assembler.create(o1)
    nk, nc, npp = op.sizes()
    n = 2 * (nk + nc + npp)
    Q = np.zeros((n, n))
    Q[: 2 * nk, 2 * nk: 2 * nk + 2 * nc] = -po.block_eval_full(a0, a1, op, "kc")
    Q[: 2 * nk, 2 * nk + 2 * nc:] = po.block_eval_full(a0, a1, op, "kp")
    Q[2 * nk + 2 * nc:, : 2 * nk] = po.block_eval_full(a0, a1, op, "pk")
    assert np.linalg.norm(Q - L @ R, 2) <= 10 * eps * np.linalg.norm(Q, 2)
    ou = po.Update.compress(a0, a1, op, eps)
    assert abs(u.k - ou.info()["k"]) <= 3


def test_els_matches_oracle_and_dense(sb, po):  # test_els.cpp:125-144
    eps = 1e-10
    g0 = sb.panelize(sb.star(5, 0.3), 10, 16)
    h = sb.hbs_invert(sb.hbs_compress(g0))
    g1, plan = sb.refine(g0, [3], 4)
    u = sb.compress_update(g0, g1, plan, eps)
    e = sb.els_build(h, g0, g1, plan, u)
    src = po.ring_sources(4, (0, 0), 3.0)
    g_new = sb.boundary_data(g1, src)
    tau = sb.els_solve(e, sb.gather_kept_added(plan, g_new))
    o0 = po.Geom.create(po.STAR, 10, prongs=5, amplitude=0.3)
    o1, op = o0.refine([3], 4)
    a1 = po.Assembler.create(o1)
    Ann = a1.full_matrix()
    ref = po.gather_kept_added(op.maps(), np.linalg.solve(Ann, o1.boundary_data(src)))
    assert rel(tau, ref) <= 1e-8
    a0 = po.Assembler.create(o0)
    oe = po.Els.build(po.Hbs.compress(a0, eps).invert(), a0, a1, op, po.Update.compress(a0, a1, op, eps))
    assert rel(tau, oe.solve(po.gather_kept_added(op.maps(), o1.boundary_data(src)))) <= 1e-9


def test_singular_woodbury_is_reported(sb):  # test_els.cpp:293-330
    g = sb.panelize(sb.circle(), 10, 16)
    h = sb.hbs_invert(sb.hbs_compress(g))
    g1, plan = sb.refine(g, [0], 2)
    n_ext = sum(2 * x for x in plan.sizes())
    e0 = sb.els_build(h, g, g1, plan,
                      sb.update_from_factors(plan, np.zeros((n_ext, 0)), np.zeros((0, n_ext))))
    rng = np.random.default_rng(0)
    u1 = rng.standard_normal(n_ext)
    y = sb.els_solve_raw(e0, u1)  # Atilde^{-1} u1
    # W = I + R Atilde^{-1} L = [[0, 0], [r.y, 1]]: loses one direction
    L = np.stack([u1, np.zeros(n_ext)], 1)
    R = np.stack([-y / (y @ y), 1e-3 * rng.standard_normal(n_ext)], 0)
    with pytest.raises(sb.SingularMatrixError, match="optimal-basis"):
        sb.els_build(h, g, g1, plan, sb.update_from_factors(plan, L, R))


def test_cfg1_els_matches_dense_and_field(sb, po):
    """BASELINE configs[0] at full size: ellipse (2, 1), 128 x 16 nodes, the 4
    panels nearest (1.99, 0) split m = 8 (A_pp is 1024 x 1024: blocked dense
    LU), 5 Stokeslets at radius 4; against the dense LU of A_nn (4992
    unknowns) and the analytic field at interior targets."""
    from paper_2108_07205_b200.configs import CONFIGS
    c = CONFIGS["cfg1"]
    g0 = sb.panelize(sb.ellipse(c.a, c.b), c.n_panels, c.q)
    panels = c.refine_panels(g0.nodes())
    assert list(panels) == [0, 1, 126, 127]
    h = sb.hbs_invert(sb.hbs_compress(g0, opts=sb.HbsOptions(eps=c.eps)))
    g1, plan = sb.refine(g0, panels, c.m)
    u = sb.compress_update(g0, g1, plan, c.eps)
    e = sb.els_build(h, g0, g1, plan, u)
    src = c.sources()[0]
    tau = sb.els_solve(e, sb.gather_kept_added(plan, sb.boundary_data(g1, src)))
    o0 = po.Geom.create(po.ELLIPSE, c.n_panels, scale=c.a, aspect=c.b / c.a)
    o1, op = o0.refine(panels, c.m)
    A = po.Assembler.create(o1).full_matrix()
    ref = po.gather_kept_added(op.maps(), np.linalg.solve(A, o1.boundary_data(src)))
    assert rel(tau, ref) <= 1e-8
    tg = c.interior_targets()[:20]
    vel = o1.evaluate_velocity(po.INTERIOR, sb.density_on_refined(e, tau), tg)
    ex = po.field_velocity(src, tg)
    assert np.max(np.linalg.norm(vel - ex, axis=1) / np.linalg.norm(ex, axis=1)) < 1e-8


@pytest.mark.parametrize("top", [2, 3, 4])
def test_collapsed_top_matches_oracle(po, tmp_path, top):
    """Solve with the top of the tree collapsed into one dense map
    (sweep.cu hbs_build_top, SBX_SWEEP_TOP=depth) against the oracle's
    level-by-level sweep on the same HBS1 factors, plain and transposed."""
    import os
    import subprocess
    import sys
    o = po.Geom.create(po.STAR, 80, prongs=5, amplitude=0.3)  # 1280 nodes: leaves at depth 5
    a = po.Assembler.create(o)
    h = po.Hbs.compress(a, 1e-10).invert()
    h.save(tmp_path / "h.hbs1")
    n = h.info()["n"]
    b = np.random.default_rng(5).standard_normal((n, 130))
    np.save(tmp_path / "b.npy", b)
    np.save(tmp_path / "x.npy", h.solve(b))
    np.save(tmp_path / "xt.npy", h.solve_t(b))
    root = str(Path(__file__).resolve().parents[1])
    env = dict(os.environ, SBX_SWEEP_TOP=str(top), PYTHONPATH=root + os.pathsep + os.environ.get("PYTHONPATH", ""))
    r = subprocess.run([sys.executable, str(Path(__file__).parent / "top_sweep_case.py"), str(tmp_path / "h.hbs1"),
                        str(tmp_path / "b.npy"), str(tmp_path / "x.npy"), str(tmp_path / "xt.npy")],
                       env=env, capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stdout + r.stderr
    assert f"top {top}" in r.stdout, r.stdout


def test_fused_app_build_bitwise(po, tmp_path):
    """The added block's HBS built with each level's inverse overlapping the
    next level's compression (hbs_compress_invert_device) gives the same
    refined solve, bit for bit, as compress-then-invert -- and a second
    fused run repeats the first (the ID rounds of the two concurrent builds
    are merged in arrival order; no engine choice may depend on it)."""
    import os
    import subprocess
    import sys
    root = str(Path(__file__).resolve().parents[1])
    out = {}
    for mode in ("fused", "unfused", "fused_again"):
        env = dict(os.environ, PYTHONPATH=root + os.pathsep + os.environ.get("PYTHONPATH", ""))
        if mode == "unfused":
            env["SBX_APP_UNFUSED"] = "1"
        r = subprocess.run([sys.executable, str(Path(__file__).parent / "app_case.py"), str(tmp_path / f"{mode}.npy")],
                           env=env, capture_output=True, text=True, timeout=600)
        assert r.returncode == 0, r.stdout + r.stderr
        out[mode] = np.load(tmp_path / f"{mode}.npy")
    assert np.array_equal(out["fused"], out["unfused"])
    assert np.array_equal(out["fused"], out["fused_again"])
    assert np.all(np.isfinite(out["fused"]))


def test_collapsed_top_auto(tmp_path):
    """Default top choice on a device-compressed 32768-unknown wall: the
    inverse's rcond gates admit the collapse (depth > 0), and the solve and
    transposed solve agree with the level-by-level sweep (SBX_SWEEP_TOP=0)."""
    import os
    import subprocess
    import sys
    root = str(Path(__file__).resolve().parents[1])
    out, tops = {}, {}
    for mode in ("auto", "off"):
        env = dict(os.environ, PYTHONPATH=root + os.pathsep + os.environ.get("PYTHONPATH", ""))
        if mode == "off":
            env["SBX_SWEEP_TOP"] = "0"
        r = subprocess.run([sys.executable, str(Path(__file__).parent / "top_auto_case.py"), str(tmp_path / f"{mode}.npy")],
                           env=env, capture_output=True, text=True, timeout=600)
        assert r.returncode == 0, r.stdout + r.stderr
        out[mode] = np.load(tmp_path / f"{mode}.npy")
        tops[mode] = int(r.stdout.split("top")[-1])
    assert tops["auto"] >= 2 and tops["off"] == 0, tops
    assert rel(out["auto"], out["off"]) < 1e-12


def test_tier1_dumped_update_factors_match_oracle(sb, po, tmp_path):
    """SURVEY 8(c) tier 1 for the ELS: the oracle's HBS1 inverse and its
    update factors L, R handed over in the reference's dump_matrix format
    (nystrom.cpp:450-477) -> device els_build / els_solve agree with the
    oracle's els_solve to 1e-12 (identical factors, different rounding)."""
    eps = 1e-10
    o0 = po.Geom.create(po.STAR, 12, prongs=5, amplitude=0.3)
    o1, op = o0.refine([3, 4], 4)
    a0, a1 = po.Assembler.create(o0), po.Assembler.create(o1)
    oh = po.Hbs.compress(a0, eps).invert()
    ou = po.Update.compress(a0, a1, op, eps)
    oe = po.Els.build(oh, a0, a1, op, ou)
    oh.save(tmp_path / "a.hbs1")
    f = ou.factors()
    po.dump_matrix(tmp_path / "L.mat", f["L"])
    po.dump_matrix(tmp_path / "R.mat", f["R"])
    g0 = sb.panelize(sb.star(5, 0.3), 12, 16)
    g1, plan = sb.refine(g0, [3, 4], 4)
    h = sb.hbs_load(tmp_path / "a.hbs1")
    u = sb.update_load(plan, tmp_path / "L.mat", tmp_path / "R.mat")
    assert u.k == ou.info()["k"]
    e = sb.els_build(h, g0, g1, plan, u)
    src = po.ring_sources(4, (0, 0), 3.0)
    G = np.stack([po.gather_kept_added(op.maps(), o1.boundary_data(s)) for s in (src, src[::-1])], 1)
    assert rel(sb.els_solve(e, G), oe.solve(G)) < 1e-12
    # and back out: the device's copy of the factors dumps to the same files
    sb.update_dump(u, tmp_path / "L2.mat", tmp_path / "R2.mat")
    assert (tmp_path / "L.mat").read_bytes() == (tmp_path / "L2.mat").read_bytes()
    assert (tmp_path / "R.mat").read_bytes() == (tmp_path / "R2.mat").read_bytes()
