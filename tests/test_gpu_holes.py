"""Single-layer components on the device (nystrom.cpp:80-172 log-corrected
Stokeslet; Mixed formulation with holes, Exterior combined field) against
the oracle, and the reference's hole-insertion assertion (test_els.cpp:168-197)."""
import numpy as np
import pytest

from test_oracle import HOLE_SOURCES, HOLE_TARGETS, density_on_refined

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def sb():
    import paper_2108_07205_b200 as sb
    sb.init(0)
    return sb


def holes_dev(sb):
    g0 = sb.panelize(sb.circle(2.0), 20, 16)
    g1, plan = sb.add_holes(g0, [(sb.circle(0.3, (-0.8, 0.0)), 10, 16), (sb.circle(0.25, (0.9, 0.3)), 10, 16),
                                 (sb.circle(0.2, (0.1, -0.9)), 10, 16)])
    return g0, g1, plan


def holes_oracle(po):
    g0 = po.Geom.create(po.CIRCLE, 20, scale=2.0)
    g1, plan = g0.add_holes([(-0.8, 0.0, 0.3, 10, 16), (0.9, 0.3, 0.25, 10, 16), (0.1, -0.9, 0.2, 10, 16)])
    return g0, g1, plan


def test_mixed_entries_match_oracle(sb, po):
    g0, g1, plan = holes_dev(sb)
    o0, o1, oplan = holes_oracle(po)
    assert np.array_equal(g1.nodes()["x"], o1.nodes()["x"])
    n = 2 * o1.n_nodes
    rng = np.random.default_rng(5)
    rows = np.concatenate([np.arange(640, 700), rng.integers(0, n, 120)])  # hole-1 panel runs + random
    cols = np.concatenate([np.arange(630, 720), rng.integers(0, n, 110)])
    A = sb.submatrix(g1, rows, cols, sb.MIXED)
    B = po.Assembler.create(o1, po.MIXED).submatrix(rows, cols)
    # wall columns (double layer + completion) are bit-identical; hole columns
    # carry log terms (device log vs libm) within a few ulps
    wall_c = cols < 640
    assert np.array_equal(A[:, wall_c], B[:, wall_c])
    assert np.max(np.abs(A - B)) <= 1e-14 * np.max(np.abs(B))


def test_exterior_entries_match_oracle(sb, po):
    g = sb.panelize(sb.star(5, 0.3), 12, 16)
    o = po.Geom.create(po.STAR, 12, prongs=5, amplitude=0.3)
    rng = np.random.default_rng(6)
    rows = np.concatenate([np.arange(0, 70), rng.integers(0, 384, 80)])
    cols = np.concatenate([np.arange(20, 90), np.arange(350, 384), rng.integers(0, 384, 60)])
    A = sb.submatrix(g, rows, cols, sb.EXTERIOR_COMBINED)
    B = po.Assembler.create(o, po.EXTERIOR).submatrix(rows, cols)
    assert np.max(np.abs(A - B)) <= 1e-14 * np.max(np.abs(B))


def test_mixed_hbs_solve_matches_dense(sb, po):  # test_hbs.cpp:128-157 on a multiply connected wall
    g0, g1, plan = holes_dev(sb)
    h = sb.hbs_invert(sb.hbs_compress(g1, sb.MIXED, opts=sb.HbsOptions(eps=1e-10)))
    o0, o1, oplan = holes_oracle(po)
    A = po.Assembler.create(o1, po.MIXED).full_matrix()
    b = np.random.default_rng(2).standard_normal(A.shape[0])
    x = sb.hbs_solve(h, b)
    assert np.linalg.norm(A @ x - b) <= 1e-7 * np.linalg.norm(b)


def test_holes_els_matches_dense_and_field(sb, po):  # test_els.cpp:168-197
    eps = 1e-10
    g0, g1, plan = holes_dev(sb)
    assert plan.sizes()[1] == 0
    h = sb.hbs_invert(sb.hbs_compress(g0, sb.MIXED, opts=sb.HbsOptions(eps=eps)))
    u = sb.compress_update(g0, g1, plan, eps, formulation=sb.MIXED)
    e = sb.els_build(h, g0, g1, plan, u, formulation=sb.MIXED)
    srcs = list(po.ring_sources(4, (0, 0), 3.5)) + HOLE_SOURCES
    g_new = sb.boundary_data(g1, srcs)
    tau = sb.els_solve(e, sb.gather_kept_added(plan, g_new))
    o0, o1, oplan = holes_oracle(po)
    A = po.Assembler.create(o1, po.MIXED).full_matrix()
    maps = oplan.maps()
    ref = po.gather_kept_added(maps, np.linalg.solve(A, o1.boundary_data(srcs)))
    assert np.linalg.norm(tau - ref) / np.linalg.norm(ref) <= 1e-8
    vel = o1.evaluate_velocity(po.MIXED, density_on_refined(maps, o1.n_nodes, tau), HOLE_TARGETS)
    exact = po.field_velocity(srcs, HOLE_TARGETS)
    assert max(np.linalg.norm(vel[i] - exact[i]) / np.linalg.norm(exact[i]) for i in range(3)) < 1e-8
    # and against the oracle's own ELS on the same inputs (T2 parity)
    a0, a1 = po.Assembler.create(o0, po.MIXED), po.Assembler.create(o1, po.MIXED)
    oe = po.Els.build(po.Hbs.compress(a0, eps).invert(), a0, a1, oplan, po.Update.compress(a0, a1, oplan, eps))
    ot = oe.solve(po.gather_kept_added(maps, o1.boundary_data(srcs)))
    assert np.linalg.norm(tau - ot) / np.linalg.norm(ot) <= 1e-9


def test_evaluate_solution_matches_oracle(sb, po):  # nystrom.cpp:408-448
    g0, g1, plan = holes_dev(sb)
    o0, o1, oplan = holes_oracle(po)
    n = 2 * o1.n_nodes
    tau = np.random.default_rng(4).standard_normal((n, 3))
    tg = np.array(HOLE_TARGETS + [(1.95, 0.0), (-0.8, 0.32)])  # two near the wall / a hole
    vel, pre, near = sb.evaluate_solution(g1, sb.MIXED, tau, tg, with_pressure=True)
    for r in range(3):
        ref = o1.evaluate_velocity(po.MIXED, tau[:, r], tg)
        assert np.max(np.abs(vel[:, :, r] - ref)) <= 1e-12 * np.max(np.abs(ref))
    assert list(near) == [False, False, False, True, True]
    # pressure: numpy restatement of evaluate_solution's pressure sum
    # (nystrom.cpp:437-440 with kernels.cpp:37-48: pressure_double on every
    # node, pressure_single on the single-layer components -- the holes under
    # MIXED), mu = 1
    nd = o1.nodes()
    x, y, nx, ny, w = nd["x"], nd["y"], nd["nx"], nd["ny"], nd["w"]
    n_wall = 20 * 16  # the wall's nodes come first; the holes carry the single layer
    sl = np.arange(o1.n_nodes) >= n_wall
    for r in range(3):
        t0, t1 = tau[0::2, r], tau[1::2, r]
        for k, (px, py) in enumerate(tg):
            rx, ry = px - x, py - y
            r2 = rx * rx + ry * ry
            rn = rx * nx + ry * ny
            pd0 = (1.0 / np.pi) * (-nx / r2 + rx * (2.0 * rn / (r2 * r2)))
            pd1 = (1.0 / np.pi) * (-ny / r2 + ry * (2.0 * rn / (r2 * r2)))
            terms = w * (pd0 * t0 + pd1 * t1) + np.where(sl, w * (rx * t0 + ry * t1) / (2.0 * np.pi * r2), 0.0)
            assert abs(pre[k, r] - terms.sum()) <= 1e-12 * np.abs(terms).sum()
