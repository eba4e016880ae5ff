"""Pins the CPU oracle (oracle/) against the reference's own test assertions.

The reference ships no golden vectors; its doctest suites pin
results through dense oracles, analytic Stokeslet fields and exact
identities.  Each test below restates one of those assertions, citing the
reference test it mirrors, and runs it against oracle/_build/liboracle.so.
scipy's LAPACK dgeqp3 is an independent cross-check of the CPQR pivots.
"""
import numpy as np
import pytest
import scipy.linalg as sla


def spectral(a):
    return np.linalg.norm(a, 2) if a.size else 0.0


def skeleton_identity_exact(k, J, P):
    return all(P[J[i], j] == (1.0 if i == j else 0.0) for i in range(k) for j in range(k))


def matrix_with_spectrum(m, n, sv, rng):
    u = np.linalg.qr(rng.standard_normal((m, len(sv))))[0]
    v = np.linalg.qr(rng.standard_normal((n, len(sv))))[0]
    return (u * sv) @ v.T


# ---------------------------------------------------------------- idlib (test_idlib.cpp)
def test_rank1_outer_product(po):  # test_idlib.cpp:48-61
    rng = np.random.default_rng(7)
    w = np.outer(rng.standard_normal(50), rng.standard_normal(30))
    k, J, P = po.row_id(w, 1e-10)
    assert k == 1 and skeleton_identity_exact(k, J, P)
    assert spectral(w - P @ w[J[:k]]) <= 1e-9 * spectral(w)


def test_identity_full_rank(po):  # test_idlib.cpp:63-73
    w = np.eye(20)
    k, J, P = po.row_id(w, 1e-10)
    assert k == 20 and skeleton_identity_exact(k, J, P)
    assert np.all(np.abs(P).sum(1) == 1.0) and np.all(P.max(1) == 1.0)
    assert np.linalg.norm(w - P @ w[J[:k]]) == 0.0


def test_dyadic_decay_rank(po):  # test_idlib.cpp:75-87
    rng = np.random.default_rng(42)
    w = matrix_with_spectrum(200, 100, 2.0 ** -np.arange(100.0), rng)
    k, J, P = po.row_id(w, 1e-10)
    assert 32 <= k <= 36 and skeleton_identity_exact(k, J, P)
    assert spectral(w - P @ w[J[:k]]) <= 1e-9 * spectral(w)


def test_wide_tall_zero(po):  # test_idlib.cpp:89-113
    rng = np.random.default_rng(3)
    sv = 10.0 ** (-2.0 * np.arange(6))
    for shape in ((12, 90), (90, 12)):
        w = matrix_with_spectrum(*shape, sv, rng)
        k, J, P = po.row_id(w, 1e-8)
        assert k == 5
        assert spectral(w - P @ w[J[:k]]) <= 1e-7 * spectral(w)
    k, J, P = po.row_id(np.zeros((8, 5)), 1e-10)
    assert k == 0 and P.shape == (8, 0)
    k, J, P = po.row_id(np.zeros((0, 4)), 1e-10)
    assert k == 0


def test_tolerance_domain(po):  # test_idlib.cpp:115-121
    w = np.eye(4)
    for bad in (0.0, -1e-3, 0.5):
        with pytest.raises(po.OracleError):
            po.row_id(w, bad)
    po.row_id(w, 0.1)


def test_low_rank_plus_noise_property(po):  # test_idlib.cpp:125-157 (300 of the 1000 draws)
    rng = np.random.default_rng(2024)
    eps = 1e-10
    for _ in range(300):
        m, n = rng.integers(10, 81), rng.integers(5, 61)
        rmax = min(m, n)
        r = rng.integers(1, max(1, rmax // 2) + 1)
        sv = 10.0 ** (-6.0 * np.arange(r) / max(r, 2))
        w = matrix_with_spectrum(m, n, sv, rng)
        noise = rng.standard_normal((m, n))
        w = w + 1e-13 * noise / np.linalg.norm(noise)
        k, J, P = po.row_id(w, eps)
        assert skeleton_identity_exact(k, J, P) and k <= rmax
        assert spectral(w - P @ w[J[:k]]) <= 10 * eps * spectral(w)


def test_randomized_agrees(po):  # test_idlib.cpp:159-176
    rng = np.random.default_rng(99)
    w = matrix_with_spectrum(400, 60, 2.0 ** (-np.arange(60) / 2.0), rng)
    kd, _, _ = po.row_id(w, 1e-10)
    k, J, P = po.randomized_row_id(w, 1e-10, 1234)
    assert abs(kd - k) <= 1 and skeleton_identity_exact(k, J, P)
    assert spectral(w - P @ w[J[:k]]) <= 1e-9 * spectral(w)
    k2, J2, P2 = po.randomized_row_id(w, 1e-10, 1234)
    assert k2 == k and np.array_equal(J2, J) and np.array_equal(P2, P)


def test_rank_forced_extends_pivots(po):  # test_idlib.cpp:203-222
    rng = np.random.default_rng(31)
    w = matrix_with_spectrum(60, 40, 10.0 ** (-0.5 * np.arange(30)), rng)
    kb, Jb, Pb = po.row_id(w, 1e-6)
    kw, Jw, Pw = po.row_id(w, forced=kb + 5)
    assert kw == kb + 5 and np.array_equal(Jw[:kb], Jb[:kb])
    assert skeleton_identity_exact(kw, Jw, Pw)
    assert spectral(w - Pw @ w[Jw[:kw]]) <= spectral(w - Pb @ w[Jb[:kb]])
    low = w[:, :3] @ rng.uniform(-1, 1, (3, 25))
    kf, Jf, Pf = po.row_id(low, forced=10)
    assert kf <= 4
    assert spectral(low - Pf @ low[Jf[:kf]]) <= 1e-10 * spectral(low)


def test_cpqr_pivots_match_lapack(po):
    """Independent cross-check: oracle pivots == LAPACK dgeqp3 on W^T."""
    rng = np.random.default_rng(5)
    for trial in range(20):
        m, n = rng.integers(20, 120), rng.integers(20, 200)
        w = matrix_with_spectrum(m, n, 10.0 ** (-12 * np.arange(min(m, n)) / min(m, n)), rng)
        k, J, _ = po.row_id(w, 1e-10)
        _, r, piv = sla.qr(w.T, mode="economic", pivoting=True)
        kl = int(np.sum(np.abs(np.diag(r)) > 1e-10 * abs(r[0, 0])))
        assert abs(k - kl) <= 1
        assert np.array_equal(J[: k - 2], piv[: k - 2])


# ---------------------------------------------------------------- quadrature / geometry
def test_gauss_rule_exact(po):  # test_quadrature.cpp
    x, w = po.gauss_rule(16)
    for p in range(32):
        exact = 0.0 if p % 2 else 2.0 / (p + 1)
        assert abs(np.sum(w * x ** p) - exact) < 1e-14


def test_log_rule_exact_on_polynomials(po):  # logquad.hpp:16-21 contract
    x, _ = po.gauss_rule(16)
    for u in (0.3, -0.77, 1.6, -2.5):
        lw = po.log_rule_weights(16, u)
        t, tw = np.polynomial.legendre.leggauss(200)
        for p in range(10):
            exact = np.sum(tw * t ** p * np.log(np.abs(t - u))) if abs(u) > 1.0 else None
            if exact is not None:
                assert abs(np.sum(lw * x ** p) - exact) < 1e-12


def test_refine_keeps_nodes_and_coarsen_inverts(po):  # test_geometry.cpp:147-187
    g0 = po.Geom.create(po.STAR, 12, prongs=5, amplitude=0.3)
    g1, plan = g0.refine([5, 2, 5], 3)
    n0, n1, m = g0.nodes(), g1.nodes(), plan.maps()
    for key in ("x", "y", "nx", "ny", "w", "curvature", "param"):
        assert np.array_equal(n0[key][m["kept_old"]], n1[key][m["kept_new"]])
    assert plan.sizes() == (10 * 16, 2 * 16, 2 * 3 * 16)
    back = g1.coarsen(plan)
    nb = back.nodes()
    for key in ("x", "y", "w"):
        assert np.array_equal(nb[key], n0[key])


# ---------------------------------------------------------------- Nystrom (test_nystrom.cpp)
def test_submatrix_matches_dense_entries(po):  # test_nystrom.cpp:169-187
    g = po.Geom.create(po.STAR, 10, prongs=3, amplitude=0.35)
    a = po.Assembler.create(g)
    A = a.full_matrix()
    rng = np.random.default_rng(1)
    rows = rng.integers(0, A.shape[0], 37)
    cols = rng.integers(0, A.shape[0], 23)
    assert np.array_equal(a.submatrix(rows, cols), A[np.ix_(rows, cols)])


def test_interior_circle_field(po):  # test_nystrom.cpp:56-68
    g = po.Geom.create(po.CIRCLE, 20)
    a = po.Assembler.create(g)
    src = po.ring_sources(5, (0, 0), 3.0)
    tau = np.linalg.solve(a.full_matrix(), g.boundary_data(src))
    tg = np.array([[0.3, 0.1], [0.4, 0.2], [-0.3, 0.4], [0.2, -0.5]])
    u = g.evaluate_velocity(po.INTERIOR, tau, tg)
    ref = po.field_velocity(src, tg)
    assert np.max(np.linalg.norm(u - ref, axis=1) / np.linalg.norm(ref, axis=1)) < 1e-9


# ---------------------------------------------------------------- HBS (test_hbs.cpp)
@pytest.mark.parametrize("case", ["interior_circle", "exterior_star"])
def test_hbs_apply_matches_dense(po, case):  # test_hbs.cpp:60-90
    if case == "interior_circle":
        g = po.Geom.create(po.CIRCLE, 10, center=(0.1, -0.2), scale=1.3)
        a = po.Assembler.create(g, po.INTERIOR, 0.8)
    else:
        g = po.Geom.create(po.STAR, 10, prongs=5, amplitude=0.3)
        a = po.Assembler.create(g, po.EXTERIOR, 1.0)
    h = po.Hbs.compress(a, 1e-10)
    A = a.full_matrix()
    assert h.info()["n"] == A.shape[0]
    assert np.linalg.norm(h.apply(np.eye(A.shape[0])) - A) / np.linalg.norm(A) < 1e-9
    v = np.random.default_rng(11).standard_normal((A.shape[0], 3))
    assert np.linalg.norm(h.apply_t(v) - A.T @ v) < 1e-9 * np.linalg.norm(A) * np.linalg.norm(v)


def test_hbs_solve_and_round_trips(po):  # test_hbs.cpp:128-157
    g = po.Geom.create(po.CIRCLE, 20)
    a = po.Assembler.create(g)
    h = po.Hbs.compress(a, 1e-10).invert()
    A = a.full_matrix()
    rng = np.random.default_rng(3)
    b = rng.standard_normal(A.shape[0])
    assert np.linalg.norm(A @ h.solve(b) - b) < 1e-7 * np.linalg.norm(b)
    v = rng.standard_normal(A.shape[0])
    assert np.linalg.norm(h.solve(h.apply(v)) - v) < 1e-6 * np.linalg.norm(v)
    assert np.linalg.norm(h.apply(h.solve(v)) - v) < 1e-6 * np.linalg.norm(v)
    assert np.linalg.norm(A.T @ h.solve_t(b) - b) < 1e-7 * np.linalg.norm(b)
    assert np.linalg.norm(h.apply(np.zeros(A.shape[0]))) == 0.0


def test_hbs_manufactured_field(po):  # test_hbs.cpp:159-184
    g = po.Geom.create(po.CIRCLE, 20)
    a = po.Assembler.create(g)
    src = po.ring_sources(5, (0, 0), 3.0)
    h = po.Hbs.compress(a, 1e-10).invert()
    tau = h.solve(g.boundary_data(src))
    tg = np.array([[0.3, 0.1], [0.4, 0.2], [-0.3, 0.4], [0.2, -0.5], [-0.5, -0.1]])
    u = g.evaluate_velocity(po.INTERIOR, tau, tg)
    ref = po.field_velocity(src, tg)
    assert np.max(np.linalg.norm(u - ref, axis=1) / np.linalg.norm(ref, axis=1)) < 1e-8


def test_hbs_tighter_tolerance_more_skeleton(po):  # test_hbs.cpp:247-260
    g = po.Geom.create(po.STAR, 20, prongs=5, amplitude=0.3)
    a = po.Assembler.create(g)
    prev = 0
    for eps in (1e-3, 1e-6, 1e-10):
        t = po.Hbs.compress(a, eps).info()["total_skeleton"]
        assert t >= prev
        prev = t
    assert prev > 0


def test_hbs_never_draws_full_block(po):  # test_hbs.cpp:262-272
    g = po.Geom.create(po.CIRCLE, 40)
    a = po.Assembler.create(g)
    info = po.Hbs.compress(a, 1e-8).info()
    assert info["n"] == 1280 and 0 < info["max_block_drawn"] < 1280 * 1280 // 4


def test_hbs1_roundtrip_bitwise(po, tmp_path):  # test_hbs.cpp:274-305
    g = po.Geom.create(po.STAR, 10, prongs=3, amplitude=0.35)
    a = po.Assembler.create(g)
    h = po.Hbs.compress(a, 1e-8).invert()
    h.save(tmp_path / "h.bin")
    back = po.Hbs.load(tmp_path / "h.bin")
    assert back.info() == h.info()
    v = np.random.default_rng(31).standard_normal((h.info()["n"], 2))
    assert np.array_equal(back.apply(v), h.apply(v))
    assert np.array_equal(back.solve(v), h.solve(v))
    (tmp_path / "bad.bin").write_bytes(b"NOPE" + b"\0" * 64)
    with pytest.raises(po.OracleError):
        po.Hbs.load(tmp_path / "bad.bin")


def test_hbs_deterministic(po):  # test_hbs.cpp:307-322
    g = po.Geom.create(po.STAR, 12, prongs=5, amplitude=0.3)
    a = po.Assembler.create(g)
    assert np.array_equal(po.Hbs.compress(a, 1e-8).node_ranks(), po.Hbs.compress(a, 1e-8).node_ranks())


# ---------------------------------------------------------------- low rank / ELS
def _refined(po, kind, n_panels, panels, m, eps=1e-10):
    g0 = po.Geom.create(po.STAR, n_panels, prongs=5, amplitude=0.3)
    g1, plan = g0.refine(panels, m)
    a0, a1 = po.Assembler.create(g0, kind), po.Assembler.create(g1, kind)
    return g0, g1, plan, a0, a1


def test_update_matches_dense(po):  # test_lowrank.cpp:64-98
    g0, g1, plan, a0, a1 = _refined(po, po.INTERIOR, 10, [2, 3], 2)
    eps = 1e-10
    nk, nc, npp = plan.sizes()
    n = 2 * (nk + nc + npp)
    Q = np.zeros((n, n))
    Q[: 2 * nk, 2 * nk: 2 * nk + 2 * nc] = -po.block_eval_full(a0, a1, plan, "kc")
    Q[: 2 * nk, 2 * nk + 2 * nc:] = po.block_eval_full(a0, a1, plan, "kp")
    Q[2 * nk + 2 * nc:, : 2 * nk] = po.block_eval_full(a0, a1, plan, "pk")
    u = po.Update.compress(a0, a1, plan, eps)
    f = u.factors()
    info = u.info()
    assert info["n_ext"] == n and 1 <= info["k"] <= info["k1"]
    nq = spectral(Q)
    assert spectral(Q - f["L1"] @ f["R1"]) <= 10 * eps * nq
    assert spectral(Q - f["L"] @ f["R"]) <= 10 * eps * nq
    sk = f["skeleton"]
    assert np.array_equal(f["L"][sk], np.eye(info["k"]))


def test_els_matches_dense_refined_solve(po):  # test_els.cpp:125-144
    eps = 1e-10
    g0, g1, plan, a0, a1 = _refined(po, po.INTERIOR, 10, [3], 4)
    h = po.Hbs.compress(a0, eps).invert()
    u = po.Update.compress(a0, a1, plan, eps)
    e = po.Els.build(h, a0, a1, plan, u)
    g_new = g1.boundary_data(po.ring_sources(4, (0, 0), 3.0))
    maps = plan.maps()
    tau = e.solve(po.gather_kept_added(maps, g_new))
    Ann = a1.full_matrix()
    ref = po.gather_kept_added(maps, np.linalg.solve(Ann, g_new))
    err = np.linalg.norm(tau - ref) / np.linalg.norm(ref)
    assert err <= 10 * eps * np.linalg.cond(Ann) and err <= 1e-8


def test_els_dummy_block_annihilates_cut_rows(po):  # test_els.cpp:146-166
    eps = 1e-10
    g0, g1, plan, a0, a1 = _refined(po, po.INTERIOR, 12, [5], 3)
    h = po.Hbs.compress(a0, eps).invert()
    e = po.Els.build(h, a0, a1, plan, po.Update.compress(a0, a1, plan, eps))
    i = e.info()
    g = po.gather_kept_added(plan.maps(), g1.boundary_data(po.ring_sources(3, (0, 0), 3.0)))
    g_ext = np.zeros(i["n_k"] + i["n_c"] + i["n_p"])
    g_ext[: i["n_k"]] = g[: i["n_k"]]
    g_ext[i["n_k"] + i["n_c"]:] = g[i["n_k"]:]
    ext = e.solve_raw(g_ext)
    tk, tc = ext[: i["n_k"]], ext[i["n_k"]: i["n_k"] + i["n_c"]]
    ack = po.block_eval_full(a0, a1, plan, "ck")
    acc = po.block_eval_full(a0, a1, plan, "cc")
    assert np.linalg.norm(ack @ tk + acc @ tc) <= 10 * eps * np.linalg.norm(ack @ tk)


def test_els_forward_apply_matches_dense(po):  # test_els.cpp:206-231
    eps = 1e-10
    g0, g1, plan, a0, a1 = _refined(po, po.EXTERIOR, 10, [2, 3], 3)
    h = po.Hbs.compress(a0, eps).invert()
    e = po.Els.build(h, a0, a1, plan, po.Update.compress(a0, a1, plan, eps))
    nk, nc, npp = plan.sizes()
    nk2, nc2, np2 = 2 * nk, 2 * nc, 2 * npp
    n = nk2 + nc2 + np2
    A = np.zeros((n, n))
    A[:nk2, :nk2] = po.block_eval_full(a0, a1, plan, "kk")
    A[nk2:nk2 + nc2, :nk2] = po.block_eval_full(a0, a1, plan, "ck")
    A[nk2:nk2 + nc2, nk2:nk2 + nc2] = po.block_eval_full(a0, a1, plan, "cc")
    A[:nk2, nk2 + nc2:] = po.block_eval_full(a0, a1, plan, "kp")
    A[nk2 + nc2:, :nk2] = po.block_eval_full(a0, a1, plan, "pk")
    A[nk2 + nc2:, nk2 + nc2:] = po.block_eval_full(a0, a1, plan, "pp")
    v = np.random.default_rng(7).standard_normal(n)
    assert np.linalg.norm(e.apply_forward(v) - A @ v) <= 10 * eps * np.linalg.norm(A, 2) * np.linalg.norm(v)


def _holes(po):
    """test_els.cpp:53-90 (make_holes): circle wall r=2, 20 panels, three holes."""
    g0 = po.Geom.create(po.CIRCLE, 20, scale=2.0)
    g1, plan = g0.add_holes([(-0.8, 0.0, 0.3, 10, 16), (0.9, 0.3, 0.25, 10, 16), (0.1, -0.9, 0.2, 10, 16)])
    return g0, g1, plan, po.Assembler.create(g0, po.MIXED), po.Assembler.create(g1, po.MIXED)


HOLE_SOURCES = [(-0.8, 0.0, 1.0, 0.5), (0.9, 0.3, -0.5, 1.0), (0.1, -0.9, 0.3, -1.0)]
HOLE_TARGETS = [(0.0, 1.2), (1.4, 0.3), (-1.3, -0.4)]


def density_on_refined(plan_maps, n_new, tau):
    """els.cpp:195-203: (kept, added) density scattered to the refined mesh."""
    out = np.zeros(2 * n_new)
    kn, an = plan_maps["kept_new"], plan_maps["added_new"]
    ks = np.stack([2 * kn, 2 * kn + 1], 1).ravel()
    as_ = np.stack([2 * an, 2 * an + 1], 1).ravel()
    out[ks] = tau[: len(ks)]
    out[as_] = tau[len(ks):]
    return out


def test_els_holes_match_dense_mixed_oracle(po):  # test_els.cpp:168-197
    eps = 1e-10
    g0, g1, plan, a0, a1 = _holes(po)
    assert plan.sizes()[1] == 0
    h = po.Hbs.compress(a0, eps).invert()
    e = po.Els.build(h, a0, a1, plan, po.Update.compress(a0, a1, plan, eps))
    srcs = list(po.ring_sources(4, (0, 0), 3.5)) + HOLE_SOURCES
    g_new = g1.boundary_data(srcs)
    maps = plan.maps()
    tau = e.solve(po.gather_kept_added(maps, g_new))
    ref = po.gather_kept_added(maps, np.linalg.solve(a1.full_matrix(), g_new))
    assert np.linalg.norm(tau - ref) / np.linalg.norm(ref) <= 1e-8
    vel = g1.evaluate_velocity(po.MIXED, density_on_refined(maps, g1.n_nodes, tau), HOLE_TARGETS)
    exact = po.field_velocity(srcs, HOLE_TARGETS)
    assert max(np.linalg.norm(vel[i] - exact[i]) / np.linalg.norm(exact[i]) for i in range(3)) < 1e-8


def _channel_geom(po, n_panels):
    import paper_2108_07205_b200 as sb  # host-only helper: the cap polynomials (numpy)
    cv = sb.channel()
    return cv, po.Geom.create(po.CHANNEL, n_panels, center=cv.center, scale=cv.scale, prongs=cv.n_prongs,
                              amplitude=cv.amplitude, aspect=cv.aspect, cos_coef=cv.cos_coef,
                              sin_coef=cv.sin_coef)


def test_channel_curve_geometry(po):
    """BASELINE configs[3]'s closed wavy channel (SBX_CHANNEL): wall nodes lie on
    y = -/+(1 + 0.2 sin(2 pi x / 4)), the caps stay outside x in [0, 8], the
    four joins sit on panel ends, and tangent, curvature and its derivative
    are continuous across them."""
    cv, o = _channel_geom(po, 256)
    nd = o.nodes()
    x, y, kap, pan = nd["x"], nd["y"], nd["curvature"], nd["panel_of"]
    # panel ranges of the four pieces (fractions 45/128, 21/128, 45/128, 17/128)
    n = 256
    b0, b1, b2 = 45 * n // 128, (45 + 21) * n // 128, (90 + 21) * n // 128
    wall = (pan < b0) | ((pan >= b1) & (pan < b2))
    assert np.max(np.abs(np.abs(y[wall]) - (1 + 0.2 * np.sin(np.pi * x[wall] / 2)))) < 1e-14
    assert np.all((x[wall] > 0) & (x[wall] < 8))
    caps = ~wall
    assert np.all((x[caps] < 1e-12) | (x[caps] > 8 - 1e-12))
    # curvature is smooth across each join: the nodes either side extrapolate to the same value
    for bj in (b0, b1, b2, n):
        left = kap[pan == (bj - 1) % n][-3:]
        right = kap[pan == bj % n][:3]
        jump = abs((2 * left[-1] - left[-2]) - (2 * right[0] - right[1]))
        assert jump < 5e-3 * (1 + abs(left[-1])), (bj, left, right)


def test_channel_hbs_manufactured_field(po):  # test_hbs.cpp:159-184 on the channel
    _, o = _channel_geom(po, 256)
    a = po.Assembler.create(o)
    h = po.Hbs.compress(a, 1e-10).invert()
    src = np.array([[x, yy, f1, f2] for (x, yy), (f1, f2) in
                    zip([(1.0, -2.6), (3.0, 2.6), (5.0, -2.6), (7.0, 2.6), (-2.5, 0.3), (10.5, -0.4)],
                        [(1.0, 0.5), (-0.3, 1.2), (0.7, -0.8), (-1.1, 0.2), (0.4, 0.9), (0.6, -0.5)])])
    tau = h.solve(o.boundary_data(src))
    tg = np.array([(x, yy) for x in (1.5, 3.5, 6.5) for yy in (-0.5, 0.0, 0.5)] + [(-0.4, 0.0), (8.5, 0.1)])
    u = o.evaluate_velocity(po.INTERIOR, tau, tg)
    ref = po.field_velocity(src, tg)
    assert np.max(np.linalg.norm(u - ref, axis=1) / np.linalg.norm(ref, axis=1)) < 1e-9
