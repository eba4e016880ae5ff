"""Diagnostic modes of the reference on the device:
svd_optimal update compression (lowrank.cpp:329-362; test_lowrank.cpp:64-131)
and the dense-oracle route of conditioning_report (els.cpp:225-270;
test_els.cpp:268-291), both through the device Jacobi SVD (svd.cu), against
the oracle's numpy restatement (pyoracle.svd_optimal) and dense numpy
condition numbers."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def sb():
    import paper_2108_07205_b200 as sb
    sb.init(0)
    return sb


def _dense_q(po, o0, o1, op):
    a0, a1 = po.Assembler.create(o0), po.Assembler.create(o1)
    nk, nc, npp = op.sizes()
    n = 2 * (nk + nc + npp)
    Q = np.zeros((n, n))
    Q[: 2 * nk, 2 * nk: 2 * nk + 2 * nc] = -po.block_eval_full(a0, a1, op, "kc")
    Q[: 2 * nk, 2 * nk + 2 * nc:] = po.block_eval_full(a0, a1, op, "kp")
    Q[2 * nk + 2 * nc:, : 2 * nk] = po.block_eval_full(a0, a1, op, "pk")
    return Q, a0, a1


@pytest.mark.parametrize("panels,m", [([3], 4), ([2, 7], 2)])
def test_svd_optimal_update(sb, po, panels, m):  # test_lowrank.cpp:64-96
    eps = 1e-10
    g0 = sb.panelize(sb.star(5, 0.3), 10, 16)
    g1, plan = sb.refine(g0, panels, m)
    v = sb.compress_update(g0, g1, plan, eps, mode=sb.SVD_OPTIMAL)
    u = sb.compress_update(g0, g1, plan, eps)
    o0 = po.Geom.create(po.STAR, 10, prongs=5, amplitude=0.3)
    o1, op = o0.refine(panels, m)
    Q, a0, a1 = _dense_q(po, o0, o1, op)
    L, R = v.factors()
    nq = np.linalg.norm(Q, 2)
    assert np.linalg.norm(Q - L @ R, 2) <= 10 * eps * nq
    vi = v.info()
    assert vi["k"] <= vi["k1"]
    assert vi["k"] <= u.k  # the diagnostic mode is at least as tight as the two-step path
    ref = po.svd_optimal(a0, a1, op, eps)
    for key in ("kc", "kp", "pk", "k1", "k"):
        assert abs(vi[key] - ref[key]) <= 1, (key, vi[key], ref[key])
    assert np.linalg.norm(L @ R - ref["L"] @ ref["R"]) <= 1e-9 * np.linalg.norm(Q)
    # the left factor has orthonormal columns (U of the final SVD)
    assert np.linalg.norm(L.T @ L - np.eye(vi["k"])) <= 1e-12 * vi["k"]
    # and the ELS built on it solves the refined system
    h = sb.hbs_invert(sb.hbs_compress(g0))
    e = sb.els_build(h, g0, g1, plan, v)
    src = po.ring_sources(4, (0, 0), 3.0)
    tau = sb.els_solve(e, sb.gather_kept_added(plan, sb.boundary_data(g1, src)))
    A = a1.full_matrix()
    dense = po.gather_kept_added(op.maps(), np.linalg.solve(A, o1.boundary_data(src)))
    assert np.linalg.norm(tau - dense) <= 1e-8 * np.linalg.norm(dense)


def test_conditioning_dense_route(sb, po):  # test_els.cpp:268-291
    eps = 1e-10
    g0 = sb.panelize(sb.star(5, 0.3), 10, 16)
    h = sb.hbs_invert(sb.hbs_compress(g0))
    g1, plan = sb.refine(g0, [3], 4)
    u = sb.compress_update(g0, g1, plan, eps)
    e = sb.els_build(h, g0, g1, plan, u)
    rep = sb.els_conditioning(e, dense=True)
    assert rep["kappa_w"] >= 1.0
    assert rep["bound_holds"] and rep["kappa_w"] <= rep["bound"]
    assert rep["kappa_ext"] > 1.0 and rep["kappa_tilde"] > 1.0
    # dense numpy oracles of the same matrices
    o0 = po.Geom.create(po.STAR, 10, prongs=5, amplitude=0.3)
    o1, op = o0.refine([3], 4)
    a0, a1 = po.Assembler.create(o0), po.Assembler.create(o1)
    mp = op.maps()
    sc = lambda v: np.stack([2 * v, 2 * v + 1], 1).reshape(-1)  # noqa: E731
    oc = np.concatenate([sc(mp["kept_old"]), sc(mp["cut_old"])])
    ad = sc(mp["added_new"])
    n = len(oc) + len(ad)
    At = np.zeros((n, n))
    At[: len(oc), : len(oc)] = a0.submatrix(oc, oc)
    At[len(oc):, len(oc):] = a1.submatrix(ad, ad)
    L, R = u.factors()
    kt = np.linalg.cond(At)
    kx = np.linalg.cond(At + L @ R)
    assert rep["kappa_tilde"] == pytest.approx(kt, rel=1e-6)
    assert rep["kappa_ext"] == pytest.approx(kx, rel=0.05)
    X, W = e.xw()
    sw = np.linalg.svd(W, compute_uv=False)
    assert rep["kappa_w"] == pytest.approx(sw[0] / sw[-1], rel=1e-8)
    for got, f in ((rep["kappa_l"], L), (rep["kappa_r"], R)):  # factor_cond (els.cpp:216-222)
        sv = np.linalg.svd(f, compute_uv=False)
        ref = sv[0] / sv[u.k - 1]
        # numerically singular factors only agree on "huge"
        assert (got > 1e12) if ref > 1e12 else got == pytest.approx(ref, rel=1e-6)
    # the estimator route lands near the dense numbers
    est = sb.els_conditioning(e)
    assert 0.3 * rep["kappa_ext"] <= est["kappa_ext"] <= 3.0 * rep["kappa_ext"]
    assert 0.3 * rep["kappa_tilde"] <= est["kappa_tilde"] <= 3.0 * rep["kappa_tilde"]
