"""§8(f) next row 1: els_apply_forward and GMRES / PGMRES-Local on the device
(els.cpp:181-186, gmres.cpp:14-126, scenario.cpp:694-727)."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def setup():
    import paper_2108_07205_b200 as sb
    sb.init(0)
    eps = 1e-10
    g0 = sb.panelize(sb.star(5, 0.3), 10, 16)
    h = sb.hbs_invert(sb.hbs_compress(g0))
    g1, plan = sb.refine(g0, [3], 4)
    u = sb.compress_update(g0, g1, plan, eps)
    e = sb.els_build(h, g0, g1, plan, u)
    return sb, g0, g1, plan, e


def test_apply_forward_matches_dense_extended(setup, po):  # test_els.cpp:206-231
    sb, g0, g1, plan, e = setup
    o0 = po.Geom.create(po.STAR, 10, prongs=5, amplitude=0.3)
    o1, op = o0.refine([3], 4)
    a0, a1 = po.Assembler.create(o0), po.Assembler.create(o1)
    nk, nc, npp = (2 * x for x in plan.sizes())
    n = nk + nc + npp
    A = np.zeros((n, n))
    A[:nk, :nk] = po.block_eval_full(a0, a1, op, "kk")
    A[nk:nk + nc, :nk] = po.block_eval_full(a0, a1, op, "ck")
    A[nk:nk + nc, nk:nk + nc] = po.block_eval_full(a0, a1, op, "cc")
    A[:nk, nk + nc:] = po.block_eval_full(a0, a1, op, "kp")
    A[nk + nc:, :nk] = po.block_eval_full(a0, a1, op, "pk")
    A[nk + nc:, nk + nc:] = po.block_eval_full(a0, a1, op, "pp")
    v = np.random.default_rng(7).standard_normal((n, 2))
    out = sb.els_apply_forward(e, v)
    assert np.linalg.norm(out - A @ v) <= 10 * 1e-10 * np.linalg.norm(A, 2) * np.linalg.norm(v)


def test_pgmres_local_converges_fast_to_the_direct_solution(setup, po):
    sb, g0, g1, plan, e = setup
    src = po.ring_sources(4, (0, 0), 3.0)
    g = sb.gather_kept_added(plan, sb.boundary_data(g1, src))
    direct = sb.els_solve(e, g)
    tau, it, hist = sb.els_gmres(e, g, precond=True, tol=1e-11)
    assert it <= 6 and hist[-1] <= 1e-11
    assert np.linalg.norm(tau - direct) <= 1e-9 * np.linalg.norm(direct)
    plain, it2, hist2 = sb.els_gmres(e, g, precond=False, tol=1e-11, max_iter=600)
    assert it2 > it
    assert np.linalg.norm(plain - direct) <= 1e-8 * np.linalg.norm(direct)


def test_gmres_budget_is_reported(setup, po):
    sb, g0, g1, plan, e = setup
    g = sb.gather_kept_added(plan, sb.boundary_data(g1, po.ring_sources(4, (0, 0), 3.0)))
    with pytest.raises(sb.ConvergenceError, match="iteration budget"):
        sb.els_gmres(e, g, precond=False, tol=1e-13, max_iter=3)
