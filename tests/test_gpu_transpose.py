"""Transposed device sweeps and ELS operators against the reference's own
assertions: hbs_apply_t vs the dense transpose and the adjoint identity
(test_hbs.cpp:60-90), hbs_solve_t inverting the transposed operator
(test_hbs.cpp:148-150), and the adjoint identities of els_solve_raw_t /
els_apply_forward_t (els.cpp:154-163, :188-193) for both A_pp branches."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def sb():
    import paper_2108_07205_b200 as sb
    sb.init(0)
    return sb


def rng_mat(n, k, seed):
    return np.random.default_rng(seed).standard_normal((n, k))


@pytest.mark.parametrize("case", ["interior", "exterior"])
def test_apply_t_matches_dense_transpose(sb, po, case):  # test_hbs.cpp:60-90
    eps = 1e-10
    if case == "interior":
        g = sb.panelize(sb.circle(1.3, (0.1, -0.2)), 10, 16)
        h = sb.hbs_compress(g, sb.INTERIOR_DIRICHLET, sb.HbsOptions(eps=eps), mu=0.8)
        o = po.Geom.create(po.CIRCLE, 10, center=(0.1, -0.2), scale=1.3)
        A = po.Assembler.create(o, po.INTERIOR, 0.8).full_matrix()
    else:
        g = sb.panelize(sb.star(5, 0.3), 10, 16)
        h = sb.hbs_compress(g, sb.EXTERIOR_COMBINED, sb.HbsOptions(eps=eps))
        o = po.Geom.create(po.STAR, 10, prongs=5, amplitude=0.3)
        A = po.Assembler.create(o, po.EXTERIOR).full_matrix()
    n = A.shape[0]
    v = rng_mat(n, 3, 11)
    At_v = sb.hbs_apply(h, v, transpose=True)
    assert np.linalg.norm(At_v - A.T @ v) < 10 * eps * np.linalg.norm(A) * np.linalg.norm(v)
    x = rng_mat(n, 1, 5)[:, 0]
    y = rng_mat(n, 1, 7)[:, 0]
    lhs = y @ sb.hbs_apply(h, x)
    rhs = x @ sb.hbs_apply(h, y, transpose=True)
    assert abs(lhs - rhs) < 1e-11 * np.linalg.norm(x) * np.linalg.norm(y) * np.linalg.norm(A)


def test_solve_t_inverts_transposed_operator(sb, po):  # test_hbs.cpp:148-150
    g = sb.panelize(sb.circle(), 20, 16)
    h = sb.hbs_invert(sb.hbs_compress(g))
    A = po.Assembler.create(po.Geom.create(po.CIRCLE, 20)).full_matrix()
    b = rng_mat(A.shape[0], 1, 3)[:, 0]
    xt = sb.hbs_solve(h, b, transpose=True)
    assert np.linalg.norm(A.T @ xt - b) < 1e-7 * np.linalg.norm(b)
    # multi-RHS (FP64 tensor-core path) and the forward solve untouched
    B = rng_mat(A.shape[0], 40, 4)
    Xt = sb.hbs_solve(h, B, transpose=True)
    assert np.linalg.norm(A.T @ Xt - B) < 1e-7 * np.linalg.norm(B)
    x = sb.hbs_solve(h, b)
    assert np.linalg.norm(A @ x - b) < 1e-7 * np.linalg.norm(b)
    # adjoint identity of the inverse sweeps
    y = rng_mat(A.shape[0], 1, 8)[:, 0]
    assert abs(y @ x - b @ sb.hbs_solve(h, y, transpose=True)) < 1e-11 * np.linalg.norm(b) * np.linalg.norm(y) * \
        np.linalg.norm(np.linalg.inv(A))


@pytest.mark.parametrize("m", [4, 80])  # dense A_pp inverse / A_pp's own HBS (2N_p > 2048)
def test_els_transposes_are_adjoints(sb, m):  # els.cpp:154-163, :188-193
    eps = 1e-10
    g0 = sb.panelize(sb.star(5, 0.3), 10, 16)
    h = sb.hbs_invert(sb.hbs_compress(g0))
    g1, plan = sb.refine(g0, [3], m)
    u = sb.compress_update(g0, g1, plan, eps)
    e = sb.els_build(h, g0, g1, plan, u)
    assert bool(e.info()["app_hbs"]) == (m == 80)
    n = e.n_ext()
    x = rng_mat(n, 2, 1)
    y = rng_mat(n, 2, 2)
    fx = sb.els_apply_forward(e, x)
    fty = sb.els_apply_forward(e, y, transpose=True)
    scale = np.linalg.norm(x) * np.linalg.norm(y) * max(np.linalg.norm(fx), 1.0)
    assert abs(np.sum(y * fx) - np.sum(fty * x)) < 1e-11 * scale
    sx = sb.els_solve_raw(e, x)
    sty = sb.els_solve_raw(e, y, transpose=True)
    scale = np.linalg.norm(x) * np.linalg.norm(y) * max(np.linalg.norm(sx) / np.linalg.norm(x), 1.0)
    assert abs(np.sum(y * sx) - np.sum(sty * x)) < 1e-10 * scale
    # the transposed solve inverts the transposed forward operator (to the
    # compression tolerance, like the forward round trip)
    r = sb.els_apply_forward(e, sty, transpose=True)
    assert np.linalg.norm(r - y) < 1e-6 * np.linalg.norm(y)
