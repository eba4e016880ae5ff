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


def test_transposed_sweeps_match_oracle_bitwise_factors(sb, po, tmp_path):
    """Tier 1: the oracle's factors loaded through HBS1; the device
    transposed sweeps against the oracle's hbs_solve_t / hbs_apply_t."""
    o = po.Geom.create(po.STAR, 12, prongs=3, amplitude=0.35)
    h = po.Hbs.compress(po.Assembler.create(o), 1e-10).invert()
    h.save(tmp_path / "t.hbs1")
    d = sb.hbs_load(tmp_path / "t.hbs1")
    b = rng_mat(d.n, 3, 6)
    rel = lambda x, y: np.linalg.norm(x - y) / np.linalg.norm(y)
    assert rel(sb.hbs_solve(d, b, transpose=True), h.solve_t(b)) < 1e-12
    assert rel(sb.hbs_apply(d, b, transpose=True), h.apply_t(b)) < 1e-12


def scalars(nodes):
    return np.stack([2 * np.asarray(nodes), 2 * np.asarray(nodes) + 1], 1).reshape(-1)


def test_conditioning_report(sb, po):  # test_els.cpp:268-291
    eps = 1e-10
    g0 = sb.panelize(sb.star(5, 0.3), 10, 16)
    h = sb.hbs_invert(sb.hbs_compress(g0))
    g1, plan = sb.refine(g0, [3], 4)
    u = sb.compress_update(g0, g1, plan, eps)
    e = sb.els_build(h, g0, g1, plan, u)
    rep = sb.els_conditioning(e)
    assert rep["kappa_w"] >= 1.0 and rep["bound_holds"] and rep["kappa_w"] <= rep["bound"]
    assert rep["kappa_ext"] > 1.0 and rep["kappa_tilde"] > 1.0
    # dense numbers (numpy SVD) of the same operators
    o0 = po.Geom.create(po.STAR, 10, prongs=5, amplitude=0.3)
    o1, op = o0.refine([3], 4)
    a0, a1 = po.Assembler.create(o0), po.Assembler.create(o1)
    m = op.maps()
    oc = np.concatenate([scalars(m["kept_old"]), scalars(m["cut_old"])])
    ad = scalars(m["added_new"])
    n = len(oc) + len(ad)
    At = np.zeros((n, n))
    At[: len(oc), : len(oc)] = a0.submatrix(oc, oc)
    At[len(oc):, len(oc):] = a1.submatrix(ad, ad)
    L, R = u.factors()
    cond = lambda a: (lambda s: s[0] / s[-1])(np.linalg.svd(a, compute_uv=False))
    k = L.shape[1]

    def factor_close(got, f):  # factor_cond (els.cpp:216-222); numerically singular factors only agree on "huge"
        s = np.linalg.svd(f, compute_uv=False)
        ref = s[0] / s[k - 1]
        return (got > 1e12 and ref > 1e12) if ref > 1e12 else abs(got / ref - 1) < 1e-6

    assert factor_close(rep["kappa_l"], L)
    assert factor_close(rep["kappa_r"], R)
    X, W = e.xw()
    assert abs(rep["kappa_w"] / cond(W) - 1) < 1e-6
    # the estimator route lands near the dense numbers (the reference's 0.3x .. 3x)
    ke, kt = cond(At + L @ R), cond(At)
    assert 0.3 * ke <= rep["kappa_ext"] <= 3.0 * ke
    assert 0.3 * kt <= rep["kappa_tilde"] <= 3.0 * kt


@pytest.mark.parametrize("nrhs", [1, 7, 32, 256])
def test_row_major_layout_bitwise(sb, nrhs):
    """SBX_ROW_MAJOR (row-major device blocks, the sweep workspace's own
    layout) gives the same bits as the column-major host path, for solves
    and applies, plain and transposed, dense and strided rows."""
    import torch
    g = sb.panelize(sb.star(5, 0.3), 64, 16)
    h = sb.hbs_invert(sb.hbs_compress(g, opts=sb.HbsOptions(eps=1e-10)))
    n = h.n
    B = rng_mat(n, nrhs, 21)
    wide = torch.zeros((n, nrhs + 3), dtype=torch.float64, device="cuda")
    wide[:, :nrhs] = torch.from_numpy(B)
    for fn in (sb.hbs_solve, sb.hbs_apply):
        for tr in (False, True):
            want = fn(h, B, transpose=tr)
            dense = fn(h, torch.from_numpy(B).cuda(), transpose=tr)          # ld == nrhs
            strided = fn(h, wide[:, :nrhs], transpose=tr)                     # ld = nrhs + 3
            colmajor = fn(h, torch.from_numpy(np.asfortranarray(B)).cuda().t().contiguous().t(), transpose=tr)
            for got in (dense, strided, colmajor):
                assert np.array_equal(got.cpu().numpy(), want), (fn.__name__, tr)
            if nrhs == 1:
                vec = fn(h, torch.from_numpy(B[:, 0]).cuda(), transpose=tr)
                assert np.array_equal(vec.cpu().numpy(), want[:, 0])
