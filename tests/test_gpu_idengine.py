"""Device ID engine (dense.cu qr_kernel / cpqr_coop_kernel + interp) against
the oracle's restatement of idlib.cpp and the reference's own ID assertions
(test_idlib.cpp)."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def sb():
    import paper_2108_07205_b200 as sb
    sb.init(0)
    return sb


def spectrum_matrix(m, n, sv, rng):
    u = np.linalg.qr(rng.standard_normal((m, len(sv))))[0]
    v = np.linalg.qr(rng.standard_normal((n, len(sv))))[0]
    return (u * sv) @ v.T


def skeleton_identity_exact(k, J, P):
    return all(P[J[i], j] == (1.0 if i == j else 0.0) for i in range(k) for j in range(k))


SHAPES = [(50, 30), (200, 100), (128, 700), (300, 5000), (2500, 300)]


@pytest.mark.parametrize("engine", [1, 2, 3])
@pytest.mark.parametrize("shape", SHAPES)
def test_row_id_matches_oracle(sb, po, engine, shape):
    m, n = shape
    rng = np.random.default_rng(m * 7 + n)
    r = min(m, n)
    w = spectrum_matrix(m, n, 10.0 ** (-14 * np.arange(r) / r), rng)
    k, J, P = sb.row_id(w, 1e-10, engine=engine)
    ko, Jo, Po = po.row_id(w, 1e-10)
    assert abs(k - ko) <= 1
    kk = min(k, ko) - 2
    assert np.array_equal(J[:kk], Jo[:kk])
    assert skeleton_identity_exact(k, J, P)
    assert np.linalg.norm(w - P @ w[J[:k]], 2) <= 10 * 1e-10 * np.linalg.norm(w, 2)


@pytest.mark.parametrize("engine", [1, 2, 3])
def test_row_id_forced_rank(sb, po, engine):  # test_idlib.cpp:203-222
    rng = np.random.default_rng(31)
    w = spectrum_matrix(60, 40, 10.0 ** (-0.5 * np.arange(30)), rng)
    kb, Jb, Pb = sb.row_id(w, 1e-6, engine=engine)
    kw, Jw, Pw = sb.row_id(w, forced=kb + 5, engine=engine)
    assert kw == kb + 5 and np.array_equal(Jw[:kb], Jb[:kb])
    low = w[:, :3] @ rng.uniform(-1, 1, (3, 25))
    kf, Jf, Pf = sb.row_id(low, forced=10, engine=engine)
    assert kf <= 4


@pytest.mark.parametrize("engine", [1, 2, 3])
def test_row_id_deterministic(sb, engine):
    rng = np.random.default_rng(9)
    w = spectrum_matrix(1200, 512, 10.0 ** (-12 * np.arange(512) / 512), rng)
    first = sb.row_id(w, 1e-10, engine=engine)
    for _ in range(4):
        again = sb.row_id(w, 1e-10, engine=engine)
        assert again[0] == first[0]
        assert np.array_equal(again[1], first[1]) and np.array_equal(again[2], first[2])


def test_row_id_edge_cases(sb):  # test_idlib.cpp:63-113
    k, J, P = sb.row_id(np.eye(20), 1e-10)
    assert k == 20 and skeleton_identity_exact(k, J, P)
    k, J, P = sb.row_id(np.zeros((8, 5)), 1e-10)
    assert k == 0
    rng = np.random.default_rng(7)
    w = np.outer(rng.standard_normal(50), rng.standard_normal(30))
    k, J, P = sb.row_id(w, 1e-10)
    assert k == 1 and skeleton_identity_exact(k, J, P)
    with pytest.raises(ValueError):
        sb.row_id(np.eye(4), 0.5)


@pytest.mark.parametrize("engine", [0, 2])
def test_row_id_very_tall_functionals(sb, po, engine):
    # W^T with 20000 functionals: the Householder vector no longer fits shared
    # memory, the cooperative engine keeps it in L2
    rng = np.random.default_rng(11)
    w = spectrum_matrix(180, 20000, 10.0 ** (-14 * np.arange(180) / 180), rng)
    k, J, P = sb.row_id(w, 1e-10, engine=engine)
    ko, Jo, Po = po.row_id(w, 1e-10)
    assert abs(k - ko) <= 1
    kk = min(k, ko) - 2
    assert np.array_equal(J[:kk], Jo[:kk])
    assert np.linalg.norm(w - P @ w[J[:k]], 2) <= 10 * 1e-10 * np.linalg.norm(w, 2)


@pytest.mark.parametrize("shape", [(50, 30), (200, 100), (128, 700), (256, 513), (40, 3000), (900, 128)])
def test_row_id_cluster_engine(sb, po, shape):
    m, n = shape
    rng = np.random.default_rng(m + 3 * n)
    r = min(m, n)
    w = spectrum_matrix(m, n, 10.0 ** (-14 * np.arange(r) / r), rng)
    k, J, P = sb.row_id(w, 1e-10, engine=4)
    ko, Jo, Po = po.row_id(w, 1e-10)
    assert abs(k - ko) <= 1
    kk = min(k, ko) - 2
    assert np.array_equal(J[:kk], Jo[:kk])
    assert skeleton_identity_exact(k, J, P)
    assert np.linalg.norm(w - P @ w[J[:k]], 2) <= 10 * 1e-10 * np.linalg.norm(w, 2)
    kw, Jw, Pw = sb.row_id(w, forced=k + 3, engine=4)
    assert np.array_equal(Jw[:k], J[:k])


@pytest.mark.parametrize("shape", [(50, 30), (200, 100), (128, 700), (256, 513), (900, 128), (256, 257),
                                   (256, 1088), (4, 9)])
def test_row_id_register_engine(sb, po, shape):
    """Register-resident cluster CPQR (engine 5): same pivots as the oracle,
    forced-rank extension keeps the eps skeleton (test_idlib.cpp:203-222)."""
    m, n = shape
    rng = np.random.default_rng(m + 5 * n)
    r = min(m, n)
    w = spectrum_matrix(m, n, 10.0 ** (-14 * np.arange(r) / r), rng)
    k, J, P = sb.row_id(w, 1e-10, engine=5)
    ko, Jo, Po = po.row_id(w, 1e-10)
    assert abs(k - ko) <= 1
    kk = min(k, ko) - 2
    assert np.array_equal(J[:kk], Jo[:kk])
    assert skeleton_identity_exact(k, J, P)
    assert np.linalg.norm(w - P @ w[J[:k]], 2) <= 10 * 1e-10 * np.linalg.norm(w, 2)
    if k + 3 <= r:
        kw, Jw, Pw = sb.row_id(w, forced=k + 3, engine=5)
        assert kw == k + 3 and np.array_equal(Jw[:k], J[:k])


@pytest.mark.parametrize("shape", [(50, 30), (200, 100), (128, 700), (256, 513), (900, 128), (256, 257),
                                   (256, 1088), (4, 9), (2000, 300)])
def test_row_id_streaming_engine(sb, po, shape):
    """Streaming one-CTA CPQR (engine 6; slab partly in shared memory, the
    rest updated in place in L2): oracle pivots and forced-rank extension."""
    m, n = shape
    rng = np.random.default_rng(m + 7 * n)
    r = min(m, n)
    w = spectrum_matrix(m, n, 10.0 ** (-14 * np.arange(r) / r), rng)
    k, J, P = sb.row_id(w, 1e-10, engine=6)
    ko, Jo, Po = po.row_id(w, 1e-10)
    assert abs(k - ko) <= 1
    kk = min(k, ko) - 2
    assert np.array_equal(J[:kk], Jo[:kk])
    assert skeleton_identity_exact(k, J, P)
    assert np.linalg.norm(w - P @ w[J[:k]], 2) <= 10 * 1e-10 * np.linalg.norm(w, 2)
    if k + 3 <= r:
        kw, Jw, Pw = sb.row_id(w, forced=k + 3, engine=6)
        assert kw == k + 3 and np.array_equal(Jw[:k], J[:k])


TALL = [(128, 700), (114, 855), (20, 1088), (64, 3000), (127, 511), (3, 9000), (96, 400), (1, 30000)]


@pytest.mark.parametrize("shape", TALL)
def test_row_id_tall_quad_tsqr(sb, po, shape):
    """Tall W^T (functionals >> candidates, n <= 128) on engine 1: the
    quad-layout TSQR + register CPQR of R0 (dense.cu tsqr_quad_kernel)
    reproduces the oracle's pivots, rank and interpolation error."""
    m, n = shape
    rng = np.random.default_rng(m * 11 + n)
    r = min(m, n)
    w = spectrum_matrix(m, n, 10.0 ** (-14 * np.arange(r) / r), rng)
    k, J, P = sb.row_id(w, 1e-10, engine=1)
    ko, Jo, Po = po.row_id(w, 1e-10)
    assert abs(k - ko) <= 1
    kk = min(k, ko) - 2
    assert np.array_equal(J[:kk], Jo[:kk])
    assert skeleton_identity_exact(k, J, P)
    assert np.linalg.norm(w - P @ w[J[:k]], 2) <= 10 * 1e-10 * np.linalg.norm(w, 2)
    kf, Jf, Pf = sb.row_id(w, forced=min(k + 3, m), engine=1)
    assert np.array_equal(Jf[:kk], Jo[:kk])


@pytest.mark.parametrize("shape", [(30, 257), (97, 257), (57, 513), (98, 513), (28, 1088), (112, 369),
                                   (128, 767), (8, 64), (4, 9), (64, 3000)])
def test_row_id_rows_engine(sb, po, shape):
    """Row-split cluster CPQR (engine 7, cpqr_rows.cu) on tall W^T (functionals
    >= 2 x candidates): same pivots and ranks as the oracle, exact skeleton
    identity, forced-rank extension keeps the eps skeleton."""
    m, n = shape
    rng = np.random.default_rng(3 * m + n)
    r = min(m, n)
    w = spectrum_matrix(m, n, 10.0 ** (-14 * np.arange(r) / r), rng)
    k, J, P = sb.row_id(w, 1e-10, engine=7)
    ko, Jo, Po = po.row_id(w, 1e-10)
    assert abs(k - ko) <= 1
    kk = min(k, ko) - 2
    assert np.array_equal(J[:kk], Jo[:kk])
    assert skeleton_identity_exact(k, J, P)
    assert np.linalg.norm(w - P @ w[J[:k]], 2) <= 10 * 1e-10 * np.linalg.norm(w, 2)
    if k + 3 <= r:
        kw, Jw, Pw = sb.row_id(w, forced=k + 3, engine=7)
        assert kw == k + 3 and np.array_equal(Jw[:k], J[:k])


@pytest.mark.parametrize("engine", [8, 9])
@pytest.mark.parametrize("shape", [(30, 257), (97, 257), (57, 513), (98, 513), (28, 1088), (112, 369),
                                   (128, 767), (8, 64), (4, 9), (64, 3000), (200, 600), (1, 40), (116, 861),
                                   (250, 1000)])
def test_row_id_push_engine(sb, po, shape, engine):
    """One-exchange row-split cluster CPQR (engines 8 and 9, cpqr_push.cu:
    pivot-column dots pushed with st.async, mbarrier transaction counts; slab
    in shared memory / in registers): same pivots and ranks as the oracle,
    exact skeleton identity, forced-rank extension keeps the eps skeleton."""
    m, n = shape
    rng = np.random.default_rng(5 * m + n)
    r = min(m, n)
    w = spectrum_matrix(m, n, 10.0 ** (-14 * np.arange(r) / r), rng)
    k, J, P = sb.row_id(w, 1e-10, engine=engine)
    ko, Jo, Po = po.row_id(w, 1e-10)
    assert abs(k - ko) <= 1
    kk = min(k, ko) - 2
    assert np.array_equal(J[:kk], Jo[:kk])
    assert skeleton_identity_exact(k, J, P)
    assert np.linalg.norm(w - P @ w[J[:k]], 2) <= 10 * 1e-10 * np.linalg.norm(w, 2)
    if k + 3 <= r:
        kw, Jw, Pw = sb.row_id(w, forced=k + 3, engine=engine)
        assert kw == k + 3 and np.array_equal(Jw[:k], J[:k])


@pytest.mark.parametrize("engine", [8, 9])
def test_row_id_push_engine_deterministic(sb, engine):
    rng = np.random.default_rng(19)
    w = spectrum_matrix(116, 861, 10.0 ** (-12 * np.arange(116) / 116), rng)
    first = sb.row_id(w, 1e-10, engine=engine)
    for _ in range(3):
        again = sb.row_id(w, 1e-10, engine=engine)
        assert again[0] == first[0]
        assert np.array_equal(again[1], first[1]) and np.array_equal(again[2], first[2])


@pytest.mark.parametrize("shape", [(30, 257), (97, 257), (57, 513), (98, 513), (112, 369), (128, 767),
                                   (8, 64), (116, 861), (110, 1172), (128, 1250), (17, 40), (1, 9)])
def test_row_id_blocked_qr_engine(sb, po, shape):
    """Blocked DMMA QR + CPQR of R0 (engine 10, bqr_kernel) on tall W^T: same
    pivots and ranks as the oracle's CPQR of W^T, exact skeleton identity,
    forced-rank extension keeps the eps skeleton."""
    m, n = shape
    rng = np.random.default_rng(7 * m + n)
    r = min(m, n)
    w = spectrum_matrix(m, n, 10.0 ** (-14 * np.arange(r) / r), rng)
    k, J, P = sb.row_id(w, 1e-10, engine=10)
    ko, Jo, Po = po.row_id(w, 1e-10)
    assert abs(k - ko) <= 1
    kk = min(k, ko) - 2
    assert np.array_equal(J[:kk], Jo[:kk])
    assert skeleton_identity_exact(k, J, P)
    assert np.linalg.norm(w - P @ w[J[:k]], 2) <= 10 * 1e-10 * np.linalg.norm(w, 2)
    if k + 3 <= r:
        kw, Jw, Pw = sb.row_id(w, forced=k + 3, engine=10)
        assert kw == k + 3 and np.array_equal(Jw[:k], J[:k])
