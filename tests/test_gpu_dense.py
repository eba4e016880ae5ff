"""Dense inverse + rcond on the device (the Woodbury operator W and the dense
A_pp go through it: els.cpp:111-127) against numpy, across the kernel
routing boundaries (register Gauss-Jordan <= 128, DMMA-tile Gauss-Jordan
<= 160, blocked LU above)."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _case(n, seed, cond=None):
    rng = np.random.default_rng(seed)
    a = rng.standard_normal((n, n))
    if cond is not None:
        u, _, vt = np.linalg.svd(a)
        a = (u * np.logspace(0, -np.log10(cond), n)) @ vt
    return a


@pytest.mark.parametrize("n", [1, 7, 64, 128, 129, 136, 146, 152, 159, 160, 161, 200, 400])
def test_dense_inverse_matches_numpy(n):
    import paper_2108_07205_b200 as sb
    sb.init(0)
    a = _case(n, 100 + n)
    inv, rc = sb.dense_inverse(a)
    ref = np.linalg.inv(a)
    kappa = np.linalg.cond(a, 1)
    assert np.linalg.norm(inv - ref) <= 1e-13 * kappa * np.linalg.norm(ref)
    assert np.linalg.norm(inv @ a - np.eye(n)) <= 1e-13 * kappa * np.sqrt(n)
    true_rc = 1.0 / kappa
    assert true_rc * 0.999 <= rc <= 3.5 * true_rc  # Hager/Higham: a lower bound of ||A^-1||_1, sharp in practice


@pytest.mark.parametrize("n", [130, 146, 160])
def test_dense_inverse_ill_conditioned_and_identity_plus_lowrank(n):
    """The W = I + R X shape of the Woodbury operator, and a 1e10 condition."""
    import paper_2108_07205_b200 as sb
    sb.init(0)
    rng = np.random.default_rng(n)
    w = np.eye(n) + rng.standard_normal((n, 12)) @ rng.standard_normal((12, n))
    inv, rc = sb.dense_inverse(w)
    assert np.linalg.norm(inv @ w - np.eye(n)) <= 1e-11
    assert rc > 1e-6
    a = _case(n, 7, cond=1e10)
    inv, rc = sb.dense_inverse(a)
    assert np.linalg.norm(inv @ a - np.eye(n)) <= 1e-4
    assert 1e-12 < rc < 1e-8


def test_dense_inverse_pivoting_needed():
    """Zero diagonal: no elimination order without row pivoting exists."""
    import paper_2108_07205_b200 as sb
    sb.init(0)
    n = 146
    rng = np.random.default_rng(3)
    a = rng.standard_normal((n, n))
    np.fill_diagonal(a, 0.0)
    a[:, 5] *= 1e-3
    inv, _ = sb.dense_inverse(a)
    assert np.linalg.norm(inv @ a - np.eye(n)) <= 1e-9


def test_dense_inverse_singular_reports_zero_rcond():
    import paper_2108_07205_b200 as sb
    sb.init(0)
    n = 146
    a = _case(n, 11)
    a[:, 17] = a[:, 3]
    _, rc = sb.dense_inverse(a)
    assert rc < 1e-13


@pytest.mark.parametrize("m,k,n", [(146, 40960, 146), (160, 8192, 65), (65, 9000, 160), (129, 20002, 131),
                                   (146, 40960, 64), (100, 16384, 40), (64, 4096, 64), (200, 10000, 100), (7, 100, 5)])
def test_matmul_matches_numpy(m, k, n):
    """The GEMM dispatcher across its routes (64 x 64 DMMA tiles, split-K,
    the thin-product kernel for W = I + R X: els.cpp:124)."""
    import paper_2108_07205_b200 as sb
    sb.init(0)
    rng = np.random.default_rng(m + k + n)
    a = rng.standard_normal((m, k))
    b = rng.standard_normal((k, n))
    c = sb.matmul(a, b)
    ref = a @ b
    assert np.linalg.norm(c - ref) <= 1e-13 * np.sqrt(k) * np.linalg.norm(ref)
    c2 = sb.matmul(a, b)
    assert np.array_equal(c, c2)  # fixed-order split-K reduction: run-to-run bitwise
