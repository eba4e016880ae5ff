"""The reference's entry-oracle plugin point, HbsSource::entries
(hbs.hpp:19-31), swapped in exactly as its tests do (test_hbs.cpp:186-245),
through sbx_hbs_compress_custom: an identity oracle passes through the
device compression untouched, and an operator with its completion term
stripped compresses accurately but is reported singular, naming the tree
node, by the inverse's rcond gate (hbs.cpp:429)."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def sb():
    import paper_2108_07205_b200 as sb
    sb.init(0)
    return sb


def test_identity_entry_oracle_passes_through(sb):  # test_hbs.cpp:186-205
    g = sb.panelize(sb.circle(1.0), 16, 16)
    calls = []

    def identity(rows, cols):
        calls.append((len(rows), len(cols)))
        return (rows[:, None] == cols[None, :]).astype(np.float64)

    op = sb.hbs_invert(sb.hbs_compress(g, entries=identity, opts=sb.HbsOptions(eps=1e-10)))
    assert calls, "the plugin was never called"
    v = np.random.default_rng(17).standard_normal(op.n)
    assert np.linalg.norm(sb.hbs_apply(op, v) - v) < 1e-12 * np.linalg.norm(v)
    assert np.linalg.norm(sb.hbs_solve(op, v) - v) < 1e-12 * np.linalg.norm(v)


def test_stripped_completion_is_singular_at_a_tree_node(sb):  # test_hbs.cpp:207-245
    g = sb.panelize(sb.circle(1.0), 20, 16)
    n = g.n_unknowns()
    idx = np.arange(n)
    A = sb.submatrix(g, idx, idx)
    nd = g.nodes()
    nrm = np.stack([nd["nx"], nd["ny"]], 1).reshape(-1)  # normal component of each scalar
    w = np.repeat(nd["w"], 2)
    A_strip = A - np.outer(nrm, w * nrm)  # drop N: n_i(r) w_j n_j(c)

    def stripped(rows, cols):
        return A_strip[np.ix_(rows, cols)]

    op = sb.hbs_compress(g, entries=stripped, with_completion=False, opts=sb.HbsOptions(eps=1e-10))
    err = np.linalg.norm(sb.hbs_apply(op, np.eye(n)) - A_strip) / np.linalg.norm(A_strip)
    assert err < 1e-9, err
    with pytest.raises(sb.SingularMatrixError, match="tree node"):
        sb.hbs_invert(op)


def test_plugin_errors_propagate(sb):
    g = sb.panelize(sb.circle(1.0), 8, 16)

    def broken(rows, cols):
        raise RuntimeError("entry oracle failed")

    with pytest.raises(RuntimeError, match="entry oracle failed"):
        sb.hbs_compress(g, entries=broken)
