"""BASELINE configs[3] (cfg4) as specified: the closed wavy channel
(SBX_CHANNEL) at full size (2048 x 16 nodes).  Device nodes equal the
oracle's bit for bit; the most refined step of the transient (gap 0.005:
panels within 5 gaps of the disk split so their length is at most the gap)
matches the oracle's refined solve to 1e-9 and the generating Stokeslet
field at fluid targets; an identity-plan step is the plain HBS solve."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def setup(po):
    import paper_2108_07205_b200 as sb
    from paper_2108_07205_b200.configs import CONFIGS
    sb.init(0)
    c = CONFIGS["cfg4"]
    cv = c.curve(sb)
    g0 = sb.panelize(cv, c.n_panels, c.q)
    o0 = po.Geom.create(po.CHANNEL, c.n_panels, c.q, center=cv.center, scale=cv.scale, prongs=cv.n_prongs,
                        amplitude=cv.amplitude, aspect=cv.aspect, cos_coef=cv.cos_coef, sin_coef=cv.sin_coef)
    return sb, c, g0, o0


def test_channel_nodes_bitwise_equal_oracle(setup):
    sb, c, g0, o0 = setup
    a, b = g0.nodes(), o0.nodes()
    for key in ("x", "y", "nx", "ny", "w", "curvature", "param"):
        assert np.array_equal(a[key], b[key]), key


def _rel(a, b):
    return float(np.linalg.norm(a - b) / np.linalg.norm(b))


def test_cfg4_refined_step_matches_oracle_and_field(setup, po):
    sb, c, g0, o0 = setup
    nd = g0.nodes()
    plen = np.zeros(c.n_panels)
    np.add.at(plen, nd["panel_of"], nd["w"])
    gap = c.gaps()[-1]
    near, m = c.step_plan(nd, plen, gap)
    assert m >= 2 and len(near) > 0
    src, tg = c.sources(), c.targets()
    h = sb.hbs_invert(sb.hbs_compress(g0, opts=sb.HbsOptions(eps=c.eps, leaf_nodes=c.leaf)))
    g1, plan = sb.refine(g0, near, m)
    upd = sb.compress_update(g0, g1, plan, c.eps)
    els = sb.els_build(h, g0, g1, plan, upd)
    tau = sb.els_solve(els, sb.gather_kept_added(plan, sb.boundary_data(g1, src)))
    # oracle, same step
    a0 = po.Assembler.create(o0)
    oh = po.Hbs.compress(a0, c.eps).invert()
    o1, op = o0.refine(near, m)
    a1 = po.Assembler.create(o1)
    oe = po.Els.build(oh, a0, a1, op, po.Update.compress(a0, a1, op, c.eps))
    otau = oe.solve(po.gather_kept_added(op.maps(), o1.boundary_data(src)))
    assert _rel(tau, otau) <= 1e-9
    vel, _, _ = sb.evaluate_solution(g1, sb.INTERIOR_DIRICHLET, sb.density_on_refined(els, tau), tg)
    ex = po.field_velocity(src, tg)
    assert np.max(np.linalg.norm(vel - ex, axis=1) / np.linalg.norm(ex, axis=1)) < 1e-9
    # identity-plan step (largest gap): the plain HBS solve, same field
    near0, m0 = c.step_plan(nd, plen, c.gaps()[0])
    assert m0 == 1
    vel0, _, _ = sb.evaluate_solution(g0, sb.INTERIOR_DIRICHLET, sb.hbs_solve(h, sb.boundary_data(g0, src)), tg)
    assert np.max(np.linalg.norm(vel0 - ex, axis=1) / np.linalg.norm(ex, axis=1)) < 1e-9
