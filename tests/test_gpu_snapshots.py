"""Snapshot batch with the update cache (reference run_snapshot_batch,
scenario.cpp:806-915): static HBS inverse once; per snapshot the panels near
a body position are refined, the update comes from the cache when the same
(panel ids, m) was seen before, and the solve is checked against the
analytic Stokeslet field.  A cached update gives bit-for-bit the same
density as a fresh compression."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def sb():
    import paper_2108_07205_b200 as sb
    sb.init(0)
    return sb


def test_snapshot_batch_with_update_cache(sb, po):
    eps, m = 1e-10, 4
    g0 = sb.panelize(sb.star(5, 0.3), 48, 16)
    h = sb.hbs_invert(sb.hbs_compress(g0, opts=sb.HbsOptions(eps=eps)))
    src = po.ring_sources(5, (0.0, 0.0), 3.0)
    tg = np.array([[0.2, 0.1], [-0.3, 0.25], [0.1, -0.4], [0.05, 0.3]])
    exact = po.field_velocity(src, tg)
    cache = sb.UpdateCache()
    nodes = g0.nodes()
    # a tour that revisits positions (the cache's reason to exist) and one
    # position away from the wall (no refinement: plain hbs_solve)
    ts = [0.3, 1.1, 0.3, 2.0, 1.1, 0.3]
    pos = [np.array([1.28 * np.cos(t) * (1 + 0.3 * np.cos(5 * t)) / 1.3,
                     1.28 * np.sin(t) * (1 + 0.3 * np.cos(5 * t)) / 1.3]) for t in ts] + [np.zeros(2)]
    hits, dens = [], {}
    for i, p in enumerate(pos):
        panels = g0.panels_near_point(p, 0.1)
        if len(panels) == 0:
            tau = sb.hbs_solve(h, sb.boundary_data(g0, src))
            vel, _, _ = sb.evaluate_solution(g0, sb.INTERIOR_DIRICHLET, tau, tg)
        else:
            g1, plan = sb.refine(g0, panels, m)
            upd, hit = cache.compress(g0, g1, plan, panels, m, eps)
            hits.append(hit)
            e = sb.els_build(h, g0, g1, plan, upd)
            tau_n = sb.els_solve(e, sb.gather_kept_added(plan, sb.boundary_data(g1, src)))
            key = tuple(panels)
            if key in dens:
                assert np.array_equal(tau_n, dens[key])
            else:
                fresh = sb.compress_update(g0, g1, plan, eps)
                assert np.array_equal(fresh.factors()[0], upd.factors()[0])
                dens[key] = tau_n
            vel, _, _ = sb.evaluate_solution(g1, sb.INTERIOR_DIRICHLET, sb.density_on_refined(e, tau_n), tg)
        err = np.max(np.linalg.norm(vel - exact, axis=1) / np.linalg.norm(exact, axis=1))
        assert err < 1e-8, (i, err)
    assert hits == [False, False, True, False, True, True]
    assert cache.stats() == {"entries": 3, "hits": 3, "misses": 3}
