"""GPU: the SPEC.md examples and invariants of solve_bilevel / update_distribution
(acceptance 3 at SPEC.md:527) on the device path.

* n = 1, N = 1 returns that sample's projected trajectory;
* elite-cost dominance of the returned record (trace_hook elites);
* weight shift-invariance and the eta = 0 refit (mean unchanged, Sigma + 1e-6 I:
  pkg/bilevel.py:175-194 always regularises);
* determinism of the drop-in path (identical seeds -> bit-identical outputs);
* convergence on the canonical static-obstacle scene (acceptance 3: elite-mean cost and
  trace(Sigma) at iteration 5 vs 1 over 50 seeds, n = 1000 / 150 / 50, gamma = 0.9).
"""

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _canon(batch=1000, n_cons=150, n_elite=50, iters=5):
    import paper_2212_02224_b200 as bd
    from paper_2212_02224_b200.harness import bilevel_config_for, canonical_scene
    from paper_2212_02224_b200.planners import PlannerEnvConfig
    env = PlannerEnvConfig(num_samples=100, max_obstacles=10)
    scene = canonical_scene(env)
    basis = bd.build_basis(10, 100, 5.0, "bernstein")
    solver = bd.LowerLevelSolver(basis, bd.TrackingWeights(), bd.ParamLayout(4), bd.ProjectionConfig(1.0, 100, 1e-3),
                                 10)
    c = bilevel_config_for(env, scene, batch_size=batch, iterations=iters)
    cfg = bd.BiLevelConfig(batch, n_cons, n_elite, iters, c.eta, 0.9, c.residual_weight, c.init_mean, c.init_cov)
    return bd, scene, solver, cfg


def test_single_sample_single_iteration_returns_its_projection():
    bd, scene, solver, cfg = _canon()
    cfg1 = bd.BiLevelConfig(1, 1, 1, 1, cfg.eta, cfg.gamma, cfg.residual_weight, cfg.init_mean, cfg.init_cov)
    res = bd.solve_bilevel(scene, solver, cfg1, np.random.default_rng(3))
    p = cfg.init_mean + np.random.default_rng(3).standard_normal((1, 8)) @ np.linalg.cholesky(cfg.init_cov).T
    _, proj = solver.solve(p, scene)
    assert res.best.index == 0 and not res.degraded
    np.testing.assert_allclose(res.best.params.to_vector(), p[0], rtol=1e-12)
    np.testing.assert_allclose(res.best.coeffs.stacked(), proj.xi[:, 0], rtol=1e-9, atol=1e-9)
    assert res.best.residual == pytest.approx(float(proj.residuals[0]), rel=1e-9, abs=1e-9)


def test_elite_cost_dominance():
    bd, scene, solver, cfg = _canon(batch=400, n_cons=100, n_elite=30, iters=3)
    augs = []
    solver_aug = {}

    def hook(it, params, proj, costs, elite):
        solver_aug[it] = (costs[elite] + cfg.residual_weight * proj.residuals[elite])
    res = bd.solve_bilevel(scene, solver, cfg, np.random.default_rng(1), trace_hook=hook)
    final = solver_aug[cfg.iterations]
    assert res.best.augmented_cost <= final.min() + 1e-9 * abs(final.min())
    assert np.all(np.diff(final) >= -1e-9 * np.abs(final[1:]))       # elites in ascending aug order


def _refit(ctx, P, costs, resid, mean, cov, eta, gamma, n, q):
    from paper_2212_02224_b200._native import ptr
    B = P.shape[0]
    mean, cov = mean.copy(), cov.copy()
    cons, el, ea, st = np.empty(n, np.int64), np.empty(q, np.int64), np.empty(q), np.empty(6)
    ctx.call("bd_rank_refit", 1, B, 8, ptr(resid), ptr(costs), ptr(P), n, q, 1.0, float(eta), float(gamma),
             ptr(mean), ptr(cov), ptr(cons), ptr(el), ptr(ea), ptr(st))
    return mean, cov, el


def test_refit_weight_shift_invariance_and_eta_zero():
    bd, scene, solver, cfg = _canon()
    rng = np.random.default_rng(7)
    B = 300
    P = np.ascontiguousarray(rng.normal(size=(B, 8)))
    costs = rng.uniform(100.0, 200.0, B)
    resid = rng.uniform(0.0, 1.0, B)
    m0, c0 = cfg.init_mean, cfg.init_cov
    m1, c1, e1 = _refit(solver.context, P, costs, resid, m0, c0, 0.7, 0.9, 100, 30)
    m2, c2, e2 = _refit(solver.context, P, costs + 1234.5, resid, m0, c0, 0.7, 0.9, 100, 30)
    np.testing.assert_array_equal(e1, e2)
    np.testing.assert_allclose(m2, m1, rtol=1e-12, atol=1e-12)
    np.testing.assert_allclose(c2, c1, rtol=1e-10, atol=1e-12)
    m3, c3, _ = _refit(solver.context, P, costs, resid, m0, c0, 0.0, 0.9, 100, 30)
    np.testing.assert_array_equal(m3, m0)
    np.testing.assert_allclose(c3, c0 + 1e-6 * np.eye(8), rtol=1e-15, atol=0)


def test_dropin_determinism_bit_identical():
    bd, scene, solver, cfg = _canon(iters=4)
    a = bd.solve_bilevel(scene, solver, cfg, np.random.default_rng(11))
    b = bd.solve_bilevel(scene, solver, cfg, np.random.default_rng(11))
    assert a.best.index == b.best.index
    np.testing.assert_array_equal(a.best.coeffs.stacked(), b.best.coeffs.stacked())
    np.testing.assert_array_equal(a.distribution.cov, b.distribution.cov)
    assert [s.elite_mean_upper_cost for s in a.diagnostics] == [s.elite_mean_upper_cost for s in b.diagnostics]


def test_acceptance3_convergence_over_50_seeds():
    bd, scene, solver, cfg = _canon()
    cost_ok = trace_ok = 0
    for seed in range(50):
        res = bd.solve_bilevel(scene, solver, cfg, np.random.default_rng(seed))
        d = res.diagnostics
        assert len(d) == 5
        cost_ok += d[4].elite_mean_upper_cost <= d[0].elite_mean_upper_cost
        trace_ok += d[4].cov_trace < d[0].cov_trace
    assert cost_ok >= 45 and trace_ok >= 45, (cost_ok, trace_ok)
