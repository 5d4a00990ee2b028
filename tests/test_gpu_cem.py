"""GPU parity of the CEM upper level (K3 select/refit, K4 sampler, the device CEM cycle)."""

import numpy as np
import pytest

import oracle as O
from tests.golden_io import load, oracle_limits, rel_err_per_sample_axis
from tests.test_gpu_parity import COST_TOL, RES_TOL, XI_TOL, _scene

pytestmark = pytest.mark.gpu


def _solver_c2(g, am_iters=100):
    import paper_2212_02224_b200 as bd
    basis = bd.build_basis(10, 100, 5.0, "bernstein")
    return bd.LowerLevelSolver(basis, bd.TrackingWeights(), bd.ParamLayout(4),
                               bd.ProjectionConfig(1.0, am_iters, 1e-3), g["ox"].shape[0])


def band_ok(ours, ref_set, r_ref, n):
    """Tie-aware set comparison: symmetric difference inside the r_(n) band."""
    rn = np.sort(r_ref)[n - 1]
    band = np.abs(r_ref - rn) <= RES_TOL * (1.0 + abs(rn))
    diff = set(map(int, ours)) ^ set(map(int, ref_set))
    return all(band[i] for i in diff), diff


def test_rank_refit_exact_on_reference_inputs():
    """Fed the reference's own residuals/costs, K3 must reproduce its sets and refit."""
    g = load("cem_c2")
    solver = _solver_c2(g)
    ctx = solver.context
    B, n, q, N, eta, gamma, w = g["cfg"]
    B, n, q = int(B), int(n), int(q)
    mean, cov = g["init_mean"].copy(), g["init_cov"].copy()
    for it in range(int(N)):
        from paper_2212_02224_b200._native import ptr
        cons = np.empty(n, np.int64)
        el = np.empty(q, np.int64)
        ea = np.empty(q)
        st = np.empty(6)
        P = np.ascontiguousarray(g["params"][it])
        ctx.call("bd_rank_refit", 1, B, 8, ptr(np.ascontiguousarray(g["residuals"][it])),
                 ptr(np.ascontiguousarray(g["costs"][it])), ptr(P), n, q, float(w), float(eta), float(gamma),
                 ptr(mean), ptr(cov), ptr(cons), ptr(el), ptr(ea), ptr(st))
        np.testing.assert_array_equal(cons, g["cons_idx"][it])
        np.testing.assert_array_equal(el, g["elite_idx"][it])
        np.testing.assert_allclose(ea, g["elite_aug"][it], rtol=1e-14)
        np.testing.assert_allclose(mean, g["mean"][it], rtol=1e-12)
        np.testing.assert_allclose(cov, g["cov"][it], rtol=1e-10, atol=1e-14)
        mean, cov = g["mean"][it].copy(), g["cov"][it].copy()


def test_rank_ties_and_nan_order():
    """Stable order with exact ties, -0 == +0, NaN last (np.argsort kind='stable')."""
    from paper_2212_02224_b200._native import ptr
    g = load("cem_c2")
    ctx = _solver_c2(g).context
    r = np.array([0.0, -0.0, 1.0, 0.0, np.nan, 0.5, 1.0, 0.0] * 4)
    c = np.arange(len(r), dtype=float)[::-1].copy()
    P = np.zeros((len(r), 8))
    n, q = 12, 5
    cons = np.empty(n, np.int64)
    el = np.empty(q, np.int64)
    ea = np.empty(q)
    mean, cov = np.zeros(8), np.eye(8)
    ctx.call("bd_rank_refit", 1, len(r), 8, ptr(r), ptr(c), ptr(P), n, q, 1.0, 0.7, 0.9, ptr(mean), ptr(cov),
             ptr(cons), ptr(el), None, None)
    ref_c, ref_e, _ = O.rank_two_stage(r, c, n, q, 1.0)
    np.testing.assert_array_equal(cons, ref_c)
    np.testing.assert_array_equal(el, ref_e)


def test_teacher_forced_config2():
    """Config 2 (B=1000, N=4, n=150, q=100) fed the reference's params each CEM iteration."""
    g = load("cem_c2")
    solver = _solver_c2(g)
    sc = _scene(g)
    B, n, q, N, eta, gamma, w = g["cfg"]
    n, q = int(n), int(q)
    for it in range(int(N)):
        _, proj = solver.solve(g["params"][it], sc)
        costs = solver.last_costs
        assert rel_err_per_sample_axis(proj.xi, g["xi"][it]) <= XI_TOL
        assert np.all(np.abs(costs - g["costs"][it]) <= COST_TOL * np.maximum(g["costs"][it], 1.0))
        r_ref = g["residuals"][it]
        assert np.all(np.abs(proj.residuals - r_ref) <= RES_TOL * (1 + r_ref))
        cons, el, ea = O.rank_two_stage(proj.residuals, costs, n, q, float(w))
        ok, diff = band_ok(cons, g["cons_idx"][it], r_ref, n)
        assert ok, f"iteration {it}: constraint-elite swaps outside the tie band: {diff}"
        assert int(el[0]) == int(g["elite_idx"][it][0]), "best index"


def test_solve_bilevel_dropin_free_running():
    """solve_bilevel with the caller's Generator reproduces the reference's run (cem_small)."""
    import paper_2212_02224_b200 as bd
    g = load("cem_small")
    solver = _solver_c2(g, am_iters=int(g["am_iters"]))
    B, n, q, N, eta, gamma, w = g["cfg"]
    cfg = bd.BiLevelConfig(int(B), int(n), int(q), int(N), eta, gamma, w, g["init_mean"], g["init_cov"])
    rng = np.random.default_rng(int(g["seed"]))
    res = solver_res = bd.solve_bilevel(_scene(g), solver, cfg, rng)
    assert not res.degraded and len(res.diagnostics) == int(N)
    assert res.best.index == int(g["best_index"])
    np.testing.assert_allclose(res.best.params.to_vector(), g["best_params"], rtol=1e-12)
    assert rel_err_per_sample_axis(res.best.coeffs.stacked()[:, None], g["best_xi"][:, None]) <= XI_TOL
    stats = np.array([[s.elite_mean_upper_cost, s.best_augmented_cost, s.cov_trace, s.residual_min,
                       s.residual_median, s.residual_max] for s in solver_res.diagnostics])
    np.testing.assert_allclose(stats[:, :3], g["stats"][:, 1:4], rtol=1e-4)
    np.testing.assert_allclose(res.distribution.mean, g["final_mean"], rtol=1e-4)
    # the caller's generator advanced exactly as the reference's
    ref_rng = np.random.default_rng(int(g["seed"]))
    ref_rng.standard_normal((int(N), int(B), 8))
    assert rng.standard_normal() == ref_rng.standard_normal()


def test_solve_bilevel_trace_hook_path():
    import paper_2212_02224_b200 as bd
    g = load("cem_small")
    solver = _solver_c2(g, am_iters=int(g["am_iters"]))
    B, n, q, N, eta, gamma, w = g["cfg"]
    cfg = bd.BiLevelConfig(int(B), int(n), int(q), int(N), eta, gamma, w, g["init_mean"], g["init_cov"])
    seen = []
    res = bd.solve_bilevel(_scene(g), solver, cfg, np.random.default_rng(int(g["seed"])),
                           trace_hook=lambda it, p, proj, c, e: seen.append((it, p.shape, proj.xi.shape, int(e[0]))))
    assert [s[0] for s in seen] == list(range(1, int(N) + 1))
    assert res.best.index == int(g["best_index"])
    np.testing.assert_allclose(res.distribution.mean, g["final_mean"], rtol=1e-4)


def test_device_rng_cycle_is_deterministic_and_contracts():
    import ctypes
    import paper_2212_02224_b200 as bd
    from paper_2212_02224_b200._native import CemConfig, ptr
    g = load("cem_c2")
    solver = _solver_c2(g)
    solver.projector._ensure_scene(_scene(g))
    cfg = CemConfig(1000, 150, 100, 4, 100, 0.7, 0.9, 1.0, 1e-3, 1234, 0)
    outs = []
    for _ in range(2):
        st = np.zeros((4, 6))
        bi = np.zeros(1, np.int64)
        done = np.zeros(1, np.int32)
        fm = np.zeros(8)
        solver.context.call("bd_cem_cycle", 1, ctypes.byref(cfg), ptr(g["init_mean"]), ptr(g["init_cov"]), None,
                            None, ptr(bi), None, None, None, None, None, ptr(st), ptr(fm), None, ptr(done))
        outs.append((st.copy(), int(bi[0]), fm.copy(), int(done[0])))
    assert outs[0][3] == 4
    np.testing.assert_array_equal(outs[0][0], outs[1][0])
    assert outs[0][1] == outs[1][1]
    assert outs[0][0][-1, 2] < outs[0][0][0, 2]      # covariance trace shrinks
    assert np.all(np.isfinite(outs[0][0]))


@pytest.mark.parametrize("case", ["c1_s0", "goal", "dense50"])
def test_evaluate_batch_baseline_planners(case):
    """BasePlanner.evaluate_batch (pkg/planners.py:233-258) on the device: best record equals the
    reference ranking of the reference's own residuals/costs (outside the tie band)."""
    import paper_2212_02224_b200 as bd
    from paper_2212_02224_b200.bilevel import evaluate_batch
    from tests.test_gpu_parity import _solver
    g = load("lower_" + case)
    solver = _solver(g)
    n, q = 150, 50
    rec, diag = evaluate_batch(solver, _scene(g), g["params"], n, q, 1.0)
    B = g["params"].shape[0]
    _, el, ea = O.rank_two_stage(g["residuals"], g["costs"], min(n, B), min(q, min(n, B)), 1.0)
    assert rec.index == int(el[0])
    assert abs(rec.augmented_cost - ea[0]) <= 1e-3 * (1 + abs(ea[0]))
    assert diag["batch"] == B and diag["proj_iterations"] == int(g["iterations_used"])


@pytest.mark.parametrize("case", ["goal", "warm", "curve"])
def test_solve_bilevel_goal_layout_and_warm_start(case):
    """solve_bilevel with the goal layout (per-sample goal rows), with a WarmStartSource for
    iteration 1 and on a curved road reproduce the reference's seeded runs
    (tests/golden/cem_variants.npz)."""
    import paper_2212_02224_b200 as bd
    g = load("cem_variants")
    layout = bd.ParamLayout(4, with_goal=(case == "goal"))
    basis = bd.build_basis(10, 100, 5.0, "bernstein")
    solver = bd.LowerLevelSolver(basis, bd.TrackingWeights(), layout, bd.ProjectionConfig(1.0, 40, 1e-3),
                                 g["ox"].shape[0])
    cfg = bd.BiLevelConfig(200, 60, 20, 3, 0.7, 0.9, 1.0, g[f"{case}_mean"], g[f"{case}_cov"])
    ws = bd.WarmStartSource(g["warm_samples"], layout) if case == "warm" else None
    scene = _scene(g)
    if case == "curve":
        from dataclasses import replace
        scene = bd.PlanningScene(scene.initial_state, replace(scene.spec, road_curvature=(g["curve_xs"], g["curve_ks"])),
                                 scene.lane_centers)
    res = bd.solve_bilevel(scene, solver, cfg, np.random.default_rng(5), warm_start=ws)
    assert not res.degraded and len(res.diagnostics) == 3
    assert res.best.index == int(g[f"{case}_best_index"])
    np.testing.assert_allclose(res.best.params.to_vector(), g[f"{case}_best_params"], rtol=1e-10, atol=1e-10)
    assert rel_err_per_sample_axis(res.best.coeffs.stacked()[:, None], g[f"{case}_best_xi"][:, None]) <= XI_TOL
    stats = np.array([[s.elite_mean_upper_cost, s.best_augmented_cost, s.cov_trace, s.residual_min,
                       s.residual_median, s.residual_max] for s in res.diagnostics])
    np.testing.assert_allclose(stats[:, :3], g[f"{case}_stats"][:, :3], rtol=1e-4)
    np.testing.assert_allclose(res.distribution.mean, g[f"{case}_final_mean"], rtol=1e-4)


def test_absurd_warm_start_rows_do_not_degrade():
    """A warm start with a few set-points far off the road (pkg/bilevel.py:249-251): they rank
    last in both implementations, the run is not degraded and elites / best / refit match."""
    import paper_2212_02224_b200 as bd
    from paper_2212_02224_b200.harness import canonical_scene
    from paper_2212_02224_b200.planners import PlannerEnvConfig
    g = load("absurd")
    scene = canonical_scene(PlannerEnvConfig(num_samples=100, max_obstacles=10))
    basis = bd.build_basis(10, 100, 5.0, "bernstein")
    solver = bd.LowerLevelSolver(basis, bd.TrackingWeights(), bd.ParamLayout(4), bd.ProjectionConfig(1.0, 100, 1e-3), 10)
    cfg = bd.BiLevelConfig(200, 60, 20, 3, 0.7, 0.9, 1.0, g["cem_mean"], g["cem_cov"])
    ws = bd.WarmStartSource(g["warm"], bd.ParamLayout(4))
    seen = []
    res = bd.solve_bilevel(scene, solver, cfg, np.random.default_rng(4), warm_start=ws,
                           trace_hook=lambda it, p, pr, c, e: seen.append(np.asarray(e).copy()))
    assert not res.degraded and not bool(g["cem_degraded"])
    assert not set(seen[0].tolist()) & {5, 50, 120, 199}
    np.testing.assert_array_equal(seen[0], g["cem_elites"][0])
    # free-running fast path: same best record and refit as the reference
    fast = bd.solve_bilevel(scene, solver, cfg, np.random.default_rng(4), warm_start=ws)
    assert not fast.degraded and len(fast.diagnostics) == 3
    assert fast.best.index == int(g["cem_best_index"])
    np.testing.assert_allclose(fast.best.params.to_vector(), g["cem_best_params"], rtol=1e-6)
    np.testing.assert_allclose(fast.distribution.mean, g["cem_final_mean"], rtol=1e-4)
    st = np.array([[s.elite_mean_upper_cost, s.best_augmented_cost, s.cov_trace, s.residual_min,
                    s.residual_median, s.residual_max] for s in fast.diagnostics])
    np.testing.assert_allclose(st[:, :5], g["cem_stats"][:, :5], rtol=1e-3, atol=1e-3)
    # iteration 1 holds the absurd rows: the reference's max is huge, the device's +inf
    assert np.isinf(st[0, 5]) and g["cem_stats"][0, 5] > 1e15
    np.testing.assert_allclose(st[1:, 5], g["cem_stats"][1:, 5], rtol=1e-3, atol=1e-3)


@pytest.mark.parametrize("B,n,q,seed", [(37, 20, 7, 0), (1000, 150, 100, 1), (4096, 600, 50, 2), (13000, 1024, 64, 3),
                                        (2000, 700, 100, 4), (3000, 850, 160, 5)])
def test_rank_refit_random_with_ties(B, n, q, seed):
    """rank_samples + update_distribution (pkg/bilevel.py:129-194) on random keys with many exact
    ties, against the oracle: constraint-elite and elite sets and order exactly, refit to 1e-12.
    B = 13000 takes the global (non-shared-memory) counting rank.  (700, 100) and (850, 160) put
    the refit kernel's dynamic shared memory in (32 KB, 36 KB], where dynamic + static exceed the
    default 48 KB (the opt-in must not be skipped there)."""
    from paper_2212_02224_b200._native import ptr
    g = load("cem_c2")
    ctx = _solver_c2(g).context
    rng = np.random.default_rng(seed)
    r = np.round(rng.exponential(1.0, B), 2)                 # residual ties
    c = np.round(rng.normal(200.0, 30.0, B), 1)              # augmented-cost ties
    r[rng.random(B) < 0.05] = 0.0
    P = np.ascontiguousarray(rng.normal(size=(B, 8)))
    mean, cov = rng.normal(size=8), np.eye(8) * 2.0 + 0.1
    m_dev, c_dev = mean.copy(), cov.copy()
    cons, el, ea, st = np.empty(n, np.int64), np.empty(q, np.int64), np.empty(q), np.empty(6)
    ctx.call("bd_rank_refit", 1, B, 8, ptr(r), ptr(c), ptr(P), n, q, 1.0, 0.7, 0.9, ptr(m_dev), ptr(c_dev),
             ptr(cons), ptr(el), ptr(ea), ptr(st))
    rc, re, ra = O.rank_two_stage(r, c, n, q, 1.0)
    np.testing.assert_array_equal(cons, rc)
    np.testing.assert_array_equal(el, re)
    np.testing.assert_array_equal(ea, ra)
    mu, C = O.refit_gaussian(mean, cov, P[re], ra, 0.7, 0.9)
    np.testing.assert_allclose(m_dev, mu, rtol=1e-12, atol=1e-13)
    np.testing.assert_allclose(c_dev, C, rtol=1e-11, atol=1e-13)
    np.testing.assert_allclose(st[[3, 4, 5]], [r.min(), np.median(r), r.max()], rtol=0, atol=0)
    assert st[1] == ra[0]


@pytest.mark.parametrize("dim,seed", [(4, 10), (10, 11), (16, 12)])
def test_rank_refit_random_other_dims(dim, seed):
    """The refit for behaviour vectors of 4 (two segments), 10 (goal layout) and 16 (the maximum)."""
    from paper_2212_02224_b200._native import ptr
    g = load("cem_c2")
    ctx = _solver_c2(g).context
    rng = np.random.default_rng(seed)
    B, n, q = 500, 120, 40
    r = np.round(rng.exponential(1.0, B), 2)
    c = np.round(rng.normal(200.0, 30.0, B), 1)
    P = np.ascontiguousarray(rng.normal(size=(B, dim)))
    A = rng.normal(size=(dim, dim))
    mean, cov = rng.normal(size=dim), A @ A.T + dim * np.eye(dim)
    m_dev, c_dev = mean.copy(), cov.copy()
    cons, el, ea, st = np.empty(n, np.int64), np.empty(q, np.int64), np.empty(q), np.empty(6)
    ctx.call("bd_rank_refit", 1, B, dim, ptr(r), ptr(c), ptr(P), n, q, 1.0, 0.6, 1.3, ptr(m_dev), ptr(c_dev),
             ptr(cons), ptr(el), ptr(ea), ptr(st))
    rc, re, ra = O.rank_two_stage(r, c, n, q, 1.0)
    np.testing.assert_array_equal(el, re)
    mu, C = O.refit_gaussian(mean, cov, P[re], ra, 0.6, 1.3)
    np.testing.assert_allclose(m_dev, mu, rtol=1e-12, atol=1e-13)
    np.testing.assert_allclose(c_dev, C, rtol=1e-11, atol=1e-12)


@pytest.mark.parametrize("seed", range(3))
def test_random_teacher_forced_cem_matches_oracle(seed):
    """Teacher-forced CEM on randomised scenes (tests/test_gpu_random_parity.py's generator):
    every iteration the device solves the oracle's samples; residuals and costs within the §8c
    tolerances, constraint-elite and elite sets exact outside the residual tie band, refit mean
    to 1e-4 when the sets agree."""
    import paper_2212_02224_b200 as bd
    from paper_2212_02224_b200._native import ptr
    from tests.test_gpu_random_parity import M, T, _random_case
    n_obs, ox, oy, lim, curv, b0, _ = _random_case(300 + seed, n_obs=10)
    B, n, q, N, am = 300, 90, 30, 3, 40
    _, W, Wd, Wdd = O.basis_matrices(10, M, T)
    qp = O.tracking_qp(W, Wd, Wdd, 4)
    aug = O.aug_qp(W, Wd, Wdd, qp.A_eq, n_obs, 1.0)
    ol = O.Limits(ox, oy, lim["a"], lim["b"], lim["v_max"], lim["a_max"], lim["kappa_max"], lim["c_max"],
                  lim["y_lb"], lim["y_ub"], lim["v_min"], curv)
    mean0 = np.concatenate([np.full(4, b0[1]), np.full(4, np.hypot(b0[2], b0[3]))])
    cov0 = np.diag(np.concatenate([np.full(4, 1.5 ** 2), np.full(4, 3.0 ** 2)]))
    tr = O.cem_cycle(qp, aug, W, Wd, Wdd, b0, ol, mean0, cov0, batch=B, n_cons=n, n_elite=q, iters=N, eta=0.7,
                     gamma=0.9, w_res=1.0, rng=np.random.default_rng(seed), am_iters=am, tol=1e-30)
    basis = bd.build_basis(10, M, T, "bernstein")
    solver = bd.LowerLevelSolver(basis, bd.TrackingWeights(), bd.ParamLayout(4), bd.ProjectionConfig(1.0, am, 1e-30),
                                 n_obs)
    spec = bd.ConstraintSpec(ox, oy, lim["a"], lim["b"], lim["v_max"], lim["a_max"], lim["kappa_max"], lim["c_max"],
                             lim["y_lb"], lim["y_ub"], lim["v_min"], curv)
    scene = bd.PlanningScene(b0, spec)
    mean, cov = mean0, cov0
    for it in range(N):
        P = np.ascontiguousarray(tr.params[it])
        _, proj = solver.solve(P, scene)
        r, c = np.asarray(proj.residuals), np.asarray(solver.last_costs)
        assert np.all(np.abs(r - tr.residuals[it]) <= RES_TOL * (1.0 + tr.residuals[it]))
        assert np.all(np.abs(c - tr.costs[it]) <= COST_TOL * np.maximum(tr.costs[it], 1.0))
        m_dev, c_dev = mean.copy(), cov.copy()
        cons, el, ea, st = np.empty(n, np.int64), np.empty(q, np.int64), np.empty(q), np.empty(6)
        solver.context.call("bd_rank_refit", 1, B, 8, ptr(np.ascontiguousarray(r)), ptr(np.ascontiguousarray(c)),
                            ptr(P), n, q, 1.0, 0.7, 0.9, ptr(m_dev), ptr(c_dev), ptr(cons), ptr(el), ptr(ea), ptr(st))
        ok, diff = band_ok(cons, tr.cons_idx[it], tr.residuals[it], n)
        assert ok, f"iteration {it}: constraint elites differ outside the tie band: {sorted(diff)}"
        if not diff and set(el.tolist()) == set(tr.elite_idx[it].tolist()):
            np.testing.assert_allclose(m_dev, tr.mean[it], rtol=1e-4, atol=1e-6)
        mean, cov = tr.mean[it], tr.cov[it]                   # teacher forcing: continue from the oracle
