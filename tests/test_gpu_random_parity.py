"""GPU: the device lower level against the float64 oracle (oracle/port.py, itself pinned to the
reference's golden vectors) on randomised scenes and set-points beyond the golden cases:
obstacle counts 0 / 3 / 10 / 20 / 50 (the last two take the sorted-window path), moving and static
obstacles, random limits, optional road curvature, every lane mapping.  Tolerances of SURVEY §8c."""

import numpy as np
import pytest

import oracle as O
from tests.golden_io import rel_err_per_sample_axis

pytestmark = pytest.mark.gpu

XI_TOL, COST_TOL, RES_TOL = 1e-4, 1e-4, 1e-3
M, T, B, ITERS = 100, 5.0, 24, 40


def _random_case(seed, m=M, horizon=T, n_obs=None):
    rng = np.random.default_rng(seed)
    n_obs = [0, 3, 10, 20, 50][seed % 5] if n_obs is None else n_obs
    lanes = int(rng.integers(2, 5))
    t = np.linspace(0.0, horizon, m)
    x0 = rng.uniform(10.0, 160.0, n_obs)
    vx = np.where(rng.random(n_obs) < 0.3, 0.0, rng.uniform(4.0, 18.0, n_obs))
    lane = rng.integers(0, lanes, n_obs) * 4.0
    drift = np.where(rng.random(n_obs) < 0.2, rng.uniform(-0.8, 0.8, n_obs), 0.0)
    ox = x0[:, None] + vx[:, None] * t[None, :]
    oy = lane[:, None] + drift[:, None] * t[None, :]
    lim = dict(a=7.0710678118654755, b=2.8284271247461903, v_max=float(rng.uniform(15.0, 25.0)),
               a_max=float(rng.uniform(4.0, 8.0)), kappa_max=float(rng.uniform(0.1, 0.3)),
               c_max=float(rng.uniform(2.0, 5.0)), y_lb=-2.0, y_ub=4.0 * lanes - 2.0,
               v_min=float(rng.uniform(0.0, 2.0)))
    curv = None
    if seed % 3 == 2:
        curv = (np.array([0.0, 40.0, 90.0, 200.0]), rng.uniform(-0.04, 0.04, 4))
    b0 = np.array([0.0, rng.uniform(0.0, 4.0), rng.uniform(5.0, 20.0), rng.uniform(-1.0, 1.0),
                   rng.uniform(-1.0, 1.0), rng.uniform(-0.5, 0.5)])
    P = np.concatenate([rng.uniform(-2.0, 4.0 * lanes - 2.0, (B, 4)), rng.uniform(0.0, 25.0, (B, 4))], axis=1)
    return n_obs, ox, oy, lim, curv, b0, P


@pytest.mark.parametrize("seed", range(20))
def test_random_scene_matches_oracle(seed):
    import paper_2212_02224_b200 as bd
    n_obs, ox, oy, lim, curv, b0, P = _random_case(seed)
    basis = bd.build_basis(10, M, T, "bernstein")
    solver = bd.LowerLevelSolver(basis, bd.TrackingWeights(), bd.ParamLayout(4),
                                 bd.ProjectionConfig(1.0, ITERS, 1e-30), n_obs)
    lanes = [0, 8, 16, 64][(seed // 5) % 4]             # auto and every forced lane mapping
    if lanes:
        solver.context.set_option("lanes_per_sample", lanes)
    spec = bd.ConstraintSpec(ox, oy, lim["a"], lim["b"], lim["v_max"], lim["a_max"], lim["kappa_max"], lim["c_max"],
                             lim["y_lb"], lim["y_ub"], lim["v_min"], curv)
    _, proj = solver.solve(P, bd.PlanningScene(b0, spec))
    costs = solver.last_costs

    _, W, Wd, Wdd = O.basis_matrices(10, M, T)
    qp = O.tracking_qp(W, Wd, Wdd, 4)
    ol = O.Limits(ox.reshape(n_obs, M), oy.reshape(n_obs, M), lim["a"], lim["b"], lim["v_max"], lim["a_max"],
                  lim["kappa_max"], lim["c_max"], lim["y_lb"], lim["y_ub"], lim["v_min"], curv)
    xb, _, bb = O.stage1(qp, P, b0)
    aug = O.aug_qp(W, Wd, Wdd, qp.A_eq, n_obs, 1.0)
    out = O.am_project(aug, W, Wd, Wdd, xb, bb, ol, 1.0, ITERS, 1e-30)
    n = W.shape[1]
    ref_cost = O.speed_cost(out["xi"][:n].T @ Wd.T, out["xi"][n:].T @ Wd.T, lim["v_max"])

    assert proj.iterations_used == out["iterations"] == ITERS
    assert rel_err_per_sample_axis(proj.xi, out["xi"]) <= XI_TOL
    assert np.all(np.abs(proj.residuals - out["residuals"]) <= RES_TOL * (1.0 + out["residuals"]))
    assert np.all(np.abs(costs - ref_cost) <= COST_TOL * np.maximum(ref_cost, 1.0))
    hist = np.asarray(proj.residual_history)                # (iterations, B) per-iteration residuals
    assert hist.shape == out["history"].shape
    assert np.all(np.abs(hist - out["history"]) <= RES_TOL * (1.0 + out["history"]))


@pytest.mark.parametrize("seed", range(5))
def test_random_goal_layout_matches_oracle(seed):
    """Goal layout (pkg/batch_qp.py:189-192, 236-238): per-sample b with the terminal rows, the
    generic stage-1 path, behaviour vectors of 10."""
    import paper_2212_02224_b200 as bd
    n_obs, ox, oy, lim, curv, b0, P8 = _random_case(100 + seed)
    rng = np.random.default_rng(seed)
    P = np.concatenate([P8, np.stack([rng.uniform(40.0, 90.0, B), rng.uniform(-2.0, 10.0, B)], axis=1)], axis=1)
    basis = bd.build_basis(10, M, T, "bernstein")
    solver = bd.LowerLevelSolver(basis, bd.TrackingWeights(), bd.ParamLayout(4, with_goal=True),
                                 bd.ProjectionConfig(1.0, ITERS, 1e-30), n_obs)
    spec = bd.ConstraintSpec(ox, oy, lim["a"], lim["b"], lim["v_max"], lim["a_max"], lim["kappa_max"], lim["c_max"],
                             lim["y_lb"], lim["y_ub"], lim["v_min"], curv)
    _, proj = solver.solve(P, bd.PlanningScene(b0, spec))
    _, W, Wd, Wdd = O.basis_matrices(10, M, T)
    qp = O.tracking_qp(W, Wd, Wdd, 4, True)
    ol = O.Limits(ox.reshape(n_obs, M), oy.reshape(n_obs, M), lim["a"], lim["b"], lim["v_max"], lim["a_max"],
                  lim["kappa_max"], lim["c_max"], lim["y_lb"], lim["y_ub"], lim["v_min"], curv)
    xb, _, bb = O.stage1(qp, P, b0)
    aug = O.aug_qp(W, Wd, Wdd, qp.A_eq, n_obs, 1.0)
    out = O.am_project(aug, W, Wd, Wdd, xb, bb, ol, 1.0, ITERS, 1e-30)
    assert rel_err_per_sample_axis(proj.xi, out["xi"]) <= XI_TOL
    assert np.all(np.abs(proj.residuals - out["residuals"]) <= RES_TOL * (1.0 + out["residuals"]))


@pytest.mark.parametrize("seed", range(5))
def test_random_planner_default_shape_matches_oracle(seed):
    """The reference planner's default shape (PlannerEnvConfig: m = 50 over 10 s, 6 obstacles),
    which runs on its own compile-time specialisation of the AM kernel."""
    import paper_2212_02224_b200 as bd
    m, horizon = 50, 10.0
    n_obs, ox, oy, lim, curv, b0, P = _random_case(200 + seed, m, horizon, n_obs=6)
    basis = bd.build_basis(10, m, horizon, "bernstein")
    solver = bd.LowerLevelSolver(basis, bd.TrackingWeights(), bd.ParamLayout(4),
                                 bd.ProjectionConfig(1.0, ITERS, 1e-30), n_obs)
    spec = bd.ConstraintSpec(ox, oy, lim["a"], lim["b"], lim["v_max"], lim["a_max"], lim["kappa_max"], lim["c_max"],
                             lim["y_lb"], lim["y_ub"], lim["v_min"], None)
    _, proj = solver.solve(P, bd.PlanningScene(b0, spec))
    _, W, Wd, Wdd = O.basis_matrices(10, m, horizon)
    qp = O.tracking_qp(W, Wd, Wdd, 4)
    ol = O.Limits(ox, oy, lim["a"], lim["b"], lim["v_max"], lim["a_max"], lim["kappa_max"], lim["c_max"],
                  lim["y_lb"], lim["y_ub"], lim["v_min"], None)
    xb, _, bb = O.stage1(qp, P, b0)
    aug = O.aug_qp(W, Wd, Wdd, qp.A_eq, n_obs, 1.0)
    out = O.am_project(aug, W, Wd, Wdd, xb, bb, ol, 1.0, ITERS, 1e-30)
    assert rel_err_per_sample_axis(proj.xi, out["xi"]) <= XI_TOL
    assert np.all(np.abs(proj.residuals - out["residuals"]) <= RES_TOL * (1.0 + out["residuals"]))
