"""Pin the CPU oracle (oracle/port.py) to vectors produced by running the reference itself."""

import math

import numpy as np
import pytest

import oracle as O
from tests.golden_io import LOWER_CASES, load, oracle_limits, rel_err_per_sample_axis


def test_basis_matches_reference():
    g = load("basis")
    for tag, args in {"b100": (10, 100, 5.0, "bernstein"), "b50": (10, 50, 10.0, "bernstein"),
                      "mono": (10, 100, 5.0, "monomial")}.items():
        t, W, Wd, Wdd = O.basis_matrices(*args)
        np.testing.assert_array_equal(t, g[tag + "_t"])
        np.testing.assert_allclose(W, g[tag + "_W"], rtol=0, atol=1e-14)
        np.testing.assert_allclose(Wd, g[tag + "_Wd"], rtol=0, atol=1e-13)
        np.testing.assert_allclose(Wdd, g[tag + "_Wdd"], rtol=0, atol=1e-12)


@pytest.mark.parametrize("goal", [False, True])
def test_qp_structure_matches_reference(goal):
    g = load("basis")
    _, W, Wd, Wdd = O.basis_matrices(10, 100, 5.0)
    qp = O.tracking_qp(W, Wd, Wdd, 4, with_goal=goal)
    p = "goal_" if goal else ""
    np.testing.assert_allclose(qp.Q, g[p + "Q"], rtol=1e-13, atol=1e-9)
    np.testing.assert_array_equal(qp.A_eq, g[p + "A_eq"])
    np.testing.assert_allclose(qp.qmx, g[p + "qmx"], rtol=1e-13, atol=1e-10)
    np.testing.assert_allclose(qp.qmy, g[p + "qmy"], rtol=1e-13, atol=1e-10)
    for n_obs in (0, 10, 50):
        aug = O.aug_qp(W, Wd, Wdd, qp.A_eq if not goal else load("basis")["A_eq"], n_obs, 1.0)
        np.testing.assert_allclose(aug.kkt, g[f"aug{n_obs}_kkt"], rtol=1e-13, atol=1e-10)


@pytest.mark.parametrize("case", LOWER_CASES)
def test_lower_level_oracle_matches_reference(case):
    g = load("lower_" + case)
    _, W, Wd, Wdd = O.basis_matrices(10, int(g["m"]), float(g["T"]))
    k_p, k_v, ws, wo, wv = g["weights"]
    qp = O.tracking_qp(W, Wd, Wdd, 4, bool(g["with_goal"]), k_p, k_v, ws, wo, wv)
    lim = oracle_limits(g)
    xb, mu, b = O.stage1(qp, g["params"], g["b0"])
    np.testing.assert_allclose(xb, g["xi_bar"], rtol=1e-10, atol=1e-9)
    np.testing.assert_allclose(mu, g["mu"], rtol=1e-8, atol=1e-6)
    aug = O.aug_qp(W, Wd, Wdd, qp.A_eq, lim.n_obs, float(g["rho"]))
    out = O.am_project(aug, W, Wd, Wdd, xb, b, lim, float(g["rho"]), int(g["max_iters"]), float(g["tol"]))
    assert out["iterations"] == int(g["iterations_used"])
    assert out["conflicts"] == int(g["clip_conflicts"])
    assert rel_err_per_sample_axis(out["xi"], g["xi"]) < 1e-9
    np.testing.assert_allclose(out["residuals"], g["residuals"], rtol=1e-7, atol=1e-9)
    np.testing.assert_allclose(out["history"], g["history"], rtol=1e-7, atol=1e-9)
    n = W.shape[1]
    c = O.speed_cost(out["xi"][:n].T @ Wd.T, out["xi"][n:].T @ Wd.T, lim.v_max)
    np.testing.assert_allclose(c, g["costs"], rtol=1e-10)


def test_cem_small_free_running_matches_reference():
    """Free-running CEM with the caller's rng reproduces the reference result exactly."""
    g = load("cem_small")
    _, W, Wd, Wdd = O.basis_matrices(10, 100, 5.0)
    qp = O.tracking_qp(W, Wd, Wdd, 4)
    lim = oracle_limits(g)
    aug = O.aug_qp(W, Wd, Wdd, qp.A_eq, lim.n_obs, 1.0)
    B, n, q, N, eta, gamma, w = g["cfg"]
    tr = O.cem_cycle(qp, aug, W, Wd, Wdd, g["b0"], lim, g["init_mean"], g["init_cov"], batch=int(B),
                     n_cons=int(n), n_elite=int(q), iters=int(N), eta=eta, gamma=gamma, w_res=w,
                     rng=np.random.default_rng(int(g["seed"])), am_iters=int(g["am_iters"]))
    np.testing.assert_allclose(np.array(tr.stats), g["stats"][:, 1:], rtol=1e-8, atol=1e-10)
    assert int(tr.elite_idx[-1][0]) == int(g["best_index"])
    np.testing.assert_allclose(tr.mean[-1], g["final_mean"], rtol=1e-9)
    np.testing.assert_allclose(tr.cov[-1], g["final_cov"], rtol=1e-8, atol=1e-12)


@pytest.mark.slow
def test_cem_c2_teacher_forced_iteration1():
    """Config-2 trace, CEM iteration 1 only (oracle at B=1000 takes ~20 s)."""
    g = load("cem_c2")
    _, W, Wd, Wdd = O.basis_matrices(10, 100, 5.0)
    qp = O.tracking_qp(W, Wd, Wdd, 4)
    lim = oracle_limits(g)
    aug = O.aug_qp(W, Wd, Wdd, qp.A_eq, lim.n_obs, 1.0)
    B, n, q, N, eta, gamma, w = g["cfg"]
    tr = O.cem_cycle(qp, aug, W, Wd, Wdd, g["b0"], lim, g["init_mean"], g["init_cov"], batch=int(B),
                     n_cons=int(n), n_elite=int(q), iters=1, eta=eta, gamma=gamma, w_res=w,
                     params_per_iter=[g["params"][0]])
    np.testing.assert_array_equal(tr.elite_idx[0], g["elite_idx"][0])
    np.testing.assert_array_equal(tr.cons_idx[0], g["cons_idx"][0])
    np.testing.assert_allclose(tr.mean[0], g["mean"][0], rtol=1e-10)


def test_dense_config4_oracle_matches_reference_subset():
    """Config 4 (tests/golden/dense_c4.npz, B = 10 000 x 50 obstacles run by the reference): the
    oracle reproduces a subset of the batch (per-sample independent: the reference's shards all
    ran the full 100 iterations) and the reference's ranking + refit on the whole batch."""
    g = load("dense_c4")
    _, W, Wd, Wdd = O.basis_matrices(10, 100, 5.0)
    qp = O.tracking_qp(W, Wd, Wdd, 4)
    lim = oracle_limits(g)
    sub = np.array([0, 1, 2, 3, 990, 4097, 9999])
    xb, _, b = O.stage1(qp, g["params"][sub], g["b0"])
    out = O.am_project(O.aug_qp(W, Wd, Wdd, qp.A_eq, 50, 1.0), W, Wd, Wdd, xb, b, lim, 1.0, 100, -1.0)
    np.testing.assert_allclose(out["residuals"], g["residuals"][sub], rtol=1e-9, atol=1e-9)
    keep = {int(k): j for j, k in enumerate(g["xi_keep_idx"])}
    have = [i for i, s in enumerate(sub) if int(s) in keep]
    assert rel_err_per_sample_axis(out["xi"][:, have], g["xi_keep"][:, [keep[int(sub[i])] for i in have]]) <= 1e-9
    n, q, w = int(g["cfg"][1]), int(g["cfg"][2]), float(g["cfg"][6])
    cons, el, ea = O.rank_two_stage(g["residuals"], g["costs"], n, q, w)
    np.testing.assert_array_equal(cons, g["cons_idx"])
    np.testing.assert_array_equal(el, g["elite_idx"])
    mu, C = O.refit_gaussian(g["init_mean"], g["init_cov"], g["params"][el], ea, float(g["cfg"][4]),
                             float(g["cfg"][5]))
    np.testing.assert_allclose(mu, g["mean"], rtol=1e-12, atol=1e-12)
    np.testing.assert_allclose(C, g["cov"], rtol=1e-12, atol=1e-12)


def test_spec_examples():
    # polar identity: xdot=3, ydot=4 -> alpha=atan2(4,3), d=5
    _, av, _, _, dv, _ = O.polar_split(np.array([[3.0]]), np.array([[4.0]]), np.zeros((1, 1)), np.zeros((1, 1)))
    assert math.isclose(dv[0, 0], 5.0) and math.isclose(av[0, 0], math.atan2(4, 3))
    # clip example: d_a=2, |sin|=0.5, kappa_max=0.2 -> v_lo contribution sqrt(5)
    lim = O.Limits(np.zeros((0, 1)), np.zeros((0, 1)), 1.0, 1.0, 20.0, 6.0, 0.2, 3.0, -2.0, 2.0, 0.0)
    _, dv, _, _ = O.coupled_clip(np.array([0.0]), np.array([0.1]), np.array([math.pi / 6]), np.array([2.0]),
                                 None, np.array([2.0]), np.array([0.0]), lim)
    assert math.isclose(dv[0], math.sqrt(5.0), rel_tol=1e-12)
    # upper cost: stationary trajectory, v_max=20, m samples -> m*400
    assert O.speed_cost(np.zeros((1, 50)), np.zeros((1, 50)), 20.0)[0] == 50 * 400.0
    # elite tie-break: residuals [3,1,2], n=2 -> {1,2}
    cons, _, _ = O.rank_two_stage(np.array([3.0, 1.0, 2.0]), np.zeros(3), 2, 1, 1.0)
    assert list(cons) == [1, 2]
    # eta = 1, single elite -> mean = p, cov = 1e-6 I
    mu, C = O.refit_gaussian(np.zeros(2), np.eye(2), np.array([[1.0, 2.0]]), np.array([5.0]), 1.0, 0.9)
    np.testing.assert_allclose(mu, [1.0, 2.0])
    np.testing.assert_allclose(C, 1e-6 * np.eye(2), atol=1e-18)
