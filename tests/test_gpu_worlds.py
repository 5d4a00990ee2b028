"""GPU: device scene construction and control emission against the
reference's build_scene / ego_flat_state / observe / controls_on_grid outputs."""

import numpy as np
import pytest

from tests.golden_io import load

pytestmark = pytest.mark.gpu


def _solver(n_obs):
    import paper_2212_02224_b200 as bd
    basis = bd.build_basis(10, 100, 5.0, "bernstein")
    return bd.LowerLevelSolver(basis, bd.TrackingWeights(), bd.ParamLayout(4), bd.ProjectionConfig(1.0, 30, 1e-3),
                               n_obs)


def _world(g, k):
    from paper_2212_02224_b200.worlds import WorldBatch
    veh = g[f"w{k}_veh"]
    return WorldBatch(g[f"w{k}_ego"][None], veh[None], np.array([veh.shape[0]], np.int32), g[f"w{k}_road"][None])


@pytest.mark.parametrize("k", range(6))
def test_build_scene_and_observe_match_reference(k):
    from paper_2212_02224_b200.worlds import PlannerEnv, build_scenes
    g = load("worlds")
    nobs, rng_, wb = g[f"w{k}_env"]
    solver = _solver(int(nobs))
    env = PlannerEnv(max_obstacles=int(nobs), obstacle_range=float(rng_), wheelbase=float(wb))
    ox, oy, b0, lim, obs = build_scenes(solver.context, solver.basis, _world(g, k), env, outputs=True)
    np.testing.assert_array_equal(ox[0], g[f"w{k}_ox"])
    np.testing.assert_array_equal(oy[0], g[f"w{k}_oy"])
    np.testing.assert_allclose(b0[0], g[f"w{k}_b0"], rtol=1e-14, atol=1e-14)
    np.testing.assert_array_equal(lim[0], g[f"w{k}_lim"])
    np.testing.assert_allclose(obs[0], g[f"w{k}_obs"], rtol=1e-13, atol=1e-13)


@pytest.mark.parametrize("k", range(24))
def test_build_scene_randomised_worlds_match_reference(k):
    """24 randomised worlds (2-5 lanes, 0-90 vehicles, 0-40 simulator steps, 1-50 obstacle rows,
    30-300 m range; tests/golden/worlds_random.npz from the reference) through the device builder."""
    from paper_2212_02224_b200.worlds import PlannerEnv, build_scenes
    g = load("worlds_random")
    nobs, rng_, wb = g[f"w{k}_env"]
    solver = _solver(int(nobs))
    env = PlannerEnv(max_obstacles=int(nobs), obstacle_range=float(rng_), wheelbase=float(wb))
    ox, oy, b0, lim, obs = build_scenes(solver.context, solver.basis, _world(g, k), env, outputs=True)
    np.testing.assert_array_equal(ox[0], g[f"w{k}_ox"])
    np.testing.assert_array_equal(oy[0], g[f"w{k}_oy"])
    np.testing.assert_allclose(b0[0], g[f"w{k}_b0"], rtol=1e-14, atol=1e-14)
    np.testing.assert_array_equal(lim[0], g[f"w{k}_lim"])
    np.testing.assert_allclose(obs[0], g[f"w{k}_obs"], rtol=1e-13, atol=1e-13)


def test_device_built_scene_drives_the_solver():
    """Scenes built on the device give the same projection as the host-uploaded reference scene."""
    import paper_2212_02224_b200 as bd
    from paper_2212_02224_b200.worlds import PlannerEnv, WorldBatch, build_scenes
    g = load("worlds")
    solver = _solver(10)
    rng = np.random.default_rng(0)
    P = np.concatenate([rng.normal(4.0, 1.5, (64, 4)), rng.normal(10.0, 3.0, (64, 4))], axis=1)
    a, b, vmin, vmax, amax, kmax, cmax, ylb, yub = g["w1_lim"]
    spec = bd.ConstraintSpec(g["w1_ox"], g["w1_oy"], a, b, vmax, amax, kmax, cmax, ylb, yub, vmin)
    _, ref = solver.solve(P, bd.PlanningScene(g["w1_b0"], spec))
    build_scenes(solver.context, solver.basis, _world(g, 1), PlannerEnv())
    solver.projector._scene_key = ("device-built",)
    xi = np.empty((64, 22))
    res = np.empty(64)
    cost = np.empty(64)
    used = np.zeros(1, np.int32)
    conf = np.zeros(1, np.int64)
    solver.context.call("bd_solve_lower", 1, 64, P, 30, 1e-3, None, None, xi, res, cost, None, used, conf)
    np.testing.assert_allclose(xi.T, ref.xi, rtol=1e-6, atol=1e-6)


def test_control_emission_matches_reference():
    from paper_2212_02224_b200.worlds import ControlEmitter, PlannerEnv
    g = load("worlds")
    solver = _solver(10)
    em = ControlEmitter(solver.context, solver.basis, 5.0, 0.1, PlannerEnv())
    np.testing.assert_array_equal(em.times, g["ctrl_times"])
    acc, ste, sing = em.emit(g["ctrl_xi"])
    np.testing.assert_array_equal(sing, g["ctrl_singular"].astype(bool))
    ok = ~sing
    np.testing.assert_allclose(acc[ok], g["ctrl_accel"][ok], rtol=1e-10, atol=1e-10)
    np.testing.assert_allclose(ste[ok], g["ctrl_steer"][ok], rtol=1e-10, atol=1e-12)


def test_control_emission_randomised_trajectories():
    """96 randomised trajectories (incl. stopping / reversing ones that hit SpeedSingularity)
    against the reference's flat_to_controls (tests/golden/worlds_random.npz)."""
    from paper_2212_02224_b200.worlds import ControlEmitter, PlannerEnv
    g = load("worlds_random")
    solver = _solver(10)
    em = ControlEmitter(solver.context, solver.basis, 5.0, 0.1, PlannerEnv())
    acc, ste, sing = em.emit(g["ctrl_xi"])
    np.testing.assert_array_equal(sing, g["ctrl_singular"].astype(bool))
    ok = ~sing
    np.testing.assert_allclose(acc[ok], g["ctrl_accel"][ok], rtol=1e-10, atol=1e-10)
    np.testing.assert_allclose(ste[ok], g["ctrl_steer"][ok], rtol=1e-10, atol=1e-12)


def test_fleet_plan_cycle_from_worlds():
    import paper_2212_02224_b200 as bd
    from paper_2212_02224_b200.fleet import FleetPlanner
    from paper_2212_02224_b200.worlds import ControlEmitter, PlannerEnv, WorldBatch
    g = load("worlds")
    ks = [0, 1, 2, 4, 5]                     # the 10-obstacle worlds
    n_max = max(g[f"w{k}_veh"].shape[0] for k in ks)
    veh = np.zeros((len(ks), n_max, 5))
    for i, k in enumerate(ks):
        veh[i, : g[f"w{k}_veh"].shape[0]] = g[f"w{k}_veh"]
    worlds = WorldBatch(np.stack([g[f"w{k}_ego"] for k in ks]), veh,
                        np.array([g[f"w{k}_veh"].shape[0] for k in ks], np.int32),
                        np.stack([g[f"w{k}_road"] for k in ks]))
    basis = bd.build_basis(10, 100, 5.0, "bernstein")
    fp = FleetPlanner(basis, bd.TrackingWeights(), bd.ParamLayout(4), bd.ProjectionConfig(1.0, 50, 1e-3), 10,
                      bd.BiLevelConfig(500, 100, 50, 3, 0.7, 0.9, 1.0))
    em = ControlEmitter(fp.context, basis, 5.0, 0.1, PlannerEnv())
    acc, ste, sing, res = fp.plan_cycle(worlds, PlannerEnv(), em, seed=3)
    assert acc.shape == (5, 50) and np.all(res.iterations_done == 3)
    assert not sing.any() and np.all(np.abs(acc) <= 6.0) and np.all(np.isfinite(ste))
    # same as planning each world alone (scene_offset keeps the Philox stream per world); a lone
    # world runs with another lane mapping, so sums differ in rounding order only
    for i in range(5):
        one = WorldBatch(worlds.ego[i:i + 1], worlds.veh[i:i + 1], worlds.n_veh[i:i + 1], worlds.road[i:i + 1])
        a1, s1, _, r1 = fp.plan_cycle(one, PlannerEnv(), em, seed=3, scene_offset=i)
        assert r1.best_index[0] == res.best_index[i]
        np.testing.assert_allclose(a1[0], acc[i], rtol=1e-4, atol=1e-4)


def test_spawned_worlds_build_the_host_recipe_scenes():
    from paper_2212_02224_b200.scenes import HighwayRecipe, highway_scene, spawn_worlds
    from paper_2212_02224_b200.worlds import PlannerEnv, build_scenes
    solver = _solver(10)
    worlds = spawn_worlds(range(5))
    ox, oy, b0, lim, _ = build_scenes(solver.context, solver.basis, worlds, PlannerEnv(), outputs=True)
    for s in range(5):
        sc = highway_scene(s)
        np.testing.assert_array_equal(ox[s], sc.spec.obstacles_x)
        np.testing.assert_array_equal(oy[s], sc.spec.obstacles_y)
        np.testing.assert_array_equal(b0[s], sc.initial_state)


@pytest.mark.parametrize("mixed", [False, True])
def test_device_built_scene_with_road_curvature(mixed):
    """road_curvature (pkg/planners.py:154): a device-built curved-road scene solves exactly like
    the host-uploaded ConstraintSpec(road_curvature=...) scene; a world without curvature in the
    same batch behaves as road_curvature=None (zero table)."""
    import paper_2212_02224_b200 as bd
    from paper_2212_02224_b200.worlds import PlannerEnv, WorldBatch, build_scenes
    g = load("worlds")
    solver = _solver(10)
    rng = np.random.default_rng(3)
    P = np.concatenate([rng.normal(4.0, 1.5, (64, 4)), rng.normal(14.0, 3.0, (64, 4))], axis=1)
    a, b, vmin, vmax, amax, kmax, cmax, ylb, yub = g["w1_lim"]
    curv = ((0.0, 40.0, 90.0, 160.0), (0.0, 0.02, 0.05, 0.01))
    spec = bd.ConstraintSpec(g["w1_ox"], g["w1_oy"], a, b, vmax, amax, kmax, cmax, ylb, yub, vmin,
                             road_curvature=(np.array(curv[0]), np.array(curv[1])))
    _, ref = solver.solve(P, bd.PlanningScene(g["w1_b0"], spec))
    w = _world(g, 1)
    if mixed:      # second world: the same world without curvature, a shorter table padded for the first
        flat = bd.ConstraintSpec(g["w1_ox"], g["w1_oy"], a, b, vmax, amax, kmax, cmax, ylb, yub, vmin)
        _, ref_flat = solver.solve(P, bd.PlanningScene(g["w1_b0"], flat))
        w = WorldBatch(np.repeat(w.ego, 2, 0), np.repeat(w.veh, 2, 0), np.repeat(w.n_veh, 2), np.repeat(w.road, 2, 0),
                       [curv, None])
    else:
        w = WorldBatch(w.ego, w.veh, w.n_veh, w.road, [curv])
    build_scenes(solver.context, solver.basis, w, PlannerEnv())
    solver.projector._scene_key = ("device-built",)
    S = w.size
    xi = np.empty((S, 64, 22))
    res, cost = np.empty((S, 64)), np.empty((S, 64))
    used, conf = np.zeros(S, np.int32), np.zeros(S, np.int64)
    solver.context.call("bd_solve_lower", S, 64, np.ascontiguousarray(np.repeat(P[None], S, 0)), 30, 1e-3, None,
                        None, xi, res, cost, None, used, conf)
    np.testing.assert_allclose(xi[0].T, ref.xi, rtol=1e-6, atol=1e-6)
    np.testing.assert_allclose(res[0], ref.residuals, rtol=1e-5, atol=1e-5)
    if mixed:
        np.testing.assert_allclose(xi[1].T, ref_flat.xi, rtol=1e-6, atol=1e-6)
        assert not np.allclose(xi[0], xi[1])
