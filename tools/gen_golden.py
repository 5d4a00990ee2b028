"""Generate golden vectors by RUNNING THE REFERENCE (development container only).

    PYTHONPATH=/root/reference/pkg/src python tools/gen_golden.py [--only NAME ...]

Writes tests/golden/*.npz.  The reference (bilevel-drive 0.1.0, pure numpy/scipy)
is imported from /root/reference/pkg/src; it does not exist on the GPU box, so the
vectors are committed and the tests read only the .npz files.

Cases:
  basis            W/Wd/Wdd, stage-1 + aug KKTs for the BASELINE basis (pkg/basis.py, pkg/batch_qp.py,
                   pkg/projection.py:189-214)
  lower_*          LowerLevelSolver.solve outputs (pkg/bilevel.py:217-225) on synthetic highway scenes
  cem_c2           teacher-forced config-2 CEM trace (B=1000, N=4, n=150, q=100) via trace_hook
                   (pkg/bilevel.py:269-270)
  cem_small        free-running solve_bilevel with default_rng(3) (B=200, N=3) for the drop-in API
  worlds           build_scene / observe / controls_on_grid outputs
  sim              simulator ticks: spawn_world + step
  episodes         run_episode with scripted planners (EpisodeLog JSONL) + suite output files
  cem_variants     solve_bilevel with the goal layout and with a warm-start source
  planners         baseline planners' plan_cycle (vanilla, grid, goal, random) on a few worlds
  dense_c4         BASELINE config 4 at its stated size: one teacher-forced CEM iteration at B = 10 000
                   x 50 obstacles (LowerLevelSolver.solve sharded over CPU processes, then the
                   reference's rank_samples + update_distribution on the whole batch)
"""

from __future__ import annotations

import argparse
import json
import math
import os
import sys
import time

import numpy as np

sys.path.insert(0, "/root/reference/pkg/src")

from bilevel_drive import batch_qp  # noqa: E402
from bilevel_drive.basis import build_basis  # noqa: E402
from bilevel_drive.batch_qp import TrackingWeights  # noqa: E402
from bilevel_drive.behavior import ParamLayout  # noqa: E402
from bilevel_drive.bench import bilevel_config_for, canonical_scene  # noqa: E402
from bilevel_drive.bilevel import (  # noqa: E402
    BiLevelConfig, LowerLevelSolver, SamplingDistribution, rank_samples, solve_bilevel,
    update_distribution, upper_cost_batch,
)
from bilevel_drive.constraints import ConstraintSpec, PlanningScene  # noqa: E402
from bilevel_drive.highway import RoadSpec, ScenarioConfig, spawn_world  # noqa: E402
from bilevel_drive.planners import PlannerEnvConfig, build_scene  # noqa: E402
from bilevel_drive.projection import ProjectionConfig  # noqa: E402

OUT = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests", "golden")


def env_for(n_obs=10, m=100, T=5.0, iters=100, obstacle_range=120.0):
    return PlannerEnvConfig(horizon=T, num_samples=m, max_obstacles=n_obs, proj_iters=iters,
                            obstacle_range=obstacle_range)


def highway_scene(env, basis, lanes, density, vehicles, seed):
    world = spawn_world(ScenarioConfig(RoadSpec(lane_count=lanes), density=density, vehicle_count=vehicles,
                                       seed=seed))
    return build_scene(world, env, basis.times)


def scene_arrays(scene):
    sp = scene.spec
    d = dict(
        ox=sp.obstacles_x, oy=sp.obstacles_y, b0=scene.initial_state, lane_centers=scene.lane_centers,
        limits=np.array([sp.ellipse_a, sp.ellipse_b, sp.v_min, sp.v_max, sp.a_max, sp.kappa_max, sp.c_max,
                         sp.y_lb, sp.y_ub]),
    )
    if sp.road_curvature is not None:
        d["curv_x"] = np.asarray(sp.road_curvature[0], float)
        d["curv_k"] = np.asarray(sp.road_curvature[1], float)
    return d


def sample_params(env, scene, B, seed):
    cfg_mean = np.concatenate([np.full(env.m_seg, scene.initial_state[1]),
                               np.full(env.m_seg, np.hypot(scene.initial_state[2], scene.initial_state[3]))])
    cfg_cov = np.diag(np.concatenate([np.full(env.m_seg, env.sigma_offset ** 2),
                                      np.full(env.m_seg, env.sigma_speed ** 2)]))
    return SamplingDistribution(cfg_mean, cfg_cov).sample(B, np.random.default_rng(seed))


def run_lower(name, scene, params, *, n_obs, m=100, T=5.0, iters=100, tol=1e-3, rho=1.0, with_goal=False,
              weights=None):
    basis = build_basis(10, m, T, "bernstein")
    layout = ParamLayout(4, with_goal=with_goal)
    weights = weights or TrackingWeights()
    solver = LowerLevelSolver(basis, weights, layout, ProjectionConfig(rho, iters, tol), n_obs)
    t0 = time.time()
    sol, proj = solver.solve(params, scene)
    dt = time.time() - t0
    xd, yd = solver.velocities(proj.xi)
    costs = upper_cost_batch(xd, yd, scene.spec.v_max)
    out = dict(
        params=params, xi_bar=sol.xi, mu=sol.mu, xi=proj.xi, residuals=proj.residuals,
        history=proj.residual_history, iterations_used=proj.iterations_used, clip_conflicts=proj.clip_conflicts,
        costs=costs, rho=rho, max_iters=iters, tol=tol, m=m, T=T, with_goal=with_goal,
        weights=np.array([weights.k_p, weights.k_v, weights.w_smooth, weights.w_offset, weights.w_speed]),
        ref_seconds=dt, **scene_arrays(scene),
    )
    np.savez_compressed(os.path.join(OUT, f"lower_{name}.npz"), **out)
    print(f"lower_{name}: B={params.shape[0]} obs={n_obs} iters_used={proj.iterations_used} "
          f"conf={proj.clip_conflicts} rmax={proj.residuals.max():.3g} rmin={proj.residuals.min():.3g} {dt:.1f}s")


def gen_basis():
    d = {}
    for tag, (order, m, T, fam) in {"b100": (10, 100, 5.0, "bernstein"), "b50": (10, 50, 10.0, "bernstein"),
                                    "mono": (10, 100, 5.0, "monomial")}.items():
        bs = build_basis(order, m, T, fam)
        d[f"{tag}_W"], d[f"{tag}_Wd"], d[f"{tag}_Wdd"], d[f"{tag}_t"] = bs.W, bs.Wdot, bs.Wddot, bs.times
    bs = build_basis(10, 100, 5.0, "bernstein")
    for goal in (False, True):
        qp = batch_qp.build_qp_structure(bs, TrackingWeights(), ParamLayout(4, with_goal=goal))
        g = "goal_" if goal else ""
        d[g + "Q"], d[g + "A_eq"], d[g + "kkt"] = qp.Q, qp.A_eq, qp.kkt
        d[g + "qmx"], d[g + "qmy"] = qp.q_map_x, qp.q_map_y
    from bilevel_drive.projection import ProjectionOperator
    qp = batch_qp.build_qp_structure(bs, TrackingWeights(), ParamLayout(4))
    for n_obs in (0, 10, 50):
        op = ProjectionOperator(bs, qp, n_obs, ProjectionConfig())
        d[f"aug{n_obs}_kkt"] = op.aug.kkt
    np.savez_compressed(os.path.join(OUT, "basis.npz"), **d)
    print("basis written")


def gen_lower():
    env = env_for()
    basis = build_basis(10, 100, 5.0, "bernstein")
    sc = highway_scene(env, basis, 4, 2.0, 24, 0)
    run_lower("c1_s0", sc, sample_params(env, sc, 100, 0), n_obs=10)
    sc = highway_scene(env, basis, 2, 1.0, 12, 1)
    run_lower("c1_s1", sc, sample_params(env, sc, 100, 1), n_obs=10)
    # canonical: 3 parked vehicles + 7 sentinels at 1e4 m (pkg/bench.py:208-242)
    sc = canonical_scene(env)
    run_lower("canon", sc, sample_params(env, sc, 100, 2), n_obs=10)
    # dense 50-obstacle scene (config 4 scene recipe, smaller batch)
    env50 = env_for(n_obs=50, obstacle_range=250.0)
    sc = highway_scene(env50, basis, 4, 3.0, 80, 0)
    run_lower("dense50", sc, sample_params(env50, sc, 48, 3), n_obs=50)
    # B = 1
    sc = highway_scene(env, basis, 4, 2.0, 24, 5)
    run_lower("b1", sc, sample_params(env, sc, 1, 5), n_obs=10, iters=30)
    # early exit: sentinel-only scene, feasible set-points
    sc0 = highway_scene(env, basis, 2, 0.5, 2, 7)
    spec = sc0.spec
    far = ConstraintSpec(obstacles_x=spec.obstacles_x * 0 + 1e4 + 100.0 * np.arange(10)[:, None],
                         obstacles_y=np.zeros_like(spec.obstacles_y), ellipse_a=spec.ellipse_a,
                         ellipse_b=spec.ellipse_b, v_max=spec.v_max, a_max=spec.a_max, kappa_max=spec.kappa_max,
                         c_max=spec.c_max, y_lb=spec.y_lb, y_ub=spec.y_ub, v_min=spec.v_min)
    sc = PlanningScene(initial_state=sc0.initial_state, spec=far, lane_centers=sc0.lane_centers)
    for tag, scale in (("early4", 0.5), ("early39", 1.0)):
        rng = np.random.default_rng(11)
        p = np.concatenate([scale * 0.3 * rng.standard_normal((16, 4)), 10.0 + scale * rng.standard_normal((16, 4))],
                           axis=1)
        run_lower(tag, sc, p, n_obs=10, iters=80)
    # curved road (tabulated kappa, np.interp semantics incl. both clamps)
    curved = ConstraintSpec(obstacles_x=spec.obstacles_x, obstacles_y=spec.obstacles_y, ellipse_a=spec.ellipse_a,
                            ellipse_b=spec.ellipse_b, v_max=spec.v_max, a_max=spec.a_max,
                            kappa_max=spec.kappa_max, c_max=spec.c_max, y_lb=spec.y_lb, y_ub=spec.y_ub,
                            v_min=3.0,
                            road_curvature=(np.array([5.0, 20.0, 40.0, 60.0]), np.array([0.01, -0.3, 0.05, 0.15])))
    sc = PlanningScene(initial_state=sc0.initial_state, spec=curved, lane_centers=sc0.lane_centers)
    run_lower("curve", sc, sample_params(env, sc, 32, 8), n_obs=10, iters=40)
    # zero obstacles
    none = ConstraintSpec(obstacles_x=np.zeros((0, 100)), obstacles_y=np.zeros((0, 100)), ellipse_a=spec.ellipse_a,
                          ellipse_b=spec.ellipse_b, v_max=spec.v_max, a_max=spec.a_max, kappa_max=spec.kappa_max,
                          c_max=spec.c_max, y_lb=spec.y_lb, y_ub=spec.y_ub, v_min=spec.v_min)
    sc = PlanningScene(initial_state=np.array([0.0, 4.0, 15.0, 0.5, 1.0, -0.2]), spec=none,
                       lane_centers=sc0.lane_centers)
    run_lower("nobs0", sc, sample_params(env, sc, 24, 9), n_obs=0, iters=25)
    # goal layout: neq = 9, per-sample b, w_offset = w_speed = 0 (pkg/planners.py:387-412)
    sc = highway_scene(env, basis, 4, 1.0, 16, 4)
    x0, v0 = sc.initial_state[0], float(np.hypot(sc.initial_state[2], sc.initial_state[3]))
    reach = max(v0, 0.3 * env.v_max) * env.horizon
    pts = np.array([np.concatenate([np.zeros(4), np.zeros(4), [x0 + f * reach, y]])
                    for f in (0.5, 0.7, 0.85, 1.0) for y in sc.lane_centers])
    w = TrackingWeights(w_offset=0.0, w_speed=0.0)
    run_lower("goal", sc, pts, n_obs=10, iters=50, with_goal=True, weights=w)


def gen_cem_c2():
    env = env_for()
    basis = build_basis(10, 100, 5.0, "bernstein")
    sc = highway_scene(env, basis, 4, 2.0, 24, 0)
    solver = LowerLevelSolver(basis, TrackingWeights(), ParamLayout(4), ProjectionConfig(1.0, 100, 1e-3), 10)
    env2 = PlannerEnvConfig(horizon=5.0, num_samples=100, max_obstacles=10, proj_iters=100, batch_size=1000,
                            constraint_elites=150, elites=100, iterations=4)
    cfg = bilevel_config_for(env2, sc, batch_size=1000, iterations=4)
    rec = {k: [] for k in ("params", "xi", "residuals", "costs", "elite_idx", "cons_idx", "elite_aug", "mean", "cov",
                           "iters_used", "conflicts", "history_max")}
    dist = [SamplingDistribution(cfg.init_mean, cfg.init_cov)]

    def hook(it, params, proj, costs, elite_idx):
        cons, el, ea = rank_samples(proj.residuals, costs, cfg.constraint_elites, cfg.elites, cfg.residual_weight)
        assert np.array_equal(el, elite_idx)
        nd = update_distribution(dist[-1], params[el], ea, cfg.eta, cfg.gamma)
        dist.append(nd)
        rec["params"].append(params)
        rec["xi"].append(proj.xi)
        rec["residuals"].append(proj.residuals)
        rec["costs"].append(costs)
        rec["elite_idx"].append(el)
        rec["cons_idx"].append(cons)
        rec["elite_aug"].append(ea)
        rec["mean"].append(nd.mean)
        rec["cov"].append(nd.cov)
        rec["iters_used"].append(proj.iterations_used)
        rec["conflicts"].append(proj.clip_conflicts)
        rec["history_max"].append(proj.residual_history.max(axis=1))
        print(f"  cem it {it}: iters={proj.iterations_used} r0={np.sum(proj.residuals == 0)}", flush=True)

    t0 = time.time()
    res = solve_bilevel(sc, solver, cfg, np.random.default_rng(0), trace_hook=hook)
    dt = time.time() - t0
    stats = np.array([[s.iteration, s.elite_mean_upper_cost, s.best_augmented_cost, s.cov_trace, s.residual_min,
                       s.residual_median, s.residual_max] for s in res.diagnostics])
    out = {k: np.array(v) for k, v in rec.items()}
    out.update(scene_arrays(sc))
    out.update(init_mean=cfg.init_mean, init_cov=cfg.init_cov, stats=stats, best_index=res.best.index,
               best_xi=np.concatenate([res.best.coeffs.cx, res.best.coeffs.cy]), best_cost=res.best.upper_cost,
               best_residual=res.best.residual, best_aug=res.best.augmented_cost,
               final_mean=res.distribution.mean, final_cov=res.distribution.cov,
               cfg=np.array([cfg.batch_size, cfg.constraint_elites, cfg.elites, cfg.iterations, cfg.eta, cfg.gamma,
                             cfg.residual_weight]), ref_seconds=dt)
    np.savez_compressed(os.path.join(OUT, "cem_c2.npz"), **out)
    print(f"cem_c2 written ({dt:.1f}s)")


def gen_cem_small():
    env = env_for(iters=40)
    basis = build_basis(10, 100, 5.0, "bernstein")
    sc = highway_scene(env, basis, 2, 1.5, 14, 3)
    solver = LowerLevelSolver(basis, TrackingWeights(), ParamLayout(4), ProjectionConfig(1.0, 40, 1e-3), 10)
    cfg = BiLevelConfig(batch_size=200, constraint_elites=60, elites=20, iterations=3, eta=0.7, gamma=0.9,
                        residual_weight=1.0,
                        init_mean=np.concatenate([np.full(4, sc.initial_state[1]), np.full(4, 10.0)]),
                        init_cov=np.diag(np.concatenate([np.full(4, 1.5 ** 2), np.full(4, 3.0 ** 2)])))
    t0 = time.time()
    res = solve_bilevel(sc, solver, cfg, np.random.default_rng(3))
    dt = time.time() - t0
    stats = np.array([[s.iteration, s.elite_mean_upper_cost, s.best_augmented_cost, s.cov_trace, s.residual_min,
                       s.residual_median, s.residual_max] for s in res.diagnostics])
    out = scene_arrays(sc)
    out.update(init_mean=cfg.init_mean, init_cov=cfg.init_cov, stats=stats, best_index=res.best.index,
               best_params=res.best.params.to_vector(),
               best_xi=np.concatenate([res.best.coeffs.cx, res.best.coeffs.cy]), best_cost=res.best.upper_cost,
               best_residual=res.best.residual, best_aug=res.best.augmented_cost,
               final_mean=res.distribution.mean, final_cov=res.distribution.cov, seed=3, am_iters=40,
               cfg=np.array([cfg.batch_size, cfg.constraint_elites, cfg.elites, cfg.iterations, cfg.eta, cfg.gamma,
                             cfg.residual_weight]), ref_seconds=dt)
    np.savez_compressed(os.path.join(OUT, "cem_small.npz"), **out)
    print(f"cem_small written ({dt:.1f}s), best idx {res.best.index}")


def gen_scenes():
    """Scenes only (for the product's synthetic scene generator parity)."""
    out = {}
    for seed in range(6):
        for lanes, dens, veh, nobs, rng_ in ((4, 2.0, 24, 10, 120.0), (4, 3.0, 80, 50, 250.0), (2, 1.0, 12, 10, 120.0)):
            env = env_for(n_obs=nobs, obstacle_range=rng_)
            basis = build_basis(10, 100, 5.0, "bernstein")
            sc = highway_scene(env, basis, lanes, dens, veh, seed)
            tag = f"s{seed}_l{lanes}_d{dens}_v{veh}_o{nobs}"
            out[tag + "_ox"], out[tag + "_oy"] = sc.spec.obstacles_x, sc.spec.obstacles_y
            out[tag + "_b0"] = sc.initial_state
            out[tag + "_lim"] = scene_arrays(sc)["limits"]
    np.savez_compressed(os.path.join(OUT, "scenes.npz"), **out)
    print("scenes written")


def gen_worlds():
    """World snapshots after a few simulator steps (nonzero heading / steer / lane changes) with the
    reference's build_scene (pkg/planners.py:116-160), ego_flat_state (:99-113) and observe
    (pkg/highway.py:208-246) outputs, plus controls_on_grid (pkg/planners.py:209-216) of the
    projected trajectories of lower_c1_s0."""
    from bilevel_drive.basis import flat_to_controls, SpeedSingularity
    from bilevel_drive.highway import observe, step
    from bilevel_drive.planners import ego_flat_state
    out = {}
    k = 0
    for lanes, dens, veh, seed, nsteps, nobs, rng_ in ((4, 2.0, 24, 0, 0, 10, 120.0), (4, 2.0, 24, 1, 17, 10, 120.0),
                                                       (2, 1.0, 12, 2, 25, 10, 120.0), (4, 3.0, 80, 3, 9, 50, 250.0),
                                                       (3, 1.5, 30, 4, 31, 10, 60.0), (2, 0.4, 3, 5, 5, 10, 120.0)):
        world = spawn_world(ScenarioConfig(RoadSpec(lane_count=lanes), density=dens, vehicle_count=veh, seed=seed))
        for t in range(nsteps):
            step(world, 0.8 * np.sin(0.3 * t), 0.03 * np.cos(0.2 * t))
        env = env_for(n_obs=nobs, obstacle_range=rng_)
        basis = build_basis(10, 100, 5.0, "bernstein")
        sc = build_scene(world, env, basis.times)
        e = world.ego
        out[f"w{k}_ego"] = np.array([e.x, e.y, e.psi, e.v, e.accel, e.steer, e.length, e.width])
        out[f"w{k}_veh"] = np.array([[v.x, v.y, v.psi, v.v, v.lateral_rate] for v in world.neighbors])
        out[f"w{k}_road"] = np.array([world.road.lane_count, world.road.lane_width])
        out[f"w{k}_env"] = np.array([nobs, rng_, env.wheelbase])
        out[f"w{k}_ox"], out[f"w{k}_oy"] = sc.spec.obstacles_x, sc.spec.obstacles_y
        out[f"w{k}_b0"] = sc.initial_state
        assert np.array_equal(sc.initial_state, ego_flat_state(world, env.wheelbase))
        out[f"w{k}_lim"] = scene_arrays(sc)["limits"]
        out[f"w{k}_obs"] = observe(world)
        k += 1
    out["n_worlds"] = k
    # control emission on the simulator grid (dt = 0.1 s over the 5 s horizon, wheelbase 2.5)
    g = np.load(os.path.join(OUT, "lower_c1_s0.npz"))
    basis = build_basis(10, 100, 5.0, "bernstein")
    times = np.arange(int(5.0 / 0.1)) * 0.1
    env = env_for()
    acc, ste, sing = [], [], []
    from bilevel_drive.basis import TrajectoryCoeffs
    xis = np.concatenate([g["xi"], g["xi_bar"], np.zeros((22, 1))], axis=1)
    for j in range(xis.shape[1]):
        try:
            c = flat_to_controls(basis, TrajectoryCoeffs.from_stacked(xis[:, j]), env.wheelbase, times=times)
            acc.append(np.clip(c.accel, -env.a_max, env.a_max))
            ste.append(np.clip(c.delta, -env.steer_limit, env.steer_limit))
            sing.append(0)
        except SpeedSingularity:
            acc.append(np.full(len(times), np.nan))
            ste.append(np.full(len(times), np.nan))
            sing.append(1)
    out.update(ctrl_xi=xis.T.copy(), ctrl_accel=np.array(acc), ctrl_steer=np.array(ste), ctrl_singular=np.array(sing),
               ctrl_times=times, ctrl_limits=np.array([env.wheelbase, env.a_max, env.steer_limit]))
    np.savez_compressed(os.path.join(OUT, "worlds.npz"), **out)
    print(f"worlds written ({k} worlds, {xis.shape[1]} control sets, {sum(sing)} singular)")


SIM_CASES = (  # lanes, density, vehicles, seed, steps, control script
    (4, 2.0, 24, 0, 60, "gentle"), (3, 1.5, 30, 4, 80, "gentle"), (4, 3.0, 80, 3, 40, "gentle"),
    (2, 1.0, 12, 2, 60, "ram"), (2, 0.4, 3, 5, 50, "swerve"), (4, 2.5, 40, 7, 100, "weave"),
)


def sim_controls(kind, t):
    if kind == "gentle":
        return 0.8 * np.sin(0.3 * t), 0.03 * np.cos(0.2 * t)
    if kind == "ram":
        return 3.0, 0.0
    if kind == "swerve":
        return 0.5, 0.12
    return 1.2 * np.sin(0.11 * t), 0.08 * np.sin(0.05 * t)       # weave


def gen_sim():
    """Closed-loop simulator ticks (pkg/highway.py:358-410): spawned world state (pkg/highway.py:168-205)
    and the full world state after every step under scripted ego controls (IDM + MOBIL neighbours,
    RK4 ego, SAT collision, lane departure)."""
    from bilevel_drive.highway import step
    out = {}
    changes = 0
    for k, (lanes, dens, nveh, seed, nsteps, kind) in enumerate(SIM_CASES):
        world = spawn_world(ScenarioConfig(RoadSpec(lane_count=lanes), density=dens, vehicle_count=nveh, seed=seed))

        def grab():
            e = world.ego
            ego = np.array([e.x, e.y, e.psi, e.v, e.accel, e.steer, e.length, e.width, e.target_speed])
            veh = np.array([[v.x, v.y, v.psi, v.v, v.lateral_rate, v.length, v.width, v.target_speed,
                             v.target_lane, v.cooldown, v.accel, v.lane_index] for v in world.neighbors])
            ws = np.array([world.time, world.step_count, float(world.collided),
                           -1.0 if world.collision_step is None else float(world.collision_step),
                           float(world.lane_departed)])
            return ego, veh, ws

        e0, v0, w0 = grab()
        egos, vehs, wss, ctrl = [], [], [], []
        for t in range(nsteps):
            a, d = sim_controls(kind, t)
            before = [v.target_lane for v in world.neighbors]
            step(world, float(a), float(d))
            changes += sum(b != v.target_lane for b, v in zip(before, world.neighbors))
            e, v, w = grab()
            egos.append(e); vehs.append(v); wss.append(w); ctrl.append((a, d))
        out[f"s{k}_road"] = np.array([lanes, world.road.lane_width, world.road.length, world.dt])
        out[f"s{k}_ego0"], out[f"s{k}_veh0"], out[f"s{k}_w0"] = e0, v0, w0
        out[f"s{k}_ego"], out[f"s{k}_veh"], out[f"s{k}_w"] = np.array(egos), np.array(vehs), np.array(wss)
        out[f"s{k}_ctrl"] = np.array(ctrl, dtype=float)
        out[f"s{k}_cfg"] = np.array([lanes, dens, nveh, seed, nsteps])
        print(f"  sim case {k}: collided={world.collided} at {world.collision_step}, departed={world.lane_departed}")
    out["n_cases"] = len(SIM_CASES)
    np.savez_compressed(os.path.join(OUT, "sim.npz"), **out)
    print(f"sim written ({len(SIM_CASES)} worlds, {changes} neighbour lane-change decisions)")


class _ScriptedPlanner:
    """Dummy planner for run_episode: cycle c returns constant (accel, steer) grids."""

    name = "scripted"

    def __init__(self, kind):
        self.kind = kind
        self.c = 0

    def reset(self):
        self.c = 0

    def plan_cycle(self, world):
        a, d = episode_controls(self.kind, self.c)
        self.c += 1
        return np.full(50, a), np.full(50, d), {"cycle": self.c - 1}


def episode_controls(kind, c):
    if kind == "cruise":
        return 0.5 * np.sin(0.7 * c), 0.02 * np.cos(0.3 * c)
    if kind == "ram":
        return 3.0, 0.0
    return 1.0, 0.0                                                      # "run": to the end of the road


EPISODE_CASES = (  # lanes, density, vehicles, seed, episode_length, road_length, planner kind
    (4, 2.0, 24, 0, 60, 1500.0, "cruise"), (2, 1.0, 12, 2, 150, 1500.0, "ram"),
    (3, 1.5, 20, 5, 150, 140.0, "run"), (4, 2.5, 40, 7, 23, 1500.0, "cruise"),
)


def gen_episodes():
    """Closed-loop run_episode (pkg/highway.py:487-532) with scripted planners: EpisodeLog JSONL
    (pkg/highway.py:436-474); plus suite outputs of write_outputs (pkg/bench.py:173-205)."""
    import tempfile
    from dataclasses import replace
    from bilevel_drive import bench as rbench
    from bilevel_drive.highway import run_episode
    out = {}
    for k, (lanes, dens, nveh, seed, length, road_len, kind) in enumerate(EPISODE_CASES):
        sc = ScenarioConfig(RoadSpec(lane_count=lanes, length=road_len), density=dens, vehicle_count=nveh,
                            seed=seed, episode_length=length, scenario_id=f"case{k}")
        log = run_episode(sc, _ScriptedPlanner(kind), replan_stride=5)
        with tempfile.TemporaryDirectory() as d:
            path = os.path.join(d, "ep.jsonl")
            log.write_jsonl(path)
            out[f"e{k}_jsonl"] = np.array(open(path).read())
        out[f"e{k}_cfg"] = np.array([lanes, dens, nveh, seed, length, road_len])
        out[f"e{k}_kind"] = np.array(kind)
        print(f"  episode {k}: steps={len(log.steps)} collided={log.collided} departed={log.lane_departed}")
    out["n_cases"] = len(EPISODE_CASES)
    # suite outputs for fixed metric rows (byte format + config fingerprint)
    env = rbench.PlannerEnvConfig(batch_size=100, iterations=3)
    suite = rbench.BenchmarkSuite(scenarios=(ScenarioConfig(RoadSpec(lane_count=3), 1.5, 20, 0, scenario_id="a"),
                                             ScenarioConfig(RoadSpec(lane_count=4), 2.0, 24, 0, scenario_id="b")),
                                  planners=("mpc-bilevel", "mpc-vanilla"), episodes_per_cell=3, env=env)
    rows = [rbench.MetricsRow("mpc-bilevel", "a", 3, 1, 1 / 3, 11.25, 0.0123, 0),
            rbench.MetricsRow("mpc-bilevel", "b", 3, 0, 0.0, float("nan"), float("nan"), 3),
            rbench.MetricsRow("mpc-vanilla", "a", 3, 2, 2 / 3, 9.876543210123, 0.5, 1),
            rbench.MetricsRow("mpc-vanilla", "b", 3, 0, 0.0, 12.0, 1e-4, 0)]
    walls = {"mpc-bilevel/a": 1.5, "mpc-bilevel/b": 2.25, "mpc-vanilla/a": 0.1}
    with tempfile.TemporaryDirectory() as d:
        paths = rbench.write_outputs(suite, rows, walls, d)
        out["suite_metrics"] = np.array(open(paths["metrics"]).read())
        out["suite_timings"] = np.array(open(paths["timings"]).read())
        out["suite_hash"] = np.array(json.load(open(paths["manifest"]))["config_hash"])
    np.savez_compressed(os.path.join(OUT, "episodes.npz"), **out)
    print("episodes written")


def gen_cem_variants():
    """solve_bilevel (pkg/bilevel.py:228-295) with the goal layout (per-sample goal rows in b,
    pkg/batch_qp.py:189-192,236-238) and with a WarmStartSource for iteration 1
    (pkg/bilevel.py:250-251), seeded default_rng(5)."""
    from bilevel_drive.behavior import WarmStartSource
    env = env_for(iters=40)
    basis = build_basis(10, 100, 5.0, "bernstein")
    sc = highway_scene(env, basis, 3, 1.5, 18, 6)
    out = scene_arrays(sc)
    y0, v0 = sc.initial_state[1], 10.0
    cases = {
        "goal": (ParamLayout(4, with_goal=True),
                 np.concatenate([np.full(4, y0), np.full(4, v0), [60.0, 4.0]]),
                 np.diag(np.concatenate([np.full(4, 1.5 ** 2), np.full(4, 3.0 ** 2), [25.0, 4.0]])), None),
        "warm": (ParamLayout(4), np.concatenate([np.full(4, y0), np.full(4, v0)]),
                 np.diag(np.concatenate([np.full(4, 1.5 ** 2), np.full(4, 3.0 ** 2)])),
                 np.random.default_rng(11).normal([y0] * 4 + [v0] * 4, [1.0] * 4 + [2.0] * 4, (37, 8))),
    }
    cases["curve"] = (ParamLayout(4), cases["warm"][1], cases["warm"][2], None)
    from dataclasses import replace as dc_replace
    curved = PlanningScene(initial_state=sc.initial_state, lane_centers=sc.lane_centers,
                           spec=dc_replace(sc.spec, road_curvature=(np.array([0.0, 30.0, 70.0, 140.0]),
                                                                    np.array([0.0, 0.03, 0.06, 0.02]))))
    out.update(curve_xs=curved.spec.road_curvature[0], curve_ks=curved.spec.road_curvature[1])
    for name, (layout, mean, cov, warm) in cases.items():
        scene = curved if name == "curve" else sc
        solver = LowerLevelSolver(basis, TrackingWeights(), layout, ProjectionConfig(1.0, 40, 1e-3), 10)
        cfg = BiLevelConfig(batch_size=200, constraint_elites=60, elites=20, iterations=3, eta=0.7, gamma=0.9,
                            residual_weight=1.0, init_mean=mean, init_cov=cov)
        ws = WarmStartSource(warm, layout) if warm is not None else None
        res = solve_bilevel(scene, solver, cfg, np.random.default_rng(5), warm_start=ws)
        stats = np.array([[s.elite_mean_upper_cost, s.best_augmented_cost, s.cov_trace, s.residual_min,
                           s.residual_median, s.residual_max] for s in res.diagnostics])
        out.update({f"{name}_mean": mean, f"{name}_cov": cov, f"{name}_best_index": res.best.index,
                    f"{name}_best_params": res.best.params.to_vector(),
                    f"{name}_best_xi": np.concatenate([res.best.coeffs.cx, res.best.coeffs.cy]),
                    f"{name}_stats": stats, f"{name}_final_mean": res.distribution.mean})
        if warm is not None:
            out[f"{name}_samples"] = warm
        print(f"  cem {name}: best {res.best.index}, cost {res.best.upper_cost:.2f}")
    np.savez_compressed(os.path.join(OUT, "cem_variants.npz"), **out)
    print("cem_variants written")


def gen_planners():
    """Baseline planners' plan_cycle (pkg/planners.py:198-216, 309-412) on spawned + stepped worlds
    with the PlannerEnvConfig defaults: controls on the 0.1 s grid and the plan diagnostics."""
    from bilevel_drive.highway import step
    from bilevel_drive.planners import make_planner
    out = {}
    worlds = []
    for k, (lanes, dens, nveh, seed, nsteps) in enumerate(((4, 2.0, 24, 0, 0), (3, 1.5, 20, 5, 13), (2, 1.0, 10, 9, 7))):
        w = spawn_world(ScenarioConfig(RoadSpec(lane_count=lanes), density=dens, vehicle_count=nveh, seed=seed))
        for t in range(nsteps):
            step(w, 0.6 * np.sin(0.4 * t), 0.02 * np.cos(0.3 * t))
        worlds.append(w)
        e = w.ego
        out[f"w{k}_ego"] = np.array([e.x, e.y, e.psi, e.v, e.accel, e.steer, e.length, e.width, e.target_speed])
        out[f"w{k}_veh"] = np.array([[v.x, v.y, v.psi, v.v, v.lateral_rate, v.length, v.width, v.target_speed,
                                      v.target_lane, v.cooldown, v.accel, v.lane_index] for v in w.neighbors])
        out[f"w{k}_road"] = np.array([w.road.lane_count, w.road.lane_width])
        out[f"w{k}_world"] = np.array([w.time, w.step_count, 0.0, -1.0, 0.0])
    env = PlannerEnvConfig()
    for k, w in enumerate(worlds):                   # MPCBiLevelPlanner: two cycles (warm mean, rng stream)
        planner = make_planner("mpc-bilevel", env, seed=k)
        for c in range(2):
            acc, ste, info = planner.plan_cycle(w)
            out[f"mpc-bilevel_{k}_{c}_accel"], out[f"mpc-bilevel_{k}_{c}_steer"] = acc, ste
            out[f"mpc-bilevel_{k}_{c}_residual"], out[f"mpc-bilevel_{k}_{c}_cost"] = info["residual"], info["upper_cost"]
            out[f"mpc-bilevel_{k}_{c}_params"] = planner._warm_mean
    for name in ("mpc-vanilla", "mpc-grid", "batch-mpc-goal", "mpc-random"):
        for k, w in enumerate(worlds):
            planner = make_planner(name, env, seed=k)
            acc, ste, info = planner.plan_cycle(w)
            out[f"{name}_{k}_accel"], out[f"{name}_{k}_steer"] = acc, ste
            out[f"{name}_{k}_residual"], out[f"{name}_{k}_cost"] = info["residual"], info["upper_cost"]
    out["n_worlds"] = len(worlds)
    np.savez_compressed(os.path.join(OUT, "planners.npz"), **out)
    print("planners written")


def gen_harness():
    """The harness callers of the path (pkg/bench.py:208-367): canonical_scene, bilevel_config_for,
    an emit_convergence_trace run, and replay_to_csv of the episode logs in episodes.npz."""
    import tempfile
    from bilevel_drive import bench as rbench
    out = {}
    env = PlannerEnvConfig(batch_size=200, iterations=4)
    sc = rbench.canonical_scene(env)
    cfg = rbench.bilevel_config_for(env, sc, batch_size=300, iterations=2)
    out.update(canon_ox=sc.spec.obstacles_x, canon_oy=sc.spec.obstacles_y, canon_b0=sc.initial_state,
               canon_lanes=sc.lane_centers, canon_limits=np.array([sc.spec.ellipse_a, sc.spec.ellipse_b, sc.spec.v_min,
                                                                   sc.spec.v_max, sc.spec.a_max, sc.spec.kappa_max,
                                                                   sc.spec.c_max, sc.spec.y_lb, sc.spec.y_ub]),
               cfg_mean=cfg.init_mean, cfg_cov=cfg.init_cov,
               cfg_sizes=np.array([cfg.batch_size, cfg.constraint_elites, cfg.elites, cfg.iterations]))
    trace = rbench.emit_convergence_trace(env, seed=3)
    out["trace_jsonl"] = np.array("".join(json.dumps(r, sort_keys=True) + "\n" for r in trace))
    eps = np.load(os.path.join(OUT, "episodes.npz"))
    with tempfile.TemporaryDirectory() as d:
        for k in range(int(eps["n_cases"])):
            log_path, csv_path = os.path.join(d, f"e{k}.jsonl"), os.path.join(d, f"e{k}.csv")
            with open(log_path, "w") as fh:
                fh.write(str(eps[f"e{k}_jsonl"]))
            rbench.replay_to_csv(log_path, csv_path)
            out[f"replay_{k}"] = np.array(open(csv_path).read())
    out["n_replays"] = int(eps["n_cases"])
    np.savez_compressed(os.path.join(OUT, "harness.npz"), **out)
    print(f"harness written ({len(trace)} trace records)")


def gen_absurd():
    """Set-points far outside any road (|offset| up to 1e300): the reference's fp64 projection
    returns huge / NaN residuals for them (pkg/projection.py:216-339, pkg/constraints.py:95-153)
    and they rank last; a CEM run with such warm-start rows (pkg/bilevel.py:249-251) is not
    degraded."""
    import warnings
    from bilevel_drive.behavior import WarmStartSource
    env = PlannerEnvConfig(num_samples=100, max_obstacles=10)
    sc = canonical_scene(env)
    basis = build_basis(10, 100, 5.0, "bernstein")
    solver = LowerLevelSolver(basis, TrackingWeights(), ParamLayout(4), ProjectionConfig(1.0, 100, 1e-3), 10)
    P = np.random.default_rng(1).normal([0] * 4 + [12] * 4, [1.5] * 4 + [3] * 4, (12, 8))
    P[3, :4] = 1e25
    P[7, 4:] = 1e300
    P[9] = -1e18
    P[10, 1] = 1e17
    with warnings.catch_warnings():
        warnings.simplefilter("ignore")
        _, proj = solver.solve(P, sc)
        xd, yd = solver.velocities(proj.xi)
    from bilevel_drive.bilevel import upper_cost_batch
    out = {"lower_params": P, "lower_resid": proj.residuals, "lower_cost": upper_cost_batch(xd, yd, sc.spec.v_max),
           "lower_xi": proj.xi}
    warm = np.random.default_rng(2).normal([0] * 4 + [12] * 4, [1.5] * 4 + [3] * 4, (200, 8))
    warm[5, :4] = 1e25
    warm[50, 4:] = -1e18
    warm[120, 1] = 1e17
    warm[199] = 3e20
    cfg = bilevel_config_for(env, sc, batch_size=200, iterations=3)
    cfg = BiLevelConfig(batch_size=200, constraint_elites=60, elites=20, iterations=3, eta=cfg.eta, gamma=cfg.gamma,
                        residual_weight=cfg.residual_weight, init_mean=cfg.init_mean, init_cov=cfg.init_cov)
    elites = []
    with warnings.catch_warnings():
        warnings.simplefilter("ignore")
        res = solve_bilevel(sc, solver, cfg, np.random.default_rng(4), warm_start=WarmStartSource(warm, ParamLayout(4)),
                            trace_hook=lambda it, p, pr, c, e: elites.append(np.asarray(e)))
    out.update(warm=warm, cem_mean=cfg.init_mean, cem_cov=cfg.init_cov, cem_best_index=res.best.index,
               cem_best_params=res.best.params.to_vector(), cem_elites=np.stack(elites), cem_degraded=res.degraded,
               cem_stats=np.array([[s.elite_mean_upper_cost, s.best_augmented_cost, s.cov_trace, s.residual_min,
                                    s.residual_median, s.residual_max] for s in res.diagnostics]),
               cem_final_mean=res.distribution.mean, cem_final_cov=res.distribution.cov)
    np.savez_compressed(os.path.join(OUT, "absurd.npz"), **out)
    print(f"absurd written: lower resid {proj.residuals[[3, 7, 9, 10]]}, cem best {res.best.index}")


def gen_worlds_random():
    """24 randomised worlds (lanes, density, vehicle count incl. none, simulator steps, obstacle
    count and range) with the reference's build_scene / ego_flat_state / observe outputs."""
    from bilevel_drive.highway import observe, step
    rng = np.random.default_rng(2026)
    out = {}
    n = 24
    for k in range(n):
        lanes = int(rng.integers(2, 6))
        dens = float(rng.uniform(0.3, 3.5))
        veh = int(rng.choice([0, 1, 2, 5, 12, 24, 40, 80, 90]))
        seed = int(rng.integers(0, 10_000))
        nsteps = int(rng.integers(0, 40))
        nobs = int(rng.choice([1, 6, 10, 25, 50]))
        rng_ = float(rng.uniform(30.0, 300.0))
        world = spawn_world(ScenarioConfig(RoadSpec(lane_count=lanes), density=dens, vehicle_count=veh, seed=seed))
        for t in range(nsteps):
            step(world, 1.2 * np.sin(0.37 * t + k), 0.05 * np.cos(0.23 * t + k))
        env = env_for(n_obs=nobs, obstacle_range=rng_)
        basis = build_basis(10, 100, 5.0, "bernstein")
        sc = build_scene(world, env, basis.times)
        e = world.ego
        out[f"w{k}_ego"] = np.array([e.x, e.y, e.psi, e.v, e.accel, e.steer, e.length, e.width])
        out[f"w{k}_veh"] = np.array([[v.x, v.y, v.psi, v.v, v.lateral_rate] for v in world.neighbors]).reshape(-1, 5)
        out[f"w{k}_road"] = np.array([world.road.lane_count, world.road.lane_width])
        out[f"w{k}_env"] = np.array([nobs, rng_, env.wheelbase])
        out[f"w{k}_ox"], out[f"w{k}_oy"] = sc.spec.obstacles_x, sc.spec.obstacles_y
        out[f"w{k}_b0"] = sc.initial_state
        out[f"w{k}_lim"] = scene_arrays(sc)["limits"]
        out[f"w{k}_obs"] = observe(world)
    out["n_worlds"] = n
    # control emission (flat_to_controls on the 0.1 s grid) of 96 randomised trajectories:
    # forward motion at 0-25 m/s with lateral wiggles, some stopping or reversing (singular)
    from bilevel_drive.basis import SpeedSingularity, TrajectoryCoeffs, flat_to_controls
    basis = build_basis(10, 100, 5.0, "bernstein")
    times = np.arange(int(5.0 / 0.1)) * 0.1
    env = env_for()
    u = np.linspace(0.0, 1.0, 11)
    xis, acc, ste, sing = [], [], [], []
    for j in range(96):
        v = rng.uniform(-3.0, 25.0) if j % 8 else rng.uniform(-0.5, 0.5)
        cx = v * 5.0 * u + rng.normal(0.0, 1.0 + 0.2 * abs(v), 11) * (u * (1 - u) * 4)
        cy = rng.uniform(-2.0, 10.0) + rng.normal(0.0, 1.5, 11)
        if j % 16 == 0:                              # standing still: SpeedSingularity
            cx, cy = np.full(11, cx[0]), np.full(11, cy[0])
        xi = np.concatenate([cx, cy])
        xis.append(xi)
        try:
            c = flat_to_controls(basis, TrajectoryCoeffs.from_stacked(xi), env.wheelbase, times=times)
            acc.append(np.clip(c.accel, -env.a_max, env.a_max))
            ste.append(np.clip(c.delta, -env.steer_limit, env.steer_limit))
            sing.append(0)
        except SpeedSingularity:
            acc.append(np.full(len(times), np.nan))
            ste.append(np.full(len(times), np.nan))
            sing.append(1)
    out.update(ctrl_xi=np.array(xis), ctrl_accel=np.array(acc), ctrl_steer=np.array(ste), ctrl_singular=np.array(sing))
    np.savez_compressed(os.path.join(OUT, "worlds_random.npz"), **out)
    print(f"worlds_random written ({n} worlds)")


def _c4_solve(args):
    """One shard of the config-4 batch through the reference's LowerLevelSolver.solve."""
    params, seed_scene = args
    env50 = env_for(n_obs=50, obstacle_range=250.0)
    basis = build_basis(10, 100, 5.0, "bernstein")
    sc = highway_scene(env50, basis, 4, 3.0, 80, seed_scene)
    solver = LowerLevelSolver(basis, TrackingWeights(), ParamLayout(4), ProjectionConfig(1.0, 100, 1e-3), 50)
    _, proj = solver.solve(params, sc)
    xd, yd = solver.velocities(proj.xi)
    return (proj.xi, proj.residuals, upper_cost_batch(xd, yd, sc.spec.v_max), proj.iterations_used,
            proj.residual_history.max(axis=1))


def gen_dense_c4(B=10_000, shards=40, keep_xi=1000):
    """BASELINE config 4 (B = 10 000 samples x 50 obstacles x 100 timesteps, 100 AM iterations):
    one CEM iteration of solve_bilevel (pkg/bilevel.py:249-292), teacher-forced from the initial
    distribution of bilevel_config_for (pkg/bench.py:245-261) drawn with default_rng(4).

    The batch is split over CPU processes.  A split solve equals the unsplit one exactly when no
    shard takes the batch-global early exit (pkg/projection.py:329): every shard then runs all
    100 iterations, so the whole batch would too, and every other operation is per sample.  This
    is checked twice: each shard's iterations_used == 100, and at B = 64 a 2-way split is
    compared with the unsplit solve (max |diff| recorded)."""
    import multiprocessing as mp
    env50 = env_for(n_obs=50, obstacle_range=250.0)
    basis = build_basis(10, 100, 5.0, "bernstein")
    sc = highway_scene(env50, basis, 4, 3.0, 80, 0)
    env2 = PlannerEnvConfig(horizon=5.0, num_samples=100, max_obstacles=50, proj_iters=100, batch_size=B,
                            constraint_elites=150, elites=100, iterations=1, obstacle_range=250.0)
    cfg = bilevel_config_for(env2, sc, batch_size=B, iterations=1)
    params = SamplingDistribution(cfg.init_mean, cfg.init_cov).sample(B, np.random.default_rng(4))
    t0 = time.time()
    with mp.get_context("fork").Pool(os.cpu_count()) as pool:
        small = pool.map(_c4_solve, [(params[:64], 0), (params[:32], 0), (params[32:64], 0)])
        parts = pool.map(_c4_solve, [(c, 0) for c in np.array_split(params, shards)])
    dt = time.time() - t0
    split_diff = max(float(np.abs(np.concatenate([small[1][0], small[2][0]], axis=1) - small[0][0]).max()),
                     float(np.abs(np.concatenate([small[1][1], small[2][1]]) - small[0][1]).max()))
    used = np.array([p[3] for p in parts])
    assert np.all(used == 100) and small[0][3] == 100, used
    xi = np.concatenate([p[0] for p in parts], axis=1)
    res = np.concatenate([p[1] for p in parts])
    costs = np.concatenate([p[2] for p in parts])
    hist_max = np.max(np.stack([p[4] for p in parts]), axis=0)
    cons, el, ea = rank_samples(res, costs, cfg.constraint_elites, cfg.elites, cfg.residual_weight)
    nd = update_distribution(SamplingDistribution(cfg.init_mean, cfg.init_cov), params[el], ea, cfg.eta, cfg.gamma)
    keep = np.unique(np.concatenate([np.arange(keep_xi), el]))
    out = dict(params=params, residuals=res, costs=costs, xi_keep_idx=keep, xi_keep=xi[:, keep],
               cons_idx=cons, elite_idx=el, elite_aug=ea, mean=nd.mean, cov=nd.cov, init_mean=cfg.init_mean,
               init_cov=cfg.init_cov, iters_used=used, history_max=hist_max, split_check_maxdiff=split_diff,
               cfg=np.array([B, cfg.constraint_elites, cfg.elites, 1, cfg.eta, cfg.gamma, cfg.residual_weight]),
               ref_seconds=dt, ref_processes=os.cpu_count(), **scene_arrays(sc))
    np.savez_compressed(os.path.join(OUT, "dense_c4.npz"), **out)
    print(f"dense_c4 written: {dt:.0f}s on {os.cpu_count()} processes, split check {split_diff:.2e}, "
          f"r=0: {int(np.sum(res == 0))}, best {el[0]}")


if __name__ == "__main__":
    ap = argparse.ArgumentParser()
    ap.add_argument("--only", nargs="*", default=None)
    a = ap.parse_args()
    os.makedirs(OUT, exist_ok=True)
    jobs = {"basis": gen_basis, "lower": gen_lower, "scenes": gen_scenes, "cem_small": gen_cem_small,
            "cem_c2": gen_cem_c2, "worlds": gen_worlds, "sim": gen_sim, "episodes": gen_episodes, "cem_variants": gen_cem_variants, "planners": gen_planners,
            "harness": gen_harness, "absurd": gen_absurd, "worlds_random": gen_worlds_random,
            "dense_c4": gen_dense_c4}
    for name, fn in jobs.items():
        if a.only is None or name in a.only:
            fn()
