"""SPEC.md acceptance criteria 2-6 measured on the device path.

    python tools/acceptance.py [--episodes 50] [--out profiles/r01/acceptance.json]

2: 50 seeded straight 2-lane scenes with 1-4 static obstacles, 250-sample batches from the
   canonical set-point distribution: batches whose 100-iteration AM reaches a batch-max residual
   <= 1e-3, and A_eq xi = b to 1e-8 for every output.
3: canonical static-obstacle scene, n=1000 / 150 / 50, gamma=0.9, N=5: seeds whose elite-mean
   cost at iteration 5 <= iteration 1 and whose trace(Sigma) decreases (of 50).
4: closed-loop collision rates over seeded episodes, dense 4-lane (density 2, 24 vehicles) for
   mpc-bilevel / mpc-random / mpc-vanilla, and sparse 2-lane (density 1, 10 vehicles).
5: mean speed of collision-free sparse 2-lane episodes, mpc-bilevel vs mpc-vanilla.
6: wall time of one Alg. 1 iteration at batch 250 and 1000 (emit_timing) and the
   factorisations during the solves.
The criteria are the SPEC's directional targets; the reference planner is the same algorithm
(closed-loop parity: DESIGN.md §4b), so these numbers describe both.
"""
import argparse
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--episodes", type=int, default=50)
ap.add_argument("--out", default=None)
a = ap.parse_args()

import paper_2212_02224_b200 as bd  # noqa: E402
from paper_2212_02224_b200 import harness  # noqa: E402
from paper_2212_02224_b200.episodes import BenchmarkSuite, run_suite  # noqa: E402
from paper_2212_02224_b200.planners import PlannerEnvConfig  # noqa: E402
from paper_2212_02224_b200.sim import RoadSpec, ScenarioConfig  # noqa: E402

out = {}
# ---- 2
env = PlannerEnvConfig(num_samples=100, max_obstacles=10)
basis = bd.build_basis(10, 100, 5.0, "bernstein")
solver = bd.LowerLevelSolver(basis, bd.TrackingWeights(), bd.ParamLayout(4), bd.ProjectionConfig(1.0, 100, 1e-3), 10)
canon = harness.canonical_scene(env)
reached, eq_ok, iters_used = 0, 0, []
for seed in range(50):
    rng = np.random.default_rng(seed)
    k = int(rng.integers(1, 5))
    ox = np.full((10, 100), 1e4) + 100.0 * np.arange(10)[:, None]
    oy = np.zeros((10, 100))
    ox[:k] = rng.uniform(30.0, 120.0, k)[:, None]
    oy[:k] = 4.0 * rng.integers(0, 2, k)[:, None]
    sp = canon.spec
    spec = bd.ConstraintSpec(ox, oy, sp.ellipse_a, sp.ellipse_b, sp.v_max, sp.a_max, sp.kappa_max, sp.c_max, sp.y_lb,
                             sp.y_ub, sp.v_min)
    scene = bd.PlanningScene(canon.initial_state, spec, canon.lane_centers)
    c = harness.bilevel_config_for(env, scene, batch_size=250)
    p = c.init_mean + rng.standard_normal((250, 8)) @ np.linalg.cholesky(c.init_cov).T
    _, proj = solver.solve(p, scene)
    reached += proj.iterations_used < 100 or float(proj.residuals.max()) <= 1e-3
    iters_used.append(int(proj.iterations_used))
    A, b = solver.qp.A_eq, scene.initial_state[:, None]
    eq_ok += bool(np.abs(A @ proj.xi - b).max() <= 1e-8 * (1 + np.abs(proj.xi).max()))
out["criterion2"] = {"scenes": 50, "batches_reaching_tol": int(reached), "eq_constraints_hold": int(eq_ok),
                     "median_iterations_used": float(np.median(iters_used)),
                     "target": ">= 45 batches reach 1e-3; all satisfy A_eq xi = b", "pass": bool(reached >= 45 and eq_ok == 50)}
# ---- 3
scene = harness.canonical_scene(env)
c = harness.bilevel_config_for(env, scene, batch_size=1000, iterations=5)
cfg = bd.BiLevelConfig(1000, 150, 50, 5, c.eta, 0.9, c.residual_weight, c.init_mean, c.init_cov)
cost_ok = trace_ok = 0
for seed in range(50):
    d = bd.solve_bilevel(scene, solver, cfg, np.random.default_rng(seed)).diagnostics
    cost_ok += d[4].elite_mean_upper_cost <= d[0].elite_mean_upper_cost
    trace_ok += d[4].cov_trace < d[0].cov_trace
out["criterion3"] = {"seeds": 50, "elite_cost_not_worse": int(cost_ok), "trace_decreases": int(trace_ok),
                     "target": ">= 45 each", "pass": bool(cost_ok >= 45 and trace_ok >= 45)}
# ---- 4 / 5
seeds = tuple(range(a.episodes))
dense = ScenarioConfig(RoadSpec(4), 2.0, 24, 0, scenario_id="dense4")
sparse = ScenarioConfig(RoadSpec(2), 1.0, 10, 0, scenario_id="sparse2")
suite = BenchmarkSuite(scenarios=(dense, sparse), planners=("mpc-bilevel", "mpc-random", "mpc-vanilla"),
                       episodes_per_cell=len(seeds), seeds=seeds, env=PlannerEnvConfig())
t0 = time.perf_counter()
rows, _, nf = run_suite(suite)
wall = time.perf_counter() - t0
rate = {(r.planner, r.scenario_id): r for r in rows}
out["criterion4"] = {
    "episodes_per_cell": len(seeds), "wall_s": wall,
    "dense4_collision_rate": {p: rate[(p, "dense4")].collision_rate for p in suite.planners},
    "sparse2_collision_rate": {p: rate[(p, "sparse2")].collision_rate for p in suite.planners},
    "target": "dense: bilevel <= random and <= vanilla; sparse: bilevel <= 0.05",
    "pass": bool(rate[("mpc-bilevel", "dense4")].collision_rate <= min(rate[("mpc-random", "dense4")].collision_rate,
                                                                     rate[("mpc-vanilla", "dense4")].collision_rate)
                 and rate[("mpc-bilevel", "sparse2")].collision_rate <= 0.05)}
bl, va = rate[("mpc-bilevel", "sparse2")].mean_speed, rate[("mpc-vanilla", "sparse2")].mean_speed
out["criterion5"] = {"sparse2_mean_speed_bilevel": bl, "sparse2_mean_speed_vanilla": va,
                     "ratio": bl / va if va == va and va else None, "target": ">= 0.9",
                     "pass": bool(va == va and bl >= 0.9 * va)}
# ---- 6
rows6 = harness.emit_timing(env, batch_sizes=(250, 1000), iteration_counts=(1, 4))
out["criterion6"] = {"rows": rows6, "target": "one iteration <= 1.0 s at 250, <= 5.0 s at 1000; no refactorisation",
                     "pass": bool(all(r["per_iteration_s"] <= (1.0 if r["batch"] == 250 else 5.0)
                                      and r["factorizations_during_solve"] == 0 for r in rows6))}
out["numerical_failure"] = bool(nf)
print(json.dumps(out, indent=1))
if a.out:
    with open(a.out, "w") as fh:
        json.dump(out, fh, indent=1)
