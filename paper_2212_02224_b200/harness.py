"""The reference harness's callers of the path, on the device (pkg/bench.py:207-353, pkg/cli.py).

* :func:`emit_timing` — the bi-level loop's wall-time table across batch sizes and CEM iteration
  counts, with the factorisation counter sampled around each solve (it must stay at zero: the
  shared KKT factorisations happen once per solver).
* :func:`emit_convergence_trace` — per-iteration convergence records on the canonical scene
  through ``solve_bilevel``'s ``trace_hook`` (elite-mean cost, residual quantiles, lateral
  envelope of the projected batch, covariance trace).
* :func:`replay_to_csv` — an episode log flattened to one row per vehicle and tick.

``python -m paper_2212_02224_b200 {bench,trace,time,replay}`` exposes them with the reference
CLI's arguments (``bench`` runs a YAML suite through :func:`.episodes.run_suite`).
"""

from __future__ import annotations

import time

import numpy as np

from . import batch_qp
from .basis import build_basis
from .behavior import ParamLayout
from .bilevel import BiLevelConfig, LowerLevelSolver, solve_bilevel
from .constraints import ConstraintSpec, PlanningScene
from .episodes import EpisodeLog
from .planners import PlannerEnvConfig
from .sim import RoadSpec

__all__ = ["canonical_scene", "bilevel_config_for", "emit_timing", "emit_convergence_trace", "replay_to_csv"]

# three parked vehicles alternating lanes on a two-lane road (longitudinal position, lane index)
_PARKED = ((45.0, 0), (80.0, 1), (120.0, 0))


def canonical_scene(env: PlannerEnvConfig) -> PlanningScene:
    """The fixed static-obstacle scene of the trace / timing runs: ego at 12 m/s in lane 0 of a
    two-lane road, the parked vehicles ahead, remaining rows far-away sentinels."""
    road = RoadSpec(lane_count=2)
    centres = np.arange(road.lane_count) * road.lane_width
    m, n_obs = env.num_samples, env.max_obstacles
    ox = np.empty((n_obs, m))
    oy = np.empty((n_obs, m))
    for i in range(n_obs):
        if i < len(_PARKED):
            x, lane = _PARKED[i]
            ox[i], oy[i] = x, centres[lane]
        else:
            ox[i], oy[i] = 1e4 + 100.0 * i, 0.0
    spec = ConstraintSpec(ox, oy, 7.0710678118654755, 2.8284271247461903, env.v_max, env.a_max, env.kappa_max,
                          env.c_max, road.y_lower, road.y_upper, env.v_min)
    return PlanningScene(np.array([0.0, 0.0, 12.0, 0.0, 0.0, 0.0]), spec, centres)


def bilevel_config_for(env: PlannerEnvConfig, scene: PlanningScene, batch_size: int | None = None,
                       iterations: int | None = None) -> BiLevelConfig:
    """Set-point distribution centred on the current lateral offset and speed of `scene`."""
    ms = env.m_seg
    b0 = scene.initial_state
    mean = np.concatenate([np.full(ms, b0[1]), np.full(ms, np.hypot(b0[2], b0[3]))])
    cov = np.diag(np.concatenate([np.full(ms, env.sigma_offset ** 2), np.full(ms, env.sigma_speed ** 2)]))
    return BiLevelConfig(env.batch_size if batch_size is None else batch_size, env.constraint_elites, env.elites,
                         env.iterations if iterations is None else iterations, env.eta, env.gamma,
                         env.residual_weight, mean, cov)


def _solver(env: PlannerEnvConfig) -> LowerLevelSolver:
    basis = build_basis(env.order, env.num_samples, env.horizon, family=env.basis_family)
    return LowerLevelSolver(basis, env.tracking_weights(), ParamLayout(env.m_seg), env.projection_config(),
                            env.max_obstacles)


def emit_timing(env: PlannerEnvConfig, batch_sizes=(250, 1000), iteration_counts=(2, 5), seed: int = 0) -> list:
    """Rows (batch, iterations, total_s, per_iteration_s, factorizations_during_solve)."""
    scene = canonical_scene(env)
    rows = []
    for batch in batch_sizes:
        solver = _solver(env)
        after_setup = batch_qp.FACTORIZATION_COUNT
        for iters in iteration_counts:
            cfg = bilevel_config_for(env, scene, batch_size=batch, iterations=iters)
            t0 = time.perf_counter()
            solve_bilevel(scene, solver, cfg, np.random.default_rng(seed))
            wall = time.perf_counter() - t0
            rows.append({"batch": batch, "iterations": iters, "total_s": wall, "per_iteration_s": wall / iters,
                         "factorizations_during_solve": batch_qp.FACTORIZATION_COUNT - after_setup})
    return rows


def emit_convergence_trace(env: PlannerEnvConfig, seed: int = 0, iterations: int | None = None) -> list:
    """One record per CEM iteration on the canonical scene (trace_hook of solve_bilevel)."""
    scene = canonical_scene(env)
    solver = _solver(env)
    cfg = bilevel_config_for(env, scene, iterations=iterations)
    n = solver.basis.num_coeffs
    W = solver.basis.W
    out = []

    def hook(it, params, proj, costs, elite_idx):
        lateral = proj.xi[n:].T @ W.T                      # (B, m) projected y(t)
        q10, q50, q90 = np.quantile(proj.residuals, [0.10, 0.50, 0.90])
        out.append({"iteration": it, "elite_mean_upper_cost": float(costs[elite_idx].mean()), "cov_trace": None,
                    "residual_q10": float(q10), "residual_q50": float(q50), "residual_q90": float(q90),
                    "y_envelope_low": lateral.min(axis=0).tolist(), "y_envelope_high": lateral.max(axis=0).tolist()})

    result = solve_bilevel(scene, solver, cfg, np.random.default_rng(seed), trace_hook=hook)
    for rec, st in zip(out, result.diagnostics):
        rec["cov_trace"] = st.cov_trace
    return out


def replay_to_csv(log_path: str, out_path: str) -> None:
    """Episode log -> rows t, vehicle, x, y, psi, v, accel, steer, collision (ego first each tick)."""
    log = EpisodeLog.read_jsonl(log_path)
    lines = ["t,vehicle,x,y,psi,v,accel,steer,collision"]
    for rec in log.steps:
        t, hit = rec["t"], int(rec["collision"])
        ex, ey, epsi, ev = rec["ego"]
        acc, steer = rec["ctrl"]
        lines.append(f"{t},ego,{ex!r},{ey!r},{epsi!r},{ev!r},{acc!r},{steer!r},{hit}")
        lines.extend(f"{t},n{k},{x!r},{y!r},{psi!r},{v!r},,,{hit}" for k, (x, y, psi, v) in enumerate(rec["neighbors"]))
    with open(out_path, "w", encoding="utf-8") as fh:
        fh.write("\n".join(lines) + "\n")
