"""Planners over a fleet of simulated worlds.

Batched restatements of the reference planners (pkg/planners.py:174-421): every planning cycle
builds all S scenes on the device from the simulator's HBM state (build_scene + ego_flat_state),
solves them in one launch sequence and emits the control grids on the device
(controls_on_grid), so a fleet of closed-loop episodes plans in one call per replan instant.

* :class:`PlannerEnvConfig` — the reference's planning-side configuration (same fields and
  defaults, pkg/planners.py:40-87).
* :class:`BatchMPCBiLevelPlanner` — MPCBiLevelPlanner (pkg/planners.py:261-306): the full CEM
  bi-level optimizer per world, warm-started from the previous cycle's best set-points.
* :class:`BatchEvaluatePlanner` subclasses — the one-sweep baselines MPCVanillaPlanner,
  MPCRandomPlanner, MPCGridPlanner and BatchMPCGoalPlanner (pkg/planners.py:309-412) on the
  same lower-level kernels (``bd_solve_lower`` over S scenes + ``bd_rank_refit`` ranking).

Differences from the reference that follow from batching (documented in DESIGN.md): the CEM
draws come from the device Philox stream keyed by (seed, cycle, world, iteration, sample) instead
of each planner's numpy Generator, so closed-loop trajectories are statistically but not
numerically those of the reference; ``solve_time`` is the wall time of the batched cycle.
"""

from __future__ import annotations

import ctypes
import math
import time
from dataclasses import dataclass

import numpy as np

from ._native import f64
from .basis import build_basis
from .batch_qp import TrackingWeights
from .behavior import ParamLayout
from .bilevel import BiLevelConfig, LowerLevelSolver, SamplingDistribution
from .fleet import FleetPlanner, FleetResult
from .projection import ProjectionConfig
from .worlds import ControlEmitter, build_scenes

__all__ = ["PlannerEnvConfig", "PlannerFailure", "BatchMPCBiLevelPlanner", "BatchMPCVanillaPlanner",
           "BatchMPCRandomPlanner", "BatchMPCGridPlanner", "BatchMPCGoalPlanner", "BATCH_PLANNER_REGISTRY",
           "make_batch_planner"]


@dataclass(frozen=True)
class PlannerEnvConfig:
    """Planning-side limits, horizon discretization, and search budgets (pkg/planners.py:40-87)."""

    v_max: float = 20.0
    a_max: float = 6.0
    kappa_max: float = 0.2
    c_max: float = 3.0
    v_min: float = 0.5
    wheelbase: float = 2.5
    horizon: float = 10.0
    num_samples: int = 50
    order: int = 10
    basis_family: str = "bernstein"
    m_seg: int = 4
    max_obstacles: int = 6
    obstacle_range: float = 120.0
    batch_size: int = 250
    constraint_elites: int = 150
    elites: int = 50
    iterations: int = 5
    eta: float = 0.7
    gamma: float = 0.9
    residual_weight: float = 1.0
    sigma_offset: float = 1.5
    sigma_speed: float = 3.0
    proj_rho: float = 1.0
    proj_iters: int = 50
    proj_tol: float = 1e-3
    k_p: float = 20.0
    k_v: float = 2.0 * math.sqrt(20.0)
    w_smooth: float = 1.0
    w_offset: float = 20.0
    w_speed: float = 20.0
    warm_start_cycles: bool = True

    def tracking_weights(self) -> TrackingWeights:
        return TrackingWeights(k_p=self.k_p, k_v=self.k_v, w_smooth=self.w_smooth, w_offset=self.w_offset,
                               w_speed=self.w_speed)

    def projection_config(self) -> ProjectionConfig:
        return ProjectionConfig(rho=self.proj_rho, max_iters=self.proj_iters, tol=self.proj_tol)

    @property
    def steer_limit(self) -> float:
        return math.atan(self.kappa_max * self.wheelbase)


class PlannerFailure(RuntimeError):
    """The planner could not produce a usable plan this cycle (pkg/planners.py:170-171)."""


@dataclass
class CyclePlan:
    """One batched planning cycle: per-world control grids, diagnostics and failures."""

    accels: np.ndarray          # S x n_ctrl
    steers: np.ndarray          # S x n_ctrl
    infos: list                 # S dicts (the reference's plan_cycle info), None where failed
    failures: list              # S failure reasons ("Type: message") or None
    solve_time: float


class _BatchPlanner:
    name = "base"
    with_goal = False

    def __init__(self, env: PlannerEnvConfig, seed: int = 0, dt: float = 0.1, device: int = 0):
        self.env = env
        self.seed = int(seed)
        self.dt = float(dt)
        self.basis = build_basis(env.order, env.num_samples, env.horizon, family=env.basis_family)
        self.layout = ParamLayout(m_seg=env.m_seg, with_goal=self.with_goal)
        self.n_ctrl = int(env.horizon / dt)
        self._setup(device)
        self.emitter = ControlEmitter(self.context, self.basis, env.horizon, dt, env)
        self.cycle = 0

    def _weights(self) -> TrackingWeights:
        return self.env.tracking_weights()

    def reset(self):
        self.cycle = 0

    # -- scene build from the simulator state (pkg/planners.py:99-160), b0 back to the host
    def _build(self, worlds) -> np.ndarray:
        b0 = build_scenes(self.context, self.basis, worlds, self.env, b0_only=True)
        self._invalidate_scene_cache()
        return b0

    @staticmethod
    def _lane_centers(road: np.ndarray) -> list:
        return [np.arange(int(n)) * w for n, w in road]

    def _initial(self, b0, centers):
        """BasePlanner.initial_distribution (pkg/planners.py:218-231) for all worlds at once: the
        lane centre nearest to y0 (first on ties, like argmin) and the speed hypot(xdot0, ydot0)."""
        env, ms = self.env, self.env.m_seg
        S = b0.shape[0]
        width = max((c.size for c in centers), default=0)
        if width == 0:
            lane_y = b0[:, 1].copy()
        else:
            tab = np.full((S, width), np.inf)
            for s, c in enumerate(centers):
                tab[s, :c.size] = c
            pick = tab[np.arange(S), np.argmin(np.abs(tab - b0[:, 1:2]), axis=1)]
            empty = np.array([c.size == 0 for c in centers])
            lane_y = np.where(empty, b0[:, 1], pick)
        mean = np.empty((S, 2 * ms))
        mean[:, :ms] = lane_y[:, None]
        mean[:, ms:] = np.hypot(b0[:, 2], b0[:, 3])[:, None]
        cov = np.diag(np.concatenate([np.full(ms, env.sigma_offset ** 2), np.full(ms, env.sigma_speed ** 2)]))
        return mean, cov

    def _emit(self, xi, ok):
        acc, ste, sing = self.emitter.emit(xi)
        failures = [None] * xi.shape[0]
        for s in np.flatnonzero(ok & sing):
            failures[s] = (f"SpeedSingularity: speed drops below the floor "
                           f"({self.emitter.eps_v:g} m/s) on the control grid")
        return acc, ste, failures

    def plan_cycle(self, state, road_host: np.ndarray) -> CyclePlan:
        """Plan every world of `state` (a SimState, device or host) once."""
        t0 = time.perf_counter()
        b0 = self._build(state.worlds)
        plan = self._plan(b0, self._lane_centers(road_host))
        plan.solve_time = time.perf_counter() - t0
        for info in plan.infos:
            if info is not None:
                info["solve_time"] = plan.solve_time
        self.cycle += 1
        return plan


class BatchMPCBiLevelPlanner(_BatchPlanner):
    """MPCBiLevelPlanner (pkg/planners.py:261-306) for S worlds per call."""

    name = "mpc-bilevel"

    def __init__(self, env: PlannerEnvConfig, seed=0, dt: float = 0.1, device: int = 0,
                 generator_seeds=None):
        """generator_seeds (one per world): draw each world's samples from its own numpy Generator
        exactly like the reference planner (default_rng(seed), reset per episode), instead of the
        device Philox stream -- closed loops then replay the reference planner's randomness."""
        self.generator_seeds = None if generator_seeds is None else [int(x) for x in generator_seeds]
        self._rngs = None
        super().__init__(env, seed, dt, device)

    def _setup(self, device):
        env = self.env
        cfg = BiLevelConfig(env.batch_size, env.constraint_elites, env.elites, env.iterations, env.eta, env.gamma,
                            env.residual_weight)
        self.fleet = FleetPlanner(self.basis, self._weights(), self.layout, env.projection_config(),
                                  env.max_obstacles, cfg, device=device)
        self.context = self.fleet.context
        self._warm = None

    def _invalidate_scene_cache(self):
        self.fleet._scenes = None
        self.fleet.solver.projector._scene_key = None

    def reset(self):
        super().reset()
        self._warm = None
        self._rngs = None

    def _draws(self, S: int):
        """(N, S*B, dim) normals from the worlds' Generators (state kept for failure rewinds)."""
        if self._rngs is None:
            if len(self.generator_seeds) != S:
                raise ValueError(f"{len(self.generator_seeds)} generator seeds for {S} worlds")
            self._rngs = [np.random.default_rng(x) for x in self.generator_seeds]
        env = self.env
        self._rng_state = [r.bit_generator.state for r in self._rngs]
        z = np.stack([r.standard_normal((env.iterations, env.batch_size, self.layout.dim)) for r in self._rngs], axis=1)
        return np.ascontiguousarray(z.reshape(env.iterations, S * env.batch_size, self.layout.dim))

    def _rewind(self, done: np.ndarray):
        """Leave each Generator where the reference's solve_bilevel would (pkg/bilevel.py:248-261)."""
        N = self.env.iterations
        for s, k in enumerate(done):
            attempted = N if k >= N else (1 if k <= 0 else k + 1)
            if attempted != N:
                self._rngs[s].bit_generator.state = self._rng_state[s]
                self._rngs[s].standard_normal((attempted, self.env.batch_size, self.layout.dim))

    def _plan(self, b0, centers) -> CyclePlan:
        env = self.env
        S = b0.shape[0]
        mean, cov = self._initial(b0, centers)
        if env.warm_start_cycles and self._warm is not None:      # pkg/planners.py:279-280
            mean = self._warm.copy()
        covs = np.repeat(cov[None], S, axis=0)
        dim, N, n2 = self.layout.dim, env.iterations, 2 * self.basis.num_coeffs
        out = FleetResult(np.zeros(S, np.int64), np.zeros((S, dim)), np.zeros((S, n2)), np.zeros(S), np.zeros(S),
                          np.zeros(S), np.zeros((S, N, 6)), np.zeros((S, dim)), np.zeros((S, dim, dim)),
                          np.zeros(S, np.int32))
        # one Philox stream per (seed, cycle): worlds are distinguished by their scene index
        cfg = self.fleet.cem_config((self.seed * 1_000_003 + self.cycle) & 0xFFFFFFFFFFFF, 0)
        z = self._draws(S) if self.generator_seeds is not None else None
        self.context.call("bd_cem_cycle", S, ctypes.byref(cfg), f64(mean), f64(covs), z, None, out.best_index,
                          out.best_params, out.best_xi, out.best_cost, out.best_residual, out.best_aug, out.stats,
                          out.final_mean, out.final_cov, out.iterations_done)
        if z is not None:
            self._rewind(out.iterations_done)
        ok = out.iterations_done > 0
        acc, ste, failures = self._emit(out.best_xi, ok)
        infos = []
        warm = mean.copy()
        for s in range(S):
            if not ok[s]:
                failures[s] = "NumericalFailure: projection failed in the first CEM iteration"
            if failures[s] is not None:
                infos.append(None)
                continue
            last = out.stats[s, out.iterations_done[s] - 1]
            warm[s] = out.best_params[s]
            infos.append({"residual": float(out.best_residual[s]), "upper_cost": float(out.best_cost[s]),
                          "elite_mean_upper_cost": float(last[0]), "cov_trace": float(last[2]),
                          "iterations": int(out.iterations_done[s]), "degraded": bool(out.iterations_done[s] < N)})
        self._warm = warm
        self.last_result = out
        return CyclePlan(acc, ste, infos, failures, 0.0)


class BatchEvaluatePlanner(_BatchPlanner):
    """One lower-level sweep per world over a set-point batch, best record by augmented cost
    (BasePlanner.evaluate_batch, pkg/planners.py:233-258), for S worlds in one launch sequence."""

    def _setup(self, device):
        env = self.env
        self.solver = LowerLevelSolver(self.basis, self._weights(), self.layout, env.projection_config(),
                                       env.max_obstacles, device=device)
        self.context = self.solver.context
        self.rngs = None

    def _invalidate_scene_cache(self):
        self.solver.projector._scene_key = ("sim", self.cycle)

    def reset(self):
        super().reset()
        self.rngs = None

    def _points(self, s, b0, centers, mean, cov) -> np.ndarray:
        raise NotImplementedError

    def _plan(self, b0, centers) -> CyclePlan:
        env = self.env
        S = b0.shape[0]
        mean, cov = self._initial(b0, centers)
        pts = [np.atleast_2d(np.asarray(self._points(s, b0, centers, mean[s], cov), float)) for s in range(S)]
        counts = [p.shape[0] for p in pts]
        B = max(counts)
        # worlds with fewer candidates (e.g. fewer lanes) are padded with copies of their first
        # point: a copy has the same residual and cost and a larger index, so it never outranks
        # the original, and the batch-global exit (max residual) is unchanged
        pts = [p if p.shape[0] == B else np.concatenate([p, np.repeat(p[:1], B - p.shape[0], axis=0)]) for p in pts]
        P = f64(np.stack(pts))                                   # S x B x dim
        dim, n2 = self.layout.dim, 2 * self.basis.num_coeffs
        xi = np.empty((S, B, n2))
        res = np.empty((S, B))
        cost = np.empty((S, B))
        used = np.zeros(S, np.int32)
        conf = np.zeros(S, np.int64)
        p = self.solver.projector
        self.context.call("bd_solve_lower", S, B, P, int(p.config.max_iters), float(p.config.tol), None, None, xi,
                          res, cost, None, used, conf)
        n = min(env.constraint_elites, B)
        q = min(env.elites, n)
        el = np.empty((S, q), np.int64)
        ea = np.empty((S, q))
        m0, c0 = np.zeros((S, dim)), np.repeat(np.eye(dim)[None], S, axis=0)
        self.context.call("bd_rank_refit", S, B, dim, res, cost, P, n, q, float(env.residual_weight), 0.5, 1.0,
                          m0, c0, None, el, ea, None)
        best = el[:, 0]
        rows = np.arange(S)
        acc, ste, failures = self._emit(xi[rows, best], np.ones(S, bool))
        infos = [None if failures[s] is not None else
                 {"residual": float(res[s, best[s]]), "upper_cost": float(cost[s, best[s]]),
                  "proj_iterations": int(used[s]), "batch": int(counts[s])} for s in range(S)]
        return CyclePlan(acc, ste, infos, failures, 0.0)


class BatchMPCVanillaPlanner(BatchEvaluatePlanner):
    """MPCVanillaPlanner (pkg/planners.py:309-325): fixed set-points (current lane, v_desired)."""

    name = "mpc-vanilla"

    def __init__(self, env: PlannerEnvConfig, seed: int = 0, dt: float = 0.1, device: int = 0,
                 v_desired: float | None = None):
        self.v_desired = v_desired
        super().__init__(env, seed, dt, device)

    def _points(self, s, b0, centers, mean, cov):
        ms = self.env.m_seg
        v_d = self.v_desired if self.v_desired is not None else self.env.v_max
        return np.concatenate([np.full(ms, mean[0]), np.full(ms, v_d)])


class BatchMPCRandomPlanner(BatchEvaluatePlanner):
    """MPCRandomPlanner (pkg/planners.py:328-338): one Gaussian batch from the initial distribution,
    drawn with each world's own numpy Generator (seeded like the reference planner)."""

    name = "mpc-random"

    def __init__(self, env: PlannerEnvConfig, seed=0, dt: float = 0.1, device: int = 0):
        super().__init__(env, 0 if np.ndim(seed) else seed, dt, device)
        self.world_seeds = seed

    def _points(self, s, b0, centers, mean, cov):
        if self.rngs is None:
            S = b0.shape[0]
            seeds = self.world_seeds if np.ndim(self.world_seeds) else [self.world_seeds] * S
            self.rngs = [np.random.default_rng(int(x)) for x in seeds]
        return SamplingDistribution(mean=mean, cov=cov).sample(self.env.batch_size, self.rngs[s])


class BatchMPCGridPlanner(BatchEvaluatePlanner):
    """MPCGridPlanner (pkg/planners.py:341-385) with its default grid: lane centres x
    (0.5, 0.75, 1.0) v_max."""

    name = "mpc-grid"

    def _points(self, s, b0, centers, mean, cov):
        env = self.env
        c = centers[s] if centers[s].size else np.array([b0[s, 1]])
        return np.array([np.concatenate([np.full(env.m_seg, y), np.full(env.m_seg, v)])
                         for y in c for v in np.array([0.5, 0.75, 1.0]) * env.v_max])


class BatchMPCGoalPlanner(BatchEvaluatePlanner):
    """BatchMPCGoalPlanner (pkg/planners.py:388-412): terminal goal positions in the equality
    constraints, tracking weights w_offset = w_speed = 0."""

    name = "batch-mpc-goal"
    with_goal = True

    def _weights(self) -> TrackingWeights:
        e = self.env
        return TrackingWeights(k_p=e.k_p, k_v=e.k_v, w_smooth=e.w_smooth, w_offset=0.0, w_speed=0.0)

    def _points(self, s, b0, centers, mean, cov):
        env = self.env
        x0 = b0[s, 0]
        v0 = float(np.hypot(b0[s, 2], b0[s, 3]))
        reach = max(v0, 0.3 * env.v_max) * env.horizon
        c = centers[s] if centers[s].size else np.array([b0[s, 1]])
        return np.array([np.concatenate([np.zeros(env.m_seg), np.zeros(env.m_seg), [x0 + f * reach, y]])
                         for f in np.array([0.5, 0.7, 0.85, 1.0]) for y in c])


BATCH_PLANNER_REGISTRY = {cls.name: cls for cls in (BatchMPCBiLevelPlanner, BatchMPCVanillaPlanner,
                                                      BatchMPCRandomPlanner, BatchMPCGridPlanner,
                                                      BatchMPCGoalPlanner)}


def make_batch_planner(name: str, env: PlannerEnvConfig, seed=0, dt: float = 0.1, device: int = 0, **kw):
    try:
        cls = BATCH_PLANNER_REGISTRY[name]
    except KeyError:
        raise ValueError(f"unknown planner {name!r}; choose from {sorted(BATCH_PLANNER_REGISTRY)}") from None
    return cls(env, seed=seed, dt=dt, device=device, **kw)
