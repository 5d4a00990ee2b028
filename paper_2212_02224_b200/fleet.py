"""Fleet planning: many independent scenes per device call (BASELINE config 5).

Each scene runs its own full CEM cycle (solve_bilevel, pkg/bilevel.py:228-295); scenes
are stacked scene-major into one launch sequence (grid.y = scene in the AM kernel, one
select/refit CTA per scene), so a few hundred scenes fill all 148 SMs.  Gaussian draws
come from the device Philox stream keyed by (seed, global scene, CEM iteration, sample),
which makes results independent of how scenes are spread over GPUs.
"""

from __future__ import annotations

import ctypes
from dataclasses import dataclass

import numpy as np

from ._native import CemConfig, f64, upload_scenes
from .basis import PolynomialBasis
from .batch_qp import TrackingWeights
from .behavior import ParamLayout
from .bilevel import BiLevelConfig, LowerLevelSolver
from .constraints import PlanningScene
from .projection import ProjectionConfig

__all__ = ["FleetPlanner", "FleetResult", "initial_distribution"]


def initial_distribution(scene: PlanningScene, m_seg: int = 4, sigma_offset: float = 1.5, sigma_speed: float = 3.0):
    """Per-scene initial Gaussian of the benchmark harness (pkg/bench.py:245-261)."""
    x0 = scene.initial_state
    mean = np.concatenate([np.full(m_seg, x0[1]), np.full(m_seg, np.hypot(x0[2], x0[3]))])
    cov = np.diag(np.concatenate([np.full(m_seg, sigma_offset**2), np.full(m_seg, sigma_speed**2)]))
    return mean, cov


@dataclass
class FleetResult:
    best_index: np.ndarray       # S
    best_params: np.ndarray      # S x dim
    best_xi: np.ndarray          # S x 2n
    best_cost: np.ndarray        # S
    best_residual: np.ndarray    # S
    best_aug: np.ndarray         # S
    stats: np.ndarray            # S x N x 6 (IterationStats fields)
    final_mean: np.ndarray       # S x dim
    final_cov: np.ndarray        # S x dim x dim
    iterations_done: np.ndarray  # S  (< N: degraded; <= 0: failed in iteration 1)


def initial_means(road: np.ndarray, b0: np.ndarray, m_seg: int) -> np.ndarray:
    """BasePlanner.initial_distribution's mean (pkg/planners.py:218-231) for S worlds at once:
    lateral set-points at the lane centre nearest to y0 (first on ties; y0 itself on a road
    without lanes), speed set-points at hypot(xdot0, ydot0).  road: S x (lanes, width, ...)."""
    S = b0.shape[0]
    lanes = road[:, 0].astype(np.int64)
    centres = np.arange(max(int(lanes.max(initial=0)), 1))[None, :] * road[:, 1:2]   # k * width, per world
    dist = np.abs(centres - b0[:, 1:2])
    dist[np.arange(centres.shape[1])[None, :] >= lanes[:, None]] = np.inf
    lane_y = np.where(lanes > 0, centres[np.arange(S), np.argmin(dist, axis=1)], b0[:, 1])
    speed = np.hypot(b0[:, 2], b0[:, 3])
    return np.concatenate([np.repeat(lane_y[:, None], m_seg, axis=1), np.repeat(speed[:, None], m_seg, axis=1)],
                          axis=1)


class FleetPlanner:
    """Batched solve_bilevel over a list of scenes sharing one basis / QP / obstacle count."""

    def __init__(self, basis: PolynomialBasis, weights: TrackingWeights, layout: ParamLayout,
                 proj_config: ProjectionConfig, num_obstacles: int, config: BiLevelConfig, device: int = 0):
        self.solver = LowerLevelSolver(basis, weights, layout, proj_config, num_obstacles, device=device)
        self.config = config
        self.layout = layout
        self._scenes = None            # the scene objects last uploaded (strong references)

    @property
    def context(self):
        return self.solver.context

    def set_scenes(self, scenes: list[PlanningScene]):
        """Upload the scenes unless they are the very objects uploaded last.  Scenes are immutable
        values; the planner keeps strong references to the uploaded ones, so an
        identity match cannot come from a recycled id() of a freed scene."""
        prev = self._scenes
        stale = self.solver.projector._scene_key is not None      # a single-scene upload since ours
        if stale or prev is None or len(prev) != len(scenes) or any(a is not b for a, b in zip(prev, scenes)):
            for sc in scenes:
                self.solver.projector._check_spec(sc.spec)
            upload_scenes(self.context, scenes, self.solver.basis.num_samples)
            self.solver.projector._scene_key = None
            self._scenes = list(scenes)

    def cem_config(self, seed: int, scene_offset: int = 0) -> CemConfig:
        c, p = self.config, self.solver.projector.config
        return CemConfig(c.batch_size, c.constraint_elites, c.elites, c.iterations, p.max_iters, c.eta, c.gamma,
                         c.residual_weight, p.tol, int(seed), int(scene_offset))

    def plan(self, scenes: list[PlanningScene], seed: int = 0, scene_offset: int = 0, init_mean=None,
             init_cov=None) -> FleetResult:
        """Plan every scene (host inputs / host outputs; copies included)."""
        S = len(scenes)
        self.set_scenes(scenes)
        dim, N, n2 = self.layout.dim, self.config.iterations, 2 * self.solver.basis.num_coeffs
        if init_mean is None or init_cov is None:
            mc = [initial_distribution(sc, self.layout.m_seg) for sc in scenes]
            init_mean = np.stack([m for m, _ in mc])
            init_cov = np.stack([c for _, c in mc])
        out = FleetResult(np.zeros(S, np.int64), np.zeros((S, dim)), np.zeros((S, n2)), np.zeros(S), np.zeros(S),
                          np.zeros(S), np.zeros((S, N, 6)), np.zeros((S, dim)), np.zeros((S, dim, dim)),
                          np.zeros(S, np.int32))
        cfg = self.cem_config(seed, scene_offset)
        self.context.call("bd_cem_cycle", S, ctypes.byref(cfg), f64(init_mean), f64(init_cov), None, None,
                          out.best_index, out.best_params, out.best_xi, out.best_cost, out.best_residual,
                          out.best_aug, out.stats, out.final_mean, out.final_cov, out.iterations_done)
        return out

    def plan_cycle(self, worlds, env, emitter, seed: int = 0, scene_offset: int = 0, sigma_offset: float = 1.5,
                   sigma_speed: float = 3.0):
        """MPCBiLevelPlanner.plan_cycle for a batch of worlds (pkg/planners.py:200-216, 276-306):
        device scene build -> device CEM cycle -> device control emission of each best trajectory.
        Returns (accels, steers, singular, FleetResult); world arrays in, controls out."""
        from .worlds import build_scenes
        b0 = build_scenes(self.context, self.solver.basis, worlds, env, b0_only=True)
        self._scenes = None              # device scenes now come from the worlds
        self.solver.projector._scene_key = None
        # BasePlanner.initial_distribution (pkg/planners.py:218-231) on the device-built initial
        # states: nearest lane centre to y0, speed = hypot(xdot0, ydot0)
        ms = self.layout.m_seg
        S = b0.shape[0]
        road = np.asarray(worlds.road.cpu() if hasattr(worlds.road, "cpu") else worlds.road)
        mean = initial_means(road, b0, ms)
        cov = np.repeat(np.diag(np.concatenate([np.full(ms, sigma_offset ** 2), np.full(ms, sigma_speed ** 2)]))[None],
                        S, axis=0)
        dim, N, n2 = self.layout.dim, self.config.iterations, 2 * self.solver.basis.num_coeffs
        out = FleetResult(np.zeros(S, np.int64), np.zeros((S, dim)), np.zeros((S, n2)), np.zeros(S), np.zeros(S),
                          np.zeros(S), np.zeros((S, N, 6)), np.zeros((S, dim)), np.zeros((S, dim, dim)),
                          np.zeros(S, np.int32))
        cfg = self.cem_config(seed, scene_offset)
        self.context.call("bd_cem_cycle", S, ctypes.byref(cfg), f64(mean), f64(cov), None, None, out.best_index,
                          out.best_params, out.best_xi, out.best_cost, out.best_residual, out.best_aug, out.stats,
                          out.final_mean, out.final_cov, out.iterations_done)
        acc, ste, sing = emitter.emit(out.best_xi)
        return acc, ste, sing, out

    def plan_device(self, S: int, seed: int, init_mean, init_cov, outputs: dict, scene_offset: int = 0):
        """Asynchronous variant on device buffers (torch tensors): scenes must already be set."""
        cfg = self.cem_config(seed, scene_offset)
        o = outputs
        self.context.call("bd_cem_cycle", S, ctypes.byref(cfg), init_mean, init_cov, None, None,
                          o.get("best_index"), o.get("best_params"), o.get("best_xi"), o.get("best_cost"),
                          o.get("best_residual"), o.get("best_aug"), o.get("stats"), o.get("final_mean"),
                          o.get("final_cov"), o.get("iterations_done"))
