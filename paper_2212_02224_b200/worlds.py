"""Steps either side of the path on the device.

* Scene construction — ``build_scene`` + ``ego_flat_state`` (pkg/planners.py:99-160) and
  ``observe`` (pkg/highway.py:208-246) for a batch of worlds in one launch (``bd_build_scenes``),
  writing the scene tiles the AM kernel reads, so a fleet of thousands of worlds goes from
  simulator state to planned trajectories without a host scene build.
* Control emission — ``controls_on_grid`` -> ``flat_to_controls`` (pkg/planners.py:209-216,
  pkg/basis.py:206-234) for a batch of trajectories (``bd_controls``).

World state travels as plain arrays (:class:`WorldBatch`); ``WorldBatch.from_worlds`` converts
the reference's ``World`` objects (duck-typed: ``world.ego``, ``world.neighbors``, ``world.road``).
"""

from __future__ import annotations

import ctypes
import math
from dataclasses import dataclass

import numpy as np

from ._native import Env, f64
from .basis import PolynomialBasis

__all__ = ["WorldBatch", "PlannerEnv", "build_scenes", "ControlEmitter", "env_struct", "curvature_tables"]


@dataclass
class WorldBatch:
    ego: np.ndarray     # S x 8: x, y, psi, v, accel, steer, length, width
    veh: np.ndarray     # S x n_max x 5: x, y, psi, v, lateral_rate (world.neighbors order)
    n_veh: np.ndarray   # S (int32)
    road: np.ndarray    # S x 2: lane_count, lane_width
    curvature: list | None = None   # per world RoadSpec.curvature ((xs...), (ks...)) or None

    @property
    def size(self) -> int:
        return self.ego.shape[0]

    @staticmethod
    def from_worlds(worlds) -> "WorldBatch":
        S = len(worlds)
        n_max = max(1, max(len(w.neighbors) for w in worlds))
        ego = np.zeros((S, 8))
        veh = np.zeros((S, n_max, 5))
        n = np.zeros(S, np.int32)
        road = np.zeros((S, 2))
        for s, w in enumerate(worlds):
            e = w.ego
            ego[s] = (e.x, e.y, e.psi, e.v, e.accel, e.steer, e.length, e.width)
            for j, v in enumerate(w.neighbors):
                veh[s, j] = (v.x, v.y, v.psi, v.v, v.lateral_rate)
            n[s] = len(w.neighbors)
            road[s] = (w.road.lane_count, w.road.lane_width)
        curv = [getattr(w.road, "curvature", None) for w in worlds]
        return WorldBatch(ego, veh, n, road, curv if any(c is not None for c in curv) else None)


@dataclass(frozen=True)
class PlannerEnv:
    """The PlannerEnvConfig fields the scene build and control emission use (pkg/planners.py:40-87)."""

    max_obstacles: int = 10
    obstacle_range: float = 120.0
    wheelbase: float = 2.5
    v_max: float = 20.0
    a_max: float = 6.0
    kappa_max: float = 0.2
    c_max: float = 3.0
    v_min: float = 0.5

    @property
    def steer_limit(self) -> float:
        return math.atan(self.kappa_max * self.wheelbase)

    def c_struct(self) -> Env:
        return Env(self.max_obstacles, self.obstacle_range, self.wheelbase, self.v_max, self.a_max, self.kappa_max,
                   self.c_max, self.v_min, 5.0, 2.0)


def build_scenes(ctx, basis: PolynomialBasis, worlds: WorldBatch, env: PlannerEnv, outputs: bool = False,
                 b0_only: bool = False):
    """Build S scenes on the device into `ctx` (replacing its scenes).  With outputs=True also
    return (ox, oy, b0, limits, observations) as host arrays; with b0_only=True return just the
    initial states b0 (S x 6, ego_flat_state)."""
    S, n_max = worlds.size, worlds.veh.shape[1]
    m = basis.num_samples
    out = (np.empty((S, env.max_obstacles, m)), np.empty((S, env.max_obstacles, m)), np.empty((S, 6)),
           np.empty((S, 9)), np.empty((S, 55))) if outputs else (None,) * 5
    if b0_only and not outputs:
        out = (None, None, np.empty((S, 6)), None, None)
    cenv = env_struct(env)
    ctx.call("bd_build_scenes", S, n_max, _dev_or(worlds.ego, np.float64), _dev_or(worlds.veh, np.float64),
             _dev_or(worlds.n_veh, np.int32), _dev_or(worlds.road, np.float64), ctypes.byref(cenv),
             f64(basis.times), *out)
    if worlds.curvature is not None and any(c is not None for c in worlds.curvature):
        cx, ck = curvature_tables(worlds.curvature)
        ctx.call("bd_set_curvature", S, cx.shape[1], cx, ck)
    return out if outputs else (out[2] if b0_only else None)


def curvature_tables(curvature: list):
    """Per-world road_curvature tables padded to one length (S x n abscissae, S x n curvatures).
    np.interp clamps beyond the last abscissa, so padding with further abscissae at the last
    curvature changes nothing; a world without curvature gets a zero table (kappa = 0 disables
    the centripetal bound and its residual term exactly as road_curvature=None does)."""
    n = max(len(c[0]) for c in curvature if c is not None)
    S = len(curvature)
    cx, ck = np.empty((S, n)), np.zeros((S, n))
    for s, c in enumerate(curvature):
        if c is None:
            cx[s] = np.arange(n, dtype=float) * 1e9 - 1e9 * (n // 2)
            continue
        xs, ks = np.asarray(c[0], float), np.asarray(c[1], float)
        if xs.shape != ks.shape or xs.ndim != 1 or xs.size < 1:
            raise ValueError("road curvature must be two equal-length 1-d sequences")
        L = xs.size
        cx[s, :L], ck[s, :L] = xs, ks
        cx[s, L:] = xs[-1] + 1e9 * np.arange(1, n - L + 1)
        ck[s, L:] = ks[-1]
    return cx, ck


def _dev_or(a, dtype):
    """Device tensors (e.g. the simulator's state) pass through; host data become contiguous arrays."""
    return a if hasattr(a, "data_ptr") else np.ascontiguousarray(a, dtype=dtype)


def env_struct(env) -> Env:
    """bd_env from a PlannerEnv or any PlannerEnvConfig-like object (duck-typed fields)."""
    if isinstance(env, PlannerEnv):
        return env.c_struct()
    return PlannerEnv(int(env.max_obstacles), float(env.obstacle_range), float(env.wheelbase), float(env.v_max),
                      float(env.a_max), float(env.kappa_max), float(env.c_max), float(env.v_min)).c_struct()


class ControlEmitter:
    """controls_on_grid for batches of trajectories on the device (pkg/planners.py:209-216)."""

    def __init__(self, ctx, basis: PolynomialBasis, horizon: float, dt: float, env: PlannerEnv, eps_v: float = 1e-3):
        self.ctx = ctx
        self.eps_v = float(eps_v)
        self.n_ctrl = int(horizon / dt)
        self.times = np.arange(self.n_ctrl) * dt
        _, Wd, Wdd = basis.matrices_at(self.times)       # host fp64 setup, once
        ctx.call("bd_set_control_grid", self.n_ctrl, f64(Wd), f64(Wdd), float(env.wheelbase), float(env.a_max),
                 float(env.steer_limit), float(eps_v))

    def emit(self, xi_rows: np.ndarray):
        """xi_rows: (count, 2n) coefficients -> (accels, steers, singular) with shapes
        (count, n_ctrl), (count, n_ctrl), (count,); singular rows raise SpeedSingularity in the
        reference and hold undefined values here."""
        X = f64(np.atleast_2d(xi_rows))
        acc = np.empty((X.shape[0], self.n_ctrl))
        ste = np.empty_like(acc)
        sing = np.zeros(X.shape[0], np.int32)
        self.ctx.call("bd_controls", X.shape[0], X, acc, ste, sing)
        return acc, ste, sing.astype(bool)
