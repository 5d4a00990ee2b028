"""Synthetic highway scenes for benchmarks and fleets.

Restates the reference's seeded scene recipe — ``spawn_world`` (pkg/highway.py:168-205)
followed by ``build_scene`` (pkg/planners.py:116-160): neighbours spread over the lanes
at density-scaled spacing, the ``max_obstacles`` nearest ones (within
``obstacle_range`` longitudinally) predicted at constant velocity over the horizon,
remaining rows padded with far sentinels.  Given the same seed it yields the same
scene as the reference (pinned by tests/test_scenes.py), without importing it.
"""

from __future__ import annotations

import math
from dataclasses import dataclass

import numpy as np

from .constraints import ConstraintSpec, PlanningScene

__all__ = ["HighwayRecipe", "highway_scene", "spawn_worlds", "SENTINEL_DISTANCE"]

SENTINEL_DISTANCE = 1e4


@dataclass(frozen=True)
class HighwayRecipe:
    lanes: int = 4
    density: float = 2.0
    vehicle_count: int = 24
    n_obs: int = 10
    obstacle_range: float = 120.0
    horizon: float = 5.0
    num_samples: int = 100
    lane_width: float = 4.0
    neighbor_speed: float = 11.0
    ego_speed: float = 10.0
    ego_lane: int = 0
    spawn_base_spacing: float = 40.0
    # PlannerEnvConfig limits (pkg/planners.py:44-48)
    v_max: float = 20.0
    a_max: float = 6.0
    kappa_max: float = 0.2
    c_max: float = 3.0
    v_min: float = 0.5


def _spawn(seed: int, r: HighwayRecipe, with_cooldown: bool = False):
    """Neighbour (x, y, v[, cooldown]) list of spawn_world (pkg/highway.py:168-205)."""
    rng = np.random.default_rng(seed)
    spacing = r.spawn_base_spacing / r.density
    cursor = [(25.0 if lane == r.ego_lane else -15.0) + spacing * 0.5 * rng.uniform(0.0, 1.0)
              for lane in range(r.lanes)]
    cars = []   # (x, y, v)
    for i in range(r.vehicle_count):
        lane = i % r.lanes
        x = cursor[lane]
        cursor[lane] = x + spacing * rng.uniform(0.85, 1.15)
        v = r.neighbor_speed * (1.0 + 0.15 * rng.uniform(-1.0, 1.0))
        cooldown = float(rng.uniform(0.0, 2.0))   # lane-change cooldown (drawn even when unused: stream alignment)
        cars.append((float(x), lane * r.lane_width, float(v), cooldown) if with_cooldown
                    else (float(x), lane * r.lane_width, float(v)))
    return cars


def spawn_worlds(seeds, recipe: HighwayRecipe = HighwayRecipe()):
    """WorldBatch of freshly spawned worlds (ego at rest on its lane, heading 0) for the device
    scene build (`worlds.build_scenes`)."""
    from .worlds import WorldBatch
    seeds = list(seeds)
    r = recipe
    S = len(seeds)
    ego = np.zeros((S, 8))
    veh = np.zeros((S, max(1, r.vehicle_count), 5))
    ego[:, 1] = r.ego_lane * r.lane_width
    ego[:, 3] = r.ego_speed
    ego[:, 6], ego[:, 7] = 5.0, 2.0
    for s, seed in enumerate(seeds):
        for j, (x, y, v) in enumerate(_spawn(seed, r)):
            veh[s, j] = (x, y, 0.0, v, 0.0)
    return WorldBatch(ego, veh, np.full(S, r.vehicle_count, np.int32), np.tile([r.lanes, r.lane_width], (S, 1)))


def highway_scene(seed: int, recipe: HighwayRecipe = HighwayRecipe()) -> PlanningScene:
    r = recipe
    ego_x, ego_y = 0.0, r.ego_lane * r.lane_width
    cars = _spawn(seed, r)
    near = sorted((c for c in cars if abs(c[0] - ego_x) <= r.obstacle_range),
                  key=lambda c: (c[0] - ego_x) ** 2 + (c[1] - ego_y) ** 2)[: r.n_obs]
    times = np.linspace(0.0, r.horizon, r.num_samples)
    ox = np.empty((r.n_obs, r.num_samples))
    oy = np.empty((r.n_obs, r.num_samples))
    for i in range(r.n_obs):
        if i < len(near):
            ox[i] = near[i][0] + near[i][2] * times
            oy[i] = near[i][1] + 0.0 * times
        else:
            ox[i] = ego_x + SENTINEL_DISTANCE + 100.0 * i
            oy[i] = 0.0
    a_axis, b_axis = math.sqrt(2.0) * 5.0, math.sqrt(2.0) * 2.0     # combined_ellipse(5, 2, 5, 2)
    spec = ConstraintSpec(obstacles_x=ox, obstacles_y=oy, ellipse_a=a_axis, ellipse_b=b_axis, v_max=r.v_max,
                          a_max=r.a_max, kappa_max=r.kappa_max, c_max=r.c_max, y_lb=-r.lane_width / 2.0,
                          y_ub=(r.lanes - 1) * r.lane_width + r.lane_width / 2.0, v_min=r.v_min)
    return PlanningScene(initial_state=np.array([ego_x, ego_y, r.ego_speed, 0.0, 0.0, 0.0]), spec=spec,
                         lane_centers=np.arange(r.lanes) * r.lane_width)
