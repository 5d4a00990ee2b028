"""Batched highway simulation on the device.

Host mirror of the reference simulator's data types and tick — ``RoadSpec`` / ``ScenarioConfig``
(pkg/highway.py:39-146), ``spawn_world`` (:168-205), ``IDMParams`` / ``MOBILParams`` (:73-89) and
``step`` (:358-410) — over a :class:`SimState` of S worlds whose arrays live in HBM between ticks.
One ``bd_sim_run`` launch advances every world by up to ``replan_stride`` ticks (the open-loop
stretch of ``run_episode``), so a fleet of episodes never round-trips its world state through
the host; :mod:`.episodes` drives the closed loop (plan -> execute -> replan).

World layout (shared with :func:`.worlds.build_scenes`, so the scene build reads the simulator's
buffers directly):

  ego      S x 8        x, y, psi, v, accel, steer, length, width
  ego_ts   S            ego target speed (its IDM v0 when it is a MOBIL follower)
  veh      S x n x 5    x, y, psi, v, lateral_rate                       (world.neighbors order)
  veh_ext  S x n x 7    length, width, target_speed, target_lane, cooldown, accel, lane_index
  n_veh    S            live neighbours per world (rows beyond are padding)
  road     S x 2        lane_count, lane_width
  world    S x 5        time, step_count, collided, collision_step (-1: none), lane_departed
"""

from __future__ import annotations

import ctypes
from dataclasses import dataclass, fields

import numpy as np

from ._native import Traffic
from .scenes import HighwayRecipe, _spawn
from .worlds import WorldBatch

__all__ = ["RoadSpec", "ScenarioConfig", "TrafficParams", "SimState", "Simulator", "SNAP_HEAD"]

SNAP_HEAD = 8        # per-tick record: time, ego x y psi v accel steer, collided, then 4 per neighbour


@dataclass(frozen=True)
class RoadSpec:
    """Straight multi-lane road (pkg/highway.py:39-66); lane i is centred at i * lane_width."""

    lane_count: int
    lane_width: float = 4.0
    length: float = 1500.0
    curvature: tuple | None = None      # ((xs...), (ks...)) for ConstraintSpec.road_curvature

    def __post_init__(self):
        if self.lane_count < 2:
            raise ValueError("need at least two lanes")
        if self.lane_width <= 2.5:
            raise ValueError("lane width must exceed vehicle width")

    @property
    def y_lower(self) -> float:
        return -self.lane_width / 2.0

    @property
    def y_upper(self) -> float:
        return (self.lane_count - 1) * self.lane_width + self.lane_width / 2.0


@dataclass(frozen=True)
class ScenarioConfig:
    """Seeded episode recipe (pkg/highway.py:92-146), same fields and dict form."""

    road: RoadSpec
    density: float
    vehicle_count: int
    seed: int
    episode_length: int = 150
    dt: float = 0.1
    neighbor_speed: float = 11.0
    ego_speed: float = 10.0
    ego_lane: int = 0
    spawn_base_spacing: float = 40.0
    scenario_id: str = "scenario"

    def __post_init__(self):
        if self.dt <= 0 or self.density <= 0:
            raise ValueError("dt and density must be positive")

    def to_dict(self) -> dict:
        return {"scenario_id": self.scenario_id, "lane_count": self.road.lane_count,
                "lane_width": self.road.lane_width, "road_length": self.road.length, "density": self.density,
                "vehicle_count": self.vehicle_count, "seed": self.seed, "episode_length": self.episode_length,
                "dt": self.dt, "neighbor_speed": self.neighbor_speed, "ego_speed": self.ego_speed,
                "ego_lane": self.ego_lane, "spawn_base_spacing": self.spawn_base_spacing}

    @staticmethod
    def from_dict(d: dict) -> "ScenarioConfig":
        road = RoadSpec(int(d["lane_count"]), float(d.get("lane_width", 4.0)), float(d.get("road_length", 1500.0)))
        return ScenarioConfig(road, float(d["density"]), int(d["vehicle_count"]), int(d.get("seed", 0)),
                              int(d.get("episode_length", 150)), float(d.get("dt", 0.1)),
                              float(d.get("neighbor_speed", 11.0)), float(d.get("ego_speed", 10.0)),
                              int(d.get("ego_lane", 0)), float(d.get("spawn_base_spacing", 40.0)),
                              str(d.get("scenario_id", "scenario")))


@dataclass(frozen=True)
class TrafficParams:
    """IDMParams + MOBILParams defaults (pkg/highway.py:73-89), tick length, ego wheelbase."""

    v0: float = 12.0
    time_headway: float = 1.5
    s0: float = 2.0
    a_max: float = 1.5
    b_comfort: float = 2.0
    delta: float = 4.0
    b_hard: float = 6.0
    politeness: float = 0.3
    b_safe: float = 4.0
    a_threshold: float = 0.1
    cooldown: float = 4.0
    dt: float = 0.1
    wheelbase: float = 2.5

    def c_struct(self) -> Traffic:
        return Traffic(*[float(getattr(self, f.name)) for f in fields(self)])


def _arr(x, dtype):
    return x if hasattr(x, "data_ptr") else np.ascontiguousarray(x, dtype=dtype)


@dataclass
class SimState:
    ego: object
    ego_ts: object
    veh: object
    veh_ext: object
    n_veh: object
    road: object
    world: object
    curvature: list | None = None      # host-side per-world road curvature tables (planning only)

    @property
    def size(self) -> int:
        return int(self.ego.shape[0])

    @property
    def n_max(self) -> int:
        return int(self.veh.shape[1])

    @property
    def worlds(self) -> WorldBatch:
        """The scene-build view (ego, veh, n_veh, road) of the same buffers."""
        return WorldBatch(self.ego, self.veh, self.n_veh, self.road, self.curvature)

    def to(self, device):
        """Copy to a torch device (e.g. "cuda:0"); device=None returns host numpy arrays."""
        import torch
        out = {}
        for f in fields(self):
            v = getattr(self, f.name)
            if f.name == "curvature":
                out[f.name] = v
                continue
            if device is None:
                out[f.name] = v.cpu().numpy() if hasattr(v, "cpu") else np.array(v)
            else:
                t = v if hasattr(v, "data_ptr") else torch.from_numpy(np.ascontiguousarray(v))
                out[f.name] = t.to(device).contiguous()
        return SimState(**out)

    @staticmethod
    def spawn(scenarios) -> "SimState":
        """spawn_world (pkg/highway.py:168-205) for each scenario, bit-exact with the reference."""
        scenarios = list(scenarios)
        S = len(scenarios)
        n_max = max(1, max(sc.vehicle_count for sc in scenarios))
        st = SimState(np.zeros((S, 8)), np.zeros(S), np.zeros((S, n_max, 5)), np.zeros((S, n_max, 7)),
                      np.zeros(S, np.int32), np.zeros((S, 2)), np.zeros((S, 5)))
        st.world[:, 3] = -1.0
        for s, sc in enumerate(scenarios):
            r = sc.road
            rec = HighwayRecipe(lanes=r.lane_count, density=sc.density, vehicle_count=sc.vehicle_count,
                                lane_width=r.lane_width, neighbor_speed=sc.neighbor_speed, ego_speed=sc.ego_speed,
                                ego_lane=sc.ego_lane, spawn_base_spacing=sc.spawn_base_spacing)
            st.ego[s] = (0.0, sc.ego_lane * r.lane_width, 0.0, sc.ego_speed, 0.0, 0.0, 5.0, 2.0)
            st.ego_ts[s] = sc.ego_speed
            for j, (x, y, v, cd) in enumerate(_spawn(sc.seed, rec, with_cooldown=True)):
                st.veh[s, j] = (x, y, 0.0, v, 0.0)
                st.veh_ext[s, j] = (5.0, 2.0, v, j % r.lane_count, cd, 0.0, j % r.lane_count)
            st.n_veh[s] = sc.vehicle_count
            st.road[s] = (r.lane_count, r.lane_width)
        curv = [sc.road.curvature for sc in scenarios]
        st.curvature = curv if any(c is not None for c in curv) else None
        return st

    @staticmethod
    def from_worlds(worlds) -> "SimState":
        """From the reference's World objects (duck-typed: ego, neighbors, road, time, step_count, ...)."""
        S = len(worlds)
        n_max = max(1, max(len(w.neighbors) for w in worlds))
        st = SimState(np.zeros((S, 8)), np.zeros(S), np.zeros((S, n_max, 5)), np.zeros((S, n_max, 7)),
                      np.zeros(S, np.int32), np.zeros((S, 2)), np.zeros((S, 5)))
        for s, w in enumerate(worlds):
            e = w.ego
            st.ego[s] = (e.x, e.y, e.psi, e.v, e.accel, e.steer, e.length, e.width)
            st.ego_ts[s] = e.target_speed
            for j, v in enumerate(w.neighbors):
                st.veh[s, j] = (v.x, v.y, v.psi, v.v, v.lateral_rate)
                st.veh_ext[s, j] = (v.length, v.width, v.target_speed, v.target_lane, v.cooldown, v.accel,
                                    v.lane_index)
            st.n_veh[s] = len(w.neighbors)
            st.road[s] = (w.road.lane_count, w.road.lane_width)
            st.world[s] = (w.time, w.step_count, float(w.collided),
                           -1.0 if w.collision_step is None else float(w.collision_step), float(w.lane_departed))
        curv = [getattr(w.road, "curvature", None) for w in worlds]
        st.curvature = curv if any(c is not None for c in curv) else None
        return st


class Simulator:
    """step / the open-loop stretch of run_episode for a SimState, on the device (bd_sim_run)."""

    def __init__(self, ctx, traffic: TrafficParams = TrafficParams()):
        self.ctx = ctx
        self.traffic = traffic
        self._c = traffic.c_struct()

    def run(self, st: SimState, controls, n_steps: int, ctrl_offset: int = 0, x_end=None, active=None,
            snapshots: bool | object = False):
        """Advance every (active) world by n_steps ticks in place.

        controls: S x n_ctrl x 2 (accel, steer); tick j uses index min(ctrl_offset + j, n_ctrl - 1)
        (pkg/highway.py:520-521).  x_end (S): stop a world after it collides or reaches
        ego.x >= x_end (run_episode, :524-529) and clear its `active` flag.  Returns
        (steps_done S, snapshots S x n_steps x (8 + 4 n_max) or None)."""
        S, n_max = st.size, st.n_max
        ctrl = _arr(controls, np.float64)
        if ctrl.shape[0] != S or ctrl.shape[-1] != 2:
            raise ValueError("controls must be S x n_ctrl x 2")
        done = np.zeros(S, np.int32)
        snap = None
        if snapshots is True:
            snap = np.empty((S, n_steps, SNAP_HEAD + 4 * n_max))
        elif snapshots is not False and snapshots is not None:
            snap = snapshots
        xe = None if x_end is None else _arr(x_end, np.float64)
        act = None if active is None else active
        if isinstance(act, np.ndarray) and act.dtype != np.int32:
            raise ValueError("active must be int32")
        self.ctx.call("bd_sim_run", S, n_max, st.ego, st.ego_ts, st.veh, st.veh_ext, _arr(st.n_veh, np.int32),
                      st.road, st.world, ctypes.byref(self._c), int(n_steps), ctrl, int(ctrl.shape[1]),
                      int(ctrl_offset), xe, act, done, snap)
        return done, snap
