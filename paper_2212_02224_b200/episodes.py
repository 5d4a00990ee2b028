"""Closed-loop episodes and benchmark suites for a fleet of worlds.

Batched restatement of ``run_episode`` (pkg/highway.py:487-532), ``EpisodeLog``
(:413-475) and the suite harness ``run_suite`` / ``write_outputs`` (pkg/bench.py:32-205).
All S episodes of a batch advance in lockstep: at every replan instant one batched planning
call (:mod:`.planners`) plans every live world from the simulator's HBM state, then one
``bd_sim_run`` launch executes the plans open loop up to the next replan instant, stopping
worlds on collision or at the end of the road.  Per-step records come back from the device as
one snapshot block per stretch and are unpacked into reference-format ``EpisodeLog`` records.
"""

from __future__ import annotations

import hashlib
import json
import os
import time
from dataclasses import dataclass, field

import numpy as np

from .planners import PlannerEnvConfig, make_batch_planner
from .sim import SNAP_HEAD, ScenarioConfig, SimState, Simulator, TrafficParams

__all__ = ["EpisodeLog", "run_episodes", "BenchmarkSuite", "MetricsRow", "run_suite", "write_outputs",
           "suite_from_dict", "load_suite", "METRICS_HEADER", "TIMINGS_HEADER"]

METRICS_HEADER = "planner,scenario,episodes,collisions,collision_rate,mean_speed,failures"
TIMINGS_HEADER = "planner,scenario,mean_solve_time,total_wall_time"


@dataclass
class EpisodeLog:
    """Per-step record of one episode plus outcome flags (pkg/highway.py:413-475, same JSONL)."""

    meta: dict
    steps: list = field(default_factory=list)
    plan_records: list = field(default_factory=list)
    collided: bool = False
    collision_step: int | None = None
    lane_departed: bool = False
    failed: bool = False
    failure_reason: str = ""

    def ego_speeds(self) -> np.ndarray:
        if isinstance(self.steps, _StepRecords):
            return self.steps.ego_speeds()
        return np.array([rec["ego"][3] for rec in self.steps])

    def mean_speed(self) -> float:
        sp = self.ego_speeds()
        return float(sp.mean()) if sp.size else 0.0

    def solve_times(self) -> list:
        return [rec["solve_time"] for rec in self.plan_records if "solve_time" in rec]

    def write_jsonl(self, path: str) -> None:
        with open(path, "w", encoding="utf-8") as fh:
            header = {"type": "meta", **self.meta, "collided": self.collided, "collision_step": self.collision_step,
                      "lane_departed": self.lane_departed, "failed": self.failed,
                      "failure_reason": self.failure_reason}
            fh.write(json.dumps(header, sort_keys=True) + "\n")
            for rec in self.plan_records:
                fh.write(json.dumps({"type": "plan", **rec}, sort_keys=True) + "\n")
            for rec in self.steps:
                fh.write(json.dumps({"type": "step", **rec}, sort_keys=True) + "\n")

    @staticmethod
    def read_jsonl(path: str) -> "EpisodeLog":
        meta, steps, plans = {}, [], []
        with open(path, "r", encoding="utf-8") as fh:
            for line in fh:
                rec = json.loads(line)
                kind = rec.pop("type")
                if kind == "meta":
                    meta = rec
                elif kind == "step":
                    steps.append(rec)
                elif kind == "plan":
                    plans.append(rec)
        log = EpisodeLog(meta=meta, steps=steps, plan_records=plans)
        log.collided = bool(meta.pop("collided", False))
        log.collision_step = meta.pop("collision_step", None)
        log.lane_departed = bool(meta.pop("lane_departed", False))
        log.failed = bool(meta.pop("failed", False))
        log.failure_reason = str(meta.pop("failure_reason", ""))
        return log


class _StepRecords(list):
    """EpisodeLog.steps filled lazily: the device snapshot blocks are kept as arrays and turned into
    the reference's per-step dicts on first read (suite metrics only need the ego speeds, which
    come straight from the arrays)."""

    def __init__(self, nv: int):
        super().__init__()
        self._nv = nv
        self._blocks = []

    def _add_block(self, block: np.ndarray) -> None:
        if self._blocks is None:
            super().extend(_snapshots(block, self._nv))
        else:
            self._blocks.append(block)

    def _fill(self) -> None:
        if self._blocks is not None:
            blocks, self._blocks = self._blocks, None
            for b in blocks:
                super().extend(_snapshots(b, self._nv))

    def ego_speeds(self) -> np.ndarray:
        if self._blocks is not None:
            return np.concatenate([b[:, 4] for b in self._blocks]) if self._blocks else np.zeros(0)
        return np.array([rec["ego"][3] for rec in self])

    def __len__(self):
        return sum(b.shape[0] for b in self._blocks) if self._blocks is not None else super().__len__()

    def __bool__(self):
        return len(self) > 0


def _materialising(name):
    base = getattr(list, name)

    def method(self, *a, **kw):
        self._fill()
        for x in a:                    # list's C fast paths read another list's storage directly
            if isinstance(x, _StepRecords):
                x._fill()
        return base(self, *a, **kw)
    method.__name__ = name
    return method


for _name in ("__iter__", "__getitem__", "__eq__", "__ne__", "__lt__", "__le__", "__gt__", "__ge__", "__contains__",
              "__reversed__", "__repr__", "append", "extend", "insert", "pop", "remove", "index", "count", "copy",
              "__add__", "__iadd__", "__mul__", "__setitem__", "__delitem__", "sort", "reverse", "clear"):
    setattr(_StepRecords, _name, _materialising(_name))


def _snapshots(block: np.ndarray, nv: int) -> list:
    """run_episode step records (pkg/highway.py:478-485) from a block of device snapshot rows
    (one C-level tolist() per block, then plain list slicing)."""
    head = block[:, :SNAP_HEAD].tolist()
    nbrs = block[:, SNAP_HEAD:SNAP_HEAD + 4 * nv].reshape(block.shape[0], nv, 4).tolist()
    return [{"t": round(h[0], 6), "ego": h[1:5], "ctrl": h[5:7], "neighbors": nb, "collision": h[7] != 0.0}
            for h, nb in zip(head, nbrs)]


def run_episodes(scenarios, planner, replan_stride: int = 5, road_end_margin: float = 60.0, device="cuda:0",
                 record_steps: bool = True) -> list:
    """run_episode (pkg/highway.py:487-532) for every scenario at once.

    `planner` is a batch planner (:func:`.planners.make_batch_planner`); its failures end the
    affected episode (failed=True, failure_reason "Type: message") and the others continue."""
    scenarios = list(scenarios)
    S = len(scenarios)
    dts = {float(sc.dt) for sc in scenarios}
    if len(dts) != 1:
        raise ValueError("all scenarios of one batch must share dt")
    dt = dts.pop()
    if abs(planner.dt - dt) > 0:
        raise ValueError(f"planner control grid dt={planner.dt} differs from the scenarios' dt={dt}")
    if planner.n_ctrl < 1:
        raise ValueError("planner horizon shorter than one tick")
    host = SimState.spawn(scenarios)
    road_host = host.road.copy()
    n_veh = host.n_veh.copy()
    st = host.to(device) if device is not None else host
    sim = Simulator(planner.context, TrafficParams(dt=dt, wheelbase=planner.env.wheelbase))
    planner.reset()
    logs = [EpisodeLog(meta={"scenario": sc.to_dict(), "planner": planner.name, "replan_stride": replan_stride},
                       steps=_StepRecords(int(n_veh[s]))) for s, sc in enumerate(scenarios)]
    lengths = np.array([sc.episode_length for sc in scenarios])
    x_end = np.array([sc.road.length - road_end_margin for sc in scenarios], dtype=np.float64)
    active = (lengths > 0).astype(np.int32)
    ctrl = None
    k = offset = 0
    while active.any():
        if k % replan_stride == 0:
            plan = planner.plan_cycle(st, road_host)
            for s in np.flatnonzero(active):
                if plan.failures[s] is not None:
                    logs[s].failed = True
                    logs[s].failure_reason = plan.failures[s]
                    active[s] = 0
                else:
                    logs[s].plan_records.append({"step": int(k), **plan.infos[s]})
            offset = 0
            if not active.any():
                break
            ctrl = np.ascontiguousarray(np.stack([plan.accels, plan.steers], axis=-1))
        n = replan_stride - (k % replan_stride)
        n = int(min(n, (lengths[active.astype(bool)] - k).min()))
        was = active.copy()
        done, snap = sim.run(st, ctrl, n, ctrl_offset=offset, x_end=x_end, active=active, snapshots=record_steps)
        if record_steps:
            for s in np.flatnonzero(was):
                if done[s]:
                    logs[s].steps._add_block(snap[s, :int(done[s])].copy())
        k += n
        offset += n
        active[(lengths <= k) & (active != 0)] = 0
    w = st.world.cpu().numpy() if hasattr(st.world, "cpu") else st.world
    for s, log in enumerate(logs):
        if w[s, 2] != 0.0 and not log.failed:
            log.collided = True
            log.collision_step = int(w[s, 3])
        log.lane_departed = bool(w[s, 4] != 0.0)
    return logs


# ----------------------------------------------------------------------------- suites
@dataclass(frozen=True)
class BenchmarkSuite:
    """pkg/bench.py:32-52: every planner over the same (scenario, seed) cells."""

    scenarios: tuple
    planners: tuple
    episodes_per_cell: int = 50
    seeds: tuple = ()
    env: PlannerEnvConfig = field(default_factory=PlannerEnvConfig)
    replan_stride: int = 5
    workers: int = 1

    def __post_init__(self):
        from .planners import BATCH_PLANNER_REGISTRY
        unknown = [p for p in self.planners if p not in BATCH_PLANNER_REGISTRY]
        if unknown:
            raise ValueError(f"unknown planners in suite: {unknown}")
        if not self.seeds:
            object.__setattr__(self, "seeds", tuple(range(self.episodes_per_cell)))
        if len(self.seeds) != self.episodes_per_cell:
            raise ValueError("seed list length must equal episodes_per_cell")


@dataclass
class MetricsRow:
    planner: str
    scenario_id: str
    episodes: int
    collisions: int
    collision_rate: float
    mean_speed: float
    mean_solve_time: float
    failures: int

    def metrics_csv(self) -> str:
        return ",".join([self.planner, self.scenario_id, str(self.episodes), str(self.collisions),
                         repr(self.collision_rate), repr(self.mean_speed), str(self.failures)])

    def timing_csv(self, wall: float) -> str:
        return ",".join([self.planner, self.scenario_id, repr(self.mean_solve_time), repr(wall)])


def suite_from_dict(data: dict, workers: int | None = None) -> BenchmarkSuite:
    env = PlannerEnvConfig(**data.get("env", {}))
    return BenchmarkSuite(scenarios=tuple(ScenarioConfig.from_dict(sc) for sc in data["scenarios"]),
                          planners=tuple(data["planners"]), episodes_per_cell=int(data.get("episodes_per_cell", 50)),
                          seeds=tuple(data.get("seeds", ())), env=env,
                          replan_stride=int(data.get("replan_stride", 5)),
                          workers=workers if workers is not None else int(data.get("workers", 1)))


def load_suite(path: str, workers: int | None = None) -> BenchmarkSuite:
    import yaml
    with open(path, "r", encoding="utf-8") as fh:
        return suite_from_dict(yaml.safe_load(fh), workers=workers)


def run_suite(suite: BenchmarkSuite, device="cuda:0"):
    """run_suite (pkg/bench.py:114-170): per planner, every (scenario, seed) episode in one
    lockstep batch (one batch per distinct dt).  Returns (rows, cell_wall, saw_numerical_failure);
    an episode's wall time is its batch's wall time divided evenly over the batch."""
    from dataclasses import replace
    rows, cell_wall, saw_nf = [], {}, False
    for pname in suite.planners:
        cells = [(sc, seed) for sc in suite.scenarios for seed in suite.seeds]
        results = [None] * len(cells)
        for dt in sorted({float(sc.dt) for sc, _ in cells}):
            idx = [i for i, (sc, _) in enumerate(cells) if float(sc.dt) == dt]
            seeds = [cells[i][1] for i in idx]
            # each episode's planner draws from its own Generator seeded like the reference's
            # make_planner(name, env, seed=seed) (mpc-bilevel and mpc-random)
            kw = {"generator_seeds": seeds} if pname == "mpc-bilevel" else {}
            planner = make_batch_planner(pname, suite.env, seed=seeds if pname == "mpc-random" else 0, dt=dt, **kw)
            t0 = time.perf_counter()
            logs = run_episodes([replace(cells[i][0], seed=cells[i][1]) for i in idx], planner,
                                replan_stride=suite.replan_stride, device=device)
            wall = (time.perf_counter() - t0) / len(idx)
            for i, log in zip(idx, logs):
                results[i] = {"wall": wall, "collided": log.collided, "failed": log.failed,
                              "mean_speed": log.mean_speed(), "solve_times": log.solve_times(),
                              "numerical_failure": "NumericalFailure" in log.failure_reason}
        n = len(suite.seeds)
        for c, sc in enumerate(suite.scenarios):
            cell = results[c * n:(c + 1) * n]
            collisions = sum(1 for r in cell if r["collided"])
            saw_nf |= any(r["numerical_failure"] for r in cell)
            clean = [r["mean_speed"] for r in cell if not r["collided"] and not r["failed"]]
            st = [t for r in cell for t in r["solve_times"]]
            rows.append(MetricsRow(pname, sc.scenario_id, len(cell), collisions, collisions / len(cell),
                                   float(np.mean(clean)) if clean else float("nan"),
                                   float(np.mean(st)) if st else float("nan"),
                                   sum(1 for r in cell if r["failed"])))
            cell_wall[f"{pname}/{sc.scenario_id}"] = float(sum(r["wall"] for r in cell))
    return rows, cell_wall, saw_nf


def _fingerprint(suite: BenchmarkSuite) -> str:
    payload = {"planners": list(suite.planners), "scenarios": [sc.to_dict() for sc in suite.scenarios],
               "episodes_per_cell": suite.episodes_per_cell, "seeds": list(suite.seeds),
               "env": {k: getattr(suite.env, k) for k in sorted(vars(suite.env))},
               "replan_stride": suite.replan_stride}
    return hashlib.sha256(json.dumps(payload, sort_keys=True).encode()).hexdigest()


def write_outputs(suite: BenchmarkSuite, rows, cell_wall: dict, out_dir: str, package_version: str | None = None):
    """metrics.csv (byte-stable), timings.csv and manifest.json in the reference's format
    (pkg/bench.py:173-205)."""
    from . import __version__
    os.makedirs(out_dir, exist_ok=True)
    paths = {k: os.path.join(out_dir, f) for k, f in
             (("metrics", "metrics.csv"), ("timings", "timings.csv"), ("manifest", "manifest.json"))}
    with open(paths["metrics"], "w", encoding="utf-8") as fh:
        fh.write(METRICS_HEADER + "\n")
        for r in rows:
            fh.write(r.metrics_csv() + "\n")
    with open(paths["timings"], "w", encoding="utf-8") as fh:
        fh.write(TIMINGS_HEADER + "\n")
        for r in rows:
            fh.write(r.timing_csv(cell_wall.get(f"{r.planner}/{r.scenario_id}", float("nan"))) + "\n")
    manifest = {"config_hash": _fingerprint(suite), "seeds": list(suite.seeds),
                "package_version": package_version or __version__, "numpy_version": np.__version__}
    with open(paths["manifest"], "w", encoding="utf-8") as fh:
        json.dump(manifest, fh, sort_keys=True, indent=2)
        fh.write("\n")
    return paths
