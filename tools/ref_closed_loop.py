"""Reference closed-loop outcomes (development container only: imports /root/reference).

    PYTHONPATH=/root/reference/pkg/src python tools/ref_closed_loop.py --seeds 0 1 ... --out FILE

Runs the reference's run_episode with MPCBiLevelPlanner(PlannerEnvConfig()) per seed (one process
per seed) and writes {seed: {steps, collided, collision_step, mean_speed, solve_time}} as JSON,
for the statistical comparison with the device closed loop (tools/closed_loop_compare.py)."""
import argparse
import json
import os
import sys
from concurrent.futures import ProcessPoolExecutor

os.environ.setdefault("OPENBLAS_NUM_THREADS", "1")
sys.path.insert(0, "/root/reference/pkg/src")


def one(args):
    seed, lanes, density, vehicles, length, planner = args
    from bilevel_drive.highway import RoadSpec, ScenarioConfig, run_episode
    from bilevel_drive.planners import PlannerEnvConfig, make_planner
    sc = ScenarioConfig(RoadSpec(lanes), density, vehicles, seed, episode_length=length)
    log = run_episode(sc, make_planner(planner, PlannerEnvConfig(), seed=0))
    return seed, {"steps": len(log.steps), "collided": log.collided, "collision_step": log.collision_step,
                  "lane_departed": log.lane_departed, "failed": log.failed, "mean_speed": log.mean_speed(),
                  "solve_time": sum(log.solve_times()) / max(1, len(log.solve_times()))}


if __name__ == "__main__":
    ap = argparse.ArgumentParser()
    ap.add_argument("--seeds", type=int, nargs="+", default=list(range(8)))
    ap.add_argument("--lanes", type=int, default=4)
    ap.add_argument("--density", type=float, default=1.0)
    ap.add_argument("--vehicles", type=int, default=12)
    ap.add_argument("--length", type=int, default=150)
    ap.add_argument("--workers", type=int, default=os.cpu_count())
    ap.add_argument("--planner", default="mpc-bilevel")
    ap.add_argument("--out", required=True)
    a = ap.parse_args()
    with ProcessPoolExecutor(a.workers) as ex:
        res = dict(ex.map(one, [(s, a.lanes, a.density, a.vehicles, a.length, a.planner) for s in a.seeds]))
    cfg = {"lanes": a.lanes, "density": a.density, "vehicles": a.vehicles, "length": a.length, "planner": a.planner}
    json.dump({"config": cfg, "episodes": {str(k): v for k, v in sorted(res.items())}}, open(a.out, "w"), indent=1)
    print(json.dumps(cfg), sum(v["collided"] for v in res.values()), "collisions of", len(res))
