"""Device closed loop vs the reference's outcomes (statistical parity of SURVEY §8f row 4).

    python tools/closed_loop_compare.py --ref profiles/r01/closed_loop/ref_d1.json [--repeats 4]

Runs run_episodes with BatchMPCBiLevelPlanner(PlannerEnvConfig()) on the reference file's
scenario config and seeds, `repeats` times with different device Philox seeds, and prints
collision rate / steps survived / mean speed beside the reference's (one seeded numpy Generator
per planner there, so individual episodes differ; the distributions should agree)."""
import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402

from paper_2212_02224_b200.episodes import run_episodes  # noqa: E402
from paper_2212_02224_b200.planners import PlannerEnvConfig, make_batch_planner  # noqa: E402
from paper_2212_02224_b200.sim import RoadSpec, ScenarioConfig  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--ref", required=True)
ap.add_argument("--repeats", type=int, default=4)
ap.add_argument("--out", default=None)
a = ap.parse_args()
ref = json.load(open(a.ref))
c = ref["config"]
seeds = sorted(int(s) for s in ref["episodes"])
scs = [ScenarioConfig(RoadSpec(c["lanes"]), c["density"], c["vehicles"], s, episode_length=c["length"]) for s in seeds]


def summary(eps):
    steps = np.array([e["steps"] for e in eps])
    col = np.array([e["collided"] for e in eps])
    return {"episodes": len(eps), "collision_rate": float(col.mean()), "mean_steps": float(steps.mean()),
            "mean_speed": float(np.mean([e["mean_speed"] for e in eps])),
            "lane_departures": int(sum(e["lane_departed"] for e in eps))}


ours = []
for r in range(a.repeats):
    planner = make_batch_planner("mpc-bilevel", PlannerEnvConfig(), seed=r)
    for lg in run_episodes(scs, planner):
        ours.append({"steps": len(lg.steps), "collided": lg.collided, "lane_departed": lg.lane_departed,
                     "mean_speed": lg.mean_speed(), "failed": lg.failed})
# the reference planner's own randomness (make_planner(..., seed=0) for every episode there)
planner = make_batch_planner("mpc-bilevel", PlannerEnvConfig(), generator_seeds=[0] * len(scs))
same = []
per_episode = []
for sd, lg in zip(seeds, run_episodes(scs, planner)):
    e = ref["episodes"][str(sd)]
    mine = {"steps": len(lg.steps), "collided": lg.collided, "lane_departed": lg.lane_departed,
            "mean_speed": lg.mean_speed(), "failed": lg.failed}
    same.append(mine)
    per_episode.append({"seed": sd, "ref_steps": e["steps"], "b200_steps": mine["steps"],
                        "ref_collided": e["collided"], "b200_collided": mine["collided"],
                        "ref_mean_speed": e["mean_speed"], "b200_mean_speed": mine["mean_speed"]})
res = {"config": c, "reference": summary(list(ref["episodes"].values())), "b200": summary(ours),
       "b200_repeats": a.repeats, "b200_reference_generators": summary(same),
       "same_outcome_episodes": int(sum(p["ref_steps"] == p["b200_steps"] and p["ref_collided"] == p["b200_collided"]
                                       for p in per_episode)),
       "per_episode_reference_generators": per_episode}
print(json.dumps(res, indent=1))
if a.out:
    json.dump(res, open(a.out, "w"), indent=1)
