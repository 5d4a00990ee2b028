"""Per-seed closed-loop outcomes on the sparse 2-lane scenario (seeds 0-7) for comparison with
profiles/r01/acceptance/ref_sparse2_*.json (tools/ref_closed_loop.py on the reference)."""
import json
import os
import sys
sys.path.insert(0, os.getcwd())
from dataclasses import replace  # noqa: E402
from paper_2212_02224_b200.episodes import run_episodes  # noqa: E402
from paper_2212_02224_b200.planners import PlannerEnvConfig, make_batch_planner  # noqa: E402
from paper_2212_02224_b200.sim import RoadSpec, ScenarioConfig  # noqa: E402
seeds = list(range(8))
base = ScenarioConfig(RoadSpec(2), 1.0, 10, 0, episode_length=150)
out = {}
for name in ("mpc-bilevel", "mpc-vanilla"):
    kw = {"generator_seeds": [0] * len(seeds)} if name == "mpc-bilevel" else {}
    planner = make_batch_planner(name, PlannerEnvConfig(), seed=0, **kw)
    logs = run_episodes([replace(base, seed=s) for s in seeds], planner)
    out[name] = {str(s): {"steps": len(l.steps), "collided": l.collided, "mean_speed": l.mean_speed()}
                 for s, l in zip(seeds, logs)}
print(json.dumps(out))
