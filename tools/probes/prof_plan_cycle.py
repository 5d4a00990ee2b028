"""Host-side cost of FleetPlanner.plan_cycle (bench.py's e2e path) for 512 worlds."""
import cProfile
import os
import pstats
import sys
import time
sys.path.insert(0, os.getcwd())
import bench  # noqa: E402
from paper_2212_02224_b200.scenes import spawn_worlds  # noqa: E402
from paper_2212_02224_b200.worlds import ControlEmitter, PlannerEnv  # noqa: E402

planner = bench.make_planner(0)
ctx = planner.context
worlds = spawn_worlds(range(10_000, 10_512))
emitter = ControlEmitter(ctx, planner.solver.basis, bench.T, 0.1, PlannerEnv())
planner.plan_cycle(worlds, PlannerEnv(), emitter, seed=1)
t0 = time.perf_counter()
for k in range(3):
    planner.plan_cycle(worlds, PlannerEnv(), emitter, seed=2 + k, scene_offset=10_000)
print("plan_cycle ms", (time.perf_counter() - t0) / 3 * 1e3)
pr = cProfile.Profile()
pr.enable()
planner.plan_cycle(worlds, PlannerEnv(), emitter, seed=9, scene_offset=10_000)
pr.disable()
pstats.Stats(pr).sort_stats("tottime").print_stats(14)
