"""Config-2 cycle: wall p50 of FleetPlanner.plan (device Philox) and solve_bilevel with the
persistent kernel on / off (diagnostic; run under ncu for the kernel durations)."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import numpy as np
import paper_2212_02224_b200 as bd
from paper_2212_02224_b200.fleet import FleetPlanner, initial_distribution
from paper_2212_02224_b200.scenes import highway_scene
reps = int(sys.argv[1]) if len(sys.argv) > 1 else 60
basis = bd.build_basis(10, 100, 5.0, "bernstein")
cfg = bd.BiLevelConfig(1000, 150, 100, 4, 0.7, 0.9, 1.0)
fp = FleetPlanner(basis, bd.TrackingWeights(), bd.ParamLayout(4), bd.ProjectionConfig(1.0, 100, 1e-3), 10, cfg)
sc = [highway_scene(0)]
solver = bd.LowerLevelSolver(basis, bd.TrackingWeights(), bd.ParamLayout(4), bd.ProjectionConfig(1.0, 100, 1e-3), 10)
mean, cov = initial_distribution(sc[0])
cfg2 = bd.BiLevelConfig(1000, 150, 100, 4, 0.7, 0.9, 1.0, mean, cov)
rem = int(sys.argv[2]) if len(sys.argv) > 2 else 1
fp.context.set_option("remainder_warp", rem)
solver.context.set_option("remainder_warp", rem)
for opt in (1, 0, 1, 0):
    fp.context.set_option("persistent_cycle", opt)
    solver.context.set_option("persistent_cycle", opt)
    for _ in range(3):
        fp.plan(sc, seed=0)
        bd.solve_bilevel(sc[0], solver, cfg2, np.random.default_rng(0))
    t = []
    for k in range(reps):
        t0 = time.perf_counter(); fp.plan(sc, seed=k); t.append(time.perf_counter() - t0)
    u = []
    for k in range(reps):
        rng = np.random.default_rng(k)
        t0 = time.perf_counter(); bd.solve_bilevel(sc[0], solver, cfg2, rng); u.append(time.perf_counter() - t0)
    print(f"remainder_warp={rem} persistent={opt}: plan p50 {np.median(t) * 1e3:.3f} ms, solve_bilevel p50 {np.median(u) * 1e3:.3f} ms")
