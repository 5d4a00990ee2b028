"""Where the config-2 CEM cycle latency goes (host draws, copies, kernels).

    python tools/latency_breakdown.py
"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402

import paper_2212_02224_b200 as bd  # noqa: E402
from paper_2212_02224_b200.fleet import FleetPlanner, initial_distribution  # noqa: E402
from paper_2212_02224_b200.scenes import highway_scene  # noqa: E402

basis = bd.build_basis(10, 100, 5.0, "bernstein")
solver = bd.LowerLevelSolver(basis, bd.TrackingWeights(), bd.ParamLayout(4), bd.ProjectionConfig(1.0, 100, 1e-3), 10)
scene = highway_scene(0)
mean, cov = initial_distribution(scene)
cfg = bd.BiLevelConfig(1000, 150, 100, 4, 0.7, 0.9, 1.0, mean, cov)


def t(fn, n=30):
    fn()
    ts = []
    for _ in range(n):
        t0 = time.perf_counter()
        fn()
        ts.append(time.perf_counter() - t0)
    return 1e3 * float(np.median(ts))


rng = np.random.default_rng(0)
print(f"numpy draws 4x1000x8: {t(lambda: rng.standard_normal((4, 1000, 8))):.3f} ms")
print(f"solve_bilevel (drop-in): {t(lambda: bd.solve_bilevel(scene, solver, cfg, rng)):.3f} ms")
fp = FleetPlanner(basis, bd.TrackingWeights(), bd.ParamLayout(4), bd.ProjectionConfig(1.0, 100, 1e-3), 10,
                  bd.BiLevelConfig(1000, 150, 100, 4, 0.7, 0.9, 1.0))
fp.set_scenes([scene])
print(f"FleetPlanner.plan (device Philox, 1 scene): {t(lambda: fp.plan([scene], seed=1)):.3f} ms")
ctx = solver.context
ctx.set_option("timing", 1)
ctx.stat("reset")
bd.solve_bilevel(scene, solver, cfg, rng)
print(f"AM kernel time per cycle: {ctx.stat('am_ms'):.3f} ms over {ctx.stat('am_launches'):.0f} launches")
for lanes in (16, 32, 64):
    ctx.set_option("lanes_per_sample", lanes)
    ctx.stat("reset")
    bd.solve_bilevel(scene, solver, cfg, rng)
    ms = ctx.stat('am_ms')
    print(f"  lanes {lanes}: AM {ms:.3f} ms, cycle {t(lambda: bd.solve_bilevel(scene, solver, cfg, rng), 15):.3f} ms")
