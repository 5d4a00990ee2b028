"""Host-side timeline of one drop-in solve_bilevel call (config 2), to see where the time
between the GPU kernels and the host-visible result goes."""
import os
import sys
import time
sys.path.insert(0, os.getcwd())
import numpy as np  # noqa: E402
import paper_2212_02224_b200 as bd  # noqa: E402
from paper_2212_02224_b200 import bilevel as B  # noqa: E402
from paper_2212_02224_b200.fleet import initial_distribution  # noqa: E402
from paper_2212_02224_b200.scenes import highway_scene  # noqa: E402

basis = bd.build_basis(10, 100, 5.0, "bernstein")
solver = bd.LowerLevelSolver(basis, bd.TrackingWeights(), bd.ParamLayout(4), bd.ProjectionConfig(1.0, 100, 1e-3), 10)
scene = highway_scene(0)
mean, cov = initial_distribution(scene)
cfg = bd.BiLevelConfig(1000, 150, 100, 4, 0.7, 0.9, 1.0, mean, cov)
rng = np.random.default_rng(0)
marks = []
orig_call = solver.context.call


def traced(name, *args):
    t0 = time.perf_counter()
    r = orig_call(name, *args)
    marks.append((name, t0, time.perf_counter()))
    return r


solver.context.call = traced
orig_normal = np.random.Generator.standard_normal
for _ in range(20):
    bd.solve_bilevel(scene, solver, cfg, rng)
rows = []
for _ in range(50):
    marks.clear()
    t0 = time.perf_counter()
    bd.solve_bilevel(scene, solver, cfg, rng)
    t1 = time.perf_counter()
    rows.append([(n, a - t0, b - t0) for n, a, b in marks] + [("total", 0.0, t1 - t0)])
med = {}
for r in rows:
    for k, (n, a, b) in enumerate(r):
        med.setdefault((k, n), []).append((a, b))
for (k, n), v in sorted(med.items()):
    a = np.median([x[0] for x in v]) * 1e6
    b = np.median([x[1] for x in v]) * 1e6
    print(f"{n:16s} start {a:8.1f} us  end {b:8.1f} us  (dur {b - a:7.1f})")
