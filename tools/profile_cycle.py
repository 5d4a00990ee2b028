"""A few config-2 CEM cycles through the drop-in solve_bilevel (for ncu launch lists)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402

import paper_2212_02224_b200 as bd  # noqa: E402
from paper_2212_02224_b200.fleet import initial_distribution  # noqa: E402
from paper_2212_02224_b200.scenes import highway_scene  # noqa: E402

basis = bd.build_basis(10, 100, 5.0, "bernstein")
solver = bd.LowerLevelSolver(basis, bd.TrackingWeights(), bd.ParamLayout(4), bd.ProjectionConfig(1.0, 100, 1e-3), 10)
scene = highway_scene(0)
mean, cov = initial_distribution(scene)
cfg = bd.BiLevelConfig(1000, 150, 100, 4, 0.7, 0.9, 1.0, mean, cov)
rng = np.random.default_rng(0)
for _ in range(int(sys.argv[1]) if len(sys.argv) > 1 else 3):
    bd.solve_bilevel(scene, solver, cfg, rng)
print("ok")
