import cProfile, pstats, sys, os
sys.path.insert(0, os.getcwd())
import numpy as np
import paper_2212_02224_b200 as bd
from paper_2212_02224_b200.fleet import initial_distribution
from paper_2212_02224_b200.scenes import highway_scene
basis = bd.build_basis(10, 100, 5.0, "bernstein")
solver = bd.LowerLevelSolver(basis, bd.TrackingWeights(), bd.ParamLayout(4), bd.ProjectionConfig(1.0, 100, 1e-3), 10)
scene = highway_scene(0); mean, cov = initial_distribution(scene)
cfg = bd.BiLevelConfig(1000, 150, 100, 4, 0.7, 0.9, 1.0, mean, cov)
rng = np.random.default_rng(0)
for _ in range(5): bd.solve_bilevel(scene, solver, cfg, rng)
pr = cProfile.Profile(); pr.enable()
for _ in range(50): bd.solve_bilevel(scene, solver, cfg, rng)
pr.disable()
st = pstats.Stats(pr); st.sort_stats("tottime").print_stats(18)
