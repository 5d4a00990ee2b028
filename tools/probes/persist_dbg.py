"""Which solve_bilevel shapes break the persistent kernel? (diagnostic; one case per process)"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import numpy as np
import paper_2212_02224_b200 as bd
from paper_2212_02224_b200.behavior import WarmStartSource
from paper_2212_02224_b200.fleet import initial_distribution
from paper_2212_02224_b200.scenes import highway_scene
N, warm, persist = int(sys.argv[1]), int(sys.argv[2]), int(sys.argv[3])
basis = bd.build_basis(10, 100, 5.0, "bernstein")
solver = bd.LowerLevelSolver(basis, bd.TrackingWeights(), bd.ParamLayout(4), bd.ProjectionConfig(1.0, 100, 1e-3), 10)
solver.context.set_option("persistent_cycle", persist)
scene = highway_scene(1)
mean, cov = initial_distribution(scene)
cfg = bd.BiLevelConfig(1000, 150, 100, N, 0.7, 0.9, 1.0, mean, cov)
ws = WarmStartSource(np.random.default_rng(9).multivariate_normal(mean, cov, 1000), solver.layout) if warm else None
if len(sys.argv) > 4:   # an earlier cycle of N' iterations on the same context first
    cfg0 = bd.BiLevelConfig(1000, 150, 100, int(sys.argv[4]), 0.7, 0.9, 1.0, mean, cov)
    bd.solve_bilevel(scene, solver, cfg0, np.random.default_rng(6), warm_start=ws)
try:
    r = bd.solve_bilevel(scene, solver, cfg, np.random.default_rng(4), warm_start=ws)
    print(f"N={N} warm={warm} persist={persist} prev={sys.argv[4:]}: best {r.best.index} cov sym {np.allclose(r.distribution.cov, r.distribution.cov.T)} "
          f"trace {np.trace(r.distribution.cov):.4f} stats {[round(s.residual_median, 5) for s in r.diagnostics]}")
except Exception as e:
    print(f"N={N} warm={warm} persist={persist}: {type(e).__name__}: {e}")
