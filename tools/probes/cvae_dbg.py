"""test_config3 sequence with the persistent kernel on / off (diagnostic)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import numpy as np
import paper_2212_02224_b200 as bd
from paper_2212_02224_b200.cvae import CVAEDecoder
from paper_2212_02224_b200.fleet import initial_distribution
from paper_2212_02224_b200.scenes import highway_scene
persist = int(sys.argv[1])
basis = bd.build_basis(10, 100, 5.0, "bernstein")
solver = bd.LowerLevelSolver(basis, bd.TrackingWeights(), bd.ParamLayout(4), bd.ProjectionConfig(1.0, 100, 1e-3), 10)
solver.context.set_option("persistent_cycle", persist)
scene = highway_scene(2)
mean, cov = initial_distribution(scene)
dec = CVAEDecoder.synthetic(3, context=solver.context)
rng = np.random.default_rng(5)
obs = np.zeros(55)
raw = dec.decode(obs, rng.standard_normal((1000, 2)))
shift = mean - raw.mean(axis=0)
ws = dec.warm_start(obs, 1000, solver.layout, np.random.default_rng(5), shift=shift)
print("warm finite", np.isfinite(ws.samples).all(), ws.samples.std(axis=0).round(3))
for N in (4, 1, 1):
    cfg = bd.BiLevelConfig(1000, 150, 100, N, 0.7, 0.9, 1.0, mean, cov)
    try:
        r = bd.solve_bilevel(scene, solver, cfg, np.random.default_rng(6), warm_start=ws)
        c = r.distribution.cov
        print(f"persist={persist} N={N}: best {r.best.index} done {len(r.diagnostics)} sym {np.allclose(c, c.T)} "
              f"diag {np.diag(c).round(4)} stats {[round(s.residual_median, 5) for s in r.diagnostics]}")
    except Exception as e:
        print(f"persist={persist} N={N}: {type(e).__name__}: {e}")
