"""Persistent CEM kernel vs launch chain: where do the two paths first differ? (diagnostic)"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import numpy as np
import paper_2212_02224_b200 as bd
from paper_2212_02224_b200.fleet import FleetPlanner
from paper_2212_02224_b200.scenes import highway_scene
basis = bd.build_basis(10, 100, 5.0, "bernstein")
for N in (1, 2, 4):
    cfg = bd.BiLevelConfig(1000, 150, 100, N, 0.7, 0.9, 1.0)
    fp = FleetPlanner(basis, bd.TrackingWeights(), bd.ParamLayout(4), bd.ProjectionConfig(1.0, 100, 1e-3), 10, cfg)
    sc = [highway_scene(5)]
    out = []
    for opt in (1, 0):
        fp.context.set_option("persistent_cycle", opt)
        r = fp.plan(sc, seed=3)
        B = 1000
        P = np.empty((B, 8)); X = np.empty((B, 22)); R = np.empty(B); C = np.empty(B)
        fp.context.call("bd_cem_last_batch", 1, B, P, X, R, C)
        out.append((r, P, X, R, C))
    (ra, Pa, Xa, Ra, Ca), (rb, Pb, Xb, Rb, Cb) = out
    print(f"N={N}: persistent_cycles={fp.context.stat('persistent_cycles')}",
          "params eq", np.array_equal(Pa, Pb), "max dP", np.abs(Pa - Pb).max(),
          "xi eq", np.array_equal(Xa, Xb), "max dxi", np.abs(Xa - Xb).max(),
          "res eq", np.array_equal(Ra, Rb), "cost eq", np.array_equal(Ca, Cb),
          "stats eq", np.array_equal(ra.stats, rb.stats))
