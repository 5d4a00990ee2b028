"""A few config-2 cycles on the per-iteration launch chain (persistent kernel off), for ncu."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import paper_2212_02224_b200 as bd
from paper_2212_02224_b200.fleet import FleetPlanner
from paper_2212_02224_b200.scenes import highway_scene
basis = bd.build_basis(10, 100, 5.0, "bernstein")
cfg = bd.BiLevelConfig(1000, 150, 100, 4, 0.7, 0.9, 1.0)
fp = FleetPlanner(basis, bd.TrackingWeights(), bd.ParamLayout(4), bd.ProjectionConfig(1.0, 100, 1e-3), 10, cfg)
fp.context.set_option("persistent_cycle", 0)
for k in range(int(sys.argv[1]) if len(sys.argv) > 1 else 2):
    fp.plan([highway_scene(0)], seed=k)
print("ok")
