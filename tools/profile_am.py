"""Run one fleet CEM cycle for profiling the AM kernel under ncu.

    python tools/profile_am.py [--scenes S] [--lanes P] [--obs N]
"""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402

import paper_2212_02224_b200 as bd  # noqa: E402
from paper_2212_02224_b200.fleet import FleetPlanner  # noqa: E402
from paper_2212_02224_b200.scenes import HighwayRecipe, highway_scene  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--scenes", type=int, default=16)
ap.add_argument("--lanes", type=int, default=0)
ap.add_argument("--obs", type=int, default=10)
ap.add_argument("--batch", type=int, default=1000)
ap.add_argument("--cycles", type=int, default=2)
ap.add_argument("--spc", type=int, default=0)
ap.add_argument("--lat", type=int, default=None)
ap.add_argument("--rem", type=int, default=None)
a = ap.parse_args()
basis = bd.build_basis(10, 100, 5.0, "bernstein")
cfg = bd.BiLevelConfig(a.batch, min(150, a.batch), min(100, a.batch), 4, 0.7, 0.9, 1.0)
fp = FleetPlanner(basis, bd.TrackingWeights(), bd.ParamLayout(4), bd.ProjectionConfig(1.0, 100, 1e-3), a.obs, cfg)
if a.lanes:
    fp.context.set_option("lanes_per_sample", a.lanes)
if a.lat is not None:
    fp.context.set_option("latency_instance", a.lat)
if a.spc:
    fp.context.set_option("samples_per_cta", a.spc)
if a.rem is not None:
    fp.context.set_option("remainder_warp", a.rem)
rec = HighwayRecipe(n_obs=a.obs, density=3.0 if a.obs > 10 else 2.0, vehicle_count=80 if a.obs > 10 else 24,
                    obstacle_range=250.0 if a.obs > 10 else 120.0)
scenes = [highway_scene(s, rec) for s in range(a.scenes)]
r = fp.plan(scenes, seed=0)
fp.context.set_option("timing", 1)
fp.context.stat("reset")
for c in range(a.cycles):
    r = fp.plan(scenes, seed=c)
ms, n, si = fp.context.stat("am_ms"), fp.context.stat("am_launches"), fp.context.stat("am_sample_iters")
print(f"S={a.scenes} B={a.batch} obs={a.obs} lanes={a.lanes or 'auto'} spc={a.spc or 'auto'}: am {ms / n:.3f} ms/launch, "
      f"{si / (ms * 1e-3) / 1e9:.3f} G sample-iters/s, done {r.iterations_done.min()} cost {float(np.mean(r.best_cost)):.1f}")
