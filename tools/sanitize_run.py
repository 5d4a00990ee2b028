"""Small invocations of every kernel family, for compute-sanitizer (memcheck / racecheck /
synccheck / initcheck):  compute-sanitizer --tool racecheck python tools/sanitize_run.py"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402

import paper_2212_02224_b200 as bd  # noqa: E402
from paper_2212_02224_b200.cvae import CVAEDecoder  # noqa: E402
from paper_2212_02224_b200.fleet import FleetPlanner  # noqa: E402
from paper_2212_02224_b200.scenes import highway_scene  # noqa: E402
from paper_2212_02224_b200.sim import RoadSpec, ScenarioConfig, SimState, Simulator  # noqa: E402
from paper_2212_02224_b200.worlds import ControlEmitter, PlannerEnv, build_scenes  # noqa: E402

basis = bd.build_basis(10, 100, 5.0, "bernstein")
cfg = bd.BiLevelConfig(96, 40, 20, 2, 0.7, 0.9, 1.0)
fp = FleetPlanner(basis, bd.TrackingWeights(), bd.ParamLayout(4), bd.ProjectionConfig(1.0, 12, 1e-3), 10, cfg)
scenes = [highway_scene(s) for s in range(2)]
for lanes in (8, 64):                                   # warp-group and two-warp mappings
    fp.context.set_option("lanes_per_sample", lanes)
    r = fp.plan(scenes, seed=1)
    assert np.all(r.iterations_done == 2)
fp.context.set_option("lanes_per_sample", 0)
solver = fp.solver
P = np.concatenate([np.random.default_rng(0).normal(4, 1.5, (40, 4)), np.random.default_rng(1).normal(10, 3, (40, 4))], 1)
solver.solve(P, scenes[0])
scs = [ScenarioConfig(RoadSpec(3), 1.5, 12, s) for s in range(3)]
st = SimState.spawn(scs)
build_scenes(fp.context, basis, st.worlds, PlannerEnv())
em = ControlEmitter(fp.context, basis, 5.0, 0.1, PlannerEnv())
acc, ste, _ = em.emit(r.best_xi)
Simulator(fp.context).run(st, np.stack([acc[:1].repeat(3, 0), ste[:1].repeat(3, 0)], -1), 6, x_end=np.full(3, 1e9),
                          active=np.ones(3, np.int32), snapshots=True)
dec = CVAEDecoder.synthetic(3, context=fp.context)
dec.decode(np.zeros(55), np.random.default_rng(2).standard_normal((130, 2)))
print("sanitize run ok")
