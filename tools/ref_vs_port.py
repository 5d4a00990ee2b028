"""Per-core speed of the reference itself against the oracle port on the same host (development
container only: the reference is not on the GPU box).

    PYTHONPATH=/root/reference/pkg/src python tools/ref_vs_port.py

The bench's reference arm times the port (oracle/, float64 numpy restatement) because the reference
cannot travel to the GPU box.  This measures both on one core here, on the reference arm's exact
unit of work -- one CEM iteration of solve_bilevel (pkg/bilevel.py:249-292) at B = 100 samples,
10 obstacles, 100 AM iterations, same scenes -- and writes profiles/r02/ref_vs_port.json.
"""

import json
import os
import sys
import time

os.environ.setdefault("OPENBLAS_NUM_THREADS", "1")
os.environ.setdefault("OMP_NUM_THREADS", "1")
import numpy as np  # noqa: E402

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, "/root/reference/pkg/src")

import bench  # noqa: E402
from bilevel_drive.basis import build_basis  # noqa: E402
from bilevel_drive.batch_qp import TrackingWeights  # noqa: E402
from bilevel_drive.behavior import ParamLayout  # noqa: E402
from bilevel_drive.bilevel import BiLevelConfig, LowerLevelSolver, solve_bilevel  # noqa: E402
from bilevel_drive.constraints import ConstraintSpec, PlanningScene  # noqa: E402
from bilevel_drive.projection import ProjectionConfig  # noqa: E402

from paper_2212_02224_b200.scenes import highway_scene  # noqa: E402


def ref_iteration(seed, B=100):
    sc = highway_scene(seed)
    sp = sc.spec
    spec = ConstraintSpec(sp.obstacles_x, sp.obstacles_y, sp.ellipse_a, sp.ellipse_b, sp.v_max, sp.a_max,
                          sp.kappa_max, sp.c_max, sp.y_lb, sp.y_ub, sp.v_min)
    scene = PlanningScene(sc.initial_state, spec)
    basis = build_basis(10, 100, 5.0, "bernstein")
    solver = LowerLevelSolver(basis, TrackingWeights(), ParamLayout(4), ProjectionConfig(1.0, 100, 1e-3), 10)
    x0 = sc.initial_state
    mean = np.concatenate([np.full(4, x0[1]), np.full(4, np.hypot(x0[2], x0[3]))])
    cov = np.diag(np.concatenate([np.full(4, 1.5 ** 2), np.full(4, 3.0 ** 2)]))
    cfg = BiLevelConfig(B, min(150, B), min(100, B), 1, 0.7, 0.9, 1.0, mean, cov)
    t0 = time.perf_counter()
    solve_bilevel(scene, solver, cfg, np.random.default_rng(seed))
    return time.perf_counter() - t0


def main(reps=5):
    ref, port = [], []
    for k in range(reps + 1):
        r = ref_iteration(1000 + k)
        p = bench._ref_worker((1000 + k, 100))
        if k:                             # first pair: warm-up (imports, caches)
            ref.append(r)
            port.append(p)
    out = {"unit": "trajectories/s per core (one CEM iteration, B=100, 10 obstacles, 100 AM iterations)",
           "reference": 100 / float(np.median(ref)), "port": 100 / float(np.median(port)),
           "reference_s": ref, "port_s": port, "reps": reps,
           "host": os.uname().nodename, "cpu": open("/proc/cpuinfo").read().split("model name")[1].split("\n")[0]
           .strip(" :\t"), "threads": "OPENBLAS_NUM_THREADS=OMP_NUM_THREADS=1, one process"}
    out["port_over_reference"] = out["port"] / out["reference"]
    os.makedirs(os.path.join(ROOT, "profiles", "r02"), exist_ok=True)
    with open(os.path.join(ROOT, "profiles", "r02", "ref_vs_port.json"), "w") as fh:
        json.dump(out, fh, indent=1)
    print(json.dumps({k: out[k] for k in ("reference", "port", "port_over_reference")}))


if __name__ == "__main__":
    main()
