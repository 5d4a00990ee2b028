"""Same config-2 plans through two library builds (BD_LIB_PATH per process): prints whether the
results are bit-identical (for refactors that must not change arithmetic)."""
import os, subprocess, sys, json
import numpy as np
if len(sys.argv) > 2 and sys.argv[1] == "--run":
    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
    import paper_2212_02224_b200 as bd
    from paper_2212_02224_b200.fleet import FleetPlanner, initial_distribution
    from paper_2212_02224_b200.scenes import highway_scene
    basis = bd.build_basis(10, 100, 5.0, "bernstein")
    out = {}
    for B, persist in [(1000, 1), (1000, 0)]:
        cfg = bd.BiLevelConfig(B, 150, 100, 4, 0.7, 0.9, 1.0)
        fp = FleetPlanner(basis, bd.TrackingWeights(), bd.ParamLayout(4), bd.ProjectionConfig(1.0, 100, 1e-3), 10, cfg)
        fp.context.set_option("persistent_cycle", persist)
        r = fp.plan([highway_scene(3)], seed=7)
        out[f"{B}_{persist}"] = [np.asarray(r.best_xi).tolist(), np.asarray(r.stats).tolist()]
    np.save(sys.argv[2], np.array(json.dumps(out)))
    sys.exit(0)
a, b = sys.argv[1], sys.argv[2]
for lib, f in [(a, "/tmp/bc_a.npy"), (b, "/tmp/bc_b.npy")]:
    subprocess.run([sys.executable, __file__, "--run", f], env={**os.environ, "BD_LIB_PATH": lib}, check=True)
ra, rb = json.loads(str(np.load("/tmp/bc_a.npy"))), json.loads(str(np.load("/tmp/bc_b.npy")))
for k in ra:
    print(k, "bit-identical" if ra[k] == rb[k] else "DIFFERENT")
