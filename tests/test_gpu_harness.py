"""GPU: the reference CLI's subcommands on the device path (pkg/cli.py:58-85, pkg/bench.py:264-353).

* ``trace`` reproduces the reference's emit_convergence_trace records on the canonical scene
  (tests/golden/harness.npz, default_rng(3), batch 200, 4 iterations).
* ``time`` writes the wall-time CSV with zero factorisations during the solves.
* ``bench`` runs a tiny YAML suite end to end and writes the three output files.
"""

import json

import numpy as np
import pytest

from tests.golden_io import load

pytestmark = pytest.mark.gpu

# the device sweep is fp32 over fp64 state: per-record tolerances
COST_RTOL = 1e-4
RESID_ATOL = 2e-3
ENVELOPE_ATOL = 2e-3


def test_trace_matches_reference(tmp_path):
    from paper_2212_02224_b200.__main__ import main
    g = load("harness")
    out = tmp_path / "trace.jsonl"
    assert main(["trace", "--output", str(out), "--seed", "3", "--batch-size", "200", "--iterations", "4"]) == 0
    ours = [json.loads(line) for line in out.read_text().splitlines()]
    ref = [json.loads(line) for line in str(g["trace_jsonl"]).splitlines()]
    assert len(ours) == len(ref) == 4
    for a, b in zip(ours, ref):
        assert sorted(a) == sorted(b)
        assert a["iteration"] == b["iteration"]
        np.testing.assert_allclose(a["elite_mean_upper_cost"], b["elite_mean_upper_cost"], rtol=COST_RTOL)
        np.testing.assert_allclose(a["cov_trace"], b["cov_trace"], rtol=COST_RTOL)
        for q in ("residual_q10", "residual_q50", "residual_q90"):
            np.testing.assert_allclose(a[q], b[q], atol=RESID_ATOL, rtol=1e-3)
        for side in ("y_envelope_low", "y_envelope_high"):
            np.testing.assert_allclose(a[side], b[side], atol=ENVELOPE_ATOL)


def test_time_reports_no_refactorisation(tmp_path):
    from paper_2212_02224_b200.__main__ import main
    out = tmp_path / "time.csv"
    assert main(["time", "--output", str(out), "--batch-sizes", "250,1000", "--iterations", "2,5"]) == 0
    lines = out.read_text().splitlines()
    assert lines[0] == "batch,iterations,total_s,per_iteration_s,factorizations_during_solve"
    rows = [line.split(",") for line in lines[1:]]
    assert [(r[0], r[1]) for r in rows] == [("250", "2"), ("250", "5"), ("1000", "2"), ("1000", "5")]
    for r in rows:
        assert float(r[2]) > 0 and abs(float(r[3]) * int(r[1]) - float(r[2])) < 1e-9
        assert r[4] == "0"


def test_bench_suite_from_yaml(tmp_path):
    import yaml
    from paper_2212_02224_b200.__main__ import main
    cfg = {"planners": ["mpc-bilevel", "mpc-vanilla"], "episodes_per_cell": 2, "replan_stride": 5,
           "env": {"batch_size": 200, "constraint_elites": 60, "elites": 20, "iterations": 2},
           "scenarios": [{"scenario_id": "tiny", "lane_count": 3, "density": 1.5, "vehicle_count": 10,
                          "episode_length": 20}]}
    path = tmp_path / "suite.yaml"
    path.write_text(yaml.safe_dump(cfg))
    outdir = tmp_path / "out"
    rc = main(["bench", "--config", str(path), "--output", str(outdir), "--seeds", "4,9"])
    assert rc == 0
    metrics = (outdir / "metrics.csv").read_text().splitlines()
    assert len(metrics) == 3 and metrics[1].startswith("mpc-bilevel,tiny,2,")
    manifest = json.loads((outdir / "manifest.json").read_text())
    assert manifest["seeds"] == [4, 9]
    assert len((outdir / "timings.csv").read_text().splitlines()) == 3


def test_bench_rerun_is_byte_identical(tmp_path):
    """SPEC acceptance 7: rerunning a suite with the same config writes a
    byte-identical metrics file (timings go to the side file)."""
    import yaml
    from paper_2212_02224_b200.__main__ import main
    cfg = {"planners": ["mpc-bilevel", "mpc-random", "mpc-vanilla"], "episodes_per_cell": 3,
           "env": {"batch_size": 300, "constraint_elites": 90, "elites": 30, "iterations": 3},
           "scenarios": [{"scenario_id": "d", "lane_count": 4, "density": 2.0, "vehicle_count": 24,
                          "episode_length": 40},
                         {"scenario_id": "s", "lane_count": 2, "density": 1.0, "vehicle_count": 10,
                          "episode_length": 40}]}
    path = tmp_path / "suite.yaml"
    path.write_text(yaml.safe_dump(cfg))
    runs = []
    for k in range(2):
        out = tmp_path / f"o{k}"
        assert main(["bench", "--config", str(path), "--output", str(out)]) == 0
        runs.append(((out / "metrics.csv").read_bytes(), (out / "manifest.json").read_bytes()))
    assert runs[0] == runs[1]
