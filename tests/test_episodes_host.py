"""CPU: episode logs and suite output files in the reference's formats (pkg/highway.py:413-475,
pkg/bench.py:56-205), pinned by tests/golden/episodes.npz."""

import os

import numpy as np

from tests.golden_io import load


def test_suite_outputs_byte_identical(tmp_path):
    from paper_2212_02224_b200.episodes import BenchmarkSuite, MetricsRow, write_outputs
    from paper_2212_02224_b200.planners import PlannerEnvConfig
    from paper_2212_02224_b200.sim import RoadSpec, ScenarioConfig
    g = load("episodes")
    suite = BenchmarkSuite(scenarios=(ScenarioConfig(RoadSpec(3), 1.5, 20, 0, scenario_id="a"),
                                      ScenarioConfig(RoadSpec(4), 2.0, 24, 0, scenario_id="b")),
                           planners=("mpc-bilevel", "mpc-vanilla"), episodes_per_cell=3,
                           env=PlannerEnvConfig(batch_size=100, iterations=3))
    rows = [MetricsRow("mpc-bilevel", "a", 3, 1, 1 / 3, 11.25, 0.0123, 0),
            MetricsRow("mpc-bilevel", "b", 3, 0, 0.0, float("nan"), float("nan"), 3),
            MetricsRow("mpc-vanilla", "a", 3, 2, 2 / 3, 9.876543210123, 0.5, 1),
            MetricsRow("mpc-vanilla", "b", 3, 0, 0.0, 12.0, 1e-4, 0)]
    walls = {"mpc-bilevel/a": 1.5, "mpc-bilevel/b": 2.25, "mpc-vanilla/a": 0.1}
    paths = write_outputs(suite, rows, walls, str(tmp_path))
    assert open(paths["metrics"]).read() == str(g["suite_metrics"])
    assert open(paths["timings"]).read() == str(g["suite_timings"])
    import json
    assert json.load(open(paths["manifest"]))["config_hash"] == str(g["suite_hash"])


def test_episode_log_jsonl_roundtrip(tmp_path):
    from paper_2212_02224_b200.episodes import EpisodeLog
    g = load("episodes")
    for k in range(int(g["n_cases"])):
        src = tmp_path / f"ref{k}.jsonl"
        src.write_text(str(g[f"e{k}_jsonl"]))
        log = EpisodeLog.read_jsonl(str(src))
        out = tmp_path / f"ours{k}.jsonl"
        log.write_jsonl(str(out))
        assert out.read_text() == src.read_text()
        assert log.mean_speed() > 0 and len(log.steps) > 0


def test_suite_validation():
    import pytest
    from paper_2212_02224_b200.episodes import BenchmarkSuite, suite_from_dict
    with pytest.raises(ValueError):
        BenchmarkSuite(scenarios=(), planners=("nope",))
    with pytest.raises(ValueError):
        BenchmarkSuite(scenarios=(), planners=("mpc-bilevel",), episodes_per_cell=2, seeds=(1,))
    s = suite_from_dict({"scenarios": [{"lane_count": 3, "density": 1.0, "vehicle_count": 5}],
                         "planners": ["mpc-grid"], "episodes_per_cell": 2, "env": {"batch_size": 64}})
    assert s.seeds == (0, 1) and s.env.batch_size == 64 and s.scenarios[0].road.lane_count == 3
