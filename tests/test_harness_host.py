"""CPU: the harness callers of the path (pkg/bench.py:208-367, pkg/cli.py) pinned by
tests/golden/harness.npz — canonical scene and CEM config exactly, replay CSV byte for byte."""

import numpy as np
import pytest

from tests.golden_io import load


def test_canonical_scene_and_config_match_reference():
    from paper_2212_02224_b200.harness import bilevel_config_for, canonical_scene
    from paper_2212_02224_b200.planners import PlannerEnvConfig
    g = load("harness")
    env = PlannerEnvConfig(batch_size=200, iterations=4)
    sc = canonical_scene(env)
    np.testing.assert_array_equal(sc.spec.obstacles_x, g["canon_ox"])
    np.testing.assert_array_equal(sc.spec.obstacles_y, g["canon_oy"])
    np.testing.assert_array_equal(sc.initial_state, g["canon_b0"])
    np.testing.assert_array_equal(sc.lane_centers, g["canon_lanes"])
    np.testing.assert_array_equal(np.array(sc.spec.limits()), g["canon_limits"])
    cfg = bilevel_config_for(env, sc, batch_size=300, iterations=2)
    np.testing.assert_array_equal(cfg.init_mean, g["cfg_mean"])
    np.testing.assert_array_equal(cfg.init_cov, g["cfg_cov"])
    assert [cfg.batch_size, cfg.constraint_elites, cfg.elites, cfg.iterations] == g["cfg_sizes"].tolist()


@pytest.mark.parametrize("via_cli", [False, True])
def test_replay_csv_byte_identical(tmp_path, via_cli):
    from paper_2212_02224_b200.__main__ import main
    from paper_2212_02224_b200.harness import replay_to_csv
    g, e = load("harness"), load("episodes")
    for k in range(int(g["n_replays"])):
        log, out = tmp_path / f"e{k}.jsonl", tmp_path / f"e{k}.csv"
        log.write_text(str(e[f"e{k}_jsonl"]))
        if via_cli:
            assert main(["replay", "--log", str(log), "--output", str(out)]) == 0
        else:
            replay_to_csv(str(log), str(out))
        assert out.read_text() == str(g[f"replay_{k}"])


def test_cli_parser_matches_reference_surface():
    from paper_2212_02224_b200.__main__ import build_parser
    p = build_parser()
    a = p.parse_args(["time", "--output", "t.csv"])
    assert (a.batch_sizes, a.iterations, a.seed) == ("250,1000", "2,5", 0)
    a = p.parse_args(["trace", "--output", "t.jsonl", "--batch-size", "64", "--iterations", "3"])
    assert (a.batch_size, a.iterations, a.seed) == (64, 3, 0)
    a = p.parse_args(["bench", "--config", "c.yaml", "--output", "d", "--seeds", "1,2"])
    assert (a.seeds, a.workers) == ("1,2", None)
    with pytest.raises(SystemExit):
        p.parse_args([])
