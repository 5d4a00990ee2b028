"""CPU: the simulator oracle is pinned to the reference's own ticks, and the product's spawn
restatement reproduces spawn_world."""

import numpy as np

from tests.golden_io import load


def test_oracle_step_matches_reference_ticks():
    from oracle import sim
    g = load("sim")
    for k in range(int(g["n_cases"])):
        ego, veh, ws, road = g[f"s{k}_ego0"], g[f"s{k}_veh0"], g[f"s{k}_w0"], g[f"s{k}_road"]
        for t, (a, d) in enumerate(g[f"s{k}_ctrl"]):
            ego, veh, ws = sim.step(ego, veh, ws, road, a, d)
            np.testing.assert_array_equal(ego, g[f"s{k}_ego"][t])
            np.testing.assert_array_equal(veh, g[f"s{k}_veh"][t])
            np.testing.assert_array_equal(ws, g[f"s{k}_w"][t])


def test_golden_covers_lane_changes_collisions_and_departures():
    g = load("sim")
    changes = sum(int(np.any(np.diff(g[f"s{k}_veh"][:, :, 8], axis=0) != 0)) for k in range(int(g["n_cases"])))
    assert changes >= 2
    assert any(g[f"s{k}_w"][-1, 2] == 1.0 for k in range(int(g["n_cases"])))
    assert any(g[f"s{k}_w"][-1, 4] == 1.0 for k in range(int(g["n_cases"])))


def test_spawn_matches_reference_spawn_world():
    from paper_2212_02224_b200.sim import RoadSpec, ScenarioConfig, SimState
    g = load("sim")
    n = int(g["n_cases"])
    scs = []
    for k in range(n):
        lanes, dens, nveh, seed, _ = g[f"s{k}_cfg"]
        scs.append(ScenarioConfig(RoadSpec(int(lanes)), float(dens), int(nveh), int(seed)))
    st = SimState.spawn(scs)
    for k in range(n):
        e0, v0 = g[f"s{k}_ego0"], g[f"s{k}_veh0"]
        nv = v0.shape[0]
        np.testing.assert_array_equal(st.ego[k], e0[:8])
        assert st.ego_ts[k] == e0[8]
        np.testing.assert_array_equal(st.veh[k, :nv], v0[:, :5])
        np.testing.assert_array_equal(st.veh_ext[k, :nv], v0[:, 5:])
        assert st.n_veh[k] == nv and np.all(st.veh[k, nv:] == 0)
        np.testing.assert_array_equal(st.world[k], g[f"s{k}_w0"])


def test_scenario_dict_roundtrip():
    from paper_2212_02224_b200.sim import RoadSpec, ScenarioConfig
    sc = ScenarioConfig(RoadSpec(3, 3.5, 900.0), 1.5, 30, 7, episode_length=80, scenario_id="x")
    assert ScenarioConfig.from_dict(sc.to_dict()) == sc


def test_curvature_tables_padding_preserves_interp():
    from paper_2212_02224_b200.worlds import curvature_tables
    tabs = [((0.0, 40.0, 90.0, 160.0), (0.0, 0.02, 0.05, 0.01)), None, ((10.0, 20.0), (0.1, -0.2)), ((5.0,), (0.3,))]
    cx, ck = curvature_tables(tabs)
    x = np.linspace(-500, 2000, 4001)
    for s, t in enumerate(tabs):
        assert np.all(np.diff(cx[s]) > 0) or cx.shape[1] == 1
        want = np.zeros_like(x) if t is None else np.interp(x, np.array(t[0]), np.array(t[1]))
        np.testing.assert_array_equal(np.interp(x, cx[s], ck[s]), want)
