"""GPU: device simulator ticks (bd_sim_run) against the reference's own step()
(tests/golden/sim.npz) and the oracle restatement."""

import numpy as np
import pytest

from tests.golden_io import load

pytestmark = pytest.mark.gpu

# continuous state: fp64 with CUDA libm transcendental (<= 2 ulp) vs glibc/numpy; discrete state exact
RTOL, ATOL = 1e-12, 1e-9


def _golden_state(g, ks):
    from paper_2212_02224_b200.sim import SimState
    S = len(ks)
    n_max = max(g[f"s{k}_veh0"].shape[0] for k in ks)
    st = SimState(np.zeros((S, 8)), np.zeros(S), np.zeros((S, n_max, 5)), np.zeros((S, n_max, 7)),
                  np.zeros(S, np.int32), np.zeros((S, 2)), np.zeros((S, 5)))
    for s, k in enumerate(ks):
        e, v = g[f"s{k}_ego0"], g[f"s{k}_veh0"]
        st.ego[s], st.ego_ts[s] = e[:8], e[8]
        st.veh[s, : len(v)], st.veh_ext[s, : len(v)] = v[:, :5], v[:, 5:]
        st.n_veh[s] = len(v)
        st.road[s] = g[f"s{k}_road"][:2]
        st.world[s] = g[f"s{k}_w0"]
    return st


def _sim():
    from paper_2212_02224_b200._native import Context
    from paper_2212_02224_b200.sim import Simulator
    return Simulator(Context(0))


def _check_tick(g, k, t, ego, veh, world, nv):
    ge, gv, gw = g[f"s{k}_ego"][t], g[f"s{k}_veh"][t], g[f"s{k}_w"][t]
    np.testing.assert_allclose(ego, ge[:8], rtol=RTOL, atol=ATOL)
    np.testing.assert_allclose(veh[:nv], gv[:, :5], rtol=RTOL, atol=ATOL)
    np.testing.assert_array_equal(world, gw)


@pytest.mark.parametrize("host_state", [True, False])
def test_device_ticks_match_reference(host_state):
    g = load("sim")
    ks = list(range(int(g["n_cases"])))
    st = _golden_state(g, ks)
    n_steps = max(len(g[f"s{k}_ctrl"]) for k in ks)
    ctrl = np.zeros((len(ks), n_steps, 2))
    for s, k in enumerate(ks):
        c = g[f"s{k}_ctrl"]
        ctrl[s, : len(c)] = c
        ctrl[s, len(c):] = c[-1]
    sim = _sim()
    if not host_state:
        st = st.to("cuda:0")
    # one tick per call for the first 10 ticks (state round trip), then the rest in one launch
    for t in range(10):
        sim.run(st, ctrl, 1, ctrl_offset=t)
        h = st.to(None)
        for s, k in enumerate(ks):
            _check_tick(g, k, t, h.ego[s], h.veh[s], h.world[s], int(h.n_veh[s]))
            np.testing.assert_array_equal(h.veh_ext[s, : h.n_veh[s], 3], g[f"s{k}_veh"][t][:, 8])
    done, snap = sim.run(st, ctrl, n_steps - 10, ctrl_offset=10, snapshots=True)
    assert np.all(done == n_steps - 10)
    h = st.to(None)
    for s, k in enumerate(ks):
        nt = len(g[f"s{k}_ctrl"])
        nv = int(h.n_veh[s])
        for t in range(10, nt):
            rec = snap[s, t - 10]
            ge, gv, gw = g[f"s{k}_ego"][t], g[f"s{k}_veh"][t], g[f"s{k}_w"][t]
            assert rec[0] == pytest.approx(gw[0], abs=1e-12) and rec[7] == gw[2]
            np.testing.assert_allclose(rec[1:7], ge[:6], rtol=RTOL, atol=ATOL)
            np.testing.assert_allclose(rec[8:8 + 4 * nv].reshape(nv, 4), gv[:, :4], rtol=RTOL, atol=ATOL)
        if nt == n_steps:
            _check_tick(g, k, nt - 1, h.ego[s], h.veh[s], h.world[s], nv)
            np.testing.assert_allclose(h.veh_ext[s, :nv], g[f"s{k}_veh"][nt - 1][:, 5:], rtol=RTOL, atol=ATOL)


def test_episode_termination_and_inactive_worlds():
    """x_end: run_episode semantics (stop after the colliding tick / at the end of the road)."""
    g = load("sim")
    ks = [3, 0, 4]                    # 3 collides at tick 40; 0 never does; 4 is parked inactive
    st = _golden_state(g, ks)
    ctrl = np.stack([np.repeat(g[f"s{k}_ctrl"][:1], 60, axis=0) for k in ks])
    ctrl[0] = g["s3_ctrl"]
    ctrl[1] = g["s0_ctrl"]
    x_end = np.array([1e9, 30.0, 1e9])
    active = np.array([1, 1, 0], np.int32)
    w4 = st.world[2].copy()
    done, snap = _sim().run(st, ctrl, 60, x_end=x_end, active=active, snapshots=True)
    assert done[0] == 40 and active[0] == 0 and st.world[0, 2] == 1.0 and st.world[0, 3] == 40
    np.testing.assert_allclose(st.ego[0], g["s3_ego"][39][:8], rtol=RTOL, atol=ATOL)
    xs = g["s0_ego"][:, 0]
    first = int(np.argmax(xs >= 30.0)) + 1
    assert done[1] == first and active[1] == 0
    assert done[2] == 0 and active[2] == 0 and np.array_equal(st.world[2], w4)


def test_random_controls_against_oracle():
    """Off-golden controls (hard braking, full steer) through a mixed batch, vs the oracle."""
    from oracle import sim as osim
    from paper_2212_02224_b200.sim import RoadSpec, ScenarioConfig, SimState
    scs = [ScenarioConfig(RoadSpec(l), d, n, s) for l, d, n, s in ((3, 2.0, 20, 11), (5, 2.5, 50, 12), (2, 1.2, 7, 13))]
    st = SimState.spawn(scs)
    rng = np.random.default_rng(0)
    ctrl = np.stack([rng.uniform(-6, 6, 30), rng.uniform(-0.4, 0.4, 30)], axis=1)[None].repeat(3, 0)
    h0 = SimState.spawn(scs)
    _sim().run(st, ctrl, 30)
    for s, sc in enumerate(scs):
        nv = sc.vehicle_count
        ego = np.concatenate([h0.ego[s], [h0.ego_ts[s]]])
        veh = np.concatenate([h0.veh[s, :nv], h0.veh_ext[s, :nv]], axis=1)
        ws = h0.world[s]
        road = np.array([sc.road.lane_count, sc.road.lane_width, sc.road.length, sc.dt])
        for t in range(30):
            ego, veh, ws = osim.step(ego, veh, ws, road, ctrl[s, t, 0], ctrl[s, t, 1])
        np.testing.assert_allclose(st.ego[s], ego[:8], rtol=1e-10, atol=1e-8)
        np.testing.assert_allclose(st.veh[s, :nv], veh[:, :5], rtol=1e-10, atol=1e-8)
        np.testing.assert_array_equal(st.veh_ext[s, :nv, 3], veh[:, 8])
        np.testing.assert_array_equal(st.world[s], ws)


def test_ragged_worlds_empty_and_crowded_against_oracle():
    """World batches with no neighbours and with more neighbours than one CTA has threads
    (the per-neighbour loops stride), and a 5-lane road, against the oracle restatement."""
    from oracle import sim as osim
    from paper_2212_02224_b200.sim import RoadSpec, ScenarioConfig, SimState
    scs = [ScenarioConfig(RoadSpec(3), 1.0, 0, 21), ScenarioConfig(RoadSpec(5), 6.0, 200, 22),
           ScenarioConfig(RoadSpec(2), 1.5, 9, 23)]
    st = SimState.spawn(scs)
    h0 = SimState.spawn(scs)
    rng = np.random.default_rng(4)
    ctrl = np.stack([rng.uniform(-2, 2, 25), rng.uniform(-0.1, 0.1, 25)], axis=1)[None].repeat(3, 0)
    _sim().run(st, ctrl, 25)
    for s, sc in enumerate(scs):
        nv = sc.vehicle_count
        ego = np.concatenate([h0.ego[s], [h0.ego_ts[s]]])
        veh = np.concatenate([h0.veh[s, :nv], h0.veh_ext[s, :nv]], axis=1)
        ws = h0.world[s]
        road = np.array([sc.road.lane_count, sc.road.lane_width, sc.road.length, sc.dt])
        for t in range(25):
            ego, veh, ws = osim.step(ego, veh, ws, road, ctrl[s, t, 0], ctrl[s, t, 1])
        np.testing.assert_allclose(st.ego[s], ego[:8], rtol=1e-10, atol=1e-8)
        if nv:
            np.testing.assert_allclose(st.veh[s, :nv], veh[:, :5], rtol=1e-10, atol=1e-8)
            np.testing.assert_array_equal(st.veh_ext[s, :nv, 3], veh[:, 8])
        np.testing.assert_array_equal(st.world[s], ws)
