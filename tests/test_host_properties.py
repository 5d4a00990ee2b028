"""CPU property tests (hypothesis) of the host-side value types and table builders."""

import numpy as np
from hypothesis import given, settings
from hypothesis import strategies as st


@settings(max_examples=60, deadline=None)
@given(n=st.integers(1, 400), m=st.integers(1, 40))
def test_segments_partition_like_array_split(n, m):
    from paper_2212_02224_b200.behavior import segment_matrix, segment_members
    if m > n:
        return
    ref = np.array_split(np.arange(n), m)
    got = segment_members(n, m)
    assert len(got) == m and all(np.array_equal(a, b) for a, b in zip(got, ref))
    S = segment_matrix(n, m)
    assert S.shape == (n, m) and np.all(S.sum(axis=1) == 1) and np.array_equal(S.sum(axis=0), [len(r) for r in ref])


@settings(max_examples=60, deadline=None)
@given(m=st.integers(1, 8), goal=st.booleans(), data=st.data())
def test_behavior_vector_roundtrip(m, goal, data):
    from paper_2212_02224_b200.behavior import BehaviorParams, ParamLayout
    lay = ParamLayout(m, goal)
    vec = np.array(data.draw(st.lists(st.floats(-1e6, 1e6), min_size=lay.dim, max_size=lay.dim)))
    p = BehaviorParams.from_vector(vec, lay)
    assert p.layout() == lay and np.array_equal(p.to_vector(), vec)
    assert len(lay.names) == lay.dim


@settings(max_examples=40, deadline=None)
@given(rows=st.integers(1, 9), n=st.integers(0, 40))
def test_warm_start_draw_is_cyclic_tile(rows, n):
    from paper_2212_02224_b200.behavior import ParamLayout, WarmStartSource
    samples = np.arange(rows * 8, dtype=float).reshape(rows, 8)
    got = WarmStartSource(samples, ParamLayout(4)).draw(n)
    want = np.tile(samples, (-(-n // rows) if n else 1, 1))[:n]
    assert np.array_equal(got, want)


@settings(max_examples=40, deadline=None)
@given(data=st.data())
def test_curvature_tables_pad_without_changing_interp(data):
    from paper_2212_02224_b200.worlds import curvature_tables
    S = data.draw(st.integers(1, 4))
    tabs = []
    for _ in range(S):
        if data.draw(st.booleans()):
            L = data.draw(st.integers(1, 6))
            xs = np.cumsum(data.draw(st.lists(st.floats(0.5, 50.0), min_size=L, max_size=L))) - 20.0
            ks = data.draw(st.lists(st.floats(-0.2, 0.2), min_size=L, max_size=L))
            tabs.append((tuple(xs), tuple(ks)))
        else:
            tabs.append(None)
    if all(t is None for t in tabs):
        return
    cx, ck = curvature_tables(tabs)
    x = np.linspace(-300, 600, 301)
    for s, t in enumerate(tabs):
        want = np.zeros_like(x) if t is None else np.interp(x, np.array(t[0]), np.array(t[1]))
        np.testing.assert_array_equal(np.interp(x, cx[s], ck[s]), want)


@settings(max_examples=30, deadline=None)
@given(lanes=st.integers(2, 6), dens=st.floats(0.3, 4.0), n=st.integers(0, 60), seed=st.integers(0, 10_000))
def test_spawn_layout_invariants(lanes, dens, n, seed):
    from paper_2212_02224_b200.sim import RoadSpec, ScenarioConfig, SimState
    st_ = SimState.spawn([ScenarioConfig(RoadSpec(lanes), dens, n, seed)])
    assert st_.n_veh[0] == n and st_.world[0, 3] == -1.0
    if n:
        lane = st_.veh_ext[0, :n, 3]
        assert np.array_equal(lane, np.arange(n) % lanes)
        assert np.array_equal(st_.veh[0, :n, 1], lane * 4.0)
        cd = st_.veh_ext[0, :n, 4]
        assert np.all((cd >= 0) & (cd < 2))
        for k in range(lanes):                  # cursors advance along each lane
            xs = st_.veh[0, :n][lane == k, 0]
            assert np.all(np.diff(xs) > 0)


@settings(max_examples=200, deadline=None)
@given(st.lists(st.floats(-20, 20), min_size=3, max_size=3), st.lists(st.floats(-20, 20), min_size=3, max_size=3),
       st.floats(2.0, 6.0), st.floats(1.5, 2.5), st.floats(2.0, 6.0), st.floats(1.5, 2.5))
def test_footprint_overlap_is_symmetric(pa, pb, la, wa, lb, wb):
    """SPEC acceptance 8 "collision-detector symmetry": the separating-axis footprint test of the
    simulator (pkg/highway.py:339-355, restated in oracle/sim.py) is symmetric."""
    from oracle.sim import overlap
    a = (pa[0], pa[1] / 4.0, pa[2] / 10.0, la, wa)
    b = (pb[0], pb[1] / 4.0, pb[2] / 10.0, lb, wb)
    assert overlap(a, b) == overlap(b, a)


@settings(max_examples=60, deadline=None)
@given(st.integers(1, 40), st.integers(0, 2**31 - 1))
def test_fleet_initial_means_match_per_world_rule(S, seed):
    """FleetPlanner.plan_cycle's vectorised initial mean equals the per-world rule of
    BasePlanner.initial_distribution (pkg/planners.py:218-231), bit for bit."""
    from paper_2212_02224_b200.fleet import initial_means
    rng = np.random.default_rng(seed)
    road = np.stack([rng.integers(0, 6, S).astype(float), rng.uniform(3.0, 5.0, S)], axis=1)
    b0 = rng.normal(size=(S, 6)) * 5.0
    b0[: S // 3, 1] = np.round(b0[: S // 3, 1])          # exact ties between two lane centres
    ref = np.empty((S, 8))
    for s in range(S):
        c = np.arange(int(road[s, 0])) * road[s, 1]
        lane_y = float(c[np.argmin(np.abs(c - b0[s, 1]))]) if c.size else b0[s, 1]
        ref[s] = np.concatenate([np.full(4, lane_y), np.full(4, float(np.hypot(b0[s, 2], b0[s, 3])))])
    np.testing.assert_array_equal(initial_means(road, b0, 4), ref)
