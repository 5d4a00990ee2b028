"""GPU: numpy's Generator(PCG64).standard_normal stream on the device (csrc/numpy_normals.cuh)
equals numpy's, and the drop-in solve_bilevel that uses it returns what the host-draw path
returns and leaves the caller's generator in exactly the same state (pkg/bilevel.py:56).

Every draw and every consumption count is bit-exact, with one measured exception: a draw from the
ziggurat's tail (|z| > r = 3.654, about 1 in 3000 draws) evaluates log1p, and CUDA's log1p and
glibc's round differently for a small fraction of arguments (1 of 10^6 draws differed, by one ulp).
The consumption -- hence the generator state -- never depends on it."""

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _ctx():
    from paper_2212_02224_b200 import numpy_stream
    from paper_2212_02224_b200._native import Context
    ctx = Context(0)
    assert numpy_stream.ensure_device_tables(ctx)
    return ctx


# 8e6 draws: each CTA owns ~7000 positions, more than its shared-memory window past the halo, so the
# walking warp slides the window (csrc/numpy_normals.cuh)
@pytest.mark.parametrize("seed,count,block", [(0, 32000, 8000), (1, 1000000, 1000), (2024, 77, 7),
                                              (5, 8000000, 1000000)])
def test_device_stream_equals_numpy(seed, count, block):
    from paper_2212_02224_b200 import numpy_stream
    ctx = _ctx()
    rng = np.random.default_rng(seed)
    rng.standard_normal(13)                      # start mid-stream
    words = numpy_stream.pcg64_state_words(rng.bit_generator)
    z = np.empty(count)
    pos = np.zeros(count // block + 1, dtype=np.int64)
    ctx.call("bd_numpy_normals", words.ctypes.data, count, block, z, pos)
    ref = np.random.Generator(np.random.PCG64(seed))
    ref.standard_normal(13)
    want = ref.standard_normal(count)
    diff = np.nonzero(z != want)[0]
    assert len(diff) <= max(1, count // 100000), len(diff)
    assert np.all(np.abs(want[diff]) > 3.6541528853610088)                  # tail draws only
    assert np.all(np.abs(z[diff] - want[diff]) <= np.spacing(np.abs(want[diff])))   # one ulp
    for b in (1, count // block):
        g = np.random.Generator(np.random.PCG64(seed))
        g.standard_normal(13 + b * block)
        h = np.random.Generator(np.random.PCG64(seed))
        h.standard_normal(13)
        h.bit_generator.advance(int(pos[b]))
        assert h.bit_generator.state == g.bit_generator.state


@pytest.mark.parametrize("warm,N", [(False, 4), (True, 4), (False, 1)])
def test_solve_bilevel_device_stream_equals_host_draws(monkeypatch, warm, N):
    import paper_2212_02224_b200 as bd
    from paper_2212_02224_b200 import bilevel as bl
    from paper_2212_02224_b200.behavior import WarmStartSource
    from paper_2212_02224_b200.fleet import initial_distribution
    from paper_2212_02224_b200.scenes import highway_scene
    basis = bd.build_basis(10, 100, 5.0, "bernstein")
    solver = bd.LowerLevelSolver(basis, bd.TrackingWeights(), bd.ParamLayout(4), bd.ProjectionConfig(1.0, 100, 1e-3),
                                 10)
    scene = highway_scene(3)
    mean, cov = initial_distribution(scene)
    cfg = bd.BiLevelConfig(1000, 150, 100, N, 0.7, 0.9, 1.0, mean, cov)
    ws = WarmStartSource(np.random.default_rng(9).multivariate_normal(mean, cov, 1000), solver.layout) if warm else None
    out = []
    for device_stream in (True, False):
        monkeypatch.setattr(bl, "_DEVICE_STREAM", device_stream)
        rng = np.random.default_rng(42)
        r = bd.solve_bilevel(scene, solver, cfg, rng, warm_start=ws)
        out.append((r, rng.bit_generator.state, rng.standard_normal()))
    (a, sa, na), (b, sb, nb) = out
    assert sa == sb and na == nb                     # generator left where the reference leaves it
    assert a.best.index == b.best.index
    # identical set-points (bar a one-ulp tail draw) -> identical results up to that ulp
    np.testing.assert_allclose(a.best.coeffs.stacked(), b.best.coeffs.stacked(), rtol=1e-12, atol=1e-12)
    np.testing.assert_allclose(a.distribution.mean, b.distribution.mean, rtol=1e-12)
    np.testing.assert_allclose([d.residual_median for d in a.diagnostics], [d.residual_median for d in b.diagnostics],
                               rtol=1e-9, atol=1e-12)


@pytest.mark.parametrize("prep", ["uint32_buffered", "mt19937"])
def test_solve_bilevel_generator_edge_cases(monkeypatch, prep):
    """A PCG64 generator holding a buffered 32-bit half (standard_normal never touches it) and a
    non-PCG64 bit generator (host draws) both end where the host-draw path leaves them."""
    import paper_2212_02224_b200 as bd
    from paper_2212_02224_b200 import bilevel as bl
    from paper_2212_02224_b200.fleet import initial_distribution
    from paper_2212_02224_b200.scenes import highway_scene
    basis = bd.build_basis(10, 100, 5.0, "bernstein")
    solver = bd.LowerLevelSolver(basis, bd.TrackingWeights(), bd.ParamLayout(4), bd.ProjectionConfig(1.0, 100, 1e-3),
                                 10)
    scene = highway_scene(4)
    mean, cov = initial_distribution(scene)
    cfg = bd.BiLevelConfig(1000, 150, 100, 2, 0.7, 0.9, 1.0, mean, cov)

    def make():
        if prep == "mt19937":
            return np.random.Generator(np.random.MT19937(5))
        g = np.random.default_rng(5)
        g.integers(0, 1000, size=3, dtype=np.uint32)          # leaves has_uint32 = 1
        return g
    out = []
    for device_stream in (True, False):
        monkeypatch.setattr(bl, "_DEVICE_STREAM", device_stream)
        rng = make()
        r = bd.solve_bilevel(scene, solver, cfg, rng)
        out.append((r.best.index, rng.bit_generator.state, rng.integers(0, 2**31), rng.standard_normal()))
    def same(a, b):
        if isinstance(a, dict):
            return a.keys() == b.keys() and all(same(a[k], b[k]) for k in a)
        if isinstance(a, np.ndarray):
            return np.array_equal(a, b)
        return a == b
    assert same(out[0][1], out[1][1])
    assert out[0][0] == out[1][0] and out[0][2] == out[1][2] and out[0][3] == out[1][3]
