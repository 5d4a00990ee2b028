"""GPU: CVAE warm-start decoder (K5) vs a float64 numpy restatement, and config 3
(decoder samples -> warm start of the device CEM cycle)."""

import numpy as np
import pytest

from oracle.cvae import decode as decode_ref
from oracle.cvae import decode_bf16

pytestmark = pytest.mark.gpu


def test_cvae_decoder_fp32_matches_float64_restatement():
    from paper_2212_02224_b200.cvae import CVAEDecoder
    dec = CVAEDecoder.synthetic(7)
    dec.ctx.set_option("cvae_tensor_cores", 0)
    rng = np.random.default_rng(0)
    obs = rng.standard_normal(55).astype(np.float32)
    z = rng.standard_normal((1000, 2)).astype(np.float32)
    got = dec.decode(obs, z)
    ref = decode_ref(dec.W, dec.b, obs, z)
    assert got.shape == (1000, 8)
    scale = np.abs(ref).max()
    np.testing.assert_allclose(got, ref, rtol=0, atol=1e-4 * scale)


@pytest.mark.parametrize("count", [1000, 128, 77])
def test_cvae_decoder_tcgen05_bf16(count):
    """Hidden layers on tcgen05 (bf16 operands, fp32 TMEM accumulation) against a float64
    restatement that rounds weights and activations to bf16 exactly where the kernel does
    (oracle.cvae.decode_bf16): what is left is the fp32 accumulation order inside the tensor core
    and the bf16 rounding flips it causes (an activation one bf16 ulp away, ~2e-3 relative, for a
    few of the 4096 activations of a sample): measured max 2.6e-3 - 4.8e-3, mean 1.3e-4 - 1.5e-4
    of the output scale.  A wrong swizzle, descriptor or epilogue mapping gives O(1) errors.  The
    bit-exact layer test below pins the GEMM itself; the plain float64 decoder bounds the total
    bf16 error."""
    from paper_2212_02224_b200.cvae import CVAEDecoder
    dec = CVAEDecoder.synthetic(7)
    rng = np.random.default_rng(1)
    obs = rng.standard_normal(55).astype(np.float32)
    z = rng.standard_normal((count, 2)).astype(np.float32)
    got = dec.decode(obs, z)
    emu = decode_bf16(dec.W, dec.b, obs, z)
    scale = np.abs(emu).max()
    err = np.abs(got - emu)
    print(f"bf16-emulated: max {err.max() / scale:.2e} mean {err.mean() / scale:.2e} of the output scale")
    assert err.max() <= 1e-2 * scale, err.max() / scale
    assert err.mean() <= 3e-4 * scale, err.mean() / scale
    ref = decode_ref(dec.W, dec.b, obs, z)
    assert np.abs(got - ref).max() <= 5e-2 * np.abs(ref).max()


def test_cvae_tcgen05_layer_bit_exact():
    """One tcgen05 hidden layer on inputs whose every product and partial sum is exact in fp32
    (multiples of 1/64 with few significant bits): any accumulation order gives the same fp32
    value, so the bf16 output must equal the float64 restatement bit for bit.  The last layer
    selects every 8th activation with weight 1.0 (exact), so the decoder output IS the tcgen05
    layer's bf16 activations.  Pins the TMA swizzle, UMMA descriptors and the TMEM epilogue."""
    from paper_2212_02224_b200.cvae import CVAEDecoder
    rng = np.random.default_rng(11)
    W0 = np.zeros((256, 57), np.float32)
    W0[:, 55:] = rng.integers(-4, 5, (256, 2)) / 64.0           # latent part; obs = 0
    b0 = (rng.integers(-8, 9, 256) / 64.0).astype(np.float32)
    W1 = (rng.integers(-7, 8, (1024, 256)) / 64.0).astype(np.float32)   # bf16-exact
    b1 = (rng.integers(-64, 65, 1024) / 4096.0).astype(np.float32)
    W2 = np.zeros((128, 1024), np.float32)
    W2[np.arange(128), 8 * np.arange(128)] = 1.0
    b2 = np.zeros(128, np.float32)
    dec = CVAEDecoder([W0, W1, W2], [b0, b1, b2])
    z = rng.integers(-3, 4, (300, 2)).astype(np.float32)
    got = dec.decode(np.zeros(55), z)
    np.testing.assert_array_equal(got, decode_bf16(dec.W, dec.b, np.zeros(55), z))
    assert np.count_nonzero(got) > 0.2 * got.size                 # ReLU leaves plenty of signal


def test_cvae_odd_sizes_and_errors():
    from paper_2212_02224_b200.cvae import CVAEDecoder
    dec = CVAEDecoder.synthetic(1, out_dim=10, hidden=(100, 70))
    rng = np.random.default_rng(1)
    obs, z = rng.standard_normal(55), rng.standard_normal((37, 2))
    np.testing.assert_allclose(dec.decode(obs, z), decode_ref(dec.W, dec.b, obs, z), atol=1e-4 * 10, rtol=1e-4)
    with pytest.raises(ValueError):
        dec.decode(np.zeros(54), z)


def test_config3_cvae_warm_start_then_cem():
    import paper_2212_02224_b200 as bd
    from paper_2212_02224_b200.cvae import CVAEDecoder
    from paper_2212_02224_b200.fleet import initial_distribution
    from paper_2212_02224_b200.scenes import highway_scene
    basis = bd.build_basis(10, 100, 5.0, "bernstein")
    solver = bd.LowerLevelSolver(basis, bd.TrackingWeights(), bd.ParamLayout(4), bd.ProjectionConfig(1.0, 100, 1e-3), 10)
    scene = highway_scene(2)
    mean, cov = initial_distribution(scene)
    dec = CVAEDecoder.synthetic(3, context=solver.context)
    rng = np.random.default_rng(5)
    obs = np.zeros(55)
    raw = dec.decode(obs, rng.standard_normal((1000, 2)))
    # map the (untrained) decoder output onto set-point units around the lane / speed mean
    shift = mean - raw.mean(axis=0)
    ws = dec.warm_start(obs, 1000, solver.layout, np.random.default_rng(5), shift=shift)
    cfg = bd.BiLevelConfig(1000, 150, 100, 4, 0.7, 0.9, 1.0, mean, cov)
    res = bd.solve_bilevel(scene, solver, cfg, np.random.default_rng(6), warm_start=ws)
    assert not res.degraded and len(res.diagnostics) == 4
    assert np.isfinite(res.best.upper_cost)
    # a one-iteration cycle ranks only the decoder's samples: its best record's set-points are
    # exactly the decoder sample at the best index
    one = bd.solve_bilevel(scene, solver, bd.BiLevelConfig(1000, 150, 100, 1, 0.7, 0.9, 1.0, mean, cov),
                           np.random.default_rng(6), warm_start=ws)
    assert len(one.diagnostics) == 1 and 0 <= one.best.index < 1000
    np.testing.assert_array_equal(one.best.params.to_vector(), ws.samples[one.best.index])


def _c3_setup(seed=2):
    import paper_2212_02224_b200 as bd
    from paper_2212_02224_b200.cvae import CVAEDecoder
    from paper_2212_02224_b200.fleet import initial_distribution
    from paper_2212_02224_b200.scenes import highway_scene
    basis = bd.build_basis(10, 100, 5.0, "bernstein")
    solver = bd.LowerLevelSolver(basis, bd.TrackingWeights(), bd.ParamLayout(4), bd.ProjectionConfig(1.0, 100, 1e-3), 10)
    scene = highway_scene(seed)
    mean, cov = initial_distribution(scene)
    dec = CVAEDecoder.synthetic(3, context=solver.context)
    return bd, solver, scene, mean, cov, dec


def _same_result(a, b):
    assert a.best.index == b.best.index and a.degraded == b.degraded
    np.testing.assert_array_equal(a.best.coeffs.stacked(), b.best.coeffs.stacked())
    np.testing.assert_array_equal(a.distribution.mean, b.distribution.mean)
    np.testing.assert_array_equal(a.distribution.cov, b.distribution.cov)
    assert [d.cov_trace for d in a.diagnostics] == [d.cov_trace for d in b.diagnostics]


def test_device_warm_start_rows_and_cycle_match_host_rows():
    """bd_cvae_warm_start keeps the rows on the device and solve_bilevel feeds them to the cycle in
    place: the rows equal decode * scale + shift computed on the host (float64, two roundings),
    the generator advances by the same count x 2 normals, and the cycle is bit-identical to the
    one fed the host copy through the reference's WarmStartSource."""
    from paper_2212_02224_b200.behavior import DeviceWarmStart, WarmStartSource
    bd, solver, scene, mean, cov, dec = _c3_setup()
    obs = np.linspace(-1.0, 1.0, 55)
    scale = np.array([1.5, 1.5, 1.5, 1.5, 2.0, 2.0, 2.0, 2.0])
    shift = mean - 0.3
    r1, r2 = np.random.default_rng(11), np.random.default_rng(11)
    ws = dec.warm_start(obs, 1000, solver.layout, r1, scale=scale, shift=shift)
    assert isinstance(ws, DeviceWarmStart) and ws.device_rows(solver.context, 1000) is not None
    z = r2.standard_normal((1000, 2))
    assert r1.bit_generator.state == r2.bit_generator.state
    want = dec.decode(obs, z) * scale + shift
    np.testing.assert_array_equal(ws.samples, want)
    cfg = bd.BiLevelConfig(1000, 150, 100, 4, 0.7, 0.9, 1.0, mean, cov)
    ga, gb = np.random.default_rng(6), np.random.default_rng(6)
    ws2 = dec.warm_start(obs, 1000, solver.layout, np.random.default_rng(11), scale=scale, shift=shift)
    a = bd.solve_bilevel(scene, solver, cfg, ga, warm_start=ws2)
    b = bd.solve_bilevel(scene, solver, cfg, gb, warm_start=WarmStartSource(want, solver.layout))
    _same_result(a, b)
    assert ga.bit_generator.state == gb.bit_generator.state


def test_device_warm_start_stale_or_short_rows_use_the_host_copy():
    """A later decode overwrites the context's device rows: the earlier source then goes through
    its host copy (same results); a batch larger than the rows repeats them cyclically (host)."""
    from paper_2212_02224_b200.behavior import WarmStartSource
    bd, solver, scene, mean, cov, dec = _c3_setup(4)
    obs = np.zeros(55)
    shift = mean.copy()
    old = dec.warm_start(obs, 1000, solver.layout, np.random.default_rng(1), shift=shift)
    dec.warm_start(obs, 1000, solver.layout, np.random.default_rng(2), shift=shift)
    assert old.device_rows(solver.context, 1000) is None
    cfg = bd.BiLevelConfig(1000, 150, 100, 2, 0.7, 0.9, 1.0, mean, cov)
    a = bd.solve_bilevel(scene, solver, cfg, np.random.default_rng(3), warm_start=old)
    b = bd.solve_bilevel(scene, solver, cfg, np.random.default_rng(3), warm_start=WarmStartSource(old.samples,
                                                                                                  solver.layout))
    _same_result(a, b)
    short = dec.warm_start(obs, 600, solver.layout, np.random.default_rng(4), shift=shift)
    assert short.device_rows(solver.context, 1000) is None
    c = bd.solve_bilevel(scene, solver, cfg, np.random.default_rng(3), warm_start=short)
    d = bd.solve_bilevel(scene, solver, cfg, np.random.default_rng(3),
                         warm_start=WarmStartSource(short.samples, solver.layout))
    _same_result(c, d)
    with pytest.raises(ValueError):
        dec.warm_start(obs, 10, bd.ParamLayout(3), np.random.default_rng(0))


def test_device_warm_start_abi_copy_and_trace_path():
    """bd_cvae_warm_start with a host `params` buffer copies the same rows the device keeps; the
    stepped solve_bilevel (trace_hook) draws a DeviceWarmStart through its host view and matches
    the reference-typed WarmStartSource."""
    import ctypes
    from paper_2212_02224_b200.behavior import WarmStartSource
    bd, solver, scene, mean, cov, dec = _c3_setup(5)
    obs = np.linspace(0.0, 2.0, 55).astype(np.float32)
    z = np.random.default_rng(3).standard_normal((300, 2)).astype(np.float32)
    shift = np.ascontiguousarray(mean, dtype=np.float64)
    host = np.empty((300, 8))
    rows = ctypes.c_void_p()
    dec.ctx.call("bd_cvae_warm_start", 300, obs.ctypes.data, z.ctypes.data, None, shift.ctypes.data, host,
                 ctypes.addressof(rows))
    assert rows.value
    np.testing.assert_array_equal(host, dec.decode(obs, z) + shift)
    ws = dec.warm_start(obs, 1000, solver.layout, np.random.default_rng(8), shift=shift)
    cfg = bd.BiLevelConfig(1000, 150, 100, 2, 0.7, 0.9, 1.0, mean, cov)
    seen = []
    a = bd.solve_bilevel(scene, solver, cfg, np.random.default_rng(2), warm_start=ws,
                         trace_hook=lambda *args: seen.append(1))
    b = bd.solve_bilevel(scene, solver, cfg, np.random.default_rng(2),
                         warm_start=WarmStartSource(ws.samples, solver.layout), trace_hook=lambda *args: None)
    assert seen
    _same_result(a, b)
