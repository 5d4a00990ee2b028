"""GPU: CVAE warm-start decoder (K5) vs a float64 numpy restatement, and config 3
(decoder samples -> warm start of the device CEM cycle)."""

import numpy as np
import pytest

from oracle.cvae import decode as decode_ref

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
    """Hidden layers on tcgen05 (bf16 operands, fp32 TMEM accumulation): bf16 rounding bound."""
    from paper_2212_02224_b200.cvae import CVAEDecoder
    dec = CVAEDecoder.synthetic(7)
    rng = np.random.default_rng(1)
    obs = rng.standard_normal(55).astype(np.float32)
    z = rng.standard_normal((count, 2)).astype(np.float32)
    got = dec.decode(obs, z)
    ref = decode_ref(dec.W, dec.b, obs, z)
    scale = np.abs(ref).max()
    err = np.abs(got - ref)
    assert err.max() <= 5e-2 * scale, err.max() / scale
    assert err.mean() <= 1e-2 * scale, err.mean() / scale


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
    # iteration 1 ranked the decoder's samples: the best record's set-points are one of them
    if res.best.index >= 0 and len(res.diagnostics) == 1:
        assert np.any(np.all(np.isclose(ws.samples, res.best.params.to_vector()), axis=1))
