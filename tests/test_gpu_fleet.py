"""GPU: device Philox stream, fleet planning (config 5) and the sharded-batch protocol (config 4)
at world size 1 on the CUDA backend."""

import numpy as np
import pytest

from oracle.philox import philox_normals
from tests.golden_io import load, rel_err_per_sample_axis
from tests.test_gpu_parity import _scene
from tests.test_parallel_gloo import OracleShardBackend

pytestmark = pytest.mark.gpu


def _fleet(batch=1000, n=150, q=100, N=4, am_iters=100, n_obs=10):
    import paper_2212_02224_b200 as bd
    from paper_2212_02224_b200.fleet import FleetPlanner
    basis = bd.build_basis(10, 100, 5.0, "bernstein")
    cfg = bd.BiLevelConfig(batch, n, q, N, 0.7, 0.9, 1.0)
    return FleetPlanner(basis, bd.TrackingWeights(), bd.ParamLayout(4), bd.ProjectionConfig(1.0, am_iters, 1e-3),
                        n_obs, cfg)


def test_device_philox_matches_numpy_restatement():
    fp = _fleet()
    P = np.empty((777, 8))
    fp.context.call("bd_sample_philox", 8, 777, np.zeros(8), np.eye(8), 1234, 3, 2, 100, P)
    Z = philox_normals(1234, 3, 2, np.arange(100, 877), 8)
    np.testing.assert_allclose(P, Z, rtol=1e-12, atol=1e-12)


def test_fleet_scenes_are_independent_of_batching():
    from paper_2212_02224_b200.scenes import highway_scene
    fp = _fleet(batch=256, n=64, q=16, N=2, am_iters=30)
    scenes = [highway_scene(s) for s in range(3)]
    allr = fp.plan(scenes, seed=9)
    for j, sc in enumerate(scenes):
        one = fp.plan([sc], seed=9, scene_offset=j)
        assert one.best_index[0] == allr.best_index[j]
        np.testing.assert_array_equal(one.best_xi[0], allr.best_xi[j])
        np.testing.assert_array_equal(one.stats[0], allr.stats[j])
    assert np.all(allr.iterations_done == 2)


def test_sharded_world1_equals_device_cem_cycle():
    import torch
    from paper_2212_02224_b200.fleet import initial_distribution
    from paper_2212_02224_b200.parallel import CudaShardBackend, ShardedCEM
    from paper_2212_02224_b200.scenes import highway_scene
    fp = _fleet(batch=512, n=100, q=50, N=3, am_iters=60)
    sc = highway_scene(4)
    mean, cov = initial_distribution(sc)
    ref = fp.plan([sc], seed=21, init_mean=mean[None], init_cov=cov[None])
    be = CudaShardBackend(fp.solver, sc)
    res = ShardedCEM(be, batch=512, n_cons=100, n_elite=50, iterations=3, eta=0.7, gamma=0.9, residual_weight=1.0,
                     am_iters=60, tol=1e-3, seed=21).run(mean, cov)
    torch.cuda.synchronize()
    assert res.best_index == int(ref.best_index[0])
    np.testing.assert_array_equal(res.best_xi, ref.best_xi[0])
    np.testing.assert_array_equal(res.mean, ref.final_mean[0])
    np.testing.assert_array_equal(res.stats, ref.stats[0])


def test_device_cem_cycle_matches_oracle_with_same_draws():
    """bd_cem_cycle (device Philox) vs the float64 oracle driven by the same Philox stream."""
    from paper_2212_02224_b200.parallel import ShardedCEM
    g = load("cem_small")
    B, n, q, N, am = 200, 60, 20, 3, 40
    fp = _fleet(batch=B, n=n, q=q, N=N, am_iters=am)
    sc = _scene(g)
    ref = ShardedCEM(OracleShardBackend(g, am), batch=B, n_cons=n, n_elite=q, iterations=N, eta=0.7, gamma=0.9,
                     residual_weight=1.0, am_iters=am, tol=1e-3, seed=17).run(g["init_mean"], g["init_cov"])
    got = fp.plan([sc], seed=17, init_mean=g["init_mean"][None], init_cov=g["init_cov"][None])
    assert int(got.best_index[0]) == ref.best_index
    assert rel_err_per_sample_axis(got.best_xi[0][:, None], ref.best_xi[:, None]) <= 1e-4
    np.testing.assert_allclose(got.final_mean[0], ref.mean, rtol=1e-4)
    np.testing.assert_allclose(got.stats[0][:, :3], ref.stats[:, :3], rtol=1e-4)


@pytest.mark.parametrize("tol", [1e-3, 5.0])
def test_sharded_p2p_exchange_world1_equals_nccl_path(tol):
    """The NVLink peer-memory exchange (fused epilogue stores, epoch signals, device exit decision)
    in a one-rank group (loopback) gives bit-identical results to the collective path; tol = 5
    makes the batch-global exit fire early, exercising the device-gated replay and its re-publish."""
    import socket

    import torch
    import torch.distributed as dist
    from paper_2212_02224_b200.fleet import initial_distribution
    from paper_2212_02224_b200.parallel import CudaShardBackend, P2PExchange, ShardedCEM
    from paper_2212_02224_b200.scenes import highway_scene
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    dist.init_process_group("nccl", init_method=f"tcp://127.0.0.1:{port}", rank=0, world_size=1,
                            device_id=torch.device("cuda:0"))
    try:
        fp = _fleet(batch=512, n=100, q=50, N=3, am_iters=60)
        sc = highway_scene(4)
        mean, cov = initial_distribution(sc)
        kw = dict(batch=512, n_cons=100, n_elite=50, iterations=3, eta=0.7, gamma=0.9, residual_weight=1.0,
                  am_iters=60, tol=tol, seed=21)
        ref = ShardedCEM(CudaShardBackend(fp.solver, sc), **kw).run(mean, cov)
        if tol > 1:
            assert min(ref.iterations_used) < 60
        be = CudaShardBackend(fp.solver, sc)
        ex = P2PExchange(fp.context, 512, 60)
        for _ in range(2):                       # epochs keep increasing across runs
            got = ShardedCEM(be, exchange=ex, **kw).run(mean, cov)
            torch.cuda.synchronize()
            assert got.best_index == ref.best_index
            np.testing.assert_array_equal(got.best_xi, ref.best_xi)
            np.testing.assert_array_equal(got.mean, ref.mean)
            np.testing.assert_array_equal(got.cov, ref.cov)
            np.testing.assert_array_equal(got.stats, ref.stats)
            assert got.iterations_used == ref.iterations_used
        assert ex.epoch == 6
    finally:
        dist.destroy_process_group()


def test_sharded_loop_keeps_device_errors():
    """The sharded loop's device error word is sticky: a non-finite set-point drawn in
    CEM iteration 2 is still reported after the loop although the later shard / refit calls of
    the loop would each have cleared it (pkg/batch_qp.py:105-106 -> ValueError), and the context
    is usable again afterwards."""
    import torch
    from paper_2212_02224_b200.fleet import initial_distribution
    from paper_2212_02224_b200.parallel import CudaShardBackend, ShardedCEM
    from paper_2212_02224_b200.scenes import highway_scene
    fp = _fleet(batch=256, n=64, q=16, N=3, am_iters=20)
    sc = highway_scene(4)
    mean, cov = initial_distribution(sc)

    class Inject(CudaShardBackend):
        def sample(self, mean, cov, seed, it, count):
            P = super().sample(mean, cov, seed, it, count)
            if it == 1:
                P[5, 0] = float("nan")
            return P

    kw = dict(batch=256, n_cons=64, n_elite=16, iterations=3, eta=0.7, gamma=0.9, residual_weight=1.0, am_iters=20,
              tol=1e-3, seed=3)
    with pytest.raises(ValueError, match="finite"):
        ShardedCEM(Inject(fp.solver, sc), **kw).run(mean, cov)
    torch.cuda.synchronize()
    res = ShardedCEM(CudaShardBackend(fp.solver, sc), **kw).run(mean, cov)
    assert np.isfinite(res.best_cost)
