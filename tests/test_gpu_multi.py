"""GPU, world size 2 (needs two visible GPUs; skipped otherwise): the multi-rank paths on real NCCL
and real NVLink peer memory, each compared bit for bit with the single-rank device run.

* ShardedCEM + CudaShardBackend (NCCL collectives): batch-global semantics of the sharded batch --
  global elites (pkg/bilevel.py:129-137), the refit (:175-194) and the batch-global early exit
  (pkg/projection.py:329) -- must give exactly the single-context bd_cem_cycle result;
* the same with P2PExchange (AM-epilogue stores into the peer's symmetric buffer, epoch signals);
* plan_fleet_distributed (config 5): scenes split over the ranks, gathered records == one rank.

Both ranks use the same lane mapping as the single-rank run (lanes_per_sample = 8) so the fp32
reduction order, and hence every bit, is shared.
"""

import multiprocessing as mp
import socket

import numpy as np
import pytest
import torch

pytestmark = [pytest.mark.gpu,
              pytest.mark.skipif(torch.cuda.device_count() < 2, reason="needs two GPUs (world size 2)")]

KW = dict(batch=512, n_cons=100, n_elite=50, iterations=3, eta=0.7, gamma=0.9, residual_weight=1.0, am_iters=60,
          seed=21)


def _fleet(device, batch=512, n=100, q=50, N=3, am_iters=60, tol=1e-3):
    import paper_2212_02224_b200 as bd
    from paper_2212_02224_b200.fleet import FleetPlanner
    basis = bd.build_basis(10, 100, 5.0, "bernstein")
    cfg = bd.BiLevelConfig(batch, n, q, N, 0.7, 0.9, 1.0)
    fp = FleetPlanner(basis, bd.TrackingWeights(), bd.ParamLayout(4), bd.ProjectionConfig(1.0, am_iters, tol), 10,
                      cfg, device=device)
    fp.context.set_option("lanes_per_sample", 8)
    return fp


def _pack(r):
    return dict(best_index=r.best_index, best_xi=r.best_xi, mean=r.mean, cov=r.cov, stats=r.stats,
                used=np.array(r.iterations_used))


def _worker(rank, world, port, tol, q):
    import torch.distributed as dist
    from paper_2212_02224_b200.fleet import initial_distribution
    from paper_2212_02224_b200.parallel import CudaShardBackend, P2PExchange, ShardedCEM, plan_fleet_distributed
    from paper_2212_02224_b200.scenes import highway_scene
    torch.cuda.set_device(rank)
    dist.init_process_group("nccl", init_method=f"tcp://127.0.0.1:{port}", rank=rank, world_size=world,
                            device_id=torch.device("cuda", rank))
    try:
        fp = _fleet(rank)
        sc = highway_scene(4)
        mean, cov = initial_distribution(sc)
        out = {"nccl": _pack(ShardedCEM(CudaShardBackend(fp.solver, sc, device=rank), tol=tol, **KW).run(mean, cov))}
        ex = P2PExchange(fp.context, KW["batch"], KW["am_iters"], device=torch.device("cuda", rank))
        be = CudaShardBackend(fp.solver, sc, device=rank)
        out["p2p"] = _pack(ShardedCEM(be, exchange=ex, tol=tol, **KW).run(mean, cov))
        fleet = _fleet(rank, batch=256, n=64, q=16, N=2, am_iters=30)
        out["fleet"] = plan_fleet_distributed(fleet, highway_scene, 6, seed=5)
        torch.cuda.synchronize()
        q.put((rank, out))
    except Exception as exc:  # noqa: BLE001
        q.put((rank, {"error": repr(exc)}))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("tol", [1e-3, 5.0])
def test_world2_sharded_and_fleet_paths_equal_single_rank(tol):
    """tol = 5 makes the batch-global exit fire early: the exit must be decided across both ranks."""
    from paper_2212_02224_b200.fleet import initial_distribution
    from paper_2212_02224_b200.scenes import highway_scene
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, tol, q)) for r in range(2)]
    for p in procs:
        p.start()
    got = dict(q.get(timeout=600) for _ in procs)
    for p in procs:
        p.join(timeout=60)
    for r in range(2):
        assert "error" not in got[r], got[r]
    # single-rank references on this process
    fp = _fleet(0, tol=tol)
    sc = highway_scene(4)
    mean, cov = initial_distribution(sc)
    ref = fp.plan([sc], seed=KW["seed"], init_mean=mean[None], init_cov=cov[None])
    for r in range(2):
        for mode in ("nccl", "p2p"):
            g = got[r][mode]
            assert g["best_index"] == int(ref.best_index[0]), (r, mode)
            np.testing.assert_array_equal(g["best_xi"], ref.best_xi[0])
            np.testing.assert_array_equal(g["mean"], ref.final_mean[0])
            np.testing.assert_array_equal(g["cov"], ref.final_cov[0])
            np.testing.assert_array_equal(g["stats"], ref.stats[0])
        np.testing.assert_array_equal(got[r]["nccl"]["used"], got[r]["p2p"]["used"])
        if tol > 1:
            assert got[r]["nccl"]["used"].min() < KW["am_iters"]
    fleet = _fleet(0, batch=256, n=64, q=16, N=2, am_iters=30)
    one = fleet.plan([highway_scene(g) for g in range(6)], seed=5)
    cols = np.concatenate([one.best_index[:, None].astype(np.float64), one.best_cost[:, None],
                           one.best_residual[:, None], one.best_aug[:, None], one.best_xi,
                           one.iterations_done[:, None].astype(np.float64)], axis=1)
    for r in range(2):
        np.testing.assert_array_equal(got[r]["fleet"], cols)
