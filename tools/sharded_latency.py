"""Config 4 through the sharded-batch protocol on one rank (ShardedCEM + CudaShardBackend) vs the
single-context CEM cycle (bd_cem_cycle) on the same scene: the protocol's overhead."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2212_02224_b200 as bd  # noqa: E402
from paper_2212_02224_b200.fleet import FleetPlanner, initial_distribution  # noqa: E402
from paper_2212_02224_b200.parallel import CudaShardBackend, P2PExchange, ShardedCEM  # noqa: E402
from paper_2212_02224_b200.scenes import HighwayRecipe, highway_scene  # noqa: E402

basis = bd.build_basis(10, 100, 5.0, "bernstein")
cfg = bd.BiLevelConfig(10_000, 150, 100, 4, 0.7, 0.9, 1.0)
fp = FleetPlanner(basis, bd.TrackingWeights(), bd.ParamLayout(4), bd.ProjectionConfig(1.0, 100, 1e-3), 50, cfg)
sc = highway_scene(0, HighwayRecipe(density=3.0, vehicle_count=80, n_obs=50, obstacle_range=250.0))
mean, cov = initial_distribution(sc)
be = CudaShardBackend(fp.solver, sc)
cem = ShardedCEM(be, batch=10_000, n_cons=150, n_elite=100, iterations=4, eta=0.7, gamma=0.9, residual_weight=1.0,
                 am_iters=100, tol=1e-3, seed=3)
cem.run(mean, cov)
torch.cuda.synchronize()
ts = []
for _ in range(5):
    t0 = time.perf_counter()
    cem.run(mean, cov)
    torch.cuda.synchronize()
    ts.append(time.perf_counter() - t0)
print(f"ShardedCEM world=1 (collective path): {1e3 * np.median(ts):.2f} ms per cycle")
import socket  # noqa: E402

import torch.distributed as dist  # noqa: E402

with socket.socket() as s:
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
dist.init_process_group("nccl", init_method=f"tcp://127.0.0.1:{port}", rank=0, world_size=1,
                        device_id=torch.device("cuda:0"))
cem.exchange = P2PExchange(fp.context, 10_000, 100)
cem.run(mean, cov)
torch.cuda.synchronize()
ts = []
for _ in range(5):
    t0 = time.perf_counter()
    cem.run(mean, cov)
    torch.cuda.synchronize()
    ts.append(time.perf_counter() - t0)
print(f"ShardedCEM world=1 (peer-memory exchange): {1e3 * np.median(ts):.2f} ms per cycle")
cem.exchange = None
dist.destroy_process_group()
fp.set_scenes([sc])
fp.plan([sc], seed=1, init_mean=mean[None], init_cov=cov[None])
ts = []
for k in range(5):
    t0 = time.perf_counter()
    fp.plan([sc], seed=2 + k, init_mean=mean[None], init_cov=cov[None])
    ts.append(time.perf_counter() - t0)
print(f"bd_cem_cycle: {1e3 * np.median(ts):.2f} ms per cycle")
