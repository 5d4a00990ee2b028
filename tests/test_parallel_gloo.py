"""Multi-rank host logic on CPU (gloo, world_size 2): the sharded-batch CEM protocol of
paper_2212_02224_b200.parallel must give the same result as one rank, and the batch-global
early exit must be decided across ranks.  The per-shard compute is a float64 oracle stand-in
(test infrastructure) because this container has no GPU."""

import os
import socket
import tempfile

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import oracle as O
from oracle.philox import philox_normals
from paper_2212_02224_b200.parallel import ShardedCEM, shard_range
from tests.golden_io import load, oracle_limits


class OracleShardBackend:
    """CPU stand-in for CudaShardBackend built on the oracle restatement."""

    def __init__(self, g, am_iters):
        _, self.W, self.Wd, self.Wdd = O.basis_matrices(10, 100, 5.0)
        self.qp = O.tracking_qp(self.W, self.Wd, self.Wdd, 4)
        self.lim = oracle_limits(g)
        self.aug = O.aug_qp(self.W, self.Wd, self.Wdd, self.qp.A_eq, self.lim.n_obs, 1.0)
        self.b0 = g["b0"]
        self.calls = []

    def tensor(self, x):
        return torch.as_tensor(np.asarray(x, dtype=np.float64))

    def sample(self, mean, cov, seed, it, count):
        z = philox_normals(seed, 0, it, np.arange(count), mean.shape[0])
        try:
            L = np.linalg.cholesky(cov.numpy())
        except np.linalg.LinAlgError:
            L = np.linalg.cholesky(cov.numpy() + 1e-5 * np.eye(cov.shape[0]))
        return torch.as_tensor(mean.numpy()[None] + z @ L.T)

    def _project(self, iters):
        pr = O.am_project(self.aug, self.W, self.Wd, self.Wdd, self._xb, self._b, self.lim, 1.0, iters, tol=-1.0)
        n = self.W.shape[1]
        cost = O.speed_cost(pr["xi"][:n].T @ self.Wd.T, pr["xi"][n:].T @ self.Wd.T, self.lim.v_max)
        return pr, cost

    def solve_shard(self, P, iters):
        self.calls.append(("solve", iters))
        self._xb, _, self._b = O.stage1(self.qp, P.numpy(), self.b0)
        pr, cost = self._project(iters)
        return {"xi": torch.as_tensor(pr["xi"].T.copy()), "residuals": torch.as_tensor(pr["residuals"]),
                "cost": torch.as_tensor(cost),
                "iter_max": torch.as_tensor(pr["history"].max(axis=1).astype(np.float32))}

    def replay_shard(self, iters, shard):
        k = int(iters[0])                      # device-gated in the CUDA backend: <= 0 keeps the first pass
        if k <= 0:
            return shard
        self.calls.append(("replay", k))
        pr, cost = self._project(k)
        return {"xi": torch.as_tensor(pr["xi"].T.copy()), "residuals": torch.as_tensor(pr["residuals"]),
                "cost": torch.as_tensor(cost)}

    def check(self):
        pass

    def rank_refit(self, resid, cost, P, mean, cov, n, q, w, eta, gamma):
        r, c = resid.numpy(), cost.numpy()
        cons, el, ea = O.rank_two_stage(r, c, n, q, w)
        mu, C = O.refit_gaussian(mean.numpy(), cov.numpy(), P.numpy()[el], ea, eta, gamma)
        st = [c[el].mean(), ea[0], np.trace(C), r.min(), np.median(r), r.max()]
        return {"mean": torch.as_tensor(mu), "cov": torch.as_tensor(C), "elite_idx": torch.as_tensor(el),
                "elite_aug": torch.as_tensor(ea), "stats": torch.as_tensor(np.array(st))}


CASE = dict(batch=40, n_cons=12, n_elite=6, iterations=2, eta=0.7, gamma=0.9, residual_weight=1.0, am_iters=12,
            tol=1e-3, seed=5)


def _run(group=None):
    g = load("lower_c1_s1")
    be = OracleShardBackend(g, CASE["am_iters"])
    cem = ShardedCEM(be, group=group, **CASE)
    mean = np.concatenate([np.full(4, g["b0"][1]), np.full(4, 10.0)])
    cov = np.diag(np.concatenate([np.full(4, 1.5 ** 2), np.full(4, 3.0 ** 2)]))
    return cem.run(mean, cov)


def _worker(rank, world, port, out):
    os.environ["OPENBLAS_NUM_THREADS"] = "1"
    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank, world_size=world)
    try:
        res = _run()
        if rank == 0:
            np.savez(out, best_index=res.best_index, best_xi=res.best_xi, mean=res.mean, cov=res.cov,
                     stats=res.stats, used=np.array(res.iterations_used))
    finally:
        dist.destroy_process_group()


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def test_shard_ranges_cover_batch():
    for total in (1, 7, 40, 1000, 10000):
        for world in (1, 2, 3, 4, 8):
            got = []
            for r in range(world):
                lo, hi, shard = shard_range(total, r, world)
                assert hi - lo <= shard
                got.extend(range(lo, hi))
            assert got == list(range(total))


@pytest.mark.slow
def test_two_rank_sharded_cem_equals_one_rank():
    ref = _run()
    with tempfile.TemporaryDirectory() as td:
        out = os.path.join(td, "r0.npz")
        mp.spawn(_worker, args=(2, _free_port(), out), nprocs=2, join=True)
        got = np.load(out)
    assert int(got["best_index"]) == ref.best_index
    np.testing.assert_allclose(got["best_xi"], ref.best_xi, rtol=1e-9, atol=1e-9)
    np.testing.assert_allclose(got["mean"], ref.mean, rtol=1e-9)
    np.testing.assert_allclose(got["cov"], ref.cov, rtol=1e-8, atol=1e-12)
    np.testing.assert_allclose(got["stats"], ref.stats, rtol=1e-8, atol=1e-10)
    assert list(got["used"]) == ref.iterations_used


class FakeBackend:
    """Scripted shard results: exercises the cross-rank early-exit decision + replay."""

    def __init__(self, rank, itmax):
        self.rank, self.itmax, self.replays = rank, itmax, []

    def tensor(self, x):
        return torch.as_tensor(np.asarray(x, dtype=np.float64))

    def sample(self, mean, cov, seed, it, count):
        return torch.arange(count * 2, dtype=torch.float64).reshape(count, 2)

    def solve_shard(self, P, iters):
        n = P.shape[0]
        return {"xi": torch.zeros(n, 22, dtype=torch.float64), "residuals": P[:, 0].clone(),
                "cost": torch.zeros(n, dtype=torch.float64), "iter_max": torch.as_tensor(self.itmax, dtype=torch.float32)}

    def replay_shard(self, iters, shard):
        if int(iters[0]) > 0:
            self.replays.append(int(iters[0]))
        return shard

    def check(self):
        pass

    def rank_refit(self, resid, cost, P, mean, cov, n, q, w, eta, gamma):
        order = torch.argsort(resid, stable=True)
        return {"mean": mean, "cov": cov, "elite_idx": order[:q], "elite_aug": resid[order[:q]],
                "stats": torch.zeros(6, dtype=torch.float64)}


def _exit_worker(rank, world, port, out):
    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank, world_size=world)
    try:
        # rank 0 converges at iteration 3, rank 1 only at iteration 6: the batch exits at 6
        itmax = [5.0, 4.0, 1e-4, 0.0, 0.0, 0.0, 0.0, 0.0] if rank == 0 else [5.0, 4.0, 3.0, 2.0, 1.0, 1e-4, 0.0, 0.0]
        be = FakeBackend(rank, itmax)
        res = ShardedCEM(be, batch=10, n_cons=4, n_elite=2, iterations=1, eta=0.5, gamma=1.0, residual_weight=1.0,
                         am_iters=8, tol=1e-3, seed=0).run(np.zeros(2), np.eye(2))
        np.save(out + f".{rank}.npy", np.array(be.replays + [res.iterations_used[0], res.best_index]))
    finally:
        dist.destroy_process_group()


def test_batch_global_exit_decided_across_ranks():
    with tempfile.TemporaryDirectory() as td:
        out = os.path.join(td, "x")
        mp.spawn(_exit_worker, args=(2, _free_port(), out), nprocs=2, join=True)
        for r in range(2):
            replays_used_best = np.load(out + f".{r}.npy")
            assert list(replays_used_best) == [6, 6, 0]
