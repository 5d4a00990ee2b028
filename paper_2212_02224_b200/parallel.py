"""Multi-GPU drivers: one process per GPU, torch.distributed (NCCL over NVLink) for the plumbing.

Two ways the path shards:

* **Fleet** (BASELINE config 5) — independent scenes, contiguous blocks of global scene ids per
  rank, each planned with :class:`~paper_2212_02224_b200.fleet.FleetPlanner`.  No collective on
  the data path; the per-scene best records are gathered once at the end (C4).

* **Sharded batch** (BASELINE config 4) — one scene whose B samples are split contiguously over
  ranks by global sample index.  Per CEM iteration (pkg/bilevel.py:249-292):

  1. every rank regenerates the *full* batch of set-points from the device Philox stream keyed
     by global sample index (bit-identical on every rank, independent of the rank count);
  2. stage 1 + AM projection on the local shard only, without the batch-global exit;
  3. C1: all-reduce(MAX) of the per-iteration shard maxima -> the reference's batch-global
     early exit (pkg/projection.py:329) decided for the whole batch; ranks replay their shard
     for exactly that many iterations if it fired;
  4. C2: all-gather of the shard (residual, cost) pairs -> full arrays on every rank;
  5. rank + refit on the full arrays, identically on every rank (C3 needs no sufficient-statistic
     exchange: every rank already holds the elite set-points), then the owner of the best sample
     broadcasts its 22 coefficients.

The protocol is written against a small backend interface so the same code runs the CUDA path
(:class:`CudaShardBackend`) and, in the CPU test-suite, an oracle stand-in over gloo.
"""

from __future__ import annotations

import math
from dataclasses import dataclass

import numpy as np
import torch
import torch.distributed as dist

__all__ = ["shard_range", "ShardedCEM", "ShardedResult", "CudaShardBackend", "plan_fleet_distributed"]


def _world(group=None):
    if dist.is_available() and dist.is_initialized():
        return dist.get_rank(group), dist.get_world_size(group)
    return 0, 1


def shard_range(total: int, rank: int, world: int) -> tuple[int, int, int]:
    """(lo, hi, shard) of the contiguous block of `total` items owned by `rank` (shard = ceil)."""
    shard = math.ceil(total / world)
    lo = min(total, rank * shard)
    return lo, min(total, lo + shard), shard


@dataclass
class ShardedResult:
    best_index: int
    best_xi: np.ndarray
    best_cost: float
    best_residual: float
    best_aug: float
    stats: np.ndarray          # N x 6 IterationStats fields
    mean: np.ndarray
    cov: np.ndarray
    iterations_used: list      # AM iterations actually run per CEM iteration


class ShardedCEM:
    """solve_bilevel over one scene with the batch sharded across the process group."""

    def __init__(self, backend, batch: int, n_cons: int, n_elite: int, iterations: int, eta: float, gamma: float,
                 residual_weight: float, am_iters: int, tol: float, seed: int, group=None, exchange=None):
        self.b = backend
        self.B, self.n, self.q, self.N = batch, n_cons, n_elite, iterations
        self.eta, self.gamma, self.w = eta, gamma, residual_weight
        self.am_iters, self.tol, self.seed = am_iters, tol, seed
        self.group = group
        self.rank, self.world = _world(group)
        self.lo, self.hi, self.shard = shard_range(batch, self.rank, self.world)
        self.exchange = exchange           # P2PExchange: NVLink peer-memory exchange instead of NCCL

    def _all_reduce_max(self, t: torch.Tensor) -> torch.Tensor:
        if self.world > 1:
            dist.all_reduce(t, op=dist.ReduceOp.MAX, group=self.group)
        return t

    def _all_gather(self, t: torch.Tensor) -> torch.Tensor:
        """Gather equal-size (padded) shards; returns the concatenation trimmed to the batch."""
        if self.world == 1:
            return t
        pad = torch.full((self.shard,) + tuple(t.shape[1:]), float("inf"), dtype=t.dtype, device=t.device)
        pad[: t.shape[0]] = t
        parts = [torch.empty_like(pad) for _ in range(self.world)]
        dist.all_gather(parts, pad, group=self.group)
        return torch.cat(parts)[: self.B]

    def _all_reduce_sum(self, t: torch.Tensor) -> torch.Tensor:
        if self.world > 1:
            dist.all_reduce(t, op=dist.ReduceOp.SUM, group=self.group)
        return t

    def run(self, init_mean, init_cov) -> ShardedResult:
        """The CEM loop with every decision on the device: the batch-global exit iteration comes
        from the all-reduced maxima as a device scalar that gates the replay kernel, the best
        sample's coefficients reach every rank through an all-reduce of owner-masked rows, and
        per-iteration records stay in device tensors until one transfer at the end -- no host
        round trip inside the loop."""
        mean = self.b.tensor(init_mean)
        cov = self.b.tensor(init_cov)
        dev = mean.device
        N = self.N
        stats = torch.zeros((N, 6), dtype=torch.float64, device=dev)
        used = torch.zeros(N, dtype=torch.int64, device=dev)
        rec = torch.zeros(5, dtype=torch.float64, device=dev)        # index, cost, residual, aug (last iteration)
        xi_best = torch.zeros(22, dtype=torch.float64, device=dev)
        ks = None
        if hasattr(self.b, "begin"):
            self.b.begin()                  # device errors accumulate over the loop (read by check())
        for it in range(N):
            P = self.b.sample(mean, cov, self.seed, it, self.B)                 # full batch, every rank
            if self.exchange is not None:
                ex = self.exchange
                epoch = ex.next_epoch()
                shard = self.b.solve_shard_p2p(P[self.lo:self.hi], self.am_iters, self.lo, epoch, self.tol)
                used[it] = shard["used"][0].to(dev)
                full = torch.stack([ex.res, ex.cost], dim=1)                      # gathered on every rank
                out = self.b.rank_refit(ex.res, ex.cost, P, mean, cov, self.n, self.q, self.w, self.eta, self.gamma)
                mean, cov = out["mean"], out["cov"]
                j = out["elite_idx"][:1]
                xi_best = self.b.best_row_p2p(j, self.lo, shard["xi"], epoch)
                pick = full.index_select(0, j)[0]
                rec = torch.stack([j[0].to(torch.float64), pick[1], pick[0], out["elite_aug"][0].to(torch.float64)])
                stats[it] = out["stats"].to(torch.float64)
                continue
            shard = self.b.solve_shard(P[self.lo:self.hi], self.am_iters)         # no exit decision
            itmax = self._all_reduce_max(shard["iter_max"].clone())              # C1
            if ks is None:
                ks = torch.arange(1, itmax.shape[0] + 1, device=itmax.device)
            hit = itmax.double() <= self.tol
            first = torch.where(hit, ks, torch.full_like(ks, self.am_iters)).min()     # used iterations
            replay = torch.where(first < self.am_iters, first, torch.zeros_like(first)).to(torch.int32).reshape(1)
            shard = self.b.replay_shard(replay, shard)                            # gated on the device
            used[it] = first.to(dev)
            rc = torch.stack([shard["residuals"], shard["cost"]], dim=1)
            full = self._all_gather(rc)                                           # C2
            out = self.b.rank_refit(full[:, 0].contiguous(), full[:, 1].contiguous(), P, mean, cov, self.n, self.q,
                                    self.w, self.eta, self.gamma)
            mean, cov = out["mean"], out["cov"]
            j = out["elite_idx"][:1]
            mine = (j >= self.lo) & (j < self.hi)
            row = shard["xi"].index_select(0, (j - self.lo).clamp(0, shard["xi"].shape[0] - 1))[0]
            xi_best = self._all_reduce_sum(row * mine.to(row.dtype))             # owner's row, zeros elsewhere
            pick = full.index_select(0, j)[0]
            rec = torch.stack([j[0].to(torch.float64), pick[1], pick[0], out["elite_aug"][0].to(torch.float64)])
            stats[it] = out["stats"].to(torch.float64)
        self.b.check()
        r = rec.cpu().numpy()
        return ShardedResult(int(r[0]), xi_best.cpu().numpy(), float(r[1]), float(r[2]), float(r[3]),
                             stats.cpu().numpy(), mean.cpu().numpy(), cov.cpu().numpy(),
                             [int(u) for u in used.cpu().numpy()])


class P2PExchange:
    """The sharded batch's exchange over NVLink peer memory (torch symmetric memory buffers,
    peer-mapped on every rank): the AM epilogue writes each (residual, cost) into every rank's
    gathered arrays, maxima and the best coefficient row follow through the same buffers with
    epoch signals (csrc/p2p_kernels.cuh) -- no NCCL call in the CEM loop."""

    def __init__(self, ctx, batch: int, iters_cap: int, group=None, device=None):
        import torch.distributed._symmetric_memory as symm
        self.group = group if group is not None else dist.group.WORLD
        self.rank, self.world = _world(group)
        al = lambda x: (x + 255) // 256 * 256  # noqa: E731
        self.res_off, self.cost_off = 0, al(8 * batch)
        self.itmax_off = al(self.cost_off + 8 * batch)
        self.xi_off = al(self.itmax_off + 4 * self.world * iters_cap)
        total = al(self.xi_off + 8 * 22 * self.world)
        dev = device if device is not None else torch.device("cuda", torch.cuda.current_device())
        self.buf = symm.empty(total, dtype=torch.uint8, device=dev)
        self.buf.zero_()
        self.hdl = symm.rendezvous(self.buf, self.group)
        ctx.call("bd_shard_p2p_set", self.world, self.rank, int(self.hdl.buffer_ptrs_dev),
                 int(self.hdl.signal_pad_ptrs_dev), self.res_off, self.cost_off, self.itmax_off, self.xi_off,
                 int(iters_cap))
        self.res = self.buf[self.res_off:self.res_off + 8 * batch].view(torch.float64)
        self.cost = self.buf[self.cost_off:self.cost_off + 8 * batch].view(torch.float64)
        self.epoch = 0
        self.iters_cap = iters_cap

    def next_epoch(self) -> int:
        self.epoch += 1
        return self.epoch


class CudaShardBackend:
    """ShardedCEM backend on the CUDA library (device tensors, C-ABI on the torch stream)."""

    def __init__(self, solver, scene, device: int | None = None):
        self.solver = solver
        self.ctx = solver.context
        self.dev = torch.device("cuda", device if device is not None else torch.cuda.current_device())
        solver.projector._check_spec(scene.spec)
        solver.projector._ensure_scene(scene)
        self.ctx.set_stream(torch.cuda.current_stream(self.dev).cuda_stream)
        self.dim = solver.layout.dim

    def tensor(self, x):
        return torch.as_tensor(np.asarray(x, dtype=np.float64), device=self.dev).contiguous()

    def sample(self, mean, cov, seed, it, count):
        P = torch.empty((count, self.dim), dtype=torch.float64, device=self.dev)
        self.ctx.call("bd_sample_philox", self.dim, count, mean, cov, int(seed), 0, int(it), 0, P)
        return P

    def solve_shard(self, P, iters):
        n = P.shape[0]
        self._xb = torch.empty((n, 22), dtype=torch.float64, device=self.dev)
        xi = torch.empty_like(self._xb)
        res = torch.empty(n, dtype=torch.float64, device=self.dev)
        cost = torch.empty_like(res)
        mx = torch.empty(iters, dtype=torch.float32, device=self.dev)
        self._iters = iters
        self.ctx.call("bd_solve_lower_shard", n, P.contiguous(), iters, self._xb, xi, res, cost, mx)
        return {"xi": xi, "residuals": res, "cost": cost, "iter_max": mx}

    def solve_shard_p2p(self, P, iters, row0, epoch, tol):
        n = P.shape[0]
        self._xb = torch.empty((n, 22), dtype=torch.float64, device=self.dev)
        xi = torch.empty_like(self._xb)
        res = torch.empty(n, dtype=torch.float64, device=self.dev)
        cost = torch.empty_like(res)
        used = torch.zeros(1, dtype=torch.int32, device=self.dev)
        self._iters = iters
        self.ctx.call("bd_solve_lower_shard_p2p", n, P.contiguous(), iters, self._xb, xi, res, cost, int(row0),
                      int(epoch), float(tol), used)
        return {"xi": xi, "residuals": res, "cost": cost, "used": used}

    def best_row_p2p(self, best, row0, xi_shard, epoch):
        out = torch.empty(22, dtype=torch.float64, device=self.dev)
        self.ctx.call("bd_shard_p2p_best_row", best.contiguous(), int(row0), xi_shard.shape[0], xi_shard, int(epoch),
                      out)
        return out

    def replay_shard(self, iters, shard):
        """Re-run the shard for iters[0] AM iterations when > 0 (device-gated, in place)."""
        n = self._xb.shape[0]
        self.ctx.call("bd_replay_shard_dev", n, self._xb, self._iters, iters.to(self.dev).contiguous(), shard["xi"],
                      shard["residuals"], shard["cost"])
        return shard

    def begin(self):
        """Sticky error word for the loop: the shard / replay / refit calls OR into it instead of
        clearing it, so a non-finite iterate, a bad right-hand side or a peer-exchange timeout in
        any iteration survives to check()."""
        self.ctx.set_option("sticky_errors", 1)

    def check(self):
        """Raise for any device error of the loop (checked once, after it)."""
        bits = self.ctx.error_bits()
        self.ctx.set_option("sticky_errors", 0)
        if bits & 16:                       # ERR_P2P_TIMEOUT: a rank never signalled
            raise RuntimeError(f"sharded CEM: peer exchange timed out (device error bits {bits:#x})")
        if bits & 4:                        # ERR_BAD_RHS
            raise ValueError(f"sharded CEM: right-hand sides must be finite (device error bits {bits:#x})")
        if bits:
            from .batch_qp import NumericalFailure
            raise NumericalFailure(f"sharded CEM: device error bits {bits:#x}")

    def rank_refit(self, resid, cost, P, mean, cov, n, q, w, eta, gamma):
        B = resid.shape[0]
        mean, cov = mean.clone(), cov.clone()
        # zero-filled: a failed iteration (device error word set) leaves them unwritten, and the loop
        # still indexes with elite 0 until check() raises after it
        el = torch.zeros(q, dtype=torch.int64, device=self.dev)
        ea = torch.zeros(q, dtype=torch.float64, device=self.dev)
        st = torch.zeros(6, dtype=torch.float64, device=self.dev)
        self.ctx.call("bd_rank_refit", 1, B, self.dim, resid, cost, P.contiguous(), n, q, float(w), float(eta),
                      float(gamma), mean, cov, None, el, ea, st)
        return {"mean": mean, "cov": cov, "elite_idx": el, "elite_aug": ea, "stats": st}


def plan_fleet_distributed(planner, scene_factory, n_scenes: int, seed: int = 0, group=None):
    """Config 5: each rank plans its contiguous block of global scene ids; the best records are
    all-gathered at the end (C4).  Returns the full FleetResult arrays on every rank."""
    rank, world = _world(group)
    lo, hi, shard = shard_range(n_scenes, rank, world)
    scenes = [scene_factory(g) for g in range(lo, hi)]
    res = planner.plan(scenes, seed=seed, scene_offset=lo)
    cols = np.concatenate([res.best_index[:, None].astype(np.float64), res.best_cost[:, None],
                           res.best_residual[:, None], res.best_aug[:, None], res.best_xi,
                           res.iterations_done[:, None].astype(np.float64)], axis=1)
    if world == 1:
        return cols
    dev = torch.device("cuda", torch.cuda.current_device()) if dist.get_backend(group) == "nccl" else torch.device("cpu")
    t = torch.full((shard, cols.shape[1]), float("nan"), dtype=torch.float64, device=dev)
    t[: cols.shape[0]] = torch.as_tensor(cols, device=dev)
    parts = [torch.empty_like(t) for _ in range(world)]
    dist.all_gather(parts, t, group=group)
    return torch.cat(parts)[:n_scenes].cpu().numpy()
