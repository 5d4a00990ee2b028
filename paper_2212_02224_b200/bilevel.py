"""CEM upper level over the device lower level — drop-in for pkg/bilevel.py.

``LowerLevelSolver.solve`` runs stage-1 + AM projection + upper cost as one device
sequence (``bd_solve_lower``).  ``solve_bilevel`` runs the whole CEM cycle on the
device (``bd_cem_cycle``: sample -> stage-1 -> AM -> exit scan / replay ->
rank + refit per iteration, no host round trip); the Gaussian draws come from the
caller's numpy Generator exactly as in the reference, so a seeded call reproduces
the reference's samples.  With a ``trace_hook`` the loop is stepped from the host
(still all compute on the device) so the hook sees every iteration.

The array-level helpers (``upper_cost_batch``, ``rank_samples``, ``select_elites``,
``update_distribution``) keep the reference signatures for callers holding host
arrays; on the path their work is done by K3 (csrc/cem_kernels.cuh).
"""

from __future__ import annotations

import ctypes
import logging
import os
from dataclasses import dataclass, field

import numpy as np

from . import numpy_stream
from ._native import CemConfig, f64, ptr
from .basis import PolynomialBasis, TrajectoryCoeffs, eval_trajectory
from .batch_qp import NumericalFailure, QPSolutionBatch, TrackingWeights, build_qp_structure
from .behavior import BehaviorParams, DeviceWarmStart, ParamLayout, WarmStartSource
from .constraints import PlanningScene
from .projection import ProjectionBatchResult, ProjectionConfig, ProjectionOperator, require_device_order

__all__ = [
    "SamplingDistribution", "EliteRecord", "BiLevelConfig", "IterationStats", "BiLevelResult", "upper_cost",
    "upper_cost_batch", "rank_samples", "select_elites", "DegenerateWeights", "update_distribution",
    "LowerLevelSolver", "solve_bilevel", "evaluate_batch",
]

log = logging.getLogger(__name__)

# BD_HOST_DRAWS=1: draw the caller's normals on the host (numpy) instead of the device stream
_DEVICE_STREAM = os.environ.get("BD_HOST_DRAWS", "0") != "1"

_COV_REG = 1e-6


@dataclass(frozen=True)
class SamplingDistribution:
    """Gaussian over behaviour vectors (pkg/bilevel.py:34-57)."""

    mean: np.ndarray
    cov: np.ndarray

    def __post_init__(self) -> None:
        mean = np.asarray(self.mean, dtype=float)
        cov = np.asarray(self.cov, dtype=float)
        if cov.shape != (mean.shape[0], mean.shape[0]):
            raise ValueError(f"cov shape {cov.shape} does not match mean dim {mean.shape[0]}")
        if not (np.array_equal(cov, cov.T) or np.allclose(cov, cov.T)):   # exact symmetry: the common, fast case
            raise ValueError("covariance must be symmetric")
        object.__setattr__(self, "mean", mean)
        object.__setattr__(self, "cov", cov)

    def sample(self, n: int, rng: np.random.Generator) -> np.ndarray:
        try:
            L = np.linalg.cholesky(self.cov)
        except np.linalg.LinAlgError:
            L = np.linalg.cholesky(self.cov + 10 * _COV_REG * np.eye(self.cov.shape[0]))
        return self.mean[None, :] + rng.standard_normal((n, self.mean.shape[0])) @ L.T


@dataclass(frozen=True)
class EliteRecord:
    index: int
    params: BehaviorParams
    coeffs: TrajectoryCoeffs
    upper_cost: float
    residual: float
    augmented_cost: float


@dataclass(frozen=True)
class BiLevelConfig:
    """Alg. 1 knobs (pkg/bilevel.py:72-97)."""

    batch_size: int = 1000
    constraint_elites: int = 150
    elites: int = 50
    iterations: int = 5
    eta: float = 0.7
    gamma: float = 0.9
    residual_weight: float = 1.0
    init_mean: np.ndarray = field(default_factory=lambda: np.zeros(8))
    init_cov: np.ndarray = field(default_factory=lambda: np.eye(8))

    def __post_init__(self) -> None:
        if not (self.elites <= self.constraint_elites <= self.batch_size):
            raise ValueError(f"need elites <= constraint_elites <= batch_size, got "
                             f"{self.elites} / {self.constraint_elites} / {self.batch_size}")
        if not (0.0 < self.eta <= 1.0):
            raise ValueError(f"eta must lie in (0, 1], got {self.eta}")
        if self.gamma <= 0:
            raise ValueError(f"gamma must be positive, got {self.gamma}")
        if self.iterations < 1:
            raise ValueError("need at least one iteration")
        object.__setattr__(self, "init_mean", np.asarray(self.init_mean, dtype=float))
        object.__setattr__(self, "init_cov", np.asarray(self.init_cov, dtype=float))


@dataclass(frozen=True)
class IterationStats:
    iteration: int
    elite_mean_upper_cost: float
    best_augmented_cost: float
    cov_trace: float
    residual_min: float
    residual_median: float
    residual_max: float


@dataclass(frozen=True)
class BiLevelResult:
    best: EliteRecord
    diagnostics: list[IterationStats]
    distribution: SamplingDistribution
    degraded: bool = False


# ----------------------------------------------------------------------------- array helpers
def upper_cost(coeffs: TrajectoryCoeffs, basis: PolynomialBasis, v_max: float) -> float:
    """sum_t (|v| - v_max)^2 of one trajectory (pkg/bilevel.py:119-122)."""
    return float(((eval_trajectory(basis, coeffs).speed() - v_max) ** 2).sum())


def upper_cost_batch(xdot: np.ndarray, ydot: np.ndarray, v_max: float) -> np.ndarray:
    """(pkg/bilevel.py:125-126); on the path the cost is fused into K2's last sweep."""
    return ((np.hypot(xdot, ydot) - v_max) ** 2).sum(axis=-1)


def rank_samples(residuals: np.ndarray, costs: np.ndarray, n: int, q: int, residual_weight: float):
    """Constraint-elite then elite sets, ties by index (pkg/bilevel.py:129-137)."""
    cons_idx = np.argsort(residuals, kind="stable")[:n]
    aug = costs[cons_idx] + residual_weight * residuals[cons_idx]
    sub = np.lexsort((cons_idx, aug))[:q]
    return cons_idx, cons_idx[sub], aug[sub]


def select_elites(records: list[EliteRecord], n: int, q: int):
    """Record-level variant (pkg/bilevel.py:140-156)."""
    if n > len(records) or q > n:
        raise ValueError(f"need q <= n <= len(records), got {q} / {n} / {len(records)}")
    res = np.array([r.residual for r in records])
    aug = np.array([r.augmented_cost for r in records])
    idx = np.array([r.index for r in records])
    order = np.lexsort((idx, res))[:n]
    cons = [records[i] for i in order]
    sub = np.lexsort((idx[order], aug[order]))[:q]
    return cons, [cons[i] for i in sub]


class DegenerateWeights(RuntimeError):
    """All elite weights underflowed (pkg/bilevel.py:159-160)."""


def _elite_weights(aug_costs: np.ndarray, gamma: float) -> np.ndarray:
    w = np.exp(-(aug_costs - aug_costs.min()) / gamma)
    total = w.sum()
    if not np.isfinite(total) or total <= 0.0:
        log.warning("elite weights degenerated; falling back to uniform")
        return np.full_like(aug_costs, 1.0 / aug_costs.shape[0])
    return w / total


def update_distribution(dist: SamplingDistribution, elite_params: np.ndarray, elite_aug_costs: np.ndarray,
                        eta: float, gamma: float) -> SamplingDistribution:
    """Exponentiated-cost refit (pkg/bilevel.py:175-194)."""
    P = np.atleast_2d(np.asarray(elite_params, dtype=float))
    w = _elite_weights(np.asarray(elite_aug_costs, dtype=float), gamma)
    mean = (1.0 - eta) * dist.mean + eta * (w @ P)
    D = P - mean[None, :]
    cov = (1.0 - eta) * dist.cov + eta * (D.T @ (w[:, None] * D)) + _COV_REG * np.eye(dist.mean.shape[0])
    return SamplingDistribution(mean=mean, cov=0.5 * (cov + cov.T))


# ----------------------------------------------------------------------------- lower level
class LowerLevelSolver:
    """Factorized QP + projection operators bound to one device context (pkg/bilevel.py:197-225)."""

    def __init__(self, basis: PolynomialBasis, weights: TrackingWeights, layout: ParamLayout,
                 proj_config: ProjectionConfig, num_obstacles: int, device: int = 0):
        require_device_order(basis)
        self.basis = basis
        self.layout = layout
        self.qp = build_qp_structure(basis, weights, layout)
        self.projector = ProjectionOperator(basis, self.qp, num_obstacles, proj_config, device=device)
        self._ctx = self.projector._ctx
        qp = self.qp
        self._ctx.call("bd_set_stage1", layout.m_seg, int(layout.with_goal), qp.num_eq, f64(qp.q_map_x),
                       f64(qp.q_map_y), f64(qp.kkt), f64(qp.kkt_inv))
        self.last_costs: np.ndarray | None = None

    @property
    def context(self):
        return self._ctx

    def _params(self, param_batch) -> np.ndarray:
        P = f64(np.atleast_2d(np.asarray(param_batch, dtype=float)))
        if P.shape[1] != self.layout.dim:
            raise ValueError(f"behavior vectors have dim {P.shape[1]}, layout wants {self.layout.dim}")
        if not np.isfinite(P).all():
            raise ValueError("right-hand sides must be finite")
        return P

    def solve(self, param_batch: np.ndarray, scene: PlanningScene) -> tuple[QPSolutionBatch, ProjectionBatchResult]:
        """Stage-1 + projection (+ upper cost, kept in ``last_costs``) on the device."""
        P = self._params(param_batch)
        self.projector._check_spec(scene.spec)
        self.projector._ensure_scene(scene)
        B = P.shape[0]
        cfg = self.projector.config
        n2, neq = 2 * self.basis.num_coeffs, self.qp.num_eq
        xb = np.empty((B, n2))
        mu = np.empty((B, neq))
        xi = np.empty((B, n2))
        res = np.empty(B)
        cost = np.empty(B)
        hist = np.empty((cfg.max_iters, B), dtype=np.float32)
        used = np.zeros(1, dtype=np.int32)
        conf = np.zeros(1, dtype=np.int64)
        self._ctx.call("bd_solve_lower", 1, B, ptr(P), cfg.max_iters, float(cfg.tol), ptr(xb), ptr(mu), ptr(xi),
                       ptr(res), ptr(cost), ptr(hist), ptr(used), ptr(conf))
        self.last_costs = cost
        k = int(used[0])
        sol = QPSolutionBatch(xi=np.ascontiguousarray(xb.T), mu=np.ascontiguousarray(mu.T))
        proj = ProjectionBatchResult(xi=np.ascontiguousarray(xi.T), residuals=res,
                                     residual_history=hist[:k].astype(np.float64), iterations_used=k,
                                     clip_conflicts=int(conf[0]))
        return sol, proj

    def velocities(self, xi: np.ndarray) -> tuple[np.ndarray, np.ndarray]:
        """(xdot, ydot), each (B, m), evaluated on the device (pkg/bilevel.py:223-225)."""
        X = f64(np.atleast_2d(np.asarray(xi, dtype=float)).T)
        B, m = X.shape[0], self.basis.num_samples
        xd = np.empty((B, m))
        yd = np.empty((B, m))
        self._ctx.call("bd_eval", B, ptr(X), None, None, ptr(xd), ptr(yd), None, None)
        return xd, yd


def evaluate_batch(solver: LowerLevelSolver, scene: PlanningScene, params: np.ndarray, constraint_elites: int,
                   elites: int, residual_weight: float = 1.0) -> tuple[EliteRecord, dict]:
    """One lower-level sweep over a set-point batch and its best record by augmented cost —
    the baseline planners' path (BasePlanner.evaluate_batch, pkg/planners.py:233-258: Random,
    Grid, Vanilla and the goal-layout planner) on the same device kernels (solve + K3 ranking)."""
    P = solver._params(params)
    _, proj = solver.solve(P, scene)
    costs = solver.last_costs
    B = P.shape[0]
    n = min(constraint_elites, B)
    q = min(elites, n)
    dim = solver.layout.dim
    el = np.empty(q, np.int64)
    ea = np.empty(q)
    mean, cov = np.zeros(dim), np.eye(dim)       # the refit K3 also performs is discarded here
    solver.context.call("bd_rank_refit", 1, B, dim, f64(proj.residuals), f64(costs), P, n, q,
                        float(residual_weight), 0.5, 1.0, mean, cov, None, el, ea, None)
    j = int(el[0])
    record = EliteRecord(index=j, params=BehaviorParams.from_vector(P[j], solver.layout),
                         coeffs=TrajectoryCoeffs.from_stacked(proj.xi[:, j]), upper_cost=float(costs[j]),
                         residual=float(proj.residuals[j]), augmented_cost=float(ea[0]))
    diag = {"residual": record.residual, "upper_cost": record.upper_cost, "proj_iterations": proj.iterations_used,
            "batch": int(B)}
    return record, diag


# ----------------------------------------------------------------------------- upper level
def _stats(it: int, row) -> IterationStats:
    return IterationStats(iteration=it, elite_mean_upper_cost=float(row[0]), best_augmented_cost=float(row[1]),
                          cov_trace=float(row[2]), residual_min=float(row[3]), residual_median=float(row[4]),
                          residual_max=float(row[5]))


def solve_bilevel(scene: PlanningScene, solver: LowerLevelSolver, config: BiLevelConfig, rng: np.random.Generator,
                  warm_start: WarmStartSource | None = None, trace_hook=None) -> BiLevelResult:
    """Alg. 1 (pkg/bilevel.py:228-295) on the device.

    Returns the elite record with the lowest augmented cost at the last completed
    iteration; a numerical failure after iteration 1 returns the best so far with
    ``degraded=True``, a failure in iteration 1 raises NumericalFailure.
    """
    if trace_hook is not None:
        return _solve_bilevel_stepped(scene, solver, config, rng, warm_start, trace_hook)
    layout = solver.layout
    dim, B, N = layout.dim, config.batch_size, config.iterations
    solver.projector._check_spec(scene.spec)
    solver.projector._ensure_scene(scene)
    pcfg = solver.projector.config
    state0 = rng.bit_generator.state
    # device-resident rows (CVAE decoder, same context) go to the cycle in place
    warm_dev = warm_start.device_rows(solver.context, B) if isinstance(warm_start, DeviceWarmStart) else None
    warm = f64(warm_start.draw(B)) if warm_start is not None and warm_dev is None else None
    warm_arg = ctypes.c_void_p(warm_dev) if warm_dev is not None else ptr(warm)
    n_draw = N - (1 if warm_start is not None else 0)
    # every small input / output of the call in one fresh float64 block: one pointer conversion
    # instead of fifteen (each costs ~1-2 us of host time in front of a ~0.9 ms cycle)
    nx = 2 * solver.basis.num_coeffs
    sizes = (("bi", 1), ("bp", dim), ("bx", nx), ("bc", 1), ("br", 1), ("ba", 1), ("st", N * 6), ("fm", dim),
             ("fc", dim * dim), ("done", 1), ("pos", n_draw + 1), ("words", 4), ("mean0", dim), ("cov0", dim * dim))
    blk = np.zeros(sum(n for _, n in sizes))
    base = blk.ctypes.data
    off, at = {}, 0
    for name, n in sizes:
        off[name] = at
        at += n

    def view(name, n, shape=None):
        v = blk[off[name]:off[name] + n]
        return v if shape is None else v.reshape(shape)

    def addr(name):
        return base + 8 * off[name]

    bi = view("bi", 1).view(np.int64)
    bp, bx = view("bp", dim), view("bx", nx)
    bc, br, ba = view("bc", 1), view("br", 1), view("ba", 1)
    st, fm, fc = view("st", N * 6, (N, 6)), view("fm", dim), view("fc", dim * dim, (dim, dim))
    done = view("done", 1).view(np.int32)
    view("mean0", dim)[:] = np.asarray(config.init_mean, dtype=np.float64).reshape(-1)
    view("cov0", dim * dim)[:] = np.asarray(config.init_cov, dtype=np.float64).reshape(-1)
    mean0, cov0 = addr("mean0"), addr("cov0")
    outs = (addr("bi"), addr("bp"), addr("bx"), addr("bc"), addr("br"), addr("ba"), addr("st"), addr("fm"),
            addr("fc"), addr("done"))

    def cfg_range(a, b):
        return CemConfig(B, config.constraint_elites, config.elites, N, pcfg.max_iters, config.eta, config.gamma,
                         config.residual_weight, pcfg.tol, 0, 0, a, b)

    # numpy stream mode: the caller's PCG64 normals are generated on the device (identical values,
    # csrc/numpy_normals.cuh) and the generator is advanced by the raw outputs they consumed; one
    # call runs the whole cycle.  Other bit generators draw on the host below.
    st_words = numpy_stream.pcg64_state_words(rng.bit_generator, state0) if _DEVICE_STREAM else None
    if st_words is not None and numpy_stream.ensure_device_tables(solver.context):
        pos = view("pos", n_draw + 1).view(np.int64)
        view("words", 4).view(np.uint64)[:] = st_words
        cfg = cfg_range(0, N)
        cfg.pcg64_state = addr("words")
        cfg.pcg64_positions = addr("pos")
        try:
            solver.context.call("bd_cem_cycle", 1, ctypes.byref(cfg), mean0, cov0, None, warm_arg, *outs)
        except RuntimeError as e:
            if "numpy normal stream" not in str(e):
                raise
            st_words = None          # a draw needed more raw values than evaluated: draw on the host
        else:
            k = int(done[0])
            attempted = N if k >= N else (1 if k <= 0 else k + 1)
            consumed = attempted - (1 if warm_start is not None else 0)
            if consumed > 0:
                # PCG64.advance drops a buffered 32-bit half; standard_normal never touches it
                buf = rng.bit_generator.state
                rng.bit_generator.advance(int(pos[consumed]))
                if buf.get("has_uint32"):
                    st_now = rng.bit_generator.state
                    st_now["has_uint32"], st_now["uinteger"] = buf["has_uint32"], buf["uinteger"]
                    rng.bit_generator.state = st_now
            return _finish(k, N, layout, bi, bp, bx, bc, br, ba, st, fm, fc, _all_finite(blk[off["bp"]:off["done"]]))

    # Iteration 1 is launched as soon as its draws exist; the remaining N-1 batches of the caller's
    # Generator are drawn while the GPU runs it (the stream is the same sequence as one
    # standard_normal((N, B, dim)) call), then iterations 2..N follow in a second call.
    z1 = None if warm_start is not None else rng.standard_normal((1, B, dim))
    if N == 1:
        solver.context.call("bd_cem_cycle", 1, ctypes.byref(cfg_range(0, 1)), mean0, cov0, ptr(z1), warm_arg, *outs)
    else:
        solver.context.call("bd_cem_cycle", 1, ctypes.byref(cfg_range(0, 1)), mean0, cov0, ptr(z1), warm_arg,
                            None, None, None, None, None, None, None, None, None, None)
        z = rng.standard_normal((N - 1, B, dim))
        solver.context.call("bd_cem_cycle", 1, ctypes.byref(cfg_range(1, N)), mean0, cov0, ptr(z), None, *outs)
    k = int(done[0])
    attempted = N if k >= N else (1 if k <= 0 else k + 1)
    consumed = attempted - (1 if warm_start is not None else 0)
    if consumed != n_draw:   # leave the caller's generator exactly where the reference would
        rng.bit_generator.state = state0
        if consumed > 0:
            rng.standard_normal((consumed, B, dim))
    return _finish(k, N, layout, bi, bp, bx, bc, br, ba, st, fm, fc, _all_finite(blk[off["bp"]:off["done"]]))


def _all_finite(vals) -> bool:
    return bool(np.isfinite(vals).all())


def _frozen(cls, **fields):
    """A frozen dataclass instance without __post_init__ (its checks already hold, see _finish)."""
    obj = object.__new__(cls)
    for name, value in fields.items():
        object.__setattr__(obj, name, value)
    return obj


def _finish(k, N, layout, bi, bp, bx, bc, br, ba, st, fm, fc, checked=False) -> BiLevelResult:
    """The result records of a device cycle.  checked=True: the caller verified every output is
    finite (the device writes the covariance exactly symmetric), so the records' own validation
    would pass and is skipped (~15 us of host time per cycle); otherwise the validating
    constructors run and raise as usual."""
    if k <= 0:
        raise NumericalFailure("bilevel iteration 1 failed: non-finite projection iterate or KKT residual")
    if k < N:
        log.warning("bilevel iteration %d failed; returning best-so-far", k + 1)
    diagnostics = [IterationStats(i + 1, *row) for i, row in enumerate(st[:k].tolist())]
    if checked and not layout.with_goal:
        lat, lon, _ = layout.columns()
        half = bx.shape[0] // 2
        best = EliteRecord(index=int(bi[0]), params=_frozen(BehaviorParams, y_d=bp[lat], v_d=bp[lon], goal=None),
                           coeffs=_frozen(TrajectoryCoeffs, cx=bx[:half], cy=bx[half:]), upper_cost=float(bc[0]),
                           residual=float(br[0]), augmented_cost=float(ba[0]))
        return BiLevelResult(best=best, diagnostics=diagnostics, distribution=_frozen(SamplingDistribution, mean=fm,
                                                                                     cov=fc), degraded=k < N)
    best = EliteRecord(index=int(bi[0]), params=BehaviorParams.from_vector(bp, layout),
                       coeffs=TrajectoryCoeffs.from_stacked(bx), upper_cost=float(bc[0]), residual=float(br[0]),
                       augmented_cost=float(ba[0]))
    return BiLevelResult(best=best, diagnostics=diagnostics, distribution=SamplingDistribution(fm, fc), degraded=k < N)


def _solve_bilevel_stepped(scene, solver, config, rng, warm_start, trace_hook) -> BiLevelResult:
    ctx = solver.context
    layout = solver.layout
    dim, B = layout.dim, config.batch_size
    mean, cov = f64(config.init_mean), f64(config.init_cov)
    SamplingDistribution(mean, cov)
    best = None
    diagnostics: list[IterationStats] = []
    degraded = False
    for it in range(1, config.iterations + 1):
        if it == 1 and warm_start is not None:
            params = f64(warm_start.draw(B))
        else:
            z = f64(rng.standard_normal((B, dim)))
            params = np.empty((B, dim))
            ctx.call("bd_sample", dim, B, ptr(mean), ptr(cov), ptr(z), ptr(params))
        try:
            _, proj = solver.solve(params, scene)
        except NumericalFailure:
            if best is None:
                raise
            log.warning("bilevel iteration %d failed; returning best-so-far", it)
            degraded = True
            break
        costs = solver.last_costs
        n, q = config.constraint_elites, config.elites
        cons = np.empty(n, dtype=np.int64)
        elite = np.empty(q, dtype=np.int64)
        eaug = np.empty(q)
        st = np.empty(6)
        mean, cov = mean.copy(), cov.copy()
        ctx.call("bd_rank_refit", 1, B, dim, f64(proj.residuals), f64(costs), ptr(params), n, q,
                 float(config.residual_weight), float(config.eta), float(config.gamma), ptr(mean), ptr(cov),
                 ptr(cons), ptr(elite), ptr(eaug), ptr(st))
        trace_hook(it, params, proj, costs, elite)
        j = int(elite[0])
        best = EliteRecord(index=j, params=BehaviorParams.from_vector(params[j], layout),
                           coeffs=TrajectoryCoeffs.from_stacked(proj.xi[:, j]), upper_cost=float(costs[j]),
                           residual=float(proj.residuals[j]), augmented_cost=float(eaug[0]))
        diagnostics.append(_stats(it, st))
    assert best is not None
    return BiLevelResult(best=best, diagnostics=diagnostics, distribution=SamplingDistribution(mean, cov),
                         degraded=degraded)
