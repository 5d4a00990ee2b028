"""Batched AM projection onto the collision / kinematic constraint set — drop-in for
pkg/projection.py.  The whole alternating-minimisation loop runs in the persistent
sm_100a kernel K2 (csrc/am_kernel.cuh); this module owns the host setup (augmented
KKT assembled and factorized once, ``FACTORIZATION_COUNT`` + 1) and the result types.
"""

from __future__ import annotations

from dataclasses import dataclass, replace

import numpy as np

from ._native import Context, f64, ptr, upload_scenes
from .basis import PolynomialBasis, TrajectoryCoeffs
from .batch_qp import QPSolutionBatch, QPStructure, structure_from_matrices
from .constraints import ConstraintSpec, PlanningScene

__all__ = [
    "ProjectionConfig", "ProjectionState", "ProjectionReport", "ProjectionBatchResult", "ProjectionOperator",
    "polar_decompose", "clip_magnitudes", "project_batch",
]

_SIN_FLOOR = 1e-8
_KAPPA_FLOOR = 1e-12


@dataclass(frozen=True)
class ProjectionConfig:
    """rho, iteration budget, residual tolerance (pkg/projection.py:38-46)."""

    rho: float = 1.0
    max_iters: int = 100
    tol: float = 1e-3

    def __post_init__(self) -> None:
        if self.rho <= 0 or self.max_iters < 1 or self.tol <= 0:
            raise ValueError("need rho > 0, max_iters >= 1, tol > 0")


@dataclass(frozen=True)
class ProjectionState:
    alpha_o: np.ndarray
    d_o: np.ndarray
    alpha_v: np.ndarray
    d_v: np.ndarray
    alpha_a: np.ndarray
    d_a: np.ndarray
    s: np.ndarray
    lam: np.ndarray
    rho: float


@dataclass(frozen=True)
class ProjectionReport:
    coeffs: TrajectoryCoeffs
    residual: float
    residual_history: np.ndarray
    iterations_used: int


@dataclass(frozen=True)
class ProjectionBatchResult:
    """Column-wise outcome of a batch (pkg/projection.py:74-97)."""

    xi: np.ndarray
    residuals: np.ndarray
    residual_history: np.ndarray
    iterations_used: int
    clip_conflicts: int

    @property
    def batch_size(self) -> int:
        return self.xi.shape[1]

    def reports(self) -> list[ProjectionReport]:
        return [ProjectionReport(coeffs=TrajectoryCoeffs.from_stacked(self.xi[:, j]),
                                 residual=float(self.residuals[j]),
                                 residual_history=self.residual_history[:, j].copy(),
                                 iterations_used=self.iterations_used) for j in range(self.batch_size)]


def polar_decompose(xdot, ydot, xddot, yddot, x=None, y=None, obstacles_x=None, obstacles_y=None,
                    ellipse=(1.0, 1.0)):
    """Closed-form polar split (pkg/projection.py:100-135).  Array utility: on the device
    path the split is fused into K2 in its trig-free residual form."""
    av, dv = np.arctan2(ydot, xdot), np.hypot(xdot, ydot)
    aa, da = np.arctan2(yddot, xddot), np.hypot(xddot, yddot)
    ao = do = None
    if obstacles_x is not None:
        if x is None or y is None:
            raise ValueError("positions are required for the obstacle split")
        a, b = ellipse
        wc = np.expand_dims(x, -2) - obstacles_x
        ws = np.expand_dims(y, -2) - obstacles_y
        ao = np.arctan2(a * ws, b * wc)
        c, s = np.cos(ao), np.sin(ao)
        den = (a * c) ** 2 + (b * s) ** 2
        do = np.where(den > 0.0, (a * wc * c + b * ws * s) / np.where(den > 0.0, den, 1.0), 0.0)
    return ao, av, aa, do, dv, da


def _clip(av, dv_raw, aa, da_raw, do_raw, da_prev, kap, spec: ConstraintSpec):
    do = None if do_raw is None else np.maximum(do_raw, 1.0)
    gap = np.abs(np.sin(aa - av))
    lo = np.maximum(spec.v_min, np.sqrt(da_prev * gap / spec.kappa_max))
    cent = kap * np.cos(av) ** 2
    hi = np.minimum(spec.v_max, np.where(cent > _KAPPA_FLOOR, np.sqrt(spec.c_max / np.maximum(cent, _KAPPA_FLOOR)),
                                         spec.v_max))
    conflicts = int(np.count_nonzero(lo > hi))
    dv = np.clip(dv_raw, np.minimum(lo, hi), hi)
    da = np.clip(da_raw, 0.0, np.minimum(spec.a_max, dv**2 * spec.kappa_max / np.maximum(gap, _SIN_FLOOR)))
    return do, dv, da, conflicts


def clip_magnitudes(state: ProjectionState, spec: ConstraintSpec, kappa_abs=None) -> ProjectionState:
    """Coupled clip windows (pkg/projection.py:138-179); array utility (fused into K2 on the path)."""
    if kappa_abs is None:
        kappa_abs = np.zeros_like(state.d_v)
    d_o, d_v, d_a, _ = _clip(state.alpha_v, state.d_v, state.alpha_a, state.d_a, state.d_o, state.d_a, kappa_abs,
                             spec)
    return replace(state, d_o=d_o, d_v=d_v, d_a=d_a)


DEVICE_ORDER = 10          # the kernels' compile-time coefficient count is order + 1 = 11 (csrc/bd_common.cuh NC)


def require_device_order(basis: PolynomialBasis) -> None:
    """The device path is built for the BASELINE basis order (10, i.e. 11 coefficients per axis);
    the reference's build_basis accepts any order >= 2 (pkg/basis.py:156-179), so another order
    is refused here, before any factorization or device work, with a message that names the limit."""
    if basis.num_coeffs != DEVICE_ORDER + 1:
        raise NotImplementedError(
            f"the B200 path supports order-{DEVICE_ORDER} bases ({DEVICE_ORDER + 1} coefficients per axis, the "
            f"BASELINE configuration); got order {basis.num_coeffs - 1}.  The reference accepts any order >= 2 "
            "(pkg/basis.py:156-179): plan with order 10 or use the reference for other orders.")


class ProjectionOperator:
    """Reusable batched projector (pkg/projection.py:182-214): the augmented KKT is
    factorized once on the host and its inverse blocks live on the device."""

    def __init__(self, basis: PolynomialBasis, qp: QPStructure, num_obstacles: int,
                 config: ProjectionConfig = ProjectionConfig(), device: int = 0, context: Context | None = None):
        if num_obstacles < 0:
            raise ValueError("num_obstacles must be nonnegative")
        require_device_order(basis)
        self.basis = basis
        self.qp = qp
        self.num_obstacles = num_obstacles
        self.config = config
        W, Wd, Wdd = basis.W, basis.Wdot, basis.Wddot
        n = basis.num_coeffs
        WtW = W.T @ W
        Qx = np.eye(n) + config.rho * (num_obstacles * WtW + Wd.T @ Wd + Wdd.T @ Wdd)
        Q = np.zeros((2 * n, 2 * n))
        Q[:n, :n] = Qx
        Q[n:, n:] = Qx + config.rho * 2.0 * WtW
        self.aug = structure_from_matrices(Q, qp.A_eq)
        self._ctx = context if context is not None else Context(device)
        self._ctx.call("bd_set_basis", basis.num_samples, n, f64(W), f64(Wd), f64(Wdd))
        self._ctx.call("bd_set_projection", num_obstacles, float(config.rho), qp.num_eq, f64(self.aug.kkt_inv),
                       f64(qp.A_eq))
        self._scene_key = None

    # ------------------------------------------------------------------ scenes
    def _ensure_scene(self, scene: PlanningScene):
        sp = scene.spec
        key = (sp.obstacles_x.tobytes(), sp.obstacles_y.tobytes(), scene.initial_state.tobytes(),
               sp.ellipse_a, sp.ellipse_b, sp.v_min, sp.v_max, sp.a_max, sp.kappa_max, sp.c_max, sp.y_lb, sp.y_ub,
               None if sp.road_curvature is None else (np.asarray(sp.road_curvature[0], float).tobytes(),
                                                       np.asarray(sp.road_curvature[1], float).tobytes()))
        if key != self._scene_key:
            upload_scenes(self._ctx, [scene], self.basis.num_samples)
            self._scene_key = key

    def _check_spec(self, spec: ConstraintSpec):
        if spec.num_samples != self.basis.num_samples:
            raise ValueError("constraint spec and basis disagree on the time grid")
        if spec.num_obstacles != self.num_obstacles:
            raise ValueError(f"operator was built for {self.num_obstacles} obstacles, spec has {spec.num_obstacles}")

    def project(self, xi_bar: np.ndarray, b_batch: np.ndarray, spec: ConstraintSpec) -> ProjectionBatchResult:
        """Project a (2n, batch) coefficient block (pkg/projection.py:216-339) on the device."""
        n = self.basis.num_coeffs
        self._check_spec(spec)
        xi_bar = np.atleast_2d(np.asarray(xi_bar, dtype=float))
        if xi_bar.shape[0] != 2 * n:
            raise ValueError(f"xi_bar must stack 2*{n} coefficient rows")
        b_batch = np.atleast_2d(np.asarray(b_batch, dtype=float))
        B = xi_bar.shape[1]
        if b_batch.shape != (self.qp.num_eq, B):
            raise ValueError(f"b_batch must be ({self.qp.num_eq}, {B})")
        self._ensure_scene(PlanningScene(initial_state=b_batch[:6, 0], spec=spec))
        return self._run(f64(xi_bar.T), f64(b_batch.T), B)

    def _run(self, xi_bar_rows: np.ndarray, b_rows, B: int, cost=None) -> ProjectionBatchResult:
        cfg = self.config
        n2 = 2 * self.basis.num_coeffs
        xi = np.empty((B, n2))
        res = np.empty(B)
        hist = np.empty((cfg.max_iters, B), dtype=np.float32)
        used = np.zeros(1, dtype=np.int32)
        conf = np.zeros(1, dtype=np.int64)
        self._ctx.call("bd_project", 1, B, ptr(xi_bar_rows), ptr(b_rows), cfg.max_iters, float(cfg.tol), ptr(xi),
                       ptr(res), ptr(cost), ptr(hist), ptr(used), ptr(conf))
        k = int(used[0])
        return ProjectionBatchResult(xi=np.ascontiguousarray(xi.T), residuals=res,
                                     residual_history=hist[:k].astype(np.float64), iterations_used=k,
                                     clip_conflicts=int(conf[0]))


def project_batch(solution: QPSolutionBatch, spec: ConstraintSpec, qp: QPStructure, config: ProjectionConfig,
                  b_batch: np.ndarray) -> list[ProjectionReport]:
    """One-shot surface that factorizes anew (pkg/projection.py:342-353)."""
    if qp.basis is None:
        raise ValueError("qp structure lacks basis metadata; build it with build_qp_structure")
    return ProjectionOperator(qp.basis, qp, spec.num_obstacles, config).project(solution.xi, b_batch, spec).reports()
