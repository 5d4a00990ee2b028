"""Sampled trajectory bases (host setup, float64) — drop-in for pkg/basis.py.

The basis is built once per solver on the host and uploaded to the device
(``bd_set_basis``); its rows feed every forward evaluation and back-projection
of the AM kernel.  Batch trajectory evaluation runs on the device
(:meth:`LowerLevelSolver.velocities`, ``bd_eval``); the single-trajectory helpers
below are convenience utilities off the hot path.
"""

from __future__ import annotations

import math
from dataclasses import dataclass

import numpy as np

__all__ = [
    "SpeedSingularity", "PolynomialBasis", "TrajectoryCoeffs", "TrajectorySamples", "FlatControls",
    "build_basis", "eval_trajectory", "curvature_from_derivatives", "flat_to_controls",
]


class SpeedSingularity(ValueError):
    """The flatness map hit a near-zero speed sample (pkg/basis.py:21-22)."""


def _bernstein(deg: int, tau: np.ndarray) -> np.ndarray:
    k = np.arange(deg + 1)
    binom = np.array([math.comb(deg, int(j)) for j in k], dtype=float)
    return binom[None, :] * tau[:, None] ** k[None, :] * (1.0 - tau[:, None]) ** (deg - k)[None, :]


def _bernstein_family(order: int, times: np.ndarray, horizon: float):
    """Bernstein rows and their time derivatives by degree elevation of the
    (order-1)/(order-2) bases (pkg/basis.py:127-150)."""
    tau = np.asarray(times, float) / horizon
    N = order
    W = _bernstein(N, tau)
    d1 = _bernstein(N - 1, tau)
    Wd = np.zeros_like(W)
    Wd[:, 1:] += d1
    Wd[:, :-1] -= d1
    Wd *= N / horizon
    d2 = _bernstein(N - 2, tau)
    Wdd = np.zeros_like(W)
    Wdd[:, 2:] += d2
    Wdd[:, 1:-1] -= 2.0 * d2
    Wdd[:, :-2] += d2
    Wdd *= N * (N - 1) / horizon**2
    return W, Wd, Wdd


def _monomial_family(order: int, times: np.ndarray, horizon: float):
    """Monomials in tau = t/T and their chain-rule derivatives (pkg/basis.py:112-124)."""
    tau = np.asarray(times, float) / horizon
    k = np.arange(order + 1)
    W = tau[:, None] ** k[None, :]
    Wd = np.zeros_like(W)
    Wdd = np.zeros_like(W)
    Wd[:, 1:] = k[1:] * tau[:, None] ** (k[1:] - 1) / horizon
    Wdd[:, 2:] = k[2:] * (k[2:] - 1) * tau[:, None] ** (k[2:] - 2) / horizon**2
    return W, Wd, Wdd


_FAMILIES = {"monomial": _monomial_family, "bernstein": _bernstein_family}


@dataclass(frozen=True)
class PolynomialBasis:
    """Basis matrices for one horizon (pkg/basis.py:25-56)."""

    order: int
    horizon: float
    times: np.ndarray
    W: np.ndarray
    Wdot: np.ndarray
    Wddot: np.ndarray
    family: str = "monomial"

    @property
    def num_samples(self) -> int:
        return self.times.shape[0]

    @property
    def num_coeffs(self) -> int:
        return self.order + 1

    def matrices_at(self, times: np.ndarray):
        return _FAMILIES[self.family](self.order, np.asarray(times, dtype=float), self.horizon)


@dataclass(frozen=True)
class TrajectoryCoeffs:
    """(c_x, c_y) of one trajectory (pkg/basis.py:59-83)."""

    cx: np.ndarray
    cy: np.ndarray

    def __post_init__(self) -> None:
        cx = np.asarray(self.cx, dtype=float)
        cy = np.asarray(self.cy, dtype=float)
        if cx.shape != cy.shape or cx.ndim != 1:
            raise ValueError(f"coefficient vectors must share one shape, got {cx.shape} / {cy.shape}")
        if not (np.isfinite(cx).all() and np.isfinite(cy).all()):
            raise ValueError("coefficients must be finite")
        object.__setattr__(self, "cx", cx)
        object.__setattr__(self, "cy", cy)

    def stacked(self) -> np.ndarray:
        return np.concatenate([self.cx, self.cy])

    @staticmethod
    def from_stacked(xi: np.ndarray) -> "TrajectoryCoeffs":
        xi = np.asarray(xi, dtype=float)
        half = xi.shape[0] // 2
        return TrajectoryCoeffs(cx=xi[:half], cy=xi[half:])


@dataclass(frozen=True)
class TrajectorySamples:
    x: np.ndarray
    y: np.ndarray
    xdot: np.ndarray
    ydot: np.ndarray
    xddot: np.ndarray
    yddot: np.ndarray

    def speed(self) -> np.ndarray:
        return np.hypot(self.xdot, self.ydot)


@dataclass(frozen=True)
class FlatControls:
    v: np.ndarray
    delta: np.ndarray
    accel: np.ndarray
    psi: np.ndarray
    kappa: np.ndarray


def _basis_problems(order: int, num_samples: int, horizon: float, family: str) -> list[str]:
    checks = [
        (order >= 2, f"polynomial order {order} is below the minimum of 2"),
        (horizon > 0, f"horizon {horizon} must be positive"),
        (num_samples >= order + 1, f"{num_samples} grid points cannot determine an order-{order} polynomial "
                                   f"(at least {order + 1} needed)"),
        (family in _FAMILIES, f"basis family {family!r} is not one of {sorted(_FAMILIES)}"),
    ]
    return [msg for ok, msg in checks if not ok]


def build_basis(order: int, num_samples: int, horizon: float, family: str = "monomial") -> PolynomialBasis:
    """Basis rows on the uniform grid linspace(0, horizon, num_samples); raises ValueError on an
    order below 2, a non-positive horizon, an under-sampled grid or an unknown family."""
    problems = _basis_problems(order, num_samples, horizon, family)
    if problems:
        raise ValueError(problems[0])
    grid = np.linspace(0.0, horizon, num_samples)
    rows = _FAMILIES[family](order, grid, horizon)
    return PolynomialBasis(order, float(horizon), grid, *rows, family=family)


def eval_trajectory(basis: PolynomialBasis, coeffs: TrajectoryCoeffs) -> TrajectorySamples:
    """Position, velocity and acceleration of one trajectory on the basis grid (host fp64; the
    batched form is ``bd_eval`` behind LowerLevelSolver.velocities)."""
    n = basis.num_coeffs
    if coeffs.cx.shape[0] != n:
        raise ValueError(f"{coeffs.cx.shape[0]} coefficients per axis for a basis of {n} functions")
    stack = np.stack([basis.W, basis.Wdot, basis.Wddot])          # (3, m, n)
    ex, ey = stack @ coeffs.cx, stack @ coeffs.cy
    return TrajectorySamples(ex[0], ey[0], ex[1], ey[1], ex[2], ey[2])


def curvature_from_derivatives(xdot, ydot, xddot, yddot) -> np.ndarray:
    """(yddot xdot - xddot ydot) / |v|^3 (pkg/basis.py:198-203)."""
    v = np.hypot(xdot, ydot)
    return (yddot * xdot - xddot * ydot) / v**3


def flat_to_controls(basis: PolynomialBasis, coeffs: TrajectoryCoeffs, wheelbase: float, eps_v: float = 1e-3,
                     times: np.ndarray | None = None) -> FlatControls:
    """Kinematic-bicycle controls implied by the flat outputs (speed, steering, longitudinal
    acceleration, heading, path curvature), on the basis grid or at `times`; SpeedSingularity
    when the speed reaches eps_v anywhere.  Batched on the device: ``bd_controls``."""
    if times is None:
        smp = eval_trajectory(basis, coeffs)
        d1 = (smp.xdot, smp.ydot)
        d2 = (smp.xddot, smp.yddot)
    else:
        _, Wd, Wdd = basis.matrices_at(times)
        d1 = (Wd @ coeffs.cx, Wd @ coeffs.cy)
        d2 = (Wdd @ coeffs.cx, Wdd @ coeffs.cy)
    speed = np.hypot(*d1)
    if (speed <= eps_v).any():
        raise SpeedSingularity(f"speed reaches {speed.min():.3g} m/s, at or below the floor {eps_v:g}")
    path_kappa = (d2[1] * d1[0] - d2[0] * d1[1]) / speed ** 3
    return FlatControls(v=speed, delta=np.arctan(path_kappa * wheelbase),
                        accel=(d1[0] * d2[0] + d1[1] * d2[1]) / speed, psi=np.arctan2(d1[1], d1[0]),
                        kappa=path_kappa)
