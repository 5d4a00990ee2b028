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


def build_basis(order: int, num_samples: int, horizon: float, family: str = "monomial") -> PolynomialBasis:
    """Uniform-grid basis on [0, horizon] (pkg/basis.py:156-179); same validation."""
    if order < 2:
        raise ValueError(f"order must be >= 2, got {order}")
    if horizon <= 0:
        raise ValueError(f"horizon must be positive, got {horizon}")
    if num_samples < order + 1:
        raise ValueError(f"num_samples={num_samples} undersamples an order-{order} polynomial "
                         f"(need at least {order + 1})")
    if family not in _FAMILIES:
        raise ValueError(f"unknown basis family {family!r}; choose from {sorted(_FAMILIES)}")
    times = np.linspace(0.0, horizon, num_samples)
    W, Wd, Wdd = _FAMILIES[family](order, times, horizon)
    return PolynomialBasis(order=order, horizon=float(horizon), times=times, W=W, Wdot=Wd, Wddot=Wdd, family=family)


def eval_trajectory(basis: PolynomialBasis, coeffs: TrajectoryCoeffs) -> TrajectorySamples:
    """One trajectory on the grid (pkg/basis.py:182-195); batches go through bd_eval."""
    if coeffs.cx.shape[0] != basis.num_coeffs:
        raise ValueError(f"coefficient length {coeffs.cx.shape[0]} does not match basis with "
                         f"{basis.num_coeffs} columns")
    M = np.stack([basis.W, basis.Wdot, basis.Wddot])
    px, py = M @ coeffs.cx, M @ coeffs.cy
    return TrajectorySamples(x=px[0], y=py[0], xdot=px[1], ydot=py[1], xddot=px[2], yddot=py[2])


def curvature_from_derivatives(xdot, ydot, xddot, yddot) -> np.ndarray:
    """(yddot xdot - xddot ydot) / |v|^3 (pkg/basis.py:198-203)."""
    v = np.hypot(xdot, ydot)
    return (yddot * xdot - xddot * ydot) / v**3


def flat_to_controls(basis: PolynomialBasis, coeffs: TrajectoryCoeffs, wheelbase: float, eps_v: float = 1e-3,
                     times: np.ndarray | None = None) -> FlatControls:
    """Bicycle controls from the flat outputs (pkg/basis.py:206-234)."""
    if times is None:
        s = eval_trajectory(basis, coeffs)
        xd, yd, xdd, ydd = s.xdot, s.ydot, s.xddot, s.yddot
    else:
        _, Wd, Wdd = basis.matrices_at(times)
        xd, yd, xdd, ydd = Wd @ coeffs.cx, Wd @ coeffs.cy, Wdd @ coeffs.cx, Wdd @ coeffs.cy
    v = np.hypot(xd, yd)
    if np.any(v <= eps_v):
        raise SpeedSingularity(f"speed drops to {v.min():.3g} m/s (floor {eps_v:g})")
    kappa = (ydd * xd - xdd * yd) / v**3
    return FlatControls(v=v, delta=np.arctan(kappa * wheelbase), accel=(xd * xdd + yd * ydd) / v,
                        psi=np.arctan2(yd, xd), kappa=kappa)
