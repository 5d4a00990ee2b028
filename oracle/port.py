"""Float64 numpy restatement of the reference hot path (oracle; tests/bench only).

Each function names the reference lines it restates
(`pkg/` = /root/reference/pkg/src/bilevel_drive/).  The restatement keeps the
reference's arithmetic (trigonometric polar split, LU solves, the direct
violation evaluator) so that it agrees with the reference to rounding; the
agreement is pinned by tests/test_oracle_golden.py against vectors produced by
the reference itself (tools/gen_golden.py).
"""

from __future__ import annotations

import math
from dataclasses import dataclass, field

import numpy as np
from scipy.linalg import lu_factor, lu_solve

__all__ = [
    "bernstein_rows", "basis_matrices", "segment_onehot", "QPData", "tracking_qp",
    "stage1", "aug_qp", "Limits", "kappa_lookup", "violation_terms", "residual_sum",
    "polar_split", "coupled_clip", "am_project", "speed_cost", "rank_two_stage",
    "softmin_weights", "refit_gaussian", "draw_gaussian", "cem_cycle", "CemTrace",
]

SIN_FLOOR = 1e-8       # pkg/projection.py:34
KAPPA_FLOOR = 1e-12    # pkg/projection.py:35
SPEED_EPS = 1e-6       # pkg/constraints.py:16
COV_REG = 1e-6         # pkg/bilevel.py:31


# --------------------------------------------------------------------------- basis
def bernstein_rows(degree: int, tau: np.ndarray) -> np.ndarray:
    """B_{k,N}(tau) columns k = 0..N (pkg/basis.py:127-133)."""
    out = np.empty((tau.shape[0], degree + 1))
    for k in range(degree + 1):
        out[:, k] = math.comb(degree, k) * tau**k * (1.0 - tau) ** (degree - k)
    return out


def basis_matrices(order: int, m: int, horizon: float, family: str = "bernstein"):
    """(times, W, Wd, Wdd) on np.linspace(0, T, m) (pkg/basis.py:112-150,156-179)."""
    times = np.linspace(0.0, horizon, m)
    tau = times / horizon
    if family == "monomial":
        W = np.empty((m, order + 1))
        Wd = np.zeros((m, order + 1))
        Wdd = np.zeros((m, order + 1))
        for k in range(order + 1):
            W[:, k] = tau**k
            if k >= 1:
                Wd[:, k] = k * tau ** (k - 1) / horizon
            if k >= 2:
                Wdd[:, k] = k * (k - 1) * tau ** (k - 2) / horizon**2
        return times, W, Wd, Wdd
    N = order
    W = bernstein_rows(N, tau)
    z = np.zeros((m, 1))
    r1 = bernstein_rows(N - 1, tau)
    Wd = N * (np.hstack([z, r1]) - np.hstack([r1, z])) / horizon
    r2 = bernstein_rows(N - 2, tau)
    Wdd = N * (N - 1) * (np.hstack([z, z, r2]) - 2 * np.hstack([z, r2, z]) + np.hstack([r2, z, z])) / horizon**2
    return times, W, Wd, Wdd


def segment_onehot(m: int, m_seg: int) -> np.ndarray:
    """One-hot (m, m_seg) map over np.array_split segments (pkg/behavior.py:81-93)."""
    S = np.zeros((m, m_seg))
    for j, idx in enumerate(np.array_split(np.arange(m), m_seg)):
        S[idx, j] = 1.0
    return S


# --------------------------------------------------------------------------- stage-1 QP
@dataclass
class QPData:
    Q: np.ndarray
    A_eq: np.ndarray
    kkt: np.ndarray
    lu: tuple
    qmx: np.ndarray | None = None
    qmy: np.ndarray | None = None
    m_seg: int = 0
    with_goal: bool = False


def _bordered(Q, A):
    """Bordered KKT + LU (pkg/batch_qp.py:125-141)."""
    n, ne = Q.shape[0], A.shape[0]
    K = np.zeros((n + ne, n + ne))
    K[:n, :n] = Q
    K[:n, n:] = A.T
    K[n:, :n] = A
    return K, lu_factor(K)


def tracking_qp(W, Wd, Wdd, m_seg: int, with_goal: bool = False, k_p=20.0, k_v=2.0 * math.sqrt(20.0),
                w_smooth=1.0, w_offset=20.0, w_speed=20.0) -> QPData:
    """Stage-1 tracking QP (pkg/batch_qp.py:152-206)."""
    n = W.shape[1]
    S = segment_onehot(W.shape[0], m_seg)
    Asp = Wdd - k_p * Wd
    Aof = Wdd - k_p * W - k_v * Wd
    Q = np.zeros((2 * n, 2 * n))
    Q[:n, :n] = w_smooth * (Wdd.T @ Wdd) + w_speed * (Asp.T @ Asp)
    Q[n:, n:] = w_smooth * (Wdd.T @ Wdd) + w_offset * (Aof.T @ Aof)
    zero = np.zeros(n)
    rows = []
    for M in (W, Wd, Wdd):
        rows.append(np.concatenate([M[0], zero]))
        rows.append(np.concatenate([zero, M[0]]))
    if with_goal:
        rows += [np.concatenate([W[-1], zero]), np.concatenate([zero, W[-1]]), np.concatenate([zero, Wd[-1]])]
    A = np.vstack(rows)
    K, lu = _bordered(Q, A)
    return QPData(Q, A, K, lu, w_speed * k_p * (Asp.T @ S), w_offset * k_p * (Aof.T @ S), m_seg, with_goal)


def stage1(qp: QPData, p: np.ndarray, b0: np.ndarray):
    """(xi (2n,B), mu (neq,B), b (neq,B)) — RHS build + LU solve (pkg/batch_qp.py:209-239,258-280)."""
    p = np.atleast_2d(np.asarray(p, dtype=float))
    ms = qp.m_seg
    q = np.concatenate([qp.qmx @ p[:, ms:2 * ms].T, qp.qmy @ p[:, :ms].T], axis=0)
    B = p.shape[0]
    b = np.repeat(np.asarray(b0, float)[:, None], B, axis=1)
    if qp.with_goal:
        b = np.vstack([b, p[:, 2 * ms], p[:, 2 * ms + 1], np.zeros(B)])
    rhs = np.vstack([-q, b])
    sol = lu_solve(qp.lu, rhs)
    n = qp.Q.shape[0]
    return sol[:n], sol[n:], b


def aug_qp(W, Wd, Wdd, A_eq, n_obs: int, rho: float) -> QPData:
    """Penalty-augmented KKT of the AM step (pkg/projection.py:189-214)."""
    n = W.shape[1]
    G = n_obs * (W.T @ W) + Wd.T @ Wd + Wdd.T @ Wdd
    Q = np.zeros((2 * n, 2 * n))
    Q[:n, :n] = np.eye(n) + rho * G
    Q[n:, n:] = Q[:n, :n] + rho * 2.0 * (W.T @ W)
    K, lu = _bordered(Q, A_eq)
    return QPData(Q, A_eq, K, lu)


# --------------------------------------------------------------------------- constraints
@dataclass
class Limits:
    """ConstraintSpec fields (pkg/constraints.py:19-72)."""
    ox: np.ndarray
    oy: np.ndarray
    a: float
    b: float
    v_max: float
    a_max: float
    kappa_max: float
    c_max: float
    y_lb: float
    y_ub: float
    v_min: float = 0.0
    curv: tuple | None = None      # (xs, ks) tabulated road curvature or None

    @property
    def n_obs(self) -> int:
        return self.ox.shape[0]


def kappa_lookup(lim: Limits, x: np.ndarray) -> np.ndarray:
    """np.interp road curvature (pkg/constraints.py:67-72)."""
    if lim.curv is None:
        return np.zeros_like(np.asarray(x, dtype=float))
    return np.interp(x, lim.curv[0], lim.curv[1])


def violation_terms(lim: Limits, X, Y, XD, YD, XDD, YDD) -> dict:
    """Per-sample positive violations by constraint (pkg/constraints.py:95-139)."""
    out = {}
    if lim.n_obs:
        dx = (X[:, None, :] - lim.ox[None]) / lim.a
        dy = (Y[:, None, :] - lim.oy[None]) / lim.b
        out["collision"] = np.maximum(1.0 - dx**2 - dy**2, 0.0).sum(axis=(1, 2))
    else:
        out["collision"] = np.zeros(X.shape[0])
    sp = np.hypot(XD, YD)
    out["velocity"] = (np.maximum(sp - lim.v_max, 0.0) + np.maximum(lim.v_min - sp, 0.0)).sum(axis=1)
    out["acceleration"] = np.maximum(np.hypot(XDD, YDD) - lim.a_max, 0.0).sum(axis=1)
    kap = np.abs(YDD * XD - XDD * YD) / np.maximum(sp, SPEED_EPS) ** 3
    out["curvature"] = np.maximum(kap - lim.kappa_max, 0.0).sum(axis=1)
    out["centripetal"] = np.maximum(XD**2 * np.abs(kappa_lookup(lim, X)) - lim.c_max, 0.0).sum(axis=1)
    out["lane"] = (np.maximum(Y - lim.y_ub, 0.0) + np.maximum(lim.y_lb - Y, 0.0)).sum(axis=1)
    return out


def residual_sum(lim: Limits, *traj) -> np.ndarray:
    """Total residual (pkg/constraints.py:142-153), summed in the reference's key order."""
    return sum(violation_terms(lim, *traj).values())


# --------------------------------------------------------------------------- AM projection
def polar_split(XD, YD, XDD, YDD, X=None, Y=None, lim: Limits | None = None):
    """(alpha_o, alpha_v, alpha_a, d_o, d_v, d_a) (pkg/projection.py:100-135)."""
    av, dv = np.arctan2(YD, XD), np.hypot(XD, YD)
    aa, da = np.arctan2(YDD, XDD), np.hypot(XDD, YDD)
    ao = do = None
    if lim is not None and lim.n_obs:
        wc = X[:, None, :] - lim.ox
        ws = Y[:, None, :] - lim.oy
        ao = np.arctan2(lim.a * ws, lim.b * wc)
        co, so = np.cos(ao), np.sin(ao)
        den = (lim.a * co) ** 2 + (lim.b * so) ** 2
        safe = np.where(den > 0.0, den, 1.0)
        do = np.where(den > 0.0, (lim.a * wc * co + lim.b * ws * so) / safe, 0.0)
    return ao, av, aa, do, dv, da


def coupled_clip(av, dv_raw, aa, da_raw, do_raw, da_prev, kap_abs, lim: Limits):
    """Clip polar magnitudes into coupled windows; returns (d_o, d_v, d_a, #conflicts)
    (pkg/projection.py:138-169)."""
    do = None if do_raw is None else np.maximum(do_raw, 1.0)
    gap = np.abs(np.sin(aa - av))
    lo = np.maximum(lim.v_min, np.sqrt(da_prev * gap / lim.kappa_max))
    cent = kap_abs * np.cos(av) ** 2
    hi = np.where(cent > KAPPA_FLOOR, np.sqrt(lim.c_max / np.maximum(cent, KAPPA_FLOOR)), lim.v_max)
    hi = np.minimum(lim.v_max, hi)
    nconf = int(np.count_nonzero(lo > hi))
    dv = np.clip(dv_raw, np.minimum(lo, hi), hi)
    ahi = np.minimum(lim.a_max, dv**2 * lim.kappa_max / np.maximum(gap, SIN_FLOOR))
    da = np.clip(da_raw, 0.0, ahi)
    return do, dv, da, nconf


def _solve_checked(aug: QPData, lin: np.ndarray, b: np.ndarray) -> np.ndarray:
    """lu_solve + 1e-8 KKT residual check (pkg/batch_qp.py:258-280); returns xi (2n,B)."""
    rhs = np.vstack([lin, b])
    sol = lu_solve(aug.lu, rhs)
    res = np.abs(aug.kkt @ sol - rhs).max(axis=0)
    if np.any(res > 1e-8 * (1.0 + np.abs(rhs).max(axis=0))):
        raise FloatingPointError("KKT residual above tolerance")
    return sol[: aug.Q.shape[0]]


def am_project(aug: QPData, W, Wd, Wdd, xi_bar, b, lim: Limits, rho=1.0, max_iters=100, tol=1e-3):
    """Alternating-minimisation projection, Alg. 2 (pkg/projection.py:216-339).

    Returns dict(xi (2n,B), residuals (B,), history (it,B), iterations, conflicts).
    """
    n, m = W.shape[1], W.shape[0]
    xi_bar = np.atleast_2d(np.asarray(xi_bar, float))
    B = xi_bar.shape[1]
    cxb, cyb = xi_bar[:n].T, xi_bar[n:].T
    fwd = lambda cx, cy: (cx @ W.T, cy @ W.T, cx @ Wd.T, cy @ Wd.T, cx @ Wdd.T, cy @ Wdd.T)
    obs = lim if lim.n_obs else None

    cx, cy = cxb.copy(), cyb.copy()
    X, Y, XD, YD, XDD, YDD = fwd(cx, cy)
    ao, av, aa, do, dv, da = polar_split(XD, YD, XDD, YDD, X, Y, obs)
    do, dv, da, conflicts = coupled_clip(av, dv, aa, da, do, np.clip(da, 0.0, lim.a_max),
                                         np.abs(kappa_lookup(lim, X)), lim)
    lx = np.zeros((B, n))
    ly = np.zeros((B, n))
    up = np.concatenate([np.full(m, lim.y_ub), np.full(m, -lim.y_lb)])
    slack = np.maximum(0.0, up[None] - np.concatenate([Y, -Y], axis=1))

    hist = np.empty((max_iters, B))
    resid = np.full(B, np.inf)
    used = 0
    for it in range(max_iters):
        used = it + 1
        tx = dv * np.cos(av) @ Wd + da * np.cos(aa) @ Wdd
        ty = dv * np.sin(av) @ Wd + da * np.sin(aa) @ Wdd
        if obs is not None:
            tx = tx + (lim.ox[None] + lim.a * do * np.cos(ao)).sum(axis=1) @ W
            ty = ty + (lim.oy[None] + lim.b * do * np.sin(ao)).sum(axis=1) @ W
        tgt = up[None] - slack
        ty = ty + (tgt[:, :m] - tgt[:, m:]) @ W
        lin_x = cxb + lx + rho * tx
        lin_y = cyb + ly + rho * ty
        xi = _solve_checked(aug, np.concatenate([lin_x, lin_y], axis=1).T, b)
        if not np.isfinite(xi).all():
            raise FloatingPointError("projection iterate is not finite")
        cx, cy = xi[:n].T, xi[n:].T
        Xp = X
        X, Y, XD, YD, XDD, YDD = fwd(cx, cy)
        ao, av, aa, do_r, dv_r, da_r = polar_split(XD, YD, XDD, YDD, X, Y, obs)
        do, dv, da, k = coupled_clip(av, dv_r, aa, da_r, do_r, da, np.abs(kappa_lookup(lim, Xp)), lim)
        conflicts += k
        lane = np.concatenate([Y, -Y], axis=1)
        slack = np.maximum(0.0, up[None] - lane)
        rl = lane - up[None] + slack
        gx = (XD - dv * np.cos(av)) @ Wd + (XDD - da * np.cos(aa)) @ Wdd
        gy = (YD - dv * np.sin(av)) @ Wd + (YDD - da * np.sin(aa)) @ Wdd
        if obs is not None:
            gx = gx + ((X[:, None, :] - lim.ox) - lim.a * do * np.cos(ao)).sum(axis=1) @ W
            gy = gy + ((Y[:, None, :] - lim.oy) - lim.b * do * np.sin(ao)).sum(axis=1) @ W
        gy = gy + (rl[:, :m] - rl[:, m:]) @ W
        lx = lx - 0.5 * rho * gx
        ly = ly - 0.5 * rho * gy
        resid = residual_sum(lim, X, Y, XD, YD, XDD, YDD)
        hist[it] = resid
        if resid.max() <= tol:
            break
    return {
        "xi": np.concatenate([cx, cy], axis=1).T,
        "residuals": resid,
        "history": hist[:used].copy(),
        "iterations": used,
        "conflicts": conflicts,
    }


# --------------------------------------------------------------------------- CEM upper level
def speed_cost(XD, YD, v_max: float) -> np.ndarray:
    """Sum_t (|v| - v_max)^2 (pkg/bilevel.py:119-126)."""
    return ((np.hypot(XD, YD) - v_max) ** 2).sum(axis=-1)


def rank_two_stage(r, c, n: int, q: int, w: float):
    """(cons_idx, elite_idx, elite_aug) with index tie-breaks (pkg/bilevel.py:129-137)."""
    cons = np.argsort(r, kind="stable")[:n]
    aug = c[cons] + w * r[cons]
    sub = np.lexsort((cons, aug))[:q]
    return cons, cons[sub], aug[sub]


def softmin_weights(aug: np.ndarray, gamma: float) -> np.ndarray:
    """exp(-(c - min c)/gamma) normalised, uniform fallback (pkg/bilevel.py:163-172)."""
    w = np.exp(-(aug - aug.min()) / gamma)
    s = w.sum()
    if not np.isfinite(s) or s <= 0.0:
        return np.full_like(aug, 1.0 / aug.shape[0])
    return w / s


def refit_gaussian(mean, cov, P, aug, eta: float, gamma: float):
    """Weighted mean/cov refit + 1e-6 I + symmetrise (pkg/bilevel.py:175-194)."""
    w = softmin_weights(np.asarray(aug, float), gamma)
    mu = (1.0 - eta) * mean + eta * (w @ P)
    D = P - mu[None]
    C = (1.0 - eta) * cov + eta * (D.T @ (w[:, None] * D)) + COV_REG * np.eye(mean.shape[0])
    return mu, 0.5 * (C + C.T)


def draw_gaussian(mean, cov, n: int, rng: np.random.Generator):
    """mu + z L^T with Cholesky fallback (pkg/bilevel.py:51-57)."""
    try:
        L = np.linalg.cholesky(cov)
    except np.linalg.LinAlgError:
        L = np.linalg.cholesky(cov + 10 * COV_REG * np.eye(cov.shape[0]))
    z = rng.standard_normal((n, mean.shape[0]))
    return mean[None] + z @ L.T


@dataclass
class CemTrace:
    params: list = field(default_factory=list)
    xi: list = field(default_factory=list)
    residuals: list = field(default_factory=list)
    costs: list = field(default_factory=list)
    cons_idx: list = field(default_factory=list)
    elite_idx: list = field(default_factory=list)
    elite_aug: list = field(default_factory=list)
    mean: list = field(default_factory=list)
    cov: list = field(default_factory=list)
    stats: list = field(default_factory=list)
    iterations_used: list = field(default_factory=list)
    conflicts: list = field(default_factory=list)


def cem_cycle(qp: QPData, aug: QPData, W, Wd, Wdd, b0, lim: Limits, mean, cov, *, batch, n_cons, n_elite,
              iters, eta, gamma, w_res, rng=None, params_per_iter=None, rho=1.0, am_iters=100, tol=1e-3):
    """CEM bi-level loop, Alg. 1 (pkg/bilevel.py:228-295).

    ``params_per_iter`` (list of (B, dim) arrays) teacher-forces the samples
    instead of drawing them from ``rng``.  Returns a CemTrace.
    """
    tr = CemTrace()
    mean = np.asarray(mean, float)
    cov = np.asarray(cov, float)
    for it in range(iters):
        P = params_per_iter[it] if params_per_iter is not None else draw_gaussian(mean, cov, batch, rng)
        xb, _, b = stage1(qp, P, b0)
        pr = am_project(aug, W, Wd, Wdd, xb, b, lim, rho, am_iters, tol)
        n = W.shape[1]
        xi = pr["xi"]
        c = speed_cost(xi[:n].T @ Wd.T, xi[n:].T @ Wd.T, lim.v_max)
        r = pr["residuals"]
        cons, el, ea = rank_two_stage(r, c, n_cons, n_elite, w_res)
        mean, cov = refit_gaussian(mean, cov, P[el], ea, eta, gamma)
        tr.params.append(P)
        tr.xi.append(xi)
        tr.residuals.append(r)
        tr.costs.append(c)
        tr.cons_idx.append(cons)
        tr.elite_idx.append(el)
        tr.elite_aug.append(ea)
        tr.mean.append(mean)
        tr.cov.append(cov)
        tr.iterations_used.append(pr["iterations"])
        tr.conflicts.append(pr["conflicts"])
        tr.stats.append([float(c[el].mean()), float(ea[0]), float(np.trace(cov)), float(r.min()),
                         float(np.median(r)), float(r.max())])
    return tr
