"""Helpers to read the committed golden vectors (tests/golden/*.npz, made by tools/gen_golden.py)."""

from __future__ import annotations

import os

import numpy as np

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")

LOWER_CASES = ["c1_s0", "c1_s1", "canon", "dense50", "b1", "early4", "early39", "curve", "nobs0", "goal"]


def load(name: str) -> dict:
    with np.load(os.path.join(GOLDEN, name + ".npz")) as z:
        return {k: z[k] for k in z.files}


def oracle_limits(g: dict):
    from oracle import Limits

    a, b, vmin, vmax, amax, kmax, cmax, ylb, yub = g["limits"]
    curv = (g["curv_x"], g["curv_k"]) if "curv_x" in g else None
    return Limits(g["ox"], g["oy"], a, b, vmax, amax, kmax, cmax, ylb, yub, vmin, curv)


def rel_err_per_sample_axis(xi, ref, n=11):
    """max over samples/axes of ||d c||_inf / max(||c_ref||_inf, 1)."""
    xi = np.asarray(xi, float)
    ref = np.asarray(ref, float)
    worst = 0.0
    for sl in (slice(0, n), slice(n, 2 * n)):
        d = np.abs(xi[sl] - ref[sl]).max(axis=0)
        s = np.maximum(np.abs(ref[sl]).max(axis=0), 1.0)
        worst = max(worst, float((d / s).max()))
    return worst
