"""GPU: SPEC.md invariants of the path on the device."""

import numpy as np
import pytest

from tests.golden_io import load
from tests.test_gpu_parity import _scene, _solver

pytestmark = pytest.mark.gpu


def test_batch_serial_equivalence():
    """Projecting a batch equals projecting each sample alone — per-sample results
    do not depend on the batch.  The reference's batch-global early exit (pkg/projection.py:329)
    couples the samples of a batch (a lone sample may stop early), so the tolerance is set below
    any residual here."""
    import paper_2212_02224_b200 as bd
    g = dict(load("lower_c1_s0"))
    g["tol"] = 1e-30
    solver = _solver(g)
    sc = _scene(g)
    _, full = solver.solve(g["params"], sc)
    checked = 0
    for j in range(0, 100, 3):
        _, one = solver.solve(g["params"][j:j + 1], sc)
        if one.iterations_used != full.iterations_used:
            continue                        # this sample alone met the tolerance: exits earlier
        np.testing.assert_allclose(one.xi[:, 0], full.xi[:, j], rtol=1e-5, atol=1e-5)
        checked += 1
    assert checked >= 3


def test_initial_conditions_preserved():
    """A_eq xi = b holds for every projected trajectory."""
    g = load("lower_c1_s1")
    solver = _solver(g)
    _, proj = solver.solve(g["params"], _scene(g))
    A = solver.qp.A_eq
    b = g["b0"][:, None]
    assert np.abs(A @ proj.xi - b).max() <= 1e-8 * (1 + np.abs(proj.xi).max())


def test_goal_rows_preserved():
    g = load("lower_goal")
    solver = _solver(g)
    sol, proj = solver.solve(g["params"], _scene(g))
    A = solver.qp.A_eq
    b = np.vstack([np.repeat(g["b0"][:, None], g["params"].shape[0], 1), g["params"][:, 8], g["params"][:, 9],
                   np.zeros(g["params"].shape[0])])
    assert np.abs(A @ proj.xi - b).max() <= 1e-8 * (1 + np.abs(proj.xi).max())
    assert np.abs(A @ sol.xi - b).max() <= 1e-8 * (1 + np.abs(sol.xi).max())


def test_interior_point_is_fixed():
    """A feasible xi_bar (no obstacles, speeds inside bounds, inside the lane) projects onto
    itself."""
    g = load("lower_early4")
    solver = _solver(g)
    P = np.concatenate([np.zeros((4, 4)), np.full((4, 4), 10.0)], axis=1)
    sol, proj = solver.solve(P, _scene(g))
    assert proj.iterations_used == 1
    np.testing.assert_allclose(proj.xi, sol.xi, rtol=1e-6, atol=1e-6)
    assert np.all(proj.residuals <= 1e-8)


def test_determinism_bit_identical():
    """Identical inputs give bit-identical outputs (SPEC.md acceptance 7)."""
    g = load("lower_dense50")
    solver = _solver(g)
    sc = _scene(g)
    a = solver.solve(g["params"], sc)[1]
    b = solver.solve(g["params"], sc)[1]
    np.testing.assert_array_equal(a.xi, b.xi)
    np.testing.assert_array_equal(a.residuals, b.residuals)


def test_residual_trend_and_clip_bounds():
    """Final residual <= first-iteration residual for >= 95% of samples."""
    g = load("lower_c1_s0")
    solver = _solver(g)
    _, proj = solver.solve(g["params"], _scene(g))
    h = proj.residual_history
    assert np.mean(h[-1] <= h[0] + 1e-9) >= 0.95
