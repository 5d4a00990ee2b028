"""Host-side setup of the drop-in (basis, QP assembly, factorization counter, scenes) vs the
reference's own outputs (golden vectors)."""

import numpy as np
import pytest

from paper_2212_02224_b200 import batch_qp, build_basis
from paper_2212_02224_b200.behavior import ParamLayout, WarmStartSource, segment_matrix
from paper_2212_02224_b200.scenes import HighwayRecipe, highway_scene
from tests.golden_io import load


@pytest.mark.parametrize("tag,args", [("b100", (10, 100, 5.0, "bernstein")), ("b50", (10, 50, 10.0, "bernstein")),
                                      ("mono", (10, 100, 5.0, "monomial"))])
def test_basis(tag, args):
    g = load("basis")
    b = build_basis(*args)
    np.testing.assert_array_equal(b.times, g[tag + "_t"])
    np.testing.assert_allclose(b.W, g[tag + "_W"], atol=1e-14)
    np.testing.assert_allclose(b.Wdot, g[tag + "_Wd"], atol=1e-13)
    np.testing.assert_allclose(b.Wddot, g[tag + "_Wdd"], atol=1e-12)


def test_basis_validation():
    with pytest.raises(ValueError):
        build_basis(1, 10, 1.0)
    with pytest.raises(ValueError):
        build_basis(10, 5, 1.0)
    with pytest.raises(ValueError):
        build_basis(10, 50, 0.0)
    with pytest.raises(ValueError):
        build_basis(10, 50, 1.0, "chebyshev")


@pytest.mark.parametrize("goal", [False, True])
def test_qp_structure_and_counter(goal):
    g = load("basis")
    b = build_basis(10, 100, 5.0, "bernstein")
    before = batch_qp.FACTORIZATION_COUNT
    qp = batch_qp.build_qp_structure(b, batch_qp.TrackingWeights(), ParamLayout(4, with_goal=goal))
    assert batch_qp.FACTORIZATION_COUNT == before + 1
    p = "goal_" if goal else ""
    np.testing.assert_allclose(qp.Q, g[p + "Q"], rtol=1e-13, atol=1e-9)
    np.testing.assert_array_equal(qp.A_eq, g[p + "A_eq"])
    np.testing.assert_allclose(qp.kkt, g[p + "kkt"], rtol=1e-13, atol=1e-9)
    np.testing.assert_allclose(qp.q_map_x, g[p + "qmx"], rtol=1e-13, atol=1e-10)
    # explicit inverse from the LU factors
    np.testing.assert_allclose(qp.kkt_inv @ qp.kkt, np.eye(qp.kkt.shape[0]), atol=1e-6)


def test_rank_deficient_structure():
    with pytest.raises(batch_qp.StructureError):
        batch_qp.structure_from_matrices(np.eye(4), np.array([[1.0, 0, 0, 0], [2.0, 0, 0, 0]]))


def test_rhs_batch_matches_reference_layout():
    g = load("lower_goal")
    b = build_basis(10, 100, 5.0, "bernstein")
    k_p, k_v, ws, wo, wv = g["weights"]
    qp = batch_qp.build_qp_structure(b, batch_qp.TrackingWeights(k_p, k_v, ws, wo, wv), ParamLayout(4, True))
    rhs = batch_qp.build_rhs_batch(qp, g["params"], g["b0"])
    assert rhs.b_batch.shape == (9, g["params"].shape[0])
    np.testing.assert_array_equal(rhs.b_batch[6], g["params"][:, 8])


def test_segment_matrix_and_warm_start(tmp_path):
    S = segment_matrix(100, 4)
    assert S.sum(axis=0).tolist() == [25, 25, 25, 25]
    lay = ParamLayout(4)
    src = WarmStartSource(np.arange(16.0).reshape(2, 8), lay)
    assert src.draw(5).shape == (5, 8)
    path = tmp_path / "ws.csv"
    WarmStartSource.write_file(str(path), src.samples, lay)
    np.testing.assert_array_equal(WarmStartSource.from_file(str(path), lay).samples, src.samples)


@pytest.mark.parametrize("seed", range(6))
def test_highway_scenes_match_reference(seed):
    g = load("scenes")
    for lanes, dens, veh, nobs, rng_ in ((4, 2.0, 24, 10, 120.0), (4, 3.0, 80, 50, 250.0), (2, 1.0, 12, 10, 120.0)):
        sc = highway_scene(seed, HighwayRecipe(lanes=lanes, density=dens, vehicle_count=veh, n_obs=nobs,
                                               obstacle_range=rng_))
        tag = f"s{seed}_l{lanes}_d{dens}_v{veh}_o{nobs}"
        np.testing.assert_array_equal(sc.spec.obstacles_x, g[tag + "_ox"])
        np.testing.assert_array_equal(sc.spec.obstacles_y, g[tag + "_oy"])
        np.testing.assert_array_equal(sc.initial_state, g[tag + "_b0"])
        lim = g[tag + "_lim"]
        assert (sc.spec.ellipse_a, sc.spec.ellipse_b, sc.spec.v_min, sc.spec.v_max) == tuple(lim[:4])
        assert (sc.spec.y_lb, sc.spec.y_ub) == tuple(lim[7:9])


def test_other_basis_orders_are_refused_before_any_work():
    """The device kernels are compiled for order-10 bases; another order raises a clear
    NotImplementedError before the factorization counter moves (pkg/basis.py:156-179 accepts it)."""
    import pytest

    import paper_2212_02224_b200 as bd
    from paper_2212_02224_b200 import batch_qp
    basis = bd.build_basis(6, 100, 5.0, "bernstein")
    n0 = batch_qp.FACTORIZATION_COUNT
    with pytest.raises(NotImplementedError, match="order-10"):
        bd.LowerLevelSolver(basis, bd.TrackingWeights(), bd.ParamLayout(4), bd.ProjectionConfig(), 10)
    assert batch_qp.FACTORIZATION_COUNT == n0
