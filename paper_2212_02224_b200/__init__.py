"""B200-native (sm_100a) hot path of the bi-level behaviour + trajectory planner
(arXiv 2212.02224), as a drop-in for the reference package `bilevel-drive`'s
optimizer API: ``LowerLevelSolver`` / ``ProjectionOperator`` / ``solve_batch`` /
``solve_bilevel`` (+ the fleet and multi-GPU drivers).

All batch compute runs in the in-tree CUDA library ``_lib/libbilevel_b200.so``
(C ABI: include/bilevel_b200.h); there is no CPU fallback.
"""

__version__ = "0.1.0"

from .basis import (  # noqa: F401
    FlatControls, PolynomialBasis, SpeedSingularity, TrajectoryCoeffs, TrajectorySamples, build_basis,
    curvature_from_derivatives, eval_trajectory, flat_to_controls,
)
from .batch_qp import (  # noqa: F401
    NumericalFailure, QPRightHandSideBatch, QPSolutionBatch, QPStructure, StructureError, TrackingWeights,
    assemble_qp, build_qp_structure, build_rhs_batch, solve_batch, structure_from_matrices,
)
from .behavior import BehaviorParams, ParamLayout, WarmStartSource, segment_matrix, segment_members  # noqa: F401
from .bilevel import (  # noqa: F401
    BiLevelConfig, BiLevelResult, DegenerateWeights, EliteRecord, IterationStats, LowerLevelSolver,
    SamplingDistribution, rank_samples, select_elites, solve_bilevel, update_distribution, upper_cost,
    upper_cost_batch,
)
from .constraints import ConstraintSpec, PlanningScene, batch_residuals, violation_breakdown  # noqa: F401
from .projection import (  # noqa: F401
    ProjectionBatchResult, ProjectionConfig, ProjectionOperator, ProjectionReport, ProjectionState,
    clip_magnitudes, polar_decompose, project_batch,
)
