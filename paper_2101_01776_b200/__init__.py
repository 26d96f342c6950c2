"""B200-native IRK stage-equation solve (drop-in for irkit's hot path).

Fully implicit Runge-Kutta (Gauss / Radau IIA / Lobatto IIIC) stage solves
with real-Schur stage decoupling, the paper's variant 0-3 linearisations and
block-2x2 preconditioned GMRES with damped-Jacobi (gamma*M - dt*L) inner
solves, on hand-written sm_100a CUDA kernels behind a C ABI
(include/irkg.h).  The public names mirror the reference package ``irkit``
(arXiv 2101.01776).
"""

from .config import PrecondSpec, SolverConfig
from .errors import (
    AssumptionViolationError,
    ConfigurationError,
    DecompositionError,
    IndexViolationError,
    IrkitError,
    KrylovBreakdownError,
    SingularMatrixError,
    StageSolveError,
    StepFailureError,
)
from .problems import (
    GridProblem,
    RunSpec,
    VorticityProblem,
    baseline_config,
    fourier_u0,
    vorticity_initial_state,
)
from .solver import (
    Block2x2System,
    DaeIntegrationResult,
    LinearOperator,
    OperatorField,
    ShiftedSolver,
    StageLinearization,
    StageState,
    VariantJacobian,
    apply_block2x2,
    block_gmres,
    build_variant_jacobian,
    combine,
    dae_integrate,
    dae_step,
    gmres,
    integrate,
    newton_like_step,
    precond_block2x2,
    solve_transformed_system,
    stage_residual,
    step,
    variant_weights,
)
from .stats import IntegrationResult, KrylovReport, SolveStats, StepStats, write_step_stats_csv
from .tableau import (
    ButcherTableau,
    EigenBlock,
    SchurForm,
    StagePrep,
    gamma_star,
    make_tableau,
    prepare_stages,
)

__all__ = [
    "AssumptionViolationError",
    "Block2x2System",
    "ButcherTableau",
    "ConfigurationError",
    "DaeIntegrationResult",
    "VorticityProblem",
    "dae_integrate",
    "dae_step",
    "vorticity_initial_state",
    "DecompositionError",
    "EigenBlock",
    "GridProblem",
    "IndexViolationError",
    "IntegrationResult",
    "IrkitError",
    "KrylovBreakdownError",
    "KrylovReport",
    "LinearOperator",
    "OperatorField",
    "PrecondSpec",
    "RunSpec",
    "SchurForm",
    "ShiftedSolver",
    "SingularMatrixError",
    "SolveStats",
    "SolverConfig",
    "StageLinearization",
    "StagePrep",
    "StageSolveError",
    "StageState",
    "StepFailureError",
    "StepStats",
    "VariantJacobian",
    "apply_block2x2",
    "build_variant_jacobian",
    "combine",
    "baseline_config",
    "block_gmres",
    "fourier_u0",
    "gamma_star",
    "gmres",
    "integrate",
    "make_tableau",
    "newton_like_step",
    "precond_block2x2",
    "prepare_stages",
    "solve_transformed_system",
    "stage_residual",
    "step",
    "variant_weights",
    "write_step_stats_csv",
]
