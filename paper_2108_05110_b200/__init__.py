"""B200-native time-stepping hot path of the ensemble MHD scheme (arXiv 2108.05110).

Public names mirror the reference package `ensmhd` (`pkg/src/ensmhd/__init__.py:11-63`)
so callers can switch by changing the import.  The time-step (`advance`, `run`)
runs on sm_100a kernels through the C ABI in include/ensmhd_b200.h; mesh and
operator setup stay on the host.
"""

from .discretization import Discretization
from .ensemble import (EnsembleConfig, EnsembleState, MemberParams, elsasser_from_primitive,
                       perturbation_factor, perturbation_factors, primitive_from_elsasser, sample_viscosities,
                       viscosity_stats)
from .mesh import Marker, Mesh, barycentric_refine, build_step_channel, build_structured_square
from .problems import (BaselineMms, PaperMmsBoundary, PaperMmsForcing, ScaledProfileBoundary, ZeroBoundary,
                       ZeroForcing, build_case, paper_mms_initial_fields, RankOneMembers, member_rows)
from .linalg import Factorization, SingularMatrixError, factorize, relative_residual
from .stepper import (Problem, RunReport, StepFailure, StepKind, StepSystem, advance, assemble_member_rhs,
                      assemble_shared_lhs, check_preconditions, energy, run, set_solver_options,
                      verify_stability_bound)

__all__ = [
    "Discretization", "EnsembleConfig", "EnsembleState", "MemberParams", "Marker", "Mesh", "Problem",
    "RunReport", "StepFailure", "StepKind", "advance", "barycentric_refine", "build_step_channel",
    "build_structured_square", "check_preconditions", "elsasser_from_primitive", "energy",
    "primitive_from_elsasser", "run", "sample_viscosities", "verify_stability_bound", "viscosity_stats",
    "perturbation_factor", "perturbation_factors", "BaselineMms", "PaperMmsForcing", "PaperMmsBoundary",
    "ZeroForcing", "ZeroBoundary", "ScaledProfileBoundary", "build_case", "paper_mms_initial_fields", "RankOneMembers", "member_rows",
    "set_solver_options", "StepSystem", "assemble_shared_lhs", "assemble_member_rhs", "Factorization",
    "SingularMatrixError", "factorize", "relative_residual",
]

__version__ = "0.1.0"
