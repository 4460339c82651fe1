"""B200-native (sm_100a, fp64) phipm/IOM2 + shallow-water hot path of
arXiv 1805.02144, behind the reference ``expintkit`` API.

The compute runs in ``libeik.so`` (CUDA, see include/eik.h); this package is
the host-side mirror of the reference's plug points (engine, steps, SWE
operators) plus the sphere grid and the configuration states.
"""

from .grid import DiscreteOperators, sphere_operators, cached_sphere_operators  # noqa: F401
from .sparse import SparseMatrix  # noqa: F401
from .phipm import (  # noqa: F401
    MatvecOperator, PhiTask, PhipmFailure, PhipmResult, as_operator,
    cost_estimate, phipm_simul_iom2,
)
from .integrators import (  # noqa: F401
    SCHEME_NAMES, EngineSeeds, SemilinearProblem, StepRecord, integrate,
    linearize, step_epi3, step_exprb42, step_exprb53, step_pexprb43,
    step_rb_euler, swe_problem,
)
from . import swe  # noqa: F401

__all__ = [
    "DiscreteOperators", "sphere_operators", "SparseMatrix", "MatvecOperator",
    "PhiTask", "PhipmFailure", "PhipmResult", "as_operator", "cost_estimate",
    "phipm_simul_iom2", "SCHEME_NAMES", "EngineSeeds", "SemilinearProblem",
    "StepRecord", "integrate", "linearize", "step_epi3", "step_exprb42",
    "step_exprb53", "step_pexprb43", "step_rb_euler", "swe_problem", "swe",
]
