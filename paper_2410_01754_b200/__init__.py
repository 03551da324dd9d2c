"""B200-native periodic FMM + Hamiltonian-interpolation electrostatics.

Drop-in for the hot path of the reference package ``lambdafmm`` 0.1.0
(arXiv 2410.01754): ``PeriodicSolver`` / ``SolverConfig`` / ``SolveResult``
(fmm/solver.py) and ``hi_energy_and_forces`` / ``build_corrections`` /
``assemble_lambda_forces`` (corrections.py), computed by hand-written sm_100a
CUDA kernels behind the C-ABI in include/lfmm.h.  There is no CPU fallback.
"""

__version__ = "0.1.0"

from .corrections import (  # noqa: F401
    CorrectionSet,
    InterpolationResult,
    SiteCorrections,
    assemble_lambda_forces,
    build_corrections,
    hi_energy_and_forces,
)
from .fmm.solver import PeriodicSolver, SolveResult, SolverConfig  # noqa: F401
from .system import LambdaState, ParticleSystem, TitratableSite, scale_charges  # noqa: F401
from .weights import expand_weights, weight_gradient, weight_gradient_matrix  # noqa: F401
