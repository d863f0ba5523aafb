"""paper_2001_04886_b200 -- B200-native s-step Orthomin / s-step GMRES (arXiv 2001.04886).

The solver hot path lives in libskrylov_b200.so (C++ host orchestration + sm_100a CUDA
kernels) behind the C ABI in include/skrylov_b200.h; this package is its reference-shaped
Python front end (sstep.py) plus the seeded input generators (problems.py).
"""
from .accounting import (  # noqa: F401
    AuditMode, AuditReport, audit, predicted_gmres, predicted_omin, run_audit, gmres_audit_slack,
    sgmres_audit_slack, somin_audit_slack,
)
from .problems import CONFIGS, Stencil, convection_diffusion, splitmix64_uniform  # noqa: F401
from .sstep import (  # noqa: F401
    BreakdownError, Context, CudaError, DeviceOperator, LogicError, SolveReport, SolverConfig, SStepBasis,
    SStepConfig, cholesky_upper, gmres_solve, gram_solve, hessenberg_lsq, krylov_block, sarnoldi, sgmres_solve,
    sgmres_solve_device, smr_solve, smr_step, solve_linear, somin_solve, somin_solve_device, ilu0_factor, DiscretizedProblem, discretize,
)

from . import sweep  # noqa: F401,E402

__version__ = "0.1.0"
