"""B200-native correction step of the multilevel local-and-parallel FEM
eigensolver (arXiv 1401.4969): hand-written sm_100a CUDA behind a C ABI
(include/mlg_b200.h), with this package as the host-side mirror of the
reference's corrector interface."""
from ._lib import ConfigError, CudaError, IoError, MlgError, SolverError, lib
from .corrector import (CorrectionState, DomainRect, EigenPair, Hierarchy, RunConfig,
                        SolveReport, StepTimings, augmented_eigensolve, coarse_eigensolve,
                        interface_solve, local_bvp_solve, local_cg_solve, multilevel_correction,
                        one_correction_step)
from . import harness

__all__ = [
    "ConfigError", "CudaError", "IoError", "MlgError", "SolverError", "lib",
    "CorrectionState", "DomainRect", "EigenPair", "Hierarchy", "RunConfig", "SolveReport",
    "StepTimings", "augmented_eigensolve", "coarse_eigensolve", "interface_solve",
    "local_bvp_solve", "local_cg_solve", "multilevel_correction", "one_correction_step", "harness",
]
