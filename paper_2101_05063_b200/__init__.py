"""B200-native batched shifted-Hessenberg robust RQ solve (arXiv 2101.05063).

Drop-in for the inverse-iteration path of the reference ``hessrq`` package:
``dhsrq3in`` / ``chsrq3in`` / ``hsrq3in`` (and the system solvers
``dhsrq3`` / ``chsrq3``) with the reference's arguments, running on
hand-written sm_100a CUDA kernels (csrc/) through the C ABI in
include/hsrq.h.  There is no CPU fallback.
"""

from .core import (
    ConfigError,
    HessenbergMatrix,
    HessrqError,
    OverflowBudget,
    RunStats,
    ScalingMatrix,
    SingularSystemError,
    SolutionBlock,
    StructuralViolationError,
    TaskError,
    TaskNode,
    TileGrid,
    Workspace,
    deinterleave_complex,
    interleave_complex,
)
from .inviter import (
    EigvecResult,
    InviterConfig,
    chsrq3in,
    converged,
    dhsrq3in,
    hsrq3in,
    starting_vector,
)
from .backsolve import chsrq3, dhsrq3
from .henry import henry_rq_solve
from .hessenberg import backmultiply, householder_hessenberg, hsrq3in_dense
from . import flops

__version__ = "0.1.0"
