"""fracprec_b200: B200-native solve phase (GMRES + block-AMG t-p-u / t-u-p
preconditioners) for the 3x3 contact/fracture-flow Jacobian of arXiv 2112.12397.

The compute path is the sm_100a shared library built from ``csrc/`` and reached
through the C ABI in ``include/fracprec_b200.h``; this package is the thin host
mirror of the reference API (see ``api.py``).
"""
from .api import (AmgConfig, BlockSystem, BlockSystemOperator, CsrMatrix, GpuPreconditioner, HostPreconditioner,
                  NumericalError, PrecondConfig, SolveStats, Workload, build_tpu, build_tup, gmres)

__all__ = ["AmgConfig", "BlockSystem", "BlockSystemOperator", "CsrMatrix", "GpuPreconditioner", "HostPreconditioner",
           "NumericalError", "PrecondConfig", "SolveStats", "Workload", "build_tpu", "build_tup", "gmres"]
