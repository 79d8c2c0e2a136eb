"""parascan-b200: B200-native temporally parallel Kalman filter and smoothers.

The hot path (element construction, the associative combine operators, the
scan variants and the two-filter combination) runs in the hand-written sm_100a
kernels of libpsk.so behind the C-ABI in include/psk.h.  This package mirrors
the reference's operator interface (see api.py) so that callers only swap the
backend object.
"""
from .api import (ContractViolation, CudaBackend, CudaError, DimensionMismatch,
                  GaussianStats, Lgssm, NotPositiveDefinite, ScanAlg, ScanSpec,
                  SingularMatrix, pkf_run, pkf_run_batch, prts_run, prts_run_batch,
                  ptfs_run, to_string)

__all__ = [
    "ContractViolation", "CudaBackend", "CudaError", "DimensionMismatch",
    "GaussianStats", "Lgssm", "NotPositiveDefinite", "ScanAlg", "ScanSpec",
    "SingularMatrix", "pkf_run", "pkf_run_batch", "prts_run", "prts_run_batch", "ptfs_run",
    "to_string",
]
