"""B200-native MCMCMI preconditioner build (drop-in for mcspai::compute_preconditioner).

Importing the package loads the sm_100a library (paper_2409_03095_b200/lib/libmcmi.so)
and fails loudly if it has not been built: there is no CPU fallback.
"""
from . import _lib
from .mcspai import (ApproxInverse, AugmentationMode, ChainBudget, CsrMatrix, DeviceError, DropMode,
                     McConfig, RngMode, RowMeta, SplitError, compute_preconditioner,
                     compute_preconditioner_serial)

_lib.load()

__all__ = [
    "ApproxInverse", "AugmentationMode", "ChainBudget", "CsrMatrix", "DeviceError", "DropMode", "McConfig",
    "RngMode", "RowMeta", "SplitError", "compute_preconditioner", "compute_preconditioner_serial",
]
