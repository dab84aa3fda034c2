"""Recovery phase on the GPU, mirroring
include/mcspai/recovery.hpp: undo the diagonal augmentation of B_hat^{-1} by n
Sherman-Morrison rank-one updates (recovery.cpp:7-33), bit-identical to the
reference; plus the dense helpers the reference's `recover` command uses
(csr_to_dense / densify_to_csr, csr.cpp:172-192).

    recovered = recover_inverse(b_hat_inv, s_diag, tol=1e-12)   # numpy n x n
    recover_inverse_device(m_tensor, s_diag, tol)                  # in place, HBM
"""
from __future__ import annotations

import ctypes as C

import numpy as np

from . import _lib as L
from .mcspai import CsrMatrix, raise_for


class RecoveryError(RuntimeError):  # recovery.hpp:9-11
    pass


def _raise(code, err):
    msg = err.value.decode(errors="replace")
    if code == L.MCMI_ERECOVERY:
        raise RecoveryError(msg)
    raise_for(code, msg)


def recover_inverse(b_hat_inv, s_diag, tol: float = 1e-12, device: int = 0) -> np.ndarray:
    """mcspai::recover_inverse(b_hat_inv, RecoveryPlan{s_diag}, tol) on a B200."""
    m = np.array(b_hat_inv, dtype=np.float64, order="C", copy=True)
    if m.ndim != 2 or m.shape[0] != m.shape[1]:
        raise ValueError("b_hat_inv must be a square matrix")
    s = np.ascontiguousarray(s_diag, np.float64)
    err = C.create_string_buffer(512)
    code = L.load().mcmi_recover_inverse(m.ctypes.data, m.shape[0], s.ctypes.data, s.size, float(tol), device,
                                         err, 512)
    _raise(code, err)
    return m


def recover_inverse_device(m, s_diag, tol: float = 1e-12, stream=None) -> None:
    """In place on a CUDA float64 (n, n) contiguous tensor."""
    s = np.ascontiguousarray(s_diag, np.float64)
    err = C.create_string_buffer(512)
    st = None if stream is None else stream.cuda_stream
    code = L.load().mcmi_recover_inverse_device(m.data_ptr(), m.shape[0], s.ctypes.data, s.size, float(tol),
                                                m.device.index, st, err, 512)
    _raise(code, err)


def csr_to_dense(m: CsrMatrix) -> np.ndarray:  # csr.cpp:186-192
    d = np.zeros((m.n, m.n))
    rows = np.repeat(np.arange(m.n), np.diff(m.row_ptr))
    d[rows, m.col_idx] = m.values
    return d


def densify_to_csr(d: np.ndarray, prune_tol: float = 0.0) -> CsrMatrix:  # csr.cpp:172-184
    r, c = np.nonzero(np.abs(d) > prune_tol)
    return CsrMatrix.from_triplets(d.shape[0], r, c, d[r, c])
