"""GPU consumer of M: left-preconditioned GMRES and
BiCGstab mirroring mcspai::gmres / bicgstab / solve (solvers.hpp:35-46,
solvers.cpp:54-244), on device-resident B and M through ``mcmi_solve_device``.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass
from enum import IntEnum

from . import _lib as L
from .mcspai import CsrMatrix, raise_for


class SolverMethod(IntEnum):  # solvers.hpp:11
    gmres = 0
    bicgstab = 1


@dataclass
class SolverConfig:  # solvers.hpp:13-18
    method: SolverMethod = SolverMethod.gmres
    rel_tol: float = 1e-6
    max_iters: int = 30000
    restart: int = 50


@dataclass
class SolveReport:  # solvers.hpp:20-30 (x returned separately)
    converged: bool
    iterations: int
    final_rel_residual: float
    breakdown: bool
    ms: float
    preconditioned: bool
    method_echo: SolverMethod


def _view(tensors, n):
    rp, ci, v = tensors
    return L.mcmi_csr_view(int(n), rp.data_ptr(), ci.data_ptr(), v.data_ptr())


def solve_device(n: int, b_tensors, m_tensors=None, rhs=None, cfg: SolverConfig | None = None,
                 device: int = 0, stream=None):
    """b_tensors / m_tensors: (row_ptr int64, col_idx int64, values f64) CUDA
    tensors; rhs: CUDA f64 tensor or None (B * ones).  Returns (x, report)."""
    import torch
    cfg = cfg or SolverConfig()
    lib = L.load()
    c = L.mcmi_solver_config()
    lib.mcmi_solver_config_default(C.byref(c))
    c.method, c.rel_tol, c.max_iters, c.restart = int(cfg.method), float(cfg.rel_tol), int(cfg.max_iters), \
        int(cfg.restart)
    x = torch.empty(max(n, 1), dtype=torch.float64, device=torch.device("cuda", device))
    bv = _view(b_tensors, n)
    mv = _view(m_tensors, n) if m_tensors is not None else None
    rep = L.mcmi_solve_report()
    err = C.create_string_buffer(512)
    s = None if stream is None else stream.cuda_stream
    code = lib.mcmi_solve_device(C.byref(bv), C.byref(mv) if mv is not None else None,
                                 rhs.data_ptr() if rhs is not None else None, x.data_ptr(), C.byref(c), device, s,
                                 C.byref(rep), err, 512)
    raise_for(code, err.value.decode(errors="replace"))
    return x[:n], SolveReport(bool(rep.converged), int(rep.iterations), float(rep.final_rel_residual),
                              bool(rep.breakdown), float(rep.ms), m_tensors is not None, SolverMethod(cfg.method))


def solve(b: CsrMatrix, m: CsrMatrix | None = None, cfg: SolverConfig | None = None, device: int = 0):
    """mcspai::solve with rhs = B * 1 (ones_product_rhs) on host CSR inputs."""
    from .engine import DeviceEngine
    bt = DeviceEngine.upload(b, device)
    mt = DeviceEngine.upload(m, device) if m is not None else None
    x, rep = solve_device(b.n, bt, mt, None, cfg, device)
    return x.cpu().numpy(), rep
