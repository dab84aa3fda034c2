"""ctypes binding of the C-ABI in include/mcmi.h (libmcmi.so, sm_100a).

The product path has no CPU fallback: if the library is missing this module
raises, and every call that cannot reach a B200 returns an error status.
"""
from __future__ import annotations

import ctypes as C
import os

from .build import LIB

_i64p = C.POINTER(C.c_int64)
_f64p = C.POINTER(C.c_double)

(MCMI_OK, MCMI_EINVAL, MCMI_ESPLIT, MCMI_ERANGE, MCMI_ECUDA, MCMI_ENOMEM, MCMI_ENODEV, MCMI_EPARSE,
 MCMI_EIO, MCMI_ERECOVERY) = range(10)

#: every symbol include/mcmi.h declares
EXPORTS = [
    "mcmi_config_default", "mcmi_build", "mcmi_build_rows", "mcmi_build_into", "mcmi_partition_rows", "mcmi_result_sizes", "mcmi_result_copy",
    "mcmi_result_stats", "mcmi_result_free", "mcmi_engine_create", "mcmi_engine_destroy",
    "mcmi_engine_build", "mcmi_copy", "mcmi_version", "mcmi_solver_config_default", "mcmi_solve_device",
    "mcmi_host_register", "mcmi_host_unregister", "mcmi_from_triplets", "mcmi_mm_parse", "mcmi_mm_read_file",
    "mcmi_host_csr_get", "mcmi_host_csr_free", "mcmi_mm_format", "mcmi_mm_write_file", "mcmi_recover_inverse",
    "mcmi_recover_inverse_device", "mcmi_scatter_shard", "mcmi_derive_chain_budget", "mcmi_augment_and_split",
    "mcmi_split_sizes", "mcmi_split_copy", "mcmi_split_free", "mcmi_transition_probabilities", "mcmi_drop_small_entries",
    "mcmi_build_start", "mcmi_job_estimate", "mcmi_job_finish", "mcmi_result_view", "mcmi_estimate_rows",
    "mcmi_retain_top_k", "mcmi_scale_columns", "mcmi_job_attach", "mcmi_result_copy_range",
]


class mcmi_config(C.Structure):
    _fields_ = [
        ("epsilon", C.c_double),
        ("delta", C.c_double),
        ("alpha", C.c_double),
        ("mode", C.c_int32),
        ("drop_mode", C.c_int32),
        ("drop_fraction", C.c_double),
        ("retain_k", C.c_int64),
        ("has_chains_override", C.c_int32),
        ("has_max_len_override", C.c_int32),
        ("chains_override", C.c_int64),
        ("max_len_override", C.c_int64),
        ("master_seed", C.c_uint64),
        ("rng_mode", C.c_int32),
        ("device", C.c_int32),
        ("flags", C.c_int32),
        ("n_gpus", C.c_int32),
    ]


MCMI_FLAG_DEG_STATS = 1
MCMI_FLAG_UNSCALED = 2


class mcmi_csr_view(C.Structure):
    _fields_ = [("n", C.c_int64), ("row_ptr", C.c_void_p), ("col_idx", C.c_void_p), ("values", C.c_void_p)]


class mcmi_stats(C.Structure):
    _fields_ = [
        ("n_chains", C.c_int64),
        ("max_len", C.c_int64),
        ("a_norm", C.c_double),
        ("rows", C.c_int64),
        ("nnz", C.c_int64),
        ("walk_steps", C.c_int64),
        ("walk_deg_sum", C.c_int64),
        ("hash_cap", C.c_int64),
        ("rows_retried", C.c_int64),
        ("ms_tables", C.c_double),
        ("ms_walk", C.c_double),
        ("ms_assemble", C.c_double),
        ("ms_total", C.c_double),
        ("launches", C.c_int64),
        ("ms_walk_kernel", C.c_double),
    ]

    def as_dict(self):
        return {k: getattr(self, k) for k, _ in self._fields_}


class mcmi_device_csr(C.Structure):
    _fields_ = [
        ("row_begin", C.c_int64),
        ("row_end", C.c_int64),
        ("nnz", C.c_int64),
        ("row_ptr", C.c_void_p),
        ("col_idx", C.c_void_p),
        ("values", C.c_void_p),
        ("chains_used", C.c_void_p),
        ("entries_before", C.c_void_p),
    ]


class mcmi_solver_config(C.Structure):
    _fields_ = [("method", C.c_int32), ("reserved", C.c_int32), ("rel_tol", C.c_double),
                ("max_iters", C.c_int64), ("restart", C.c_int64)]


class mcmi_solve_report(C.Structure):
    _fields_ = [("converged", C.c_int32), ("breakdown", C.c_int32), ("iterations", C.c_int64),
                ("final_rel_residual", C.c_double), ("ms", C.c_double)]


_lib = None


def load(path: str | None = None):
    """Loads libmcmi.so; raises if it has not been built (no fallback)."""
    global _lib
    if _lib is not None:
        return _lib
    # MCMI_LIB_PATH: an alternative build of the same library (A/B kernel experiments)
    path = path or os.environ.get("MCMI_LIB_PATH") or LIB
    if not os.path.exists(path):
        raise ImportError(
            f"{path} not found: the CUDA library is required (run `python paper_2409_03095_b200/build.py` or `python __graft_entry__.py`)")
    L = C.CDLL(path)
    L.mcmi_config_default.argtypes = [C.POINTER(mcmi_config)]
    L.mcmi_config_default.restype = None
    L.mcmi_build.argtypes = [C.POINTER(mcmi_csr_view), C.POINTER(mcmi_config), C.POINTER(C.c_void_p),
                             C.c_char_p, C.c_size_t]
    L.mcmi_build_rows.argtypes = [C.POINTER(mcmi_csr_view), C.POINTER(mcmi_config), C.c_int64, C.c_int64,
                                  C.POINTER(C.c_void_p), C.c_char_p, C.c_size_t]
    L.mcmi_build_into.argtypes = [C.POINTER(mcmi_csr_view), C.POINTER(mcmi_config), C.c_int64, C.c_int64,
                                  C.c_void_p, C.c_void_p, C.c_void_p, C.c_int64, C.c_void_p, C.c_void_p,
                                  C.POINTER(C.c_int64), C.POINTER(mcmi_stats), C.c_char_p, C.c_size_t]
    L.mcmi_partition_rows.argtypes = [C.c_void_p, C.c_int64, C.c_int64, C.c_int, C.c_void_p]
    L.mcmi_result_sizes.argtypes = [C.c_void_p, _i64p, _i64p]
    L.mcmi_derive_chain_budget.argtypes = [C.c_void_p, C.c_double, _i64p, _i64p, C.c_char_p, C.c_size_t]
    L.mcmi_augment_and_split.argtypes = [C.c_void_p, C.c_double, C.c_int32, C.c_int, C.POINTER(C.c_void_p),
                                         C.c_char_p, C.c_size_t]
    L.mcmi_split_sizes.argtypes = [C.c_void_p, _i64p, _i64p, _i64p, _f64p]
    L.mcmi_split_copy.argtypes = [C.c_void_p] + [C.c_void_p] * 9
    L.mcmi_split_free.argtypes = [C.c_void_p]
    L.mcmi_split_free.restype = None
    L.mcmi_drop_small_entries.argtypes = [C.c_void_p, C.c_double, C.c_int32, C.c_int, C.c_void_p, C.c_void_p,
                                          C.c_void_p, _i64p, C.c_char_p, C.c_size_t]
    L.mcmi_transition_probabilities.argtypes = [C.c_void_p, C.c_int, C.c_void_p, C.c_void_p, C.c_void_p, _i64p,
                                                C.c_char_p, C.c_size_t]
    L.mcmi_result_copy.argtypes = [C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p,
                                   _i64p, _i64p]
    L.mcmi_result_view.argtypes = [C.c_void_p] + [C.POINTER(C.c_void_p)] * 5
    L.mcmi_build_start.argtypes = [C.POINTER(mcmi_csr_view), C.POINTER(mcmi_config), C.c_int64, C.c_int64,
                                   C.POINTER(C.c_void_p), C.c_char_p, C.c_size_t]
    L.mcmi_job_estimate.argtypes = [C.c_void_p, _i64p]
    L.mcmi_retain_top_k.argtypes = [C.POINTER(mcmi_csr_view), C.c_int64, C.c_void_p, C.c_int, C.c_void_p,
                                    C.c_void_p, C.c_void_p, _i64p, C.c_char_p, C.c_size_t]
    L.mcmi_scale_columns.argtypes = [C.POINTER(mcmi_csr_view), C.c_void_p, C.c_int64, C.c_int, C.c_void_p,
                                     C.c_char_p, C.c_size_t]
    L.mcmi_estimate_rows.argtypes = [C.POINTER(mcmi_csr_view), C.c_void_p, C.c_int64, C.c_int64, C.c_int64,
                                     C.c_int64, C.c_double, C.c_uint64, C.c_int32, C.c_int, C.POINTER(C.c_void_p),
                                     C.c_char_p, C.c_size_t]
    L.mcmi_job_finish.argtypes = [C.c_void_p, C.POINTER(C.c_void_p), _i64p, C.c_char_p, C.c_size_t]
    L.mcmi_job_attach.argtypes = [C.c_void_p, C.c_void_p, C.c_void_p, C.c_int64]
    L.mcmi_result_copy_range.argtypes = [C.c_void_p, C.c_int64, C.c_int64, C.c_void_p, C.c_void_p]
    L.mcmi_result_stats.argtypes = [C.c_void_p, C.POINTER(mcmi_stats)]
    L.mcmi_result_free.argtypes = [C.c_void_p]
    L.mcmi_result_free.restype = None
    L.mcmi_engine_create.argtypes = [C.c_int, C.POINTER(C.c_void_p), C.c_char_p, C.c_size_t]
    L.mcmi_engine_destroy.argtypes = [C.c_void_p]
    L.mcmi_engine_destroy.restype = None
    L.mcmi_engine_build.argtypes = [C.c_void_p, C.POINTER(mcmi_csr_view), C.POINTER(mcmi_config), C.c_int64,
                                    C.c_int64, C.c_void_p, C.POINTER(mcmi_device_csr), C.POINTER(mcmi_stats),
                                    C.c_char_p, C.c_size_t]
    L.mcmi_copy.argtypes = [C.c_void_p, C.c_void_p, C.c_size_t, C.c_void_p]
    L.mcmi_version.restype = C.c_char_p
    L.mcmi_host_register.argtypes = [C.c_void_p, C.c_size_t]
    L.mcmi_host_unregister.argtypes = [C.c_void_p]
    L.mcmi_solver_config_default.argtypes = [C.POINTER(mcmi_solver_config)]
    L.mcmi_solver_config_default.restype = None
    L.mcmi_solve_device.argtypes = [C.POINTER(mcmi_csr_view), C.POINTER(mcmi_csr_view), C.c_void_p, C.c_void_p,
                                    C.POINTER(mcmi_solver_config), C.c_int, C.c_void_p,
                                    C.POINTER(mcmi_solve_report), C.c_char_p, C.c_size_t]
    L.mcmi_from_triplets.argtypes = [C.c_int64, C.c_void_p, C.c_void_p, C.c_void_p, C.c_int64,
                                     C.POINTER(C.c_void_p), C.c_char_p, C.c_size_t]
    L.mcmi_mm_parse.argtypes = [C.c_char_p, C.c_size_t, C.POINTER(C.c_void_p), C.c_char_p, C.c_size_t]
    L.mcmi_mm_read_file.argtypes = [C.c_char_p, C.POINTER(C.c_void_p), C.c_char_p, C.c_size_t]
    L.mcmi_host_csr_get.argtypes = [C.c_void_p, C.POINTER(mcmi_csr_view)]
    L.mcmi_host_csr_get.restype = None
    L.mcmi_host_csr_free.argtypes = [C.c_void_p]
    L.mcmi_host_csr_free.restype = None
    L.mcmi_mm_format.argtypes = [C.POINTER(mcmi_csr_view), C.c_void_p, C.c_size_t, C.POINTER(C.c_size_t),
                                 C.c_char_p, C.c_size_t]
    L.mcmi_mm_write_file.argtypes = [C.POINTER(mcmi_csr_view), C.c_char_p, C.c_char_p, C.c_size_t]
    L.mcmi_recover_inverse.argtypes = [C.c_void_p, C.c_int64, C.c_void_p, C.c_int64, C.c_double, C.c_int,
                                       C.c_char_p, C.c_size_t]
    L.mcmi_recover_inverse_device.argtypes = [C.c_void_p, C.c_int64, C.c_void_p, C.c_int64, C.c_double, C.c_int,
                                              C.c_void_p, C.c_char_p, C.c_size_t]
    L.mcmi_scatter_shard.argtypes = [C.c_void_p, C.c_void_p, C.c_void_p, C.c_int64, C.c_int64, C.c_int64,
                                     C.c_int64, C.c_int64, C.c_int64, C.POINTER(C.c_void_p), C.c_int, C.c_void_p]
    _lib = L
    return L
