"""ctypes binding of the plain-C restatement (oracle/_build/libmcmi_oracle.so).

TEST INFRASTRUCTURE ONLY: imported by tests/, __graft_entry__.smoke() and the
cpu_baseline leg of bench.py — never by the product package.
"""
from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "_build", "libmcmi_oracle.so")

_i64p = C.POINTER(C.c_int64)
_f64p = C.POINTER(C.c_double)


class OrcConfig(C.Structure):
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


class OracleError(RuntimeError):
    def __init__(self, code, msg):
        super().__init__(msg)
        self.code = code


_lib = None


def build():
    import subprocess
    subprocess.run(["make", "-s", "-C", _HERE, "oracle"], check=True)


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            build()
        L = C.CDLL(LIB_PATH)
        L.orc_build.argtypes = [C.c_int64, _i64p, _i64p, _f64p, C.POINTER(OrcConfig), C.c_int64,
                                C.c_int64, C.POINTER(C.c_void_p), C.c_char_p, C.c_size_t]
        L.orc_result_sizes.argtypes = [C.c_void_p, _i64p, _i64p]
        L.orc_result_copy.argtypes = [C.c_void_p, _i64p, _i64p, _f64p, _i64p, _i64p, _i64p, _i64p,
                                      _i64p, _i64p, _f64p]
        L.orc_result_free.argtypes = [C.c_void_p]
        L.orc_philox.argtypes = [C.POINTER(C.c_uint32), C.POINTER(C.c_uint32), C.POINTER(C.c_uint32)]
        _lib = L
    return _lib


def make_config(**kw) -> OrcConfig:
    c = OrcConfig(epsilon=0.0625, delta=0.0625, alpha=5.0, mode=1, drop_mode=0, drop_fraction=0.0,
                  retain_k=0, has_chains_override=0, has_max_len_override=0, chains_override=0,
                  max_len_override=0, master_seed=0, rng_mode=0, device=0, flags=0, n_gpus=0)
    for k, v in kw.items():
        if k == "chains_override":
            if v is not None:
                c.has_chains_override, c.chains_override = 1, int(v)
        elif k == "max_len_override":
            if v is not None:
                c.has_max_len_override, c.max_len_override = 1, int(v)
        elif k == "deg_stats":
            continue
        else:
            setattr(c, k, v)
    return c


@dataclass
class OracleResult:
    row_ptr: np.ndarray
    col_idx: np.ndarray
    values: np.ndarray
    chains_used: np.ndarray
    entries_before: np.ndarray
    n_chains: int
    max_len: int
    walk_steps: int
    walk_deg_sum: int
    a_norm: float


def compute_preconditioner(n, row_ptr, col_idx, values, row_begin=0, row_end=-1, **cfg) -> OracleResult:
    L = lib()
    c = make_config(**cfg)
    rp = np.ascontiguousarray(row_ptr, np.int64)
    ci = np.ascontiguousarray(col_idx, np.int64)
    v = np.ascontiguousarray(values, np.float64)
    if ci.size == 0:
        ci, v = np.zeros(1, np.int64), np.zeros(1)
    h = C.c_void_p()
    err = C.create_string_buffer(512)
    code = L.orc_build(n, rp.ctypes.data_as(_i64p), ci.ctypes.data_as(_i64p), v.ctypes.data_as(_f64p),
                       C.byref(c), row_begin, row_end, C.byref(h), err, 512)
    if code:
        raise OracleError(code, err.value.decode())
    try:
        nr, nnz = C.c_int64(), C.c_int64()
        L.orc_result_sizes(h, C.byref(nr), C.byref(nnz))
        orp = np.empty(nr.value + 1, np.int64)
        oci = np.empty(max(nnz.value, 1), np.int64)
        ov = np.empty(max(nnz.value, 1))
        cu = np.empty(max(nr.value, 1), np.int64)
        eb = np.empty(max(nr.value, 1), np.int64)
        nc, ml, ws, wd = C.c_int64(), C.c_int64(), C.c_int64(), C.c_int64()
        an = C.c_double()
        L.orc_result_copy(h, orp.ctypes.data_as(_i64p), oci.ctypes.data_as(_i64p), ov.ctypes.data_as(_f64p),
                          cu.ctypes.data_as(_i64p), eb.ctypes.data_as(_i64p), C.byref(nc), C.byref(ml),
                          C.byref(ws), C.byref(wd), C.byref(an))
    finally:
        L.orc_result_free(h)
    return OracleResult(orp, oci[: nnz.value], ov[: nnz.value], cu[: nr.value], eb[: nr.value],
                        nc.value, ml.value, ws.value, wd.value, an.value)


def philox(ctr, key):
    L = lib()
    c = (C.c_uint32 * 4)(*ctr)
    k = (C.c_uint32 * 2)(*key)
    o = (C.c_uint32 * 4)()
    L.orc_philox(c, k, o)
    return list(o)


def write_mm_bytes(n, row_ptr, col_idx, values) -> bytes:
    """write_matrix_market (matrix_market.cpp:155-169) formatting, '%.17g'."""
    out = [b"%%MatrixMarket matrix coordinate real general\n",
           b"%d %d %d\n" % (n, n, int(row_ptr[-1]))]
    rp = np.asarray(row_ptr)
    ci = np.asarray(col_idx)
    v = np.asarray(values)
    rows = np.repeat(np.arange(n, dtype=np.int64), np.diff(rp))
    out.extend(b"%d %d %.17g\n" % (int(r) + 1, int(c) + 1, float(x)) for r, c, x in zip(rows, ci, v))
    return b"".join(out)
