"""ctypes binding of oracle/_ref/libmcspai_ref.so — TEST INFRASTRUCTURE ONLY.

The library is the unmodified reference (``/root/reference/proj/src``) compiled
by ``oracle/Makefile`` plus ``oracle/ref_shim.cpp``.  Only ``tests/``,
``__graft_entry__.smoke()`` and ``bench.py`` (cpu_baseline leg and
``--impl reference``) import this module; the product never does.
"""
from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "_ref", "libmcspai_ref.so")

_i64p = C.POINTER(C.c_int64)
_f64p = C.POINTER(C.c_double)


class RefConfig(C.Structure):
    """Mirror of mcspai::McConfig (mc_engine.hpp:15-26)."""

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
    ]


class RefError(RuntimeError):
    def __init__(self, code: int, msg: str):
        super().__init__(msg)
        self.code = code  # 1 invalid_argument, 2 SplitError, 3 out_of_range, 4 other


_lib = None


def available() -> bool:
    return os.path.exists(LIB_PATH)


def lib():
    global _lib
    if _lib is None:
        if not available():
            raise FileNotFoundError(f"{LIB_PATH} missing: run `make -C oracle ref`")
        L = C.CDLL(LIB_PATH)
        L.ref_build.argtypes = [C.c_int64, _i64p, _i64p, _f64p, C.POINTER(RefConfig),
                                C.c_int, C.c_int, C.POINTER(C.c_void_p), C.c_char_p, C.c_size_t]
        L.ref_build_timed.argtypes = [C.c_int64, _i64p, _i64p, _f64p, C.POINTER(RefConfig), C.c_int, C.c_int,
                                      C.POINTER(C.c_void_p), C.POINTER(C.c_double), C.c_char_p, C.c_size_t]
        L.ref_result_sizes.argtypes = [C.c_void_p, _i64p, _i64p]
        L.ref_result_copy.argtypes = [C.c_void_p, _i64p, _i64p, _f64p, _i64p, _i64p, _i64p, _i64p]
        L.ref_result_write_mm.argtypes = [C.c_void_p, C.c_char_p, C.c_char_p, C.c_size_t]
        L.ref_result_free.argtypes = [C.c_void_p]
        L.ref_csr_sizes.argtypes = [C.c_void_p, _i64p, _i64p]
        L.ref_csr_copy.argtypes = [C.c_void_p, _i64p, _i64p, _f64p]
        L.ref_csr_free.argtypes = [C.c_void_p]
        L.ref_gen.argtypes = [C.c_int, C.c_int64, C.c_double, C.c_double, C.c_double, C.c_uint64]
        L.ref_gen.restype = C.c_void_p
        L.ref_write_mm.argtypes = [C.c_int64, _i64p, _i64p, _f64p, C.c_char_p, C.c_char_p, C.c_size_t]
        L.ref_read_mm.argtypes = [C.c_char_p, C.POINTER(C.c_void_p), C.c_char_p, C.c_size_t]
        L.ref_parse_mm.argtypes = [C.c_char_p, C.c_size_t, C.POINTER(C.c_void_p), C.c_char_p, C.c_size_t]
        L.ref_format_mm.argtypes = [C.c_int64, _i64p, _i64p, _f64p, C.POINTER(C.c_size_t)]
        L.ref_format_mm.restype = C.c_void_p
        L.ref_free_buf.argtypes = [C.c_void_p]
        L.ref_recover.argtypes = [C.c_int64, _f64p, _f64p, C.c_int64, C.c_double, _f64p, C.c_char_p, C.c_size_t]
        L.ref_dense_inverse.argtypes = [C.c_int64, _f64p, _f64p, C.c_char_p, C.c_size_t]
        L.ref_from_triplets.argtypes = [C.c_int64, _i64p, _i64p, _f64p, C.c_int64, C.POINTER(C.c_void_p),
                                        C.c_char_p, C.c_size_t]
        L.ref_drop.argtypes = [C.c_int64, _i64p, _i64p, _f64p, C.c_double, C.c_int,
                               C.POINTER(C.c_void_p), C.c_char_p, C.c_size_t]
        L.ref_split.argtypes = [C.c_int64, _i64p, _i64p, _f64p, C.c_double, C.c_int,
                                C.POINTER(C.c_void_p), C.c_char_p, C.c_size_t]
        L.ref_split_matrix.argtypes = [C.c_void_p, C.c_int]
        L.ref_split_matrix.restype = C.c_void_p
        L.ref_split_diag.argtypes = [C.c_void_p, _f64p, _f64p, _f64p]
        L.ref_split_free.argtypes = [C.c_void_p]
        L.ref_split_from_ap.argtypes = [C.c_int64, _i64p, _i64p, _f64p, _f64p]
        L.ref_split_from_ap.restype = C.c_void_p
        L.ref_budget.argtypes = [C.POINTER(RefConfig), C.c_double, _i64p, _i64p, C.c_char_p, C.c_size_t]
        L.ref_estimate_row.argtypes = [C.c_void_p, C.c_int64, C.c_int64, C.c_int64, C.c_double,
                                       C.c_uint64, _i64p, _f64p, C.c_int64]
        L.ref_estimate_row.restype = C.c_int64
        L.ref_retain_top_k.argtypes = [C.c_int64, _i64p, _f64p, C.c_int64, C.c_int64]
        L.ref_retain_top_k.restype = C.c_int64
        L.ref_rng_u32.argtypes = [C.c_uint64, C.c_uint64, C.c_int64, C.POINTER(C.c_uint32)]
        L.ref_rng_double.argtypes = [C.c_uint64, C.c_uint64, C.c_int64, _f64p]
        L.ref_max_threads.restype = C.c_int
        L.ref_solve.argtypes = [C.c_int64, _i64p, _i64p, _f64p, C.c_int64, _i64p, _i64p, _f64p, C.c_int,
                                C.c_double, C.c_int64, C.c_int64, _i64p, C.POINTER(C.c_int), _f64p,
                                C.c_char_p, C.c_size_t]
        _lib = L
    return _lib


def _p(a, t):
    return a.ctypes.data_as(t)


@dataclass
class Csr:
    n: int
    row_ptr: np.ndarray  # int64[n+1]
    col_idx: np.ndarray  # int64[nnz]
    values: np.ndarray  # float64[nnz]

    @property
    def nnz(self) -> int:
        return int(self.row_ptr[-1])

    def args(self):
        rp = np.ascontiguousarray(self.row_ptr, dtype=np.int64)
        ci = np.ascontiguousarray(self.col_idx, dtype=np.int64)
        v = np.ascontiguousarray(self.values, dtype=np.float64)
        if ci.size == 0:
            ci = np.zeros(1, np.int64)
            v = np.zeros(1, np.float64)
        return rp, ci, v


def _csr_from_handle(h) -> Csr:
    L = lib()
    n, nnz = C.c_int64(), C.c_int64()
    L.ref_csr_sizes(h, C.byref(n), C.byref(nnz))
    rp = np.empty(n.value + 1, np.int64)
    ci = np.empty(max(nnz.value, 1), np.int64)
    v = np.empty(max(nnz.value, 1), np.float64)
    L.ref_csr_copy(h, _p(rp, _i64p), _p(ci, _i64p), _p(v, _f64p))
    return Csr(n.value, rp, ci[: nnz.value], v[: nnz.value])


def make_config(**kw) -> RefConfig:
    c = RefConfig(epsilon=0.0625, delta=0.0625, alpha=5.0, mode=1, drop_mode=0,
                  drop_fraction=0.0, retain_k=0, has_chains_override=0,
                  has_max_len_override=0, chains_override=0, max_len_override=0,
                  master_seed=0)
    for k, v in kw.items():
        if k == "chains_override":
            if v is not None:
                c.has_chains_override, c.chains_override = 1, int(v)
        elif k == "max_len_override":
            if v is not None:
                c.has_max_len_override, c.max_len_override = 1, int(v)
        elif k in ("rng_mode", "device"):
            continue
        else:
            setattr(c, k, v)
    return c


@dataclass
class RefResult:
    m: Csr
    chains_used: np.ndarray
    entries_before: np.ndarray
    n_chains: int
    max_len: int
    build_s: float = 0.0  #: wall time of the reference call alone (ref_build_timed)


def _check(code, err):
    if code:
        raise RefError(code, err.value.decode(errors="replace"))


def compute_preconditioner(b: Csr, n_threads: int = 0, serial: bool = False,
                           mm_path: str | None = None, copy: bool = True, **cfg) -> RefResult:
    """The reference's compute_preconditioner(_serial) on b.  ``build_s`` is
    the wall time of that call alone; copy=False skips copying M out (timing
    runs)."""
    L = lib()
    c = make_config(**cfg)
    rp, ci, v = b.args()
    h = C.c_void_p()
    err = C.create_string_buffer(512)
    secs = C.c_double(0.0)
    code = L.ref_build_timed(b.n, _p(rp, _i64p), _p(ci, _i64p), _p(v, _f64p), C.byref(c),
                             n_threads, int(serial), C.byref(h), C.byref(secs), err, 512)
    _check(code, err)
    if not copy:
        L.ref_result_free(h)
        return RefResult(Csr(b.n, np.zeros(1, np.int64), np.zeros(0, np.int64), np.zeros(0)),
                         np.zeros(0, np.int64), np.zeros(0, np.int64), 0, 0, secs.value)
    try:
        n, nnz = C.c_int64(), C.c_int64()
        L.ref_result_sizes(h, C.byref(n), C.byref(nnz))
        orp = np.empty(n.value + 1, np.int64)
        oci = np.empty(max(nnz.value, 1), np.int64)
        ov = np.empty(max(nnz.value, 1), np.float64)
        cu = np.empty(max(n.value, 1), np.int64)
        eb = np.empty(max(n.value, 1), np.int64)
        nc, ml = C.c_int64(), C.c_int64()
        L.ref_result_copy(h, _p(orp, _i64p), _p(oci, _i64p), _p(ov, _f64p), _p(cu, _i64p),
                          _p(eb, _i64p), C.byref(nc), C.byref(ml))
        if mm_path:
            _check(L.ref_result_write_mm(h, mm_path.encode(), err, 512), err)
    finally:
        L.ref_result_free(h)
    return RefResult(Csr(n.value, orp, oci[: nnz.value], ov[: nnz.value]),
                     cu[: n.value], eb[: n.value], nc.value, ml.value, secs.value)


# generator kinds (ref_shim.cpp ref_gen)
def gen_tridiagonal(n):
    return _gen(0, n)


def gen_convection_diffusion(grid, conv_x=20.0, conv_y=10.0):
    return _gen(1, grid, conv_x, conv_y)


def gen_brusselator(grid):
    return _gen(2, grid)


def gen_random_ddm(n, fill, seed):
    return _gen(3, n, fill, seed=seed)


def gen_broad_spectrum(n, nnz_per_row, lo, hi, seed):
    return _gen(4, n, float(nnz_per_row), lo, hi, seed)


def _gen(kind, a, x=0.0, y=0.0, z=0.0, seed=0) -> Csr:
    L = lib()
    h = L.ref_gen(kind, a, x, y, z, seed)
    try:
        return _csr_from_handle(h)
    finally:
        L.ref_csr_free(h)


def write_mm(m: Csr, path: str):
    L = lib()
    rp, ci, v = m.args()
    err = C.create_string_buffer(512)
    _check(L.ref_write_mm(m.n, _p(rp, _i64p), _p(ci, _i64p), _p(v, _f64p), path.encode(), err, 512), err)


def read_mm(path: str) -> Csr:
    L = lib()
    h = C.c_void_p()
    err = C.create_string_buffer(512)
    _check(L.ref_read_mm(path.encode(), C.byref(h), err, 512), err)
    try:
        return _csr_from_handle(h)
    finally:
        L.ref_csr_free(h)


def parse_mm(text: bytes) -> Csr:
    """parse_matrix_market (matrix_market.cpp:27-147) over an in-memory text."""
    L = lib()
    h = C.c_void_p()
    err = C.create_string_buffer(512)
    _check(L.ref_parse_mm(text, len(text), C.byref(h), err, 512), err)
    try:
        return _csr_from_handle(h)
    finally:
        L.ref_csr_free(h)


def format_mm(m: Csr) -> bytes:
    """write_matrix_market (matrix_market.cpp:155-169) into memory."""
    L = lib()
    rp, ci, v = m.args()
    n = C.c_size_t()
    p = L.ref_format_mm(m.n, _p(rp, _i64p), _p(ci, _i64p), _p(v, _f64p), C.byref(n))
    try:
        return C.string_at(p, n.value)
    finally:
        L.ref_free_buf(p)


def recover_inverse(m, s_diag, tol: float = 1e-12):
    """recover_inverse (recovery.cpp:7-33) on a dense row-major n x n matrix."""
    L = lib()
    a = np.ascontiguousarray(m, np.float64)
    s = np.ascontiguousarray(s_diag, np.float64)
    out = np.empty_like(a)
    err = C.create_string_buffer(512)
    _check(L.ref_recover(a.shape[0], _p(a, _f64p), _p(s, _f64p), s.size, tol, _p(out, _f64p), err, 512), err)
    return out


def dense_inverse(m):
    """dense_inverse (dense_solve.cpp): Gauss-Jordan with partial pivoting."""
    L = lib()
    a = np.ascontiguousarray(m, np.float64)
    out = np.empty_like(a)
    err = C.create_string_buffer(512)
    _check(L.ref_dense_inverse(a.shape[0], _p(a, _f64p), _p(out, _f64p), err, 512), err)
    return out


def from_triplets(n: int, rows, cols, vals) -> Csr:
    """CsrMatrix::from_triplets (csr.cpp:17-58)."""
    L = lib()
    r = np.ascontiguousarray(rows, np.int64)
    c = np.ascontiguousarray(cols, np.int64)
    v = np.ascontiguousarray(vals, np.float64)
    h = C.c_void_p()
    err = C.create_string_buffer(512)
    _check(L.ref_from_triplets(n, _p(r, _i64p), _p(c, _i64p), _p(v, _f64p), r.size, C.byref(h), err, 512), err)
    try:
        return _csr_from_handle(h)
    finally:
        L.ref_csr_free(h)


def drop_small_entries(m: Csr, p: float, drop_mode: int = 0) -> Csr:
    L = lib()
    rp, ci, v = m.args()
    h = C.c_void_p()
    err = C.create_string_buffer(512)
    _check(L.ref_drop(m.n, _p(rp, _i64p), _p(ci, _i64p), _p(v, _f64p), p, drop_mode,
                      C.byref(h), err, 512), err)
    try:
        return _csr_from_handle(h)
    finally:
        L.ref_csr_free(h)


@dataclass
class RefSplit:
    b_hat: Csr
    a: Csr
    p: Csr
    b1_diag: np.ndarray
    s_diag: np.ndarray
    a_norm: float
    handle: int = 0


def augment_and_split(b: Csr, alpha: float, mode: int = 1, keep_handle=False) -> RefSplit:
    L = lib()
    rp, ci, v = b.args()
    h = C.c_void_p()
    err = C.create_string_buffer(512)
    _check(L.ref_split(b.n, _p(rp, _i64p), _p(ci, _i64p), _p(v, _f64p), alpha, mode,
                       C.byref(h), err, 512), err)
    mats = [_csr_from_handle(L.ref_split_matrix(h, w)) for w in range(3)]
    b1 = np.empty(max(b.n, 1))
    s = np.empty(max(b.n, 1))
    an = C.c_double()
    L.ref_split_diag(h, _p(b1, _f64p), _p(s, _f64p), C.byref(an))
    out = RefSplit(*mats, b1[: b.n], s[: b.n], an.value)
    if keep_handle:
        out.handle = h.value
    else:
        L.ref_split_free(h)
    return out


def free_split(sp: RefSplit):
    if sp.handle:
        lib().ref_split_free(C.c_void_p(sp.handle))
        sp.handle = 0


def derive_chain_budget(a_norm: float, **cfg):
    L = lib()
    c = make_config(**cfg)
    nc, ml = C.c_int64(), C.c_int64()
    err = C.create_string_buffer(512)
    _check(L.ref_budget(C.byref(c), a_norm, C.byref(nc), C.byref(ml), err, 512), err)
    return nc.value, ml.value


def estimate_row(sp: RefSplit, r: int, n_chains: int, max_len: int, delta: float, seed: int):
    L = lib()
    cap = sp.a.n
    cols = np.empty(max(cap, 1), np.int64)
    vals = np.empty(max(cap, 1), np.float64)
    ln = L.ref_estimate_row(C.c_void_p(sp.handle), r, n_chains, max_len, delta, seed,
                            _p(cols, _i64p), _p(vals, _f64p), cap)
    return cols[:ln].copy(), vals[:ln].copy()


def retain_top_k(cols, vals, k: int, diag_col: int):
    L = lib()
    c = np.ascontiguousarray(cols, np.int64).copy()
    v = np.ascontiguousarray(vals, np.float64).copy()
    ln = L.ref_retain_top_k(len(c), _p(c, _i64p), _p(v, _f64p), k, diag_col)
    return c[:ln], v[:ln]


def rng_u32(seed: int, sid: int, count: int) -> np.ndarray:
    out = np.empty(count, np.uint32)
    lib().ref_rng_u32(seed, sid, count, out.ctypes.data_as(C.POINTER(C.c_uint32)))
    return out


def rng_double(seed: int, sid: int, count: int) -> np.ndarray:
    out = np.empty(count, np.float64)
    lib().ref_rng_double(seed, sid, count, _p(out, _f64p))
    return out


def max_threads() -> int:
    return lib().ref_max_threads()


def solve(b: Csr, m: Csr | None, method: str = "gmres", rel_tol: float = 1e-6, max_iters: int = 30000,
          restart: int = 50):
    """mcspai::solve (solvers.cpp:240-244) with rhs = B*1 (ones_product_rhs):
    returns (iterations, converged, final_rel_residual)."""
    L = lib()
    rp, ci, v = b.args()
    if m is not None:
        mrp, mci, mv = m.args()
        nm = m.n
    else:
        mrp, mci, mv = np.zeros(1, np.int64), np.zeros(1, np.int64), np.zeros(1)
        nm = -1
    it, conv, res = C.c_int64(), C.c_int(), C.c_double()
    err = C.create_string_buffer(512)
    _check(L.ref_solve(b.n, _p(rp, _i64p), _p(ci, _i64p), _p(v, _f64p), nm, _p(mrp, _i64p), _p(mci, _i64p),
                       _p(mv, _f64p), 0 if method == "gmres" else 1, rel_tol, max_iters, restart,
                       C.byref(it), C.byref(conv), C.byref(res), err, 512), err)
    return it.value, bool(conv.value), res.value


def split_from_ap(n, row_ptr, col_idx, a_values, p_values):
    """A hand-built SplitSystem handle (split.a, split.p on A's pattern); free with free_split."""
    rp = np.ascontiguousarray(row_ptr, np.int64)
    ci = np.ascontiguousarray(col_idx if len(col_idx) else np.zeros(1, np.int64), np.int64)
    av = np.ascontiguousarray(a_values if len(a_values) else np.zeros(1), np.float64)
    pv = np.ascontiguousarray(p_values if len(p_values) else np.zeros(1), np.float64)
    h = lib().ref_split_from_ap(n, _p(rp, _i64p), _p(ci, _i64p), _p(av, _f64p), _p(pv, _f64p))
    a = Csr(n, rp, ci[: rp[-1]], av[: rp[-1]])
    return RefSplit(a, a, Csr(n, rp, ci[: rp[-1]], pv[: rp[-1]]), np.ones(n), np.zeros(n), 0.5, handle=h)
