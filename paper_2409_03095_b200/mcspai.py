"""Python mirror of the reference's preconditioner-build interface.

Same names, argument meaning and error behaviour as
``/root/reference/proj/include/mcspai/mc_engine.hpp`` and ``split.hpp`` /
``csr.hpp``, so the parity tests read like the reference's own tests:

=========================  ===============================================
reference (C++)            here
=========================  ===============================================
``McConfig``               :class:`McConfig` (+ ``rng_mode``, ``device``, ``n_gpus``)
``CsrMatrix``              :class:`CsrMatrix` (int64 / float64 numpy)
``ApproxInverse``          :class:`ApproxInverse`
``RowMeta``                :class:`RowMeta` (column arrays)
``ChainBudget``            :class:`ChainBudget`
``compute_preconditioner`` :func:`compute_preconditioner`
``std::invalid_argument``  :class:`ValueError`
``SplitError``             :class:`SplitError`
``std::out_of_range``      :class:`IndexError`
=========================  ===============================================

Every call goes through the C-ABI (include/mcmi.h) into the sm_100a kernels.
``n_threads`` is accepted for signature compatibility.  A host build uses
``McConfig.n_gpus`` GPUs of this process (row blocks, one host thread per
GPU); one process per GPU with device-resident shards is
:mod:`paper_2409_03095_b200.distributed`.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, field
from enum import IntEnum
from typing import Optional

import numpy as np

from . import _lib as L

index_t = np.int64


class AugmentationMode(IntEnum):  # split.hpp:9-12
    plain = 0
    sign_aware = 1


class DropMode(IntEnum):  # csr.hpp:61-64
    value_range = 0
    count_quantile = 1


class RngMode(IntEnum):
    reference = 0  #: RngStream(seed, row): byte-identical to the reference
    keyed = 1  #: Philox keyed by (row, chain, step)


class SplitError(RuntimeError):
    """mcspai::SplitError (split.hpp:14-16)."""


class ParseError(RuntimeError):  # matrix_market.hpp:12-14
    pass


class DeviceError(RuntimeError):
    """CUDA runtime / device failure (no CPU fallback exists)."""


@dataclass
class McConfig:  # mc_engine.hpp:15-26
    epsilon: float = 0.0625
    delta: float = 0.0625
    alpha: float = 5.0
    mode: AugmentationMode = AugmentationMode.sign_aware
    drop_fraction: float = 0.0
    drop_mode: DropMode = DropMode.value_range
    retain_k: int = 0
    chains_override: Optional[int] = None
    max_len_override: Optional[int] = None
    master_seed: int = 0
    rng_mode: RngMode = RngMode.reference
    device: int = 0
    #: GPUs of a host build (row blocks on devices device..device+n_gpus-1, one
    #: host thread each); 0 = env MCMI_GPUS, else 1.  M does not depend on it.
    n_gpus: int = 0
    deg_stats: bool = False  #: also count sum deg(s) over steps (stats["walk_deg_sum"]); ~4% slower
    #: rows of (I - A)^-1 as estimate_row returns them: no scale_columns, no zero prune
    unscaled: bool = False

    def to_c(self) -> L.mcmi_config:
        c = L.mcmi_config()
        c.epsilon = float(self.epsilon)
        c.delta = float(self.delta)
        c.alpha = float(self.alpha)
        c.mode = int(self.mode)
        c.drop_mode = int(self.drop_mode)
        c.drop_fraction = float(self.drop_fraction)
        c.retain_k = int(self.retain_k)
        c.has_chains_override = int(self.chains_override is not None)
        c.chains_override = int(self.chains_override or 0)
        c.has_max_len_override = int(self.max_len_override is not None)
        c.max_len_override = int(self.max_len_override or 0)
        c.master_seed = int(self.master_seed) & 0xFFFFFFFFFFFFFFFF
        c.rng_mode = int(self.rng_mode)
        c.device = int(self.device)
        c.n_gpus = int(self.n_gpus)
        c.flags = (L.MCMI_FLAG_DEG_STATS if self.deg_stats else 0) | (L.MCMI_FLAG_UNSCALED if self.unscaled else 0)
        return c

    def oracle_kwargs(self) -> dict:
        """Field dict accepted by oracle.make_config / ref.make_config (tests)."""
        return dict(epsilon=self.epsilon, delta=self.delta, alpha=self.alpha, mode=int(self.mode),
                    drop_fraction=self.drop_fraction, drop_mode=int(self.drop_mode),
                    retain_k=int(self.retain_k), chains_override=self.chains_override,
                    max_len_override=self.max_len_override, master_seed=int(self.master_seed),
                    rng_mode=int(self.rng_mode))


@dataclass
class CsrMatrix:  # csr.hpp:16-40
    n: int = 0
    row_ptr: np.ndarray = field(default_factory=lambda: np.zeros(1, np.int64))
    col_idx: np.ndarray = field(default_factory=lambda: np.zeros(0, np.int64))
    values: np.ndarray = field(default_factory=lambda: np.zeros(0, np.float64))

    def __post_init__(self):
        self.row_ptr = np.ascontiguousarray(self.row_ptr, dtype=np.int64)
        self.col_idx = np.ascontiguousarray(self.col_idx, dtype=np.int64)
        self.values = np.ascontiguousarray(self.values, dtype=np.float64)

    def nnz(self) -> int:
        return int(self.values.size)

    def row_begin(self, i: int) -> int:
        return int(self.row_ptr[i])

    def row_end(self, i: int) -> int:
        return int(self.row_ptr[i + 1])

    def at(self, i: int, j: int) -> float:
        a, b = self.row_ptr[i], self.row_ptr[i + 1]
        k = a + np.searchsorted(self.col_idx[a:b], j)
        return float(self.values[k]) if k < b and self.col_idx[k] == j else 0.0

    def __eq__(self, other) -> bool:  # `operator== = default`
        return (isinstance(other, CsrMatrix) and self.n == other.n
                and np.array_equal(self.row_ptr, other.row_ptr)
                and np.array_equal(self.col_idx, other.col_idx)
                and np.array_equal(self.values.view(np.uint64), other.values.view(np.uint64)))

    @staticmethod
    def identity(n: int) -> "CsrMatrix":
        return CsrMatrix(n, np.arange(n + 1), np.arange(n), np.ones(n))

    @staticmethod
    def from_triplets(n, rows, cols, vals) -> "CsrMatrix":
        """csr.cpp:17-58 (native, mcmi_from_triplets): sort by (row, col), sum
        duplicates in the reference's sort order, prune exact zeros."""
        rows = np.ascontiguousarray(rows, np.int64)
        cols = np.ascontiguousarray(cols, np.int64)
        vals = np.ascontiguousarray(vals, np.float64)
        if not (rows.size == cols.size == vals.size):
            raise ValueError("triplet arrays must have equal length")
        h = C.c_void_p()
        err = C.create_string_buffer(512)
        code = L.load().mcmi_from_triplets(int(n), rows.ctypes.data, cols.ctypes.data, vals.ctypes.data,
                                           rows.size, C.byref(h), err, 512)
        raise_for(code, err.value.decode(errors="replace"))
        return host_csr_take(h)


def host_csr_take(h) -> CsrMatrix:
    """Copies a library-owned mcmi_host_csr into a CsrMatrix and frees it."""
    lib = L.load()
    try:
        v = L.mcmi_csr_view()
        lib.mcmi_host_csr_get(h, C.byref(v))
        n = int(v.n)
        nnz = 0
        rp = np.zeros(max(n, 0) + 1, np.int64)
        if n > 0:
            C.memmove(rp.ctypes.data, v.row_ptr, (n + 1) * 8)
            nnz = int(rp[-1])
        ci = np.empty(nnz, np.int64)
        vals = np.empty(nnz, np.float64)
        if nnz:
            C.memmove(ci.ctypes.data, v.col_idx, nnz * 8)
            C.memmove(vals.ctypes.data, v.values, nnz * 8)
        return CsrMatrix(n, rp, ci, vals)
    finally:
        lib.mcmi_host_csr_free(h)


@dataclass
class ChainBudget:  # mc_engine.hpp:28-31
    n_chains: int = 1
    max_len: int = 1


@dataclass
class RowMeta:  # mc_engine.hpp:33-36, one array entry per row
    chains_used: np.ndarray
    entries_before_retention: np.ndarray


@dataclass
class ApproxInverse:  # mc_engine.hpp:39-45
    m: CsrMatrix
    row_meta: RowMeta
    config_echo: McConfig
    budget_echo: ChainBudget
    seed_echo: int
    stats: dict = field(default_factory=dict)


def raise_for(code: int, msg: str):
    if code == L.MCMI_OK:
        return
    if code == L.MCMI_EINVAL:
        raise ValueError(msg)
    if code == L.MCMI_ESPLIT:
        raise SplitError(msg)
    if code == L.MCMI_ERANGE:
        raise IndexError(msg)
    if code == L.MCMI_ENOMEM:
        raise MemoryError(msg)
    if code == L.MCMI_EPARSE:
        raise ParseError(msg)
    if code == L.MCMI_EIO:
        raise RuntimeError(msg)
    raise DeviceError(f"[status {code}] {msg}")


def compute_preconditioner(b: CsrMatrix, cfg: McConfig | None = None, n_threads: int = 0,
                           out: dict | None = None, rows: tuple[int, int] | None = None) -> ApproxInverse:
    """mcspai::compute_preconditioner (mc_engine.hpp:80-81) on a B200.

    ``out`` may hold preallocated (pinned) numpy arrays ``row_ptr``,
    ``col_idx``, ``values`` of sufficient size to receive the result without
    an extra allocation (used by the end-to-end benchmark).  ``rows`` =
    (begin, end) builds only that row shard (``mcmi_build_rows``).
    """
    del n_threads
    cfg = cfg or McConfig()
    if b.row_ptr.size != b.n + 1 or (b.n > 0 and (b.col_idx.size < b.row_ptr[-1] or b.values.size < b.row_ptr[-1])):
        raise ValueError("CsrMatrix arrays are inconsistent with row_ptr (need n+1 row pointers and "
                         "row_ptr[n] column indices and values)")
    lib = L.load()
    view = L.mcmi_csr_view(int(b.n), b.row_ptr.ctypes.data, b.col_idx.ctypes.data if b.col_idx.size else None,
                           b.values.ctypes.data if b.values.size else None)
    c = cfg.to_c()
    h = C.c_void_p()
    err = C.create_string_buffer(1024)
    lo, hi = rows if rows is not None else (0, -1)
    if out is not None and out.get("values") is not None:
        # streamed build into the caller's (pinned) arrays: the device->host copy
        # of each row chunk overlaps the walks of the next (mcmi_build_into)
        nrows = (b.n if hi < 0 else hi) - lo
        cap = int(min(out["col_idx"].size, out["values"].size))
        rp, ci, v = out["row_ptr"][: nrows + 1], out["col_idx"], out["values"]
        cu, eb = np.empty(max(nrows, 1), np.int64), np.empty(max(nrows, 1), np.int64)
        nnz = C.c_int64()
        st = L.mcmi_stats()
        code = lib.mcmi_build_into(C.byref(view), C.byref(c), lo, hi, rp.ctypes.data, ci.ctypes.data,
                                   v.ctypes.data, cap, cu.ctypes.data, eb.ctypes.data, C.byref(nnz),
                                   C.byref(st), err, 1024)
        if not (code == L.MCMI_ENOMEM and nnz.value > cap):  # too small: fall back to the handle path
            raise_for(code, err.value.decode(errors="replace"))
            k = nnz.value
            return ApproxInverse(CsrMatrix(nrows, rp, ci[:k], v[:k]), RowMeta(cu[:nrows], eb[:nrows]), cfg,
                                 ChainBudget(st.n_chains, st.max_len), int(cfg.master_seed), st.as_dict())
    code = lib.mcmi_build_rows(C.byref(view), C.byref(c), lo, hi, C.byref(h), err, 1024)
    raise_for(code, err.value.decode(errors="replace"))
    owner = _ResultOwner(h)
    n, nnz = C.c_int64(), C.c_int64()
    lib.mcmi_result_sizes(h, C.byref(n), C.byref(nnz))
    n, nnz = n.value, nnz.value
    st = L.mcmi_stats()
    lib.mcmi_result_stats(h, C.byref(st))
    if out is not None and out.get("values") is not None and out["values"].size >= nnz:
        # caller arrays: one multi-threaded host copy out of the result
        rp, ci, v = out["row_ptr"][: n + 1], out["col_idx"][:nnz], out["values"][:nnz]
        cu, eb = np.empty(n, np.int64), np.empty(n, np.int64)
        nc, ml = C.c_int64(), C.c_int64()
        raise_for(lib.mcmi_result_copy(h, rp.ctypes.data, ci.ctypes.data if nnz else None,
                                       v.ctypes.data if nnz else None, cu.ctypes.data if n else None,
                                       eb.ctypes.data if n else None, C.byref(nc), C.byref(ml)), "result copy failed")
    else:
        # zero copy: numpy views of the library's page-locked result arrays,
        # which stay alive (and out of the library's pool) while any view does
        rp, ci, v, cu, eb = owner.arrays(n, nnz)
    return ApproxInverse(CsrMatrix(n, rp, ci, v), RowMeta(cu, eb), cfg, ChainBudget(st.n_chains, st.max_len),
                         int(cfg.master_seed), st.as_dict())


class _ResultOwner:
    """Owns an mcmi_result; numpy views of its host arrays keep it alive."""

    def __init__(self, h):
        self.h = h
        self.lib = L.load()

    def arrays(self, n, nnz):
        ptrs = [C.c_void_p() for _ in range(5)]
        raise_for(self.lib.mcmi_result_view(self.h, *[C.byref(p) for p in ptrs]), "result view failed")

        def view(ptr, count, ctype, dtype):
            if count <= 0 or not ptr.value:
                return np.zeros(max(count, 0), dtype)
            buf = (ctype * count).from_address(ptr.value)
            buf._owner = self  # the ctypes buffer (numpy's base) keeps the result alive
            return np.frombuffer(buf, dtype=dtype)

        return (view(ptrs[0], n + 1, C.c_int64, np.int64), view(ptrs[1], nnz, C.c_int64, np.int64),
                view(ptrs[2], nnz, C.c_double, np.float64), view(ptrs[3], n, C.c_int64, np.int64),
                view(ptrs[4], n, C.c_int64, np.int64))

    def __del__(self):
        try:
            if self.h:
                self.lib.mcmi_result_free(self.h)
                self.h = None
        except Exception:  # noqa: BLE001 — interpreter shutdown
            pass


def host_register(*arrays):
    """Page-locks numpy arrays for the library's DMA (mcmi_host_register) so
    streamed builds into them overlap the device->host copy with the walks."""
    lib = L.load()
    for a in arrays:
        if a is not None and a.size:
            raise_for(lib.mcmi_host_register(a.ctypes.data, a.nbytes), "cudaHostRegister failed")


def host_unregister(*arrays):
    lib = L.load()
    for a in arrays:
        if a is not None and a.size:
            lib.mcmi_host_unregister(a.ctypes.data)


def compute_preconditioner_serial(b: CsrMatrix, cfg: McConfig | None = None) -> ApproxInverse:
    """The reference's serial twin (mc_engine.hpp:85-86): same contract, so
    the same device build (the result is independent of execution layout)."""
    return compute_preconditioner(b, cfg)


# ------------------------------------------------------------ fine-grained API
# The reference's public building blocks (mc_engine.hpp:55-74, split.hpp:21-39),
# on the same device code as the build.

def _view(m: CsrMatrix) -> L.mcmi_csr_view:
    if m.row_ptr.size != m.n + 1:
        raise ValueError("CsrMatrix arrays are inconsistent with row_ptr")
    return L.mcmi_csr_view(int(m.n), m.row_ptr.ctypes.data, m.col_idx.ctypes.data if m.col_idx.size else None,
                           m.values.ctypes.data if m.values.size else None)


def derive_chain_budget(cfg: McConfig, a_norm: float) -> ChainBudget:
    """mcspai::derive_chain_budget (mc_engine.hpp:55): host arithmetic with
    glibc log/ceil, the code the build itself runs."""
    c = cfg.to_c()
    nc, ml = C.c_int64(), C.c_int64()
    err = C.create_string_buffer(256)
    raise_for(L.load().mcmi_derive_chain_budget(C.byref(c), float(a_norm), C.byref(nc), C.byref(ml), err, 256),
              err.value.decode(errors="replace"))
    return ChainBudget(nc.value, ml.value)


@dataclass
class SplitSystem:  # split.hpp:21-28
    b_hat: CsrMatrix
    b1_diag: np.ndarray
    a: CsrMatrix
    p: CsrMatrix
    s_diag: np.ndarray
    a_norm: float
    #: (B, alpha, mode) it was derived from: estimate_row rebuilds the device
    #: tables from these (the device never holds a SplitSystem between calls)
    source: tuple = field(default=None, repr=False, compare=False)


def augment_and_split(b: CsrMatrix, alpha: float, mode: AugmentationMode = AugmentationMode.sign_aware,
                      device: int = 0) -> SplitSystem:
    """mcspai::augment_and_split (split.hpp:34-35) on the GPU."""
    lib = L.load()
    h = C.c_void_p()
    err = C.create_string_buffer(512)
    raise_for(lib.mcmi_augment_and_split(C.byref(_view(b)), float(alpha), int(mode), int(device), C.byref(h), err, 512),
              err.value.decode(errors="replace"))
    try:
        n, nb, na, an = C.c_int64(), C.c_int64(), C.c_int64(), C.c_double()
        lib.mcmi_split_sizes(h, C.byref(n), C.byref(nb), C.byref(na), C.byref(an))
        n, nb, na = n.value, nb.value, na.value
        brp, bci, bv = np.empty(n + 1, np.int64), np.empty(nb, np.int64), np.empty(nb)
        arp, aci, av, pv = np.empty(n + 1, np.int64), np.empty(na, np.int64), np.empty(na), np.empty(na)
        b1, sd = np.empty(n), np.empty(n)
        ptr = lambda x: x.ctypes.data if x.size else None  # noqa: E731
        lib.mcmi_split_copy(h, ptr(brp), ptr(bci), ptr(bv), ptr(b1), ptr(arp), ptr(aci), ptr(av), ptr(pv), ptr(sd))
    finally:
        lib.mcmi_split_free(h)
    return SplitSystem(CsrMatrix(n, brp, bci, bv), b1, CsrMatrix(n, arp, aci, av), CsrMatrix(n, arp.copy(), aci.copy(), pv),
                       sd, an.value, source=(b, float(alpha), AugmentationMode(int(mode)), int(device)))


def transition_probabilities(a: CsrMatrix, device: int = 0) -> CsrMatrix:
    """mcspai::transition_probabilities (split.hpp:39) on the GPU."""
    n, nnz = a.n, int(a.row_ptr[-1]) if a.n > 0 else 0
    rp, ci, v = np.zeros(n + 1, np.int64), np.empty(nnz, np.int64), np.empty(nnz)
    k = C.c_int64()
    err = C.create_string_buffer(512)
    raise_for(L.load().mcmi_transition_probabilities(C.byref(_view(a)), int(device), rp.ctypes.data,
                                                     ci.ctypes.data if nnz else None, v.ctypes.data if nnz else None,
                                                     C.byref(k), err, 512),
              err.value.decode(errors="replace"))
    return CsrMatrix(n, rp, ci[: k.value].copy(), v[: k.value].copy())


def drop_small_entries(m: CsrMatrix, p: float, mode: DropMode = DropMode.value_range, device: int = 0) -> CsrMatrix:
    """mcspai::drop_small_entries (csr.hpp:76-77) on the GPU: the build's drop
    filter (value range or count quantile, diagonal never dropped)."""
    n, nnz = m.n, int(m.row_ptr[-1]) if m.n > 0 else 0
    rp, ci, v = np.zeros(n + 1, np.int64), np.empty(nnz, np.int64), np.empty(nnz)
    k = C.c_int64()
    err = C.create_string_buffer(512)
    raise_for(L.load().mcmi_drop_small_entries(C.byref(_view(m)), float(p), int(mode), int(device), rp.ctypes.data,
                                               ci.ctypes.data if nnz else None, v.ctypes.data if nnz else None,
                                               C.byref(k), err, 512),
              err.value.decode(errors="replace"))
    return CsrMatrix(n, rp, ci[: k.value].copy(), v[: k.value].copy())


@dataclass
class RngStream:  # rng.hpp:17-30: RngStream(seed, stream_id)
    seed: int
    stream_id: int


def estimate_rows(split: SplitSystem, row_begin: int, row_end: int, budget: ChainBudget, delta: float, seed: int,
                  rng_mode: RngMode = RngMode.reference, device: int = 0) -> CsrMatrix:
    """mcspai::estimate_row (mc_engine.hpp:63-65) for rows [row_begin, row_end)
    at once, on the GPU (``mcmi_estimate_rows``): row r is estimate_row(split,
    r, budget, delta, RngStream(seed, r)) — columns sorted, unscaled, nothing
    pruned.  Uses only split.a and split.p (a hand-built SplitSystem works, as
    in the reference's tests, test_mc_engine.cpp:112-127)."""
    a, p = split.a, split.p
    if not (p.n == a.n and np.array_equal(p.row_ptr, a.row_ptr) and np.array_equal(p.col_idx, a.col_idx)):
        raise ValueError("estimate_row: P must have A's sparsity pattern (transition_probabilities(A))")
    lib = L.load()
    h = C.c_void_p()
    err = C.create_string_buffer(512)
    pv = np.ascontiguousarray(p.values, np.float64)
    raise_for(lib.mcmi_estimate_rows(C.byref(_view(a)), pv.ctypes.data if pv.size else None, int(row_begin),
                                     int(row_end), int(budget.n_chains), int(budget.max_len), float(delta),
                                     int(seed) & 0xFFFFFFFFFFFFFFFF, int(rng_mode), int(device), C.byref(h), err, 512),
              err.value.decode(errors="replace"))
    owner = _ResultOwner(h)
    n, nnz = C.c_int64(), C.c_int64()
    lib.mcmi_result_sizes(h, C.byref(n), C.byref(nnz))
    rp, ci, v, _, _ = owner.arrays(n.value, nnz.value)
    return CsrMatrix(n.value, rp.copy(), ci.copy(), v.copy())


def estimate_row(split: SplitSystem, r: int, budget: ChainBudget, delta: float, stream: RngStream):
    """mcspai::estimate_row (mc_engine.hpp:63-65): row r of (I - A)^-1 as
    (column, value) pairs, column-sorted, from budget.n_chains walks, on the
    build's walk kernel (``mcmi_estimate_rows``).  The device keys row r's
    draws by RngStream(seed, r), the stream compute_preconditioner gives that
    row (mc_engine.cpp:168); other stream ids are not supported."""
    if int(stream.stream_id) != int(r):
        raise ValueError("estimate_row: the device draws row r from RngStream(seed, r); stream_id must equal r")
    if not 0 <= r < split.a.n:
        raise IndexError("row out of range")
    m = estimate_rows(split, r, r + 1, budget, delta, stream.seed,
                      device=split.source[3] if split.source else 0)
    return list(zip(m.col_idx.tolist(), m.values.tolist()))


def retain_top_k_rows(m: CsrMatrix, k: int, diag_cols=None, device: int = 0) -> CsrMatrix:
    """mcspai::retain_top_k (mc_engine.hpp:70) on every row of ``m`` at once, on
    the GPU (``mcmi_retain_top_k``): row r keeps its k entries ranked first by
    (column == diag_cols[r] first, |value| descending, column ascending), in
    their original order; ``diag_cols`` defaults to r."""
    n, nnz = m.n, int(m.row_ptr[-1]) if m.n > 0 else 0
    rp, ci, v = np.zeros(n + 1, np.int64), np.empty(nnz, np.int64), np.empty(nnz)
    d = None if diag_cols is None else np.ascontiguousarray(diag_cols, np.int64)
    if d is not None and d.size != n:
        raise ValueError("diag_cols needs one column per row")
    got = C.c_int64()
    err = C.create_string_buffer(512)
    raise_for(L.load().mcmi_retain_top_k(C.byref(_view(m)), int(k), d.ctypes.data if d is not None and n else None,
                                         int(device), rp.ctypes.data, ci.ctypes.data if nnz else None,
                                         v.ctypes.data if nnz else None, C.byref(got), err, 512),
              err.value.decode(errors="replace"))
    return CsrMatrix(n, rp, ci[: got.value].copy(), v[: got.value].copy())


def retain_top_k(row, k: int, diag_col: int, device: int = 0):
    """mcspai::retain_top_k(SparseRow, k, diag_col) (mc_engine.hpp:70): a list of
    (column, value) pairs in, the kept pairs out."""
    row = list(row)
    m = CsrMatrix(1, np.array([0, len(row)]), np.array([c for c, _ in row], np.int64),
                  np.array([x for _, x in row], np.float64))
    out = retain_top_k_rows(m, k, [diag_col], device)
    return list(zip(out.col_idx.tolist(), out.values.tolist()))


def scale_columns_rows(m: CsrMatrix, b1_diag, device: int = 0) -> CsrMatrix:
    """mcspai::scale_columns (mc_engine.hpp:74) on every entry of ``m``:
    value / b1_diag[column], on the GPU (``mcmi_scale_columns``)."""
    b1 = np.ascontiguousarray(b1_diag, np.float64)
    nnz = int(m.row_ptr[-1]) if m.n > 0 else 0
    out = np.empty(nnz)
    err = C.create_string_buffer(512)
    raise_for(L.load().mcmi_scale_columns(C.byref(_view(m)), b1.ctypes.data if b1.size else None, b1.size,
                                          int(device), out.ctypes.data if nnz else None, err, 512),
              err.value.decode(errors="replace"))
    return CsrMatrix(m.n, m.row_ptr.copy(), m.col_idx.copy(), out)


def scale_columns(row: list, b1_diag, device: int = 0) -> None:
    """mcspai::scale_columns(SparseRow&, b1_diag) (mc_engine.hpp:74): in place on
    a list of (column, value) pairs."""
    m = CsrMatrix(1, np.array([0, len(row)]), np.array([c for c, _ in row], np.int64),
                  np.array([x for _, x in row], np.float64))
    out = scale_columns_rows(m, b1_diag, device)
    row[:] = list(zip(out.col_idx.tolist(), out.values.tolist()))
