"""Synthetic inputs for the BASELINE.json configs (numpy; not on the hot path).

``convection_diffusion`` and ``tridiagonal`` reproduce the reference
generators bit-for-bit (synthetic.cpp:9-72; checked in tests against
the reference library in tests/test_generators.py).  The others are new shapes the reference lacks:

* ``laplacian3d``     7-point 3D Laplacian (diag 6, off -1)          — config C3
* ``stencil27``       sym_r6_a11-style symmetric 27-point stencil with a
                      symmetric hash-keyed value jitter              — config C2
* ``powerlaw``        power-law row lengths, uniform random columns,
                      log-uniform magnitudes                          — config C5

All return a :class:`~paper_2409_03095_b200.mcspai.CsrMatrix` with sorted,
duplicate-free rows (the from_triplets invariants, csr.hpp:12-15).  The module
needs only numpy, so bench.py's reference arm and the golden-vector scripts
import it by file path, without the package (which maps libmcmi.so).
"""
from __future__ import annotations

import numpy as np

try:
    from .mcspai import CsrMatrix
except ImportError:  # loaded by file path (bench.py --impl reference, tests/golden): no product import

    class CsrMatrix:  # type: ignore[no-redef]  # the fields of mcspai.CsrMatrix (csr.hpp:16-21)
        def __init__(self, n, row_ptr, col_idx, values):
            self.n, self.row_ptr, self.col_idx, self.values = int(n), row_ptr, col_idx, values

        def nnz(self) -> int:
            return int(self.values.size)

_M64 = np.uint64(0xFFFFFFFFFFFFFFFF)


def _splitmix64(x: np.ndarray) -> np.ndarray:
    x = x.astype(np.uint64, copy=True)
    with np.errstate(over="ignore"):
        x += np.uint64(0x9E3779B97F4A7C15)
        z = x
        z = (z ^ (z >> np.uint64(30))) * np.uint64(0xBF58476D1CE4E5B9)
        z = (z ^ (z >> np.uint64(27))) * np.uint64(0x94D049BB133111EB)
        z = z ^ (z >> np.uint64(31))
    return z


def _u01(x: np.ndarray) -> np.ndarray:
    return (_splitmix64(x) >> np.uint64(11)).astype(np.float64) * 2.0 ** -53


def tridiagonal(n: int) -> CsrMatrix:
    """make_tridiagonal (synthetic.cpp:9-29)."""
    rows, cols, vals = [], [], []
    i = np.arange(n)
    rows = np.concatenate([i[1:], i, i[:-1]])
    cols = np.concatenate([i[1:] - 1, i, i[:-1] + 1])
    vals = np.concatenate([np.full(n - 1, -1.0), np.full(n, 2.0), np.full(n - 1, -1.0)])
    order = np.lexsort((cols, rows))
    rp = np.zeros(n + 1, np.int64)
    np.add.at(rp, rows + 1, 1)
    return CsrMatrix(n, np.cumsum(rp), cols[order], vals[order])


def _grid_csr(n: int, cols: np.ndarray, vals: np.ndarray, valid: np.ndarray) -> CsrMatrix:
    """cols/vals/valid: (n, k) with columns already increasing along axis 1."""
    counts = valid.sum(axis=1)
    rp = np.zeros(n + 1, np.int64)
    np.cumsum(counts, out=rp[1:])
    return CsrMatrix(n, rp, cols[valid], vals[valid])


def convection_diffusion(grid: int, conv_x: float = 20.0, conv_y: float = 10.0) -> CsrMatrix:
    """make_convection_diffusion (synthetic.cpp:31-72), same IEEE arithmetic."""
    n = grid * grid
    h = 1.0 / float(grid + 1)
    diff = 1.0 / (h * h)
    cx = conv_x / h
    cy = conv_y / h
    i = np.arange(n, dtype=np.int64)
    ix, iy = i % grid, i // grid
    # column order: (iy-1), (ix-1), diag, (ix+1), (iy+1)
    cols = np.stack([i - grid, i - 1, i, i + 1, i + grid], axis=1)
    valid = np.stack([iy > 0, ix > 0, np.ones(n, bool), ix + 1 < grid, iy + 1 < grid], axis=1)
    diag = 4.0 * diff + cx + cy
    vals = np.empty((n, 5))
    vals[:, 0] = -diff - cy
    vals[:, 1] = -diff - cx
    vals[:, 2] = diag
    vals[:, 3] = -diff
    vals[:, 4] = -diff
    keep = valid & (vals != 0.0)  # from_triplets prunes exact zeros
    return _grid_csr(n, cols, vals, keep)


def laplacian3d(nx: int, ny: int | None = None, nz: int | None = None) -> CsrMatrix:
    """7-point 3D Laplacian, diag 6, off-diagonal -1 (config C3 at 100^3)."""
    ny = nx if ny is None else ny
    nz = nx if nz is None else nz
    n = nx * ny * nz
    i = np.arange(n, dtype=np.int64)
    x, y, z = i % nx, (i // nx) % ny, i // (nx * ny)
    sxy = nx * ny
    cols = np.stack([i - sxy, i - nx, i - 1, i, i + 1, i + nx, i + sxy], axis=1)
    valid = np.stack([z > 0, y > 0, x > 0, np.ones(n, bool), x + 1 < nx, y + 1 < ny, z + 1 < nz], axis=1)
    vals = np.full((n, 7), -1.0)
    vals[:, 3] = 6.0
    return _grid_csr(n, cols, vals, valid)


def stencil27(nx: int = 110, ny: int = 110, nz: int = 109, seed: int = 11) -> CsrMatrix:
    """sym_r6_a11-style stand-in: symmetric 27-point stencil,
    n = 110*110*109 = 1,318,900 (paper: 1,314,306 rows, 28 nnz/row).

    b_ij = -(0.5 + u(min(i,j), max(i,j), seed)) off the diagonal (u uniform in
    [0,1) from a symmetric hash), b_ii = sum_j |b_ij| + 1: symmetric, strictly
    diagonally dominant.
    """
    n = nx * ny * nz
    i = np.arange(n, dtype=np.int64)
    x, y, z = i % nx, (i // nx) % ny, i // (nx * ny)
    offs = [(dz, dy, dx) for dz in (-1, 0, 1) for dy in (-1, 0, 1) for dx in (-1, 0, 1)]
    cols = np.empty((n, 27), np.int64)
    valid = np.empty((n, 27), bool)
    for k, (dz, dy, dx) in enumerate(offs):
        cols[:, k] = i + dx + nx * dy + nx * ny * dz
        valid[:, k] = ((x + dx >= 0) & (x + dx < nx) & (y + dy >= 0) & (y + dy < ny)
                       & (z + dz >= 0) & (z + dz < nz))
    lo = np.minimum(i[:, None], cols)
    hi = np.maximum(i[:, None], cols)
    key = (lo.astype(np.uint64) * np.uint64(n) + hi.astype(np.uint64)) ^ np.uint64(seed * 0x9E3779B1)
    vals = -(0.5 + _u01(key))
    vals[~valid] = 0.0
    vals[:, 13] = 0.0
    diag = np.abs(vals).sum(axis=1) + 1.0
    vals[:, 13] = diag
    return _grid_csr(n, cols, vals, valid)


def powerlaw(n: int, gamma: float = 2.1, dmin: int = 2, dmax: int = 2000, seed: int = 5,
             lo: float = 1e-4, hi: float = 1.0) -> CsrMatrix:
    """Power-law row lengths (config C5, modelled on make_broad_spectrum,
    synthetic.cpp:162-191): deg ~ d^-gamma on [dmin, dmax], uniform random
    columns (duplicates merged, self-loops dropped), log-uniform |v| in
    [lo, hi] with random sign (hash of (row, col)), diag = 1.1*rowsum + 1."""
    i = np.arange(n, dtype=np.uint64)
    base = np.uint64(seed) * np.uint64(0x100000001B3)
    u = _u01(i ^ base)
    a = 1.0 - gamma
    d = ((dmax ** a - dmin ** a) * u + dmin ** a) ** (1.0 / a)  # inverse CDF
    deg = np.clip(np.floor(d).astype(np.int64), dmin, dmax)
    rows = np.repeat(np.arange(n, dtype=np.int64), deg)
    e = np.arange(rows.size, dtype=np.uint64)
    cols = (_u01(e * np.uint64(3) + base + np.uint64(1)) * n).astype(np.int64)
    key = np.sort(rows * n + cols)  # sorted by (row, col)
    key = key[np.concatenate(([True], key[1:] != key[:-1]))]  # duplicates merged
    rows, cols = key // n, key % n
    off = cols != rows
    key, rows, cols = key[off], rows[off], cols[off]
    h = key.astype(np.uint64) ^ base
    mag = np.exp(np.log(lo) + (np.log(hi) - np.log(lo)) * _u01(h * np.uint64(5) + np.uint64(7)))
    vals = np.where(_u01(h * np.uint64(5) + np.uint64(9)) < 0.5, -mag, mag)
    rowsum = np.bincount(rows, weights=np.abs(vals), minlength=n)
    diag_key = np.arange(n, dtype=np.int64) * (n + 1)
    pos = np.searchsorted(key, diag_key)
    cols = np.insert(cols, pos, np.arange(n, dtype=np.int64))
    vals = np.insert(vals, pos, 1.1 * rowsum + 1.0)
    counts = np.bincount(rows, minlength=n) + 1
    rp = np.zeros(n + 1, np.int64)
    np.cumsum(counts, out=rp[1:])
    return CsrMatrix(n, rp, cols, vals)


#: BASELINE.json configs -> (generator, McConfig overrides)
CONFIGS = {
    "c1_poisson2d_100": (lambda: convection_diffusion(100, 0.0, 0.0), {}),
    "c2_sym27_1p3m": (lambda: stencil27(), {"epsilon": 0.01, "delta": 0.01}),
    "c2_sym27_default": (lambda: stencil27(), {}),
    "c3_lap3d_100": (lambda: laplacian3d(100), {}),
    "c3_lap3d_100_heavy": (lambda: laplacian3d(100), {"epsilon": 0.01, "delta": 0.01, "alpha": 1.5}),
    "c4_convdiff_1000": (lambda: convection_diffusion(1000), {}),
    # C5: one point of the eps/delta sweep (tools/c5_sweep.py runs the grid)
    "c5_powerlaw_4m": (lambda: powerlaw(4_000_000),
                       {"alpha": 0.1, "delta": 1e-300, "chains_override": 100, "max_len_override": 8,
                        "retain_k": 32}),
    # the C5 grid's wide corner (bench.py builds its leading 12,500 rows)
    "c5_powerlaw_4m_1e4x32": (lambda: powerlaw(4_000_000),
                              {"alpha": 0.1, "delta": 1e-300, "chains_override": 10000, "max_len_override": 32,
                               "retain_k": 32}),
}

