"""Shared test helpers (fixture loading, Matrix Market hashing)."""
from __future__ import annotations

import hashlib
import json
import os

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
GOLDEN = os.path.join(HERE, "golden")

_inputs = None


def goldens() -> dict:
    with open(os.path.join(GOLDEN, "goldens.json")) as f:
        return json.load(f)


def golden_input(spec: str):
    """(n, row_ptr, col_idx, values) frozen by tests/golden/make_goldens.py."""
    global _inputs
    if _inputs is None:
        _inputs = np.load(os.path.join(GOLDEN, "inputs.npz"))
    rp = _inputs[f"{spec}/row_ptr"]
    return len(rp) - 1, rp, _inputs[f"{spec}/col_idx"], _inputs[f"{spec}/values"]


def mm_bytes(n, row_ptr, col_idx, values) -> bytes:
    """write_matrix_market (matrix_market.cpp:155-169): '%lld %lld %.17g'."""
    rp = np.asarray(row_ptr)
    rows = np.repeat(np.arange(n, dtype=np.int64), np.diff(rp)) + 1
    cols = np.asarray(col_idx) + 1
    out = [b"%%MatrixMarket matrix coordinate real general\n", b"%d %d %d\n" % (n, n, int(rp[-1]))]
    out.extend(b"%d %d %.17g\n" % (int(r), int(c), float(v)) for r, c, v in zip(rows, cols, values))
    return b"".join(out)


def mm_sha256(n, row_ptr, col_idx, values) -> str:
    return hashlib.sha256(mm_bytes(n, row_ptr, col_idx, values)).hexdigest()


def arr_sha256(a) -> str:
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def bits_equal(a, b) -> bool:
    a = np.ascontiguousarray(a, np.float64)
    b = np.ascontiguousarray(b, np.float64)
    return a.shape == b.shape and np.array_equal(a.view(np.uint64), b.view(np.uint64))
