"""Matrix Market I/O (§8f rank 2), mirroring include/mcspai/matrix_market.hpp.

    parse_matrix_market(text)            matrix_market.cpp:27-147
    read_matrix_market_file(path)        matrix_market.cpp:149-153
    write_matrix_market(m[, out])        matrix_market.cpp:155-169
    write_matrix_market_file(m, path)    matrix_market.cpp:171-177

All four run in the native library (paper_2409_03095_b200/csrc/mmio.cpp,
multi-threaded) and produce the reference's results byte for byte: the same
CsrMatrix (duplicates summed in the reference's order) or the same ParseError
text naming the line, and the same "%lld %lld %.17g" output.
"""
from __future__ import annotations

import ctypes as C
import os

from . import _lib as L
from .mcspai import CsrMatrix, ParseError, host_csr_take, raise_for

__all__ = ["ParseError", "parse_matrix_market", "read_matrix_market_file", "write_matrix_market",
           "write_matrix_market_file", "format_matrix_market"]


def _err():
    return C.create_string_buffer(512)


def parse_matrix_market(text) -> CsrMatrix:
    """Parses Matrix Market text (str or bytes)."""
    if isinstance(text, str):
        text = text.encode()
    h = C.c_void_p()
    err = _err()
    code = L.load().mcmi_mm_parse(text, len(text), C.byref(h), err, 512)
    raise_for(code, err.value.decode(errors="replace"))
    return host_csr_take(h)


def read_matrix_market_file(path) -> CsrMatrix:
    h = C.c_void_p()
    err = _err()
    code = L.load().mcmi_mm_read_file(os.fsencode(path), C.byref(h), err, 512)
    raise_for(code, err.value.decode(errors="replace"))
    return host_csr_take(h)


def _view(m: CsrMatrix) -> L.mcmi_csr_view:
    if m.row_ptr.size != m.n + 1 and m.n > 0:
        raise ValueError("row_ptr must hold n + 1 entries")
    return L.mcmi_csr_view(m.n, m.row_ptr.ctypes.data, m.col_idx.ctypes.data, m.values.ctypes.data)


def format_matrix_market(m: CsrMatrix) -> bytes:
    """The bytes write_matrix_market emits for m (one formatting pass when the
    text fits the usual ~48 bytes per entry, a second one otherwise)."""
    lib = L.load()
    v = _view(m)
    err = _err()
    got = C.c_size_t()
    cap = 128 + 48 * m.nnz()
    for _ in range(2):
        buf = C.create_string_buffer(cap)
        code = lib.mcmi_mm_format(C.byref(v), buf, cap, C.byref(got), err, 512)
        if code == L.MCMI_ENOMEM and got.value > cap:
            cap = got.value
            continue
        raise_for(code, err.value.decode(errors="replace"))
        return buf.raw[: got.value]
    raise MemoryError("matrix market: formatting buffer")


def write_matrix_market(m: CsrMatrix, out=None):
    """Writes m to the binary or text stream `out`; returns the text if out is None."""
    data = format_matrix_market(m)
    if out is None:
        return data.decode()
    try:
        out.write(data)
    except TypeError:
        out.write(data.decode())
    return None


def write_matrix_market_file(m: CsrMatrix, path) -> None:
    err = _err()
    v = _view(m)
    code = L.load().mcmi_mm_write_file(C.byref(v), os.fsencode(path), err, 512)
    raise_for(code, err.value.decode(errors="replace"))
