"""Device-resident builds: B already in HBM (torch tensors), M left in HBM.

Thin wrapper over ``mcmi_engine_*`` (include/mcmi.h).  torch provides the
device memory, streams and (in :mod:`.distributed`) NCCL; the build itself is
the sm_100a pipeline behind the C-ABI.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass

from . import _lib as L
from .mcspai import CsrMatrix, McConfig, raise_for


@dataclass
class DeviceCsr:
    """Shard [row_begin, row_end) of M; pointers owned by the engine."""
    raw: L.mcmi_device_csr
    stats: dict

    @property
    def nnz(self) -> int:
        return int(self.raw.nnz)

    @property
    def rows(self) -> int:
        return int(self.raw.row_end - self.raw.row_begin)


class DeviceEngine:
    def __init__(self, device: int = 0):
        self.lib = L.load()
        self.device = device
        h = C.c_void_p()
        err = C.create_string_buffer(512)
        raise_for(self.lib.mcmi_engine_create(device, C.byref(h), err, 512), err.value.decode())
        self.h = h

    def close(self):
        if self.h:
            self.lib.mcmi_engine_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    @staticmethod
    def upload(b: CsrMatrix, device: int = 0):
        """H2D of B in the reference layout (int64 / float64)."""
        import torch
        dev = torch.device("cuda", device)
        return (torch.from_numpy(b.row_ptr).to(dev), torch.from_numpy(b.col_idx).to(dev),
                torch.from_numpy(b.values).to(dev))

    def build(self, n: int, row_ptr, col_idx, values, cfg: McConfig, row_begin: int = 0,
              row_end: int = -1, stream=None) -> DeviceCsr:
        """``row_ptr``/``col_idx``/``values``: device tensors (or raw pointers).

        Runs on ``stream`` (a torch stream or a raw cudaStream_t); by default on
        torch's current stream of the engine's device, so B tensors still being
        produced by queued torch work are complete before the build reads them."""
        ptr = lambda t: t if isinstance(t, int) else t.data_ptr()  # noqa: E731
        if stream is None:
            import torch
            stream = torch.cuda.current_stream(torch.device("cuda", self.device))
        view = L.mcmi_csr_view(int(n), ptr(row_ptr), ptr(col_idx), ptr(values))
        c = cfg.to_c()
        out = L.mcmi_device_csr()
        st = L.mcmi_stats()
        err = C.create_string_buffer(1024)
        s = None if stream is None else (stream if isinstance(stream, int) else stream.cuda_stream)
        code = self.lib.mcmi_engine_build(self.h, C.byref(view), C.byref(c), row_begin, row_end, s,
                                          C.byref(out), C.byref(st), err, 1024)
        raise_for(code, err.value.decode(errors="replace"))
        return DeviceCsr(out, st.as_dict())

    def to_tensors(self, d: DeviceCsr, stream=None):
        """Copies the engine-owned shard into fresh torch tensors (same device)."""
        import torch
        dev = torch.device("cuda", self.device)
        rows, nnz = d.rows, d.nnz
        rp = torch.empty(rows + 1, dtype=torch.int64, device=dev)
        ci = torch.empty(max(nnz, 1), dtype=torch.int64, device=dev)
        v = torch.empty(max(nnz, 1), dtype=torch.float64, device=dev)
        cu = torch.empty(max(rows, 1), dtype=torch.int64, device=dev)
        eb = torch.empty(max(rows, 1), dtype=torch.int64, device=dev)
        if stream is None:
            stream = torch.cuda.current_stream(dev)
        s = stream if isinstance(stream, int) else stream.cuda_stream
        for dst, src, nb in ((rp, d.raw.row_ptr, 8 * (rows + 1)), (ci, d.raw.col_idx, 8 * nnz),
                             (v, d.raw.values, 8 * nnz), (cu, d.raw.chains_used, 8 * rows),
                             (eb, d.raw.entries_before, 8 * rows)):
            if nb:
                raise_for(self.lib.mcmi_copy(dst.data_ptr(), src, nb, s), "copy out")
        return rp, ci[:nnz], v[:nnz], cu[:rows], eb[:rows]
