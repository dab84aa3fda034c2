"""Sharded multi-GPU build: one process per GPU, rows block-partitioned,
transition tables replicated, shards assembled on every GPU.

SURVEY.md §8e: rows are independent (mc_engine.cpp:164-178), so rank g builds
rows [r_g, r_{g+1}) of M from its own replica of B; a rank-ordered
concatenation equals the reference's row-ordered assembly
(mc_engine.cpp:214-220), so M is byte-identical for any number of GPUs.

Two assemblies:
  * ``assemble_p2p`` (default on GPUs): one kernel per rank
    (``mcmi_scatter_shard``, csrc/scatter.cu) stores the rank's shard straight
    into every GPU's symmetric M buffer over NVLink peer memory, then a
    symmetric-memory barrier; no padding, staging or concatenation passes.
  * ``allgatherv_csr``: NCCL has no all-gather-v, so shards are padded to the
    largest shard and gathered with one ``all_gather_into_tensor`` per array,
    then trimmed.  It is the reference point for the fused path and runs on
    gloo (CPU tensors) for the host-side tests.
"""
from __future__ import annotations

import numpy as np


def partition_rows(row_ptr: np.ndarray, world: int) -> list[tuple[int, int]]:
    """Contiguous row blocks balanced on cost(r) = 1 + nnz(r) (a proxy for
    the walk work of a row: steps scale with the reachable neighbourhood).
    The library's own partition (``mcmi_partition_rows``), so one process per
    GPU and one process over several GPUs (``McConfig.n_gpus``) cut the same
    blocks."""
    from . import _lib as L
    rp = np.ascontiguousarray(row_ptr, np.int64)
    n = rp.size - 1
    edges = np.zeros(world + 1, np.int64)
    code = L.load().mcmi_partition_rows(rp.ctypes.data, 0, n, int(world), edges.ctypes.data)
    if code != L.MCMI_OK:
        raise ValueError(f"mcmi_partition_rows failed with status {code}")
    return [(int(edges[g]), int(edges[g + 1])) for g in range(world)]


def _gather_padded(t, dist, group=None):
    import torch
    world = dist.get_world_size(group)
    if t.is_cuda:
        out = torch.empty(world * t.numel(), dtype=t.dtype, device=t.device)
        dist.all_gather_into_tensor(out, t.contiguous(), group=group)
        return [out[g * t.numel():(g + 1) * t.numel()] for g in range(world)]
    parts = [torch.empty_like(t) for _ in range(world)]
    dist.all_gather(parts, t.contiguous(), group=group)
    return parts


def allgatherv_csr(row_ptr, col_idx, values, dist, group=None):
    """All-gather variable-size CSR row shards (rank order) into the full M.

    row_ptr: int64 [rows_g + 1] starting at 0; col_idx int64 [nnz_g];
    values float64 [nnz_g].  Returns (row_ptr, col_idx, values) of the
    concatenation on every rank (same device as the inputs).
    """
    import torch
    dev = col_idx.device
    sizes = torch.tensor([col_idx.numel(), row_ptr.numel() - 1], dtype=torch.int64, device=dev)
    all_sizes = torch.stack(_gather_padded(sizes, dist, group)).cpu()
    mx_nnz = max(int(all_sizes[:, 0].max()), 1)
    mx_rows = int(all_sizes[:, 1].max())

    def pad(t, length, dtype):
        p = torch.zeros(length, dtype=dtype, device=dev)
        p[: t.numel()] = t
        return p

    cols = _gather_padded(pad(col_idx, mx_nnz, torch.int64), dist, group)
    vals = _gather_padded(pad(values, mx_nnz, torch.float64), dist, group)
    rps = _gather_padded(pad(row_ptr, mx_rows + 1, torch.int64), dist, group)
    out_c, out_v, out_r, off = [], [], [], 0
    for g in range(all_sizes.shape[0]):
        k, r = int(all_sizes[g, 0]), int(all_sizes[g, 1])
        out_c.append(cols[g][:k])
        out_v.append(vals[g][:k])
        out_r.append(rps[g][:r] + off)
        off += k
    out_r.append(torch.tensor([off], dtype=torch.int64, device=dev))
    return torch.cat(out_r), torch.cat(out_c), torch.cat(out_v)


def build_sharded(b, cfg, dist, engine=None, device=None, stream=None, tensors=None, assembly="p2p", sym=None):
    """Builds this rank's row block on its GPU and assembles M on every rank.

    ``tensors``: B already on the device (row_ptr, col_idx, values).
    ``assembly``: "p2p" (fused peer-store kernel into symmetric memory; pass a
    ``SymmetricM`` as ``sym`` to reuse its buffer across builds) or "nccl".
    Returns (row_ptr, col_idx, values, stats) as device tensors (for "p2p",
    views of the symmetric buffer, valid until its next assembly).
    """
    import torch

    from .engine import DeviceEngine
    rank, world = dist.get_rank(), dist.get_world_size()
    dev = device if device is not None else torch.device("cuda", torch.cuda.current_device())
    eng = engine or DeviceEngine(dev.index)
    rp, ci, v = tensors if tensors is not None else DeviceEngine.upload(b, dev.index)
    lo, hi = partition_rows(b.row_ptr, world)[rank]
    d = eng.build(b.n, rp, ci, v, cfg, lo, hi, stream=stream)
    if assembly == "p2p":
        mrp, mci, mv = assemble_p2p(d, lo, hi, b.n, dist, sym or SymmetricM(dev, dist), stream)
    else:
        srp, sci, sv, _, _ = eng.to_tensors(d, stream=stream)
        mrp, mci, mv = allgatherv_csr(srp, sci, sv, dist)
    return mrp, mci, mv, d.stats


# ---------------------------------------------------------------- fused (P2P)

def p2p_layout(n: int, nnz_total: int) -> tuple[int, int, int]:
    """Byte offsets (col_idx, values) and total size of the symmetric M buffer:
    [row_ptr n+1 int64][col_idx nnz int64][values nnz f64], 16-byte aligned."""
    a16 = lambda x: (x + 15) // 16 * 16  # noqa: E731
    col_at = a16(8 * (n + 1))
    val_at = col_at + a16(8 * nnz_total)
    return col_at, val_at, val_at + a16(8 * nnz_total)


class SymmetricM:
    """The per-process symmetric buffer that receives M (torch symmetric
    memory: allocated on every rank, mapped into every peer).  Grows
    collectively (every rank sees the same sizes)."""

    def __init__(self, device, dist, group=None):
        self.device = device
        self.dist = dist
        self.group = group or dist.group.WORLD
        self.buf = None
        self.handle = None

    def ensure(self, nbytes: int):
        import torch
        import torch.distributed._symmetric_memory as symm
        if self.buf is not None and self.buf.numel() >= nbytes:
            return
        try:
            symm.enable_symm_mem_for_group(self.group.group_name)
        except Exception:  # noqa: BLE001 — already enabled / not needed on newer torch
            pass
        self.handle = None
        self.buf = symm.empty(max(nbytes, 16) + (1 << 20), dtype=torch.uint8, device=self.device)
        self.handle = symm.rendezvous(self.buf, self.group)

    def peer_ptrs(self):
        return list(self.handle.buffer_ptrs)


def assemble_p2p(shard, lo: int, hi: int, n: int, dist, sym: SymmetricM, stream=None):
    """Assembles M on every rank from this rank's device shard (an engine
    DeviceCsr) with one peer-store kernel.  Returns (row_ptr, col_idx, values)
    views of the symmetric buffer (valid until the next assembly)."""
    import ctypes as C

    import torch

    from . import _lib as L
    lib = L.load()
    dev = sym.device
    world = dist.get_world_size(sym.group)
    sizes = torch.tensor([shard.nnz], dtype=torch.int64, device=dev)
    all_sizes = [torch.empty_like(sizes) for _ in range(world)]
    dist.all_gather(all_sizes, sizes, group=sym.group)
    nnzs = [int(x.item()) for x in all_sizes]
    rank = dist.get_rank(sym.group)
    nnz_off, total = sum(nnzs[:rank]), sum(nnzs)
    col_at, val_at, nbytes = p2p_layout(n, total)
    sym.ensure(nbytes)
    ptrs = sym.peer_ptrs()
    arr = (C.c_void_p * len(ptrs))(*ptrs)
    st = (stream or torch.cuda.current_stream(dev))
    raw = shard.raw
    code = lib.mcmi_scatter_shard(raw.row_ptr, raw.col_idx, raw.values, hi - lo, shard.nnz, lo, nnz_off, n, total,
                                  arr, len(ptrs), st.cuda_stream)
    if code != L.MCMI_OK:
        raise RuntimeError(f"mcmi_scatter_shard failed with status {code}")
    with torch.cuda.stream(st):
        sym.handle.barrier()
    b = sym.buf
    rp = b[: 8 * (n + 1)].view(torch.int64)
    ci = b[col_at: col_at + 8 * total].view(torch.int64)
    v = b[val_at: val_at + 8 * total].view(torch.float64)
    return rp, ci, v
