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
  * ``allgatherv_csr``: the all-gather-v as grouped point-to-point transfers
    (every shard sent straight into its slice of every rank's output; NCCL
    send/recv in one group).  It is the reference point for the fused path and
    runs on gloo (CPU tensors) for the host-side tests.
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


def _gather_sizes(t, dist, group=None):
    """All-gather of one small fixed-size tensor per rank -> [world, ...]."""
    import torch
    world = dist.get_world_size(group)
    if t.is_cuda:
        out = torch.empty(world * t.numel(), dtype=t.dtype, device=t.device)
        dist.all_gather_into_tensor(out, t.contiguous(), group=group)
        return out.view(world, -1)
    parts = [torch.empty_like(t) for _ in range(world)]
    dist.all_gather(parts, t.contiguous(), group=group)
    return torch.stack(parts)


def allgatherv_csr(row_ptr, col_idx, values, dist, group=None):
    """All-gather-v of variable-size CSR row shards (rank order) into the full M.

    row_ptr: int64 [rows_g + 1] starting at 0; col_idx int64 [nnz_g];
    values float64 [nnz_g].  One all-gather of (nnz_g, rows_g), then every rank
    sends its shard to every peer and receives each peer's shard straight into
    that peer's slice of the output (grouped point-to-point: NCCL send/recv
    inside one group) — no padding, no trimming, no concatenation
    pass.  The received row pointers are shifted by their shard's entry offset
    on the device.  Returns (row_ptr, col_idx, values) of the concatenation on
    every rank (same device as the inputs).
    """
    import torch
    dev = col_idx.device
    world, rank = dist.get_world_size(group), dist.get_rank(group)
    rows = row_ptr.numel() - 1
    sizes = _gather_sizes(torch.tensor([col_idx.numel(), rows], dtype=torch.int64, device=dev), dist, group).cpu()
    nnzs, rowss = [int(x) for x in sizes[:, 0]], [int(x) for x in sizes[:, 1]]
    nnz_off = [sum(nnzs[:g]) for g in range(world)]
    row_off = [sum(rowss[:g]) for g in range(world)]
    total_nnz, total_rows = sum(nnzs), sum(rowss)
    out_c = torch.empty(max(total_nnz, 1), dtype=torch.int64, device=dev)
    out_v = torch.empty(max(total_nnz, 1), dtype=torch.float64, device=dev)
    out_r = torch.empty(total_rows + 1, dtype=torch.int64, device=dev)

    def my(t, off, cnt):
        return t[off: off + cnt]

    my(out_c, nnz_off[rank], nnzs[rank]).copy_(col_idx[: nnzs[rank]])
    my(out_v, nnz_off[rank], nnzs[rank]).copy_(values[: nnzs[rank]])
    my(out_r, row_off[rank], rows).copy_(row_ptr[:rows])
    ops = []
    for peer in range(world):
        if peer == rank:
            continue
        # the same (cols, values, row pointers) order on both sides of every pair
        for t, cnt in ((col_idx, nnzs[rank]), (values, nnzs[rank]), (row_ptr, rows)):
            if cnt:
                ops.append(dist.P2POp(dist.isend, t[:cnt].contiguous(), peer, group))
        for t, off, cnt in ((out_c, nnz_off[peer], nnzs[peer]), (out_v, nnz_off[peer], nnzs[peer]),
                            (out_r, row_off[peer], rowss[peer])):
            if cnt:
                ops.append(dist.P2POp(dist.irecv, my(t, off, cnt), peer, group))
    if ops:
        for req in dist.batch_isend_irecv(ops):
            req.wait()
    if total_rows:
        shift = torch.repeat_interleave(torch.tensor(nnz_off, dtype=torch.int64, device=dev),
                                        torch.tensor(rowss, dtype=torch.int64, device=dev))
        out_r[:total_rows] += shift
    out_r[total_rows] = total_nnz
    return out_r, out_c[:total_nnz], out_v[:total_nnz]


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


#: symmetric-memory barrier timeout (the rendezvous is bounded by the process
#: group's store timeout: bench.py creates its group with a 180 s timeout)
P2P_BARRIER_TIMEOUT_MS = 60_000


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
        # bounded: a peer that never arrives fails the step instead of hanging the job
        sym.handle.barrier(channel=0, timeout_ms=P2P_BARRIER_TIMEOUT_MS)
    b = sym.buf
    rp = b[: 8 * (n + 1)].view(torch.int64)
    ci = b[col_at: col_at + 8 * total].view(torch.int64)
    v = b[val_at: val_at + 8 * total].view(torch.float64)
    return rp, ci, v
