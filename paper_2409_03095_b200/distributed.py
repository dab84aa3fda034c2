"""Sharded multi-GPU build: one process per GPU, rows block-partitioned,
transition tables replicated, shards assembled with an all-gather.

SURVEY.md §8e: rows are independent (mc_engine.cpp:164-178), so rank g builds
rows [r_g, r_{g+1}) of M from its own replica of B; a rank-ordered
concatenation equals the reference's row-ordered assembly
(mc_engine.cpp:214-220), so M is byte-identical for any number of GPUs.

NCCL has no all-gather-v; shards are padded to the largest shard and gathered
with one ``all_gather_into_tensor`` per array (NVLink/NVSwitch bandwidth makes
the padding cheap for balanced shards), then trimmed on device.  The same code
runs on gloo (CPU tensors) for the host-side tests.
"""
from __future__ import annotations

import numpy as np


def partition_rows(row_ptr: np.ndarray, world: int) -> list[tuple[int, int]]:
    """Contiguous row blocks balanced on cost(r) = 1 + nnz(r) (a proxy for
    the walk work of a row: steps scale with the reachable neighbourhood)."""
    rp = np.asarray(row_ptr, np.int64)
    n = rp.size - 1
    cost = np.arange(n + 1, dtype=np.float64) + rp.astype(np.float64)  # prefix of 1 + nnz(r)
    total = cost[-1]
    edges = [0]
    for g in range(1, world):
        edges.append(int(np.searchsorted(cost, total * g / world, side="left")))
    edges.append(n)
    for g in range(1, len(edges)):
        edges[g] = max(edges[g], edges[g - 1])
    return [(edges[g], edges[g + 1]) for g in range(world)]


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


def build_sharded(b, cfg, dist, engine=None, device=None, stream=None, tensors=None):
    """Builds this rank's row block on its GPU and assembles M on every rank.

    ``tensors``: B already on the device (row_ptr, col_idx, values).
    Returns (row_ptr, col_idx, values, stats) as device tensors.
    """
    import torch

    from .engine import DeviceEngine
    rank, world = dist.get_rank(), dist.get_world_size()
    dev = device if device is not None else torch.device("cuda", torch.cuda.current_device())
    eng = engine or DeviceEngine(dev.index)
    rp, ci, v = tensors if tensors is not None else DeviceEngine.upload(b, dev.index)
    lo, hi = partition_rows(b.row_ptr, world)[rank]
    d = eng.build(b.n, rp, ci, v, cfg, lo, hi, stream=stream)
    srp, sci, sv, _, _ = eng.to_tensors(d, stream=stream)
    mrp, mci, mv = allgatherv_csr(srp, sci, sv, dist)
    return mrp, mci, mv, d.stats
