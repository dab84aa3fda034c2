"""Host-side multi-rank logic on CPU (gloo, world_size 2): the row partition
and the all-gather-v assembly reproduce the single-process M exactly.  The
shards come from the oracle's row-range build (the GPU shards are checked
against the same oracle in tests/test_gpu_parity.py)."""
import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp

from helpers import golden_input


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, spec, cfg, q):
    import torch
    import torch.distributed as dist

    from oracle import oracle
    from paper_2409_03095_b200.distributed import allgatherv_csr, partition_rows
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    n, rp, ci, v = golden_input(spec)
    lo, hi = partition_rows(rp, world)[rank]
    shard = oracle.compute_preconditioner(n, rp, ci, v, row_begin=lo, row_end=hi, **cfg)
    mrp, mci, mv = allgatherv_csr(torch.from_numpy(shard.row_ptr), torch.from_numpy(shard.col_idx),
                                  torch.from_numpy(shard.values), dist)
    if rank == 0:
        q.put((mrp.numpy(), mci.numpy(), mv.numpy()))
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_gloo_allgatherv_equals_full_build(oracle_mod, world):
    spec = "convdiff:64:20:10"
    cfg = dict(master_seed=7)
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, spec, cfg, q)) for r in range(world)]
    for p in procs:
        p.start()
    got = q.get(timeout=300)
    for p in procs:
        p.join(timeout=300)
        assert p.exitcode == 0
    n, rp, ci, v = golden_input(spec)
    full = oracle_mod.compute_preconditioner(n, rp, ci, v, **cfg)
    assert np.array_equal(got[0], full.row_ptr)
    assert np.array_equal(got[1], full.col_idx)
    assert np.array_equal(got[2].view(np.uint64), full.values.view(np.uint64))


def test_partition_rows_balanced_and_contiguous():
    from paper_2409_03095_b200.distributed import partition_rows
    n, rp, _, _ = golden_input("broad:1024:24:1e-4:1:7")
    for world in (1, 2, 4, 8):
        parts = partition_rows(rp, world)
        assert parts[0][0] == 0 and parts[-1][1] == n
        assert all(parts[g][1] == parts[g + 1][0] for g in range(world - 1))
        cost = [(hi - lo) + int(rp[hi] - rp[lo]) for lo, hi in parts]
        assert max(cost) - min(cost) <= 2 * (1 + int(np.diff(rp).max()))


def _partition_numpy(rp, lo, hi, world):
    """Restatement of the partition rule: block g starts at the first row whose
    cost prefix (cost = 1 + nnz per row) reaches total * g / world."""
    rp = np.asarray(rp, np.int64)
    idx = np.arange(lo, hi + 1)
    cost = (idx - lo).astype(np.float64) + (rp[lo:hi + 1] - rp[lo]).astype(np.float64)
    total = cost[-1] if hi > lo else 0.0
    edges = [lo]
    for g in range(1, world):
        e = lo + int(np.searchsorted(cost, total * g / world, side="left")) if hi > lo else lo
        edges.append(max(min(e, hi), edges[-1]))
    edges.append(hi)
    return edges


def test_library_partition_matches_restatement():
    """mcmi_partition_rows (used by host builds over several GPUs and by
    distributed.partition_rows) against the numpy restatement: sub-ranges,
    empty rows, more parts than rows."""
    from paper_2409_03095_b200 import _lib as L
    lib = L.load()
    rng = np.random.default_rng(3)
    for trial in range(60):
        n = int(rng.integers(0, 400))
        deg = rng.integers(0, 40, size=n) * (rng.random(n) < 0.8)
        rp = np.concatenate([[0], np.cumsum(deg)]).astype(np.int64)
        lo = int(rng.integers(0, n + 1))
        hi = int(rng.integers(lo, n + 1))
        world = int(rng.integers(1, 12))
        edges = np.zeros(world + 1, np.int64)
        assert lib.mcmi_partition_rows(rp.ctypes.data, lo, hi, world, edges.ctypes.data) == L.MCMI_OK
        assert edges.tolist() == _partition_numpy(rp, lo, hi, world), (trial, n, lo, hi, world)
    bad = np.zeros(3, np.int64)
    assert lib.mcmi_partition_rows(bad.ctypes.data, 0, 2, 0, bad.ctypes.data) == L.MCMI_EINVAL
    assert lib.mcmi_partition_rows(bad.ctypes.data, 2, 1, 2, bad.ctypes.data) == L.MCMI_EINVAL


def _shard(g, seed):
    """Synthetic CSR shard of rank g (some shards empty, some with rows but no entries)."""
    rng = np.random.default_rng(seed * 100 + g)
    rows = int(rng.choice([0, 1, 5, 40]))
    counts = rng.integers(0, 6, size=rows) * (rng.random(rows) < 0.7)
    rp = np.concatenate([[0], np.cumsum(counts)]).astype(np.int64)
    return rp, rng.integers(0, 1000, size=int(rp[-1])).astype(np.int64), rng.normal(size=int(rp[-1]))


def _worker_ragged(rank, world, port, seed, q):
    import torch
    import torch.distributed as dist

    from paper_2409_03095_b200.distributed import allgatherv_csr
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    rp, ci, v = _shard(rank, seed)
    mrp, mci, mv = allgatherv_csr(torch.from_numpy(rp), torch.from_numpy(ci), torch.from_numpy(v), dist)
    q.put((rank, mrp.numpy(), mci.numpy(), mv.numpy()))
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("world,seed", [(2, 1), (3, 2), (4, 3), (4, 4)])
def test_gloo_allgatherv_ragged_and_empty_shards(world, seed):
    """The grouped point-to-point all-gather-v on shards of any size (empty,
    rows without entries): every rank ends with the rank-ordered concatenation,
    row pointers shifted by the entries before them."""
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker_ragged, args=(r, world, port, seed, q)) for r in range(world)]
    for p in procs:
        p.start()
    got = [q.get(timeout=300) for _ in range(world)]
    for p in procs:
        p.join(timeout=300)
        assert p.exitcode == 0
    parts = [_shard(g, seed) for g in range(world)]
    want_rp, off = [np.zeros(1, np.int64)], 0
    for rp, _, _ in parts:
        want_rp.append(rp[1:] + off)
        off += int(rp[-1])
    want_rp = np.concatenate(want_rp)
    want_ci = np.concatenate([p[1] for p in parts])
    want_v = np.concatenate([p[2] for p in parts])
    for _, rp, ci, v in got:
        assert np.array_equal(rp, want_rp)
        assert np.array_equal(ci, want_ci)
        assert np.array_equal(v.view(np.uint64), want_v.view(np.uint64))
