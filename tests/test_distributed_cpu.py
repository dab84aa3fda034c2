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
