"""Fused multi-GPU assembly: mcmi_scatter_shard's peer stores and
global offsets, exercised on one GPU with several local buffers standing in for
the peers' symmetric buffers, and the full symmetric-memory path under
torchrun with one rank (tools/p2p_check.py)."""
import ctypes as C
import os
import subprocess
import sys

import numpy as np
import pytest

pytestmark = pytest.mark.gpu
REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def torch_mod():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    return torch


@pytest.mark.parametrize("n,parts,seed", [(1000, 2, 0), (999, 3, 1), (4097, 5, 2), (7, 4, 3)])
def test_scatter_shards_into_peer_buffers(torch_mod, n, parts, seed):
    torch = torch_mod
    from paper_2409_03095_b200 import _lib as L
    from paper_2409_03095_b200.distributed import p2p_layout, partition_rows
    rng = np.random.default_rng(seed)
    cnt = rng.integers(0, 9, n)
    rp = np.zeros(n + 1, np.int64)
    np.cumsum(cnt, out=rp[1:])
    nnz = int(rp[-1])
    ci = rng.integers(0, n, nnz).astype(np.int64)
    v = rng.standard_normal(nnz)
    col_at, val_at, nbytes = p2p_layout(n, nnz)
    dev = torch.device("cuda", 0)
    bufs = [torch.full((nbytes,), 0xAB, dtype=torch.uint8, device=dev) for _ in range(parts)]
    ptrs = (C.c_void_p * parts)(*[b.data_ptr() for b in bufs])
    lib = L.load()
    for lo, hi in partition_rows(rp, parts):
        srp = torch.from_numpy(rp[lo:hi + 1] - rp[lo]).to(dev)
        sci = torch.from_numpy(ci[rp[lo]:rp[hi]].copy()).to(dev)
        sv = torch.from_numpy(v[rp[lo]:rp[hi]].copy()).to(dev)
        code = lib.mcmi_scatter_shard(srp.data_ptr(), sci.data_ptr() if sci.numel() else None,
                                      sv.data_ptr() if sv.numel() else None, hi - lo, int(rp[hi] - rp[lo]), lo,
                                      int(rp[lo]), n, nnz, ptrs, parts, None)
        assert code == 0
    torch.cuda.synchronize()
    for b in bufs:
        h = b.cpu().numpy()
        assert np.array_equal(h[: 8 * (n + 1)].view(np.int64), rp)
        assert np.array_equal(h[col_at: col_at + 8 * nnz].view(np.int64), ci)
        assert np.array_equal(h[val_at: val_at + 8 * nnz].view(np.uint64), v.view(np.uint64))


def test_scatter_rejects_bad_offsets(torch_mod):
    from paper_2409_03095_b200 import _lib as L
    lib = L.load()
    ptrs = (C.c_void_p * 1)(None)
    assert lib.mcmi_scatter_shard(None, None, None, 1, 0, 0, 0, 1, 0, ptrs, 1, None) == L.MCMI_EINVAL


def test_symmetric_memory_assembly_torchrun(torch_mod):
    r = subprocess.run([sys.executable, "-m", "torch.distributed.run", "--nproc-per-node", "1", "--master-addr",
                        "127.0.0.1", "--master-port", "29517", os.path.join(REPO, "tools", "p2p_check.py"),
                        "c3_lap3d_100"], capture_output=True, text=True, timeout=600, cwd=REPO)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-3000:]
    assert "OK" in r.stdout
