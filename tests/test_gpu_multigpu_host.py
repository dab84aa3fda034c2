"""Host builds over several GPUs of one process (McConfig.n_gpus):
row blocks built concurrently, one host thread and engine per shard, copied
to their global offsets.  Rows are independent (mc_engine.cpp:164-178), so M,
RowMeta and the step count must equal the single-GPU build bit for bit.

This box has one GPU: MCMI_SHARD_WRAP=1 maps every shard onto it (several
engines on one device, running concurrently).  The kernels of different
shards never wait on each other, so this exercises exactly the partition,
concurrent build and offset-copy logic that runs on distinct GPUs.
"""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu


@pytest.fixture
def wrap(monkeypatch):
    monkeypatch.setenv("MCMI_SHARD_WRAP", "1")
    monkeypatch.delenv("MCMI_GPUS", raising=False)


def _same(a, b):
    assert a.m.n == b.m.n
    assert np.array_equal(a.m.row_ptr, b.m.row_ptr)
    assert np.array_equal(a.m.col_idx, b.m.col_idx)
    assert np.array_equal(a.m.values.view(np.uint64), b.m.values.view(np.uint64))
    assert np.array_equal(a.row_meta.chains_used, b.row_meta.chains_used)
    assert np.array_equal(a.row_meta.entries_before_retention, b.row_meta.entries_before_retention)
    assert a.budget_echo == b.budget_echo
    assert a.stats["walk_steps"] == b.stats["walk_steps"]
    assert a.stats["nnz"] == b.stats["nnz"] == a.m.nnz()


def _matrices():
    from paper_2409_03095_b200 import generators as G
    return {"convdiff40": G.convection_diffusion(40), "lap3d_12": G.laplacian3d(12),
            "powerlaw3000": G.powerlaw(3000, dmax=200, seed=3)}


@pytest.mark.parametrize("name", ["convdiff40", "lap3d_12", "powerlaw3000"])
@pytest.mark.parametrize("g", [2, 3, 8])
@pytest.mark.parametrize("rng", [0, 1])
def test_sharded_host_build_equals_single(wrap, name, g, rng):
    from paper_2409_03095_b200.mcspai import McConfig, compute_preconditioner
    b = _matrices()[name]
    kw = dict(master_seed=11, rng_mode=rng, retain_k=8 if name == "powerlaw3000" else 0,
              alpha=1.5 if name == "powerlaw3000" else 5.0)
    one = compute_preconditioner(b, McConfig(n_gpus=1, **kw))
    many = compute_preconditioner(b, McConfig(n_gpus=g, **kw))
    _same(one, many)


@pytest.mark.parametrize("g", [2, 4])
def test_sharded_build_into_host_arrays(wrap, g):
    """mcmi_build_into with several GPUs: shards copied straight to their
    offsets in the caller's arrays."""
    from paper_2409_03095_b200 import generators as G
    from paper_2409_03095_b200.mcspai import McConfig, compute_preconditioner
    b = G.convection_diffusion(50)
    one = compute_preconditioner(b, McConfig(n_gpus=1, master_seed=3))
    cap = one.m.nnz() + 17
    out = {"row_ptr": np.full(b.n + 1, -7, np.int64), "col_idx": np.full(cap, -7, np.int64),
           "values": np.full(cap, np.nan)}
    many = compute_preconditioner(b, McConfig(n_gpus=g, master_seed=3), out=out)
    _same(one, many)
    # too small: the call reports the size and the wrapper falls back to the handle path
    small = {"row_ptr": np.empty(b.n + 1, np.int64), "col_idx": np.empty(10, np.int64), "values": np.empty(10)}
    _same(one, compute_preconditioner(b, McConfig(n_gpus=g, master_seed=3), out=small))


@pytest.mark.parametrize("rows", [(0, 1), (5, 905), (1000, 1600), (1600, 1600)])
def test_sharded_row_range(wrap, rows):
    from paper_2409_03095_b200 import generators as G
    from paper_2409_03095_b200.mcspai import McConfig, compute_preconditioner
    b = G.convection_diffusion(40)
    one = compute_preconditioner(b, McConfig(n_gpus=1, master_seed=5), rows=rows)
    many = compute_preconditioner(b, McConfig(n_gpus=3, master_seed=5), rows=rows)
    _same(one, many)


def test_more_gpus_than_rows(wrap):
    from paper_2409_03095_b200 import generators as G
    from paper_2409_03095_b200.mcspai import McConfig, compute_preconditioner
    b = G.tridiagonal(3)
    _same(compute_preconditioner(b, McConfig(n_gpus=1)), compute_preconditioner(b, McConfig(n_gpus=8)))


def test_env_gpu_count(monkeypatch):
    """n_gpus = 0 reads MCMI_GPUS (the drop-in's knob: no code change)."""
    from paper_2409_03095_b200 import generators as G
    from paper_2409_03095_b200.mcspai import McConfig, compute_preconditioner
    b = G.convection_diffusion(30)
    monkeypatch.setenv("MCMI_SHARD_WRAP", "1")
    monkeypatch.setenv("MCMI_GPUS", "3")
    _same(compute_preconditioner(b, McConfig(n_gpus=1)), compute_preconditioner(b, McConfig()))


def test_too_many_gpus_is_an_error(monkeypatch):
    import torch

    from paper_2409_03095_b200 import generators as G
    from paper_2409_03095_b200.mcspai import DeviceError, McConfig, compute_preconditioner
    monkeypatch.delenv("MCMI_SHARD_WRAP", raising=False)
    count = torch.cuda.device_count()
    with pytest.raises(DeviceError, match="visible"):
        compute_preconditioner(G.convection_diffusion(10), McConfig(n_gpus=count + 1))


def test_errors_propagate_from_shards(wrap):
    """A split error raised by the shards is reported once, as the single build does."""
    from paper_2409_03095_b200.mcspai import CsrMatrix, McConfig, SplitError, compute_preconditioner
    n = 6
    rp = np.arange(n + 1)
    b = CsrMatrix(n, rp, np.arange(n), np.array([1.0, -2.0, 1.0, 1.0, 1.0, 1.0]))  # row 1: -2 + alpha*||B|| = 0
    with pytest.raises(SplitError) as one:
        compute_preconditioner(b, McConfig(n_gpus=1, alpha=1.0, mode=0))
    with pytest.raises(SplitError) as many:
        compute_preconditioner(b, McConfig(n_gpus=3, alpha=1.0, mode=0))
    assert str(one.value) == str(many.value)
