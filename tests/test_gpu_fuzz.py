"""Randomised differential parity: random sparse matrices (random and
structured patterns, explicit zeros, missing diagonals, empty rows, negative
diagonals) x random McConfig (every field, both RNG keyings) built on the GPU
and compared bit for bit with the oracle, and for rng_mode=reference also with
the unmodified reference library.  Error cases must raise the same error class
as the reference."""
import numpy as np
import pytest

from helpers import bits_equal

pytestmark = pytest.mark.gpu

N_CASES = 400


def random_matrix(rng: np.random.Generator):
    from paper_2409_03095_b200.mcspai import CsrMatrix
    n = int(rng.choice([1, 2, 3, 5, 8, 17, 40, 97, 250]))
    kind = rng.integers(0, 4)
    rows, cols, vals = [], [], []
    for i in range(n):
        if kind == 0:  # random fill
            k = rng.integers(0, min(n, 12) + 1)
            cs = rng.choice(n, size=k, replace=False) if k else []
        elif kind == 1:  # banded
            cs = [j for j in range(max(0, i - 2), min(n, i + 3))]
        elif kind == 2:  # power-law-ish hubs
            k = min(n, int(rng.pareto(1.5)) + 1)
            cs = rng.choice(n, size=k, replace=False)
        else:  # single off-diagonal (zero-variance walks)
            cs = [(i + 1) % n] if n > 1 else []
        for j in cs:
            rows.append(i)
            cols.append(int(j))
            v = rng.uniform(-1, 1) * 10.0 ** rng.uniform(-4, 1)
            if rng.random() < 0.03:
                v = 0.0  # explicit zero (pruned by from_triplets)
            vals.append(v)
        if rng.random() < 0.9:  # diagonal (sometimes missing, sometimes negative)
            rows.append(i)
            cols.append(i)
            vals.append(rng.uniform(0.5, 20.0) * (-1 if rng.random() < 0.3 else 1))
    return CsrMatrix.from_triplets(n, rows, cols, vals)


def random_config(rng: np.random.Generator, mc):
    cfg = mc.McConfig(
        epsilon=float(rng.choice([0.5, 0.2, 0.1, 0.05, 0.02])),
        delta=float(rng.choice([0.5, 0.1, 0.01, 1e-3, 1e-9])),
        alpha=float(rng.choice([0.3, 1.0, 1.5, 2.0, 5.0])),
        mode=mc.AugmentationMode(int(rng.integers(0, 2))),
        drop_fraction=float(rng.choice([0.0, 0.0, 0.1, 0.5, 1.0])),
        drop_mode=mc.DropMode(int(rng.integers(0, 2))),
        retain_k=int(rng.choice([0, 0, 1, 3, 8, 40])),
        chains_override=int(rng.choice([1, 7, 33, 200])) if rng.random() < 0.3 else None,
        max_len_override=int(rng.choice([0, 1, 2, 5, 40])) if rng.random() < 0.3 else None,
        master_seed=int(rng.integers(0, 2**63)),
        rng_mode=mc.RngMode(int(rng.integers(0, 2))),
    )
    return cfg


@pytest.fixture(scope="module")
def env():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from oracle import oracle, ref
    from paper_2409_03095_b200 import mcspai
    return mcspai, oracle, ref if ref.available() else None


@pytest.mark.parametrize("seed", [20261018, 7, 99])
def test_random_differential(env, seed):
    mc, oracle, ref = env
    rng = np.random.default_rng(seed)
    checked = errors = 0
    for case in range(N_CASES):
        b = random_matrix(rng)
        cfg = random_config(rng, mc)
        try:
            want = oracle.compute_preconditioner(b.n, b.row_ptr, b.col_idx, b.values, **cfg.oracle_kwargs())
            want_err = None
        except oracle.OracleError as e:
            want, want_err = None, e.code
        try:
            got = mc.compute_preconditioner(b, cfg)
            got_err = None
        except ValueError:
            got, got_err = None, 1
        except mc.SplitError:
            got, got_err = None, 2
        ctx = f"case {case}: n={b.n} cfg={cfg}"
        assert got_err == want_err, ctx
        if want_err is not None:
            errors += 1
            continue
        assert np.array_equal(got.m.row_ptr, want.row_ptr), ctx
        assert np.array_equal(got.m.col_idx, want.col_idx), ctx
        assert bits_equal(got.m.values, want.values), ctx
        assert np.array_equal(got.row_meta.chains_used, want.chains_used), ctx
        assert np.array_equal(got.row_meta.entries_before_retention, want.entries_before), ctx
        assert got.stats["walk_steps"] == want.walk_steps, ctx
        if ref is not None and int(cfg.rng_mode) == 0:
            kw = {k: v for k, v in cfg.oracle_kwargs().items() if k != "rng_mode"}
            r = ref.compute_preconditioner(ref.Csr(b.n, b.row_ptr, b.col_idx, b.values), **kw)
            assert np.array_equal(got.m.col_idx, r.m.col_idx) and bits_equal(got.m.values, r.m.values), ctx
        checked += 1
    assert checked >= N_CASES // 2 and errors >= 1
