"""Pins the CPU oracle (oracle/mcmi_oracle.c) before it is trusted as the
checker: Random123 known-answer vectors, the reference's own exact unit-test
values, the BASELINE.md golden hashes, and direct equality with the
UNMODIFIED reference library (oracle/_ref) on every golden case.
"""
import numpy as np
import pytest

from helpers import bits_equal, golden_input, goldens, mm_sha256

# SURVEY.md §8c, verified against Random123 philox4x32_10
PHILOX_KAT = [
    ([0, 0, 0, 0], [0, 0], [0x6627E8D5, 0xE169C58D, 0xBC57AC4C, 0x9B00DBD8]),
    ([0xFFFFFFFF] * 4, [0xFFFFFFFF] * 2, [0x408F276D, 0x41C83B0E, 0xA20BC7C6, 0x6D5451FD]),
    ([0x243F6A88, 0x85A308D3, 0x13198A2E, 0x03707344], [0xA4093822, 0x299F31D0],
     [0xD16CFE09, 0x94FDCCEB, 0x5001E420, 0x24126EA1]),
]

BASELINE_MD_HASHES = {
    "poisson2d_100_default_seed0": "43c063c12da4b2c49ed338aa62fa1249149bbee5b6c1d43fc056aa8564c2f670",
    "rdb2048_acc6": "eec0935147fda558747341140fd63cff09edb5c2bb9afd8dbe368bb0262bcb2a",
    "convdiff_64_default_seed7": "d02541a0dce21ae8703072f82efb25d2af5371b47e0906a59a1d507fc3da43bb",
    "broad1024_bench": "c5853ebc8619bf72f9f077cad299219ca0f0928c0489d7d4a51702725012b033",
}


@pytest.mark.parametrize("ctr,key,want", PHILOX_KAT)
def test_philox_known_answers(oracle_mod, ctr, key, want):
    assert oracle_mod.philox(ctr, key) == want


def test_stream_matches_reference(ref_mod):
    # RngStream(0x0123456789abcdef, 5) first words and RngStream(42,0).next_double()
    assert ref_mod.rng_u32(0x0123456789ABCDEF, 5, 4).tolist() == [0xB341ED12, 0x7899C9CC, 0x8D35F144, 0x68EBA6FB]
    assert ref_mod.rng_double(42, 0, 1)[0] == 0.46858651833910492


def test_goldens_agree_with_baseline_md():
    g = goldens()
    for name, h in BASELINE_MD_HASHES.items():
        assert g[name]["mm_sha256"] == h


@pytest.mark.parametrize("name", sorted(goldens()))
def test_oracle_matches_golden(oracle_mod, name):
    case = goldens()[name]
    n, rp, ci, v = golden_input(case["input"])
    r = oracle_mod.compute_preconditioner(n, rp, ci, v, **case["config"])
    assert r.n_chains == case["n_chains"] and r.max_len == case["max_len"]
    assert int(r.row_ptr[-1]) == case["nnz"]
    assert mm_sha256(n, r.row_ptr, r.col_idx, r.values) == case["mm_sha256"]


@pytest.mark.parametrize("name", sorted(goldens()))
def test_oracle_matches_reference_library(oracle_mod, ref_mod, name):
    case = goldens()[name]
    n, rp, ci, v = golden_input(case["input"])
    r = oracle_mod.compute_preconditioner(n, rp, ci, v, **case["config"])
    b = ref_mod.Csr(n, rp, ci, v)
    want = ref_mod.compute_preconditioner(b, serial=True, **case["config"])
    assert np.array_equal(r.row_ptr, want.m.row_ptr)
    assert np.array_equal(r.col_idx, want.m.col_idx)
    assert bits_equal(r.values, want.m.values)
    assert np.array_equal(r.chains_used, want.chains_used)
    assert np.array_equal(r.entries_before, want.entries_before)


def _mat(n, rows, cols, vals):
    from paper_2409_03095_b200.mcspai import CsrMatrix
    return CsrMatrix.from_triplets(n, rows, cols, vals)


def test_budget_kat(oracle_mod):
    # test_mc_engine.cpp:80-86: eps=.05, delta=.01, ||A||=.5 -> N=728, L=7.
    # A 2x2 system with ||A|| = 0.5 exactly: b = [[1, .5],[.5, 1]], alpha s.t. b_hat_ii = 1
    # is not reachable with alpha > 0, so use rows whose off-diagonal / b_hat = 0.5:
    # b = [[1, -3],[0, 1]], ||B|| = 4, alpha = .5 -> b_hat_00 = 3, a_01 = 1.
    # Instead pin the formula through the reference on the same a_norm values.
    from oracle import ref
    if not ref.available():
        pytest.skip("oracle/_ref missing")
    assert ref.derive_chain_budget(0.5, epsilon=0.05, delta=0.01) == (728, 7)
    assert ref.derive_chain_budget(0.0, epsilon=0.6745) == (1, 1)
    assert ref.derive_chain_budget(0.5, epsilon=0.5, chains_override=1000, max_len_override=3) == (1000, 3)


def test_identity_pipeline(oracle_mod):
    # test_mc_engine.cpp:222-230: identity, alpha = 1 -> M = 0.5 I, one entry per row
    m = _mat(6, range(6), range(6), [1.0] * 6)
    r = oracle_mod.compute_preconditioner(6, m.row_ptr, m.col_idx, m.values, alpha=1.0)
    assert np.array_equal(r.col_idx, np.arange(6)) and np.all(r.values == 0.5)
    assert np.all(r.entries_before == 1)
    assert np.all(r.chains_used == 1)  # chain 0 consumed no randomness


def test_zero_variance_matches_neumann(oracle_mod):
    # acceptance.cpp:124-162 / test_mc_engine.cpp:129-148 circulant shift
    n = 5
    m = _mat(n, list(range(5)) * 2, list(range(5)) + [1, 2, 3, 4, 0],
             [2.0, -2.0, 2.0, 2.0, -2.0, 0.7, -0.6, 0.5, 0.9, -0.8])
    for seed in (0, 7, 1234567):
        r = oracle_mod.compute_preconditioner(n, m.row_ptr, m.col_idx, m.values, epsilon=0.1, delta=0.05,
                                              alpha=1.5, master_seed=seed)
        assert np.all(r.chains_used == 1)
    r0 = oracle_mod.compute_preconditioner(n, m.row_ptr, m.col_idx, m.values, epsilon=0.1, delta=0.05, alpha=1.5)
    r1 = oracle_mod.compute_preconditioner(n, m.row_ptr, m.col_idx, m.values, epsilon=0.1, delta=0.05, alpha=1.5,
                                           master_seed=99)
    assert bits_equal(r0.values, r1.values)


def test_error_behaviour(oracle_mod):
    from oracle.oracle import OracleError
    # plain mode cancelling a negative diagonal (test_mc_split.cpp:89-94)
    m = _mat(2, [0, 1], [0, 1], [-1.0, 1.0])
    with pytest.raises(OracleError) as e:
        oracle_mod.compute_preconditioner(2, m.row_ptr, m.col_idx, m.values, alpha=1.0, mode=0)
    assert e.value.code == 2 and "degenerate diagonal after augmentation at row 0" in str(e.value)
    # dominance failure (test_mc_split.cpp:104-111)
    m = _mat(2, [0, 0, 1], [0, 1, 1], [-10.0, 10.0, 1.0])
    with pytest.raises(OracleError) as e:
        oracle_mod.compute_preconditioner(2, m.row_ptr, m.col_idx, m.values, alpha=1.0, mode=0)
    assert e.value.code == 2 and "diagonal dominance failure" in str(e.value)
    with pytest.raises(OracleError) as e:
        oracle_mod.compute_preconditioner(2, m.row_ptr, m.col_idx, m.values, drop_fraction=1.5)
    assert e.value.code == 1
    with pytest.raises(OracleError) as e:
        oracle_mod.compute_preconditioner(2, m.row_ptr, m.col_idx, m.values, alpha=0.0)
    assert e.value.code == 1


def test_keyed_mode_differs_but_same_pattern_rules(oracle_mod):
    n, rp, ci, v = golden_input("convdiff:64:20:10")
    a = oracle_mod.compute_preconditioner(n, rp, ci, v, master_seed=7, rng_mode=0)
    b = oracle_mod.compute_preconditioner(n, rp, ci, v, master_seed=7, rng_mode=1)
    assert not bits_equal(a.values, b.values)
    # same estimator: agree within Monte Carlo error on the diagonal
    da = a.values[np.searchsorted(a.col_idx[a.row_ptr[0]:a.row_ptr[1]], 0)]
    db = b.values[np.searchsorted(b.col_idx[b.row_ptr[0]:b.row_ptr[1]], 0)]
    assert abs(da - db) / abs(da) < 0.05


def test_row_range_is_slice_of_full(oracle_mod):
    n, rp, ci, v = golden_input("convdiff:64:20:10")
    full = oracle_mod.compute_preconditioner(n, rp, ci, v, master_seed=7)
    part = oracle_mod.compute_preconditioner(n, rp, ci, v, master_seed=7, row_begin=1000, row_end=1500)
    lo, hi = full.row_ptr[1000], full.row_ptr[1500]
    assert np.array_equal(part.row_ptr, full.row_ptr[1000:1501] - lo)
    assert np.array_equal(part.col_idx, full.col_idx[lo:hi])
    assert bits_equal(part.values, full.values[lo:hi])
