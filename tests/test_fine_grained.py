"""The reference's fine-grained public functions (derive_chain_budget,
augment_and_split, transition_probabilities, estimate_row), checked against
the unmodified reference (oracle/_ref) bit for bit, with its error types and
messages.  derive_chain_budget is host code and runs here; the others run the
device kernels (@gpu)."""
import numpy as np
import pytest

from helpers import bits_equal


def _ref_csr(ref, m):
    return ref.Csr(m.n, m.row_ptr, m.col_idx, m.values)


def _same_csr(got, want):
    assert got.n == want.n
    assert np.array_equal(got.row_ptr, want.row_ptr)
    assert np.array_equal(got.col_idx, want.col_idx)
    assert bits_equal(got.values, want.values)


# ------------------------------------------------------------ host (CPU suite)

@pytest.mark.parametrize("a_norm", [0.0, 1e-300, 1 / 11, 0.25, 0.5, 0.9, 0.999999, 1 - 2 ** -52])
@pytest.mark.parametrize("eps,delta", [(0.0625, 0.0625), (0.01, 0.01), (0.5, 1e-300), (1e-4, 0.9)])
def test_derive_chain_budget_matches_reference(ref_mod, a_norm, eps, delta):
    from paper_2409_03095_b200.mcspai import McConfig, derive_chain_budget
    got = derive_chain_budget(McConfig(epsilon=eps, delta=delta), a_norm)
    assert (got.n_chains, got.max_len) == ref_mod.derive_chain_budget(a_norm, epsilon=eps, delta=delta)


def test_derive_chain_budget_overrides_and_errors(ref_mod):
    from paper_2409_03095_b200.mcspai import McConfig, derive_chain_budget
    for kw in (dict(chains_override=7), dict(max_len_override=3), dict(chains_override=0, max_len_override=0),
               dict(chains_override=-5)):
        got = derive_chain_budget(McConfig(**kw), 0.3)
        assert (got.n_chains, got.max_len) == ref_mod.derive_chain_budget(0.3, **kw)
    for bad in (1.0, 1.5, -0.1, float("nan")):
        with pytest.raises(ValueError, match=r"\|\|A\|\| must lie in \[0,1\)"):
            derive_chain_budget(McConfig(), bad)
        with pytest.raises(Exception):
            ref_mod.derive_chain_budget(bad)


# ------------------------------------------------------------ device (B200)

def _matrices():
    from paper_2409_03095_b200 import generators as G
    from paper_2409_03095_b200.mcspai import CsrMatrix
    rng = np.random.default_rng(9)
    out = {"convdiff20": G.convection_diffusion(20), "lap3d_6": G.laplacian3d(6),
           "powerlaw500": G.powerlaw(500, dmax=50, seed=2)}
    # missing diagonals, duplicate diagonal entries, negative diagonals, empty rows
    n = 60
    rows, cols, vals = [], [], []
    for i in range(n):
        if i % 7:  # every 7th row has no diagonal
            rows.append(i), cols.append(i), vals.append(float(rng.choice([-1, 1])) * (4.0 + rng.random()))
        for j in rng.choice(n, size=int(rng.integers(0, 4)), replace=False):
            if j != i:
                rows.append(i), cols.append(int(j)), vals.append(float(rng.normal()))
    order = np.lexsort((cols, rows))
    r, c, v = np.array(rows)[order], np.array(cols)[order], np.array(vals)[order]
    rp = np.zeros(n + 1, np.int64)
    np.add.at(rp, r + 1, 1)
    out["ragged60"] = CsrMatrix(n, np.cumsum(rp), c, v)
    # a duplicated diagonal entry (only the first is augmented) and an explicit zero
    out["dupdiag"] = CsrMatrix(3, np.array([0, 3, 5, 7]), np.array([0, 0, 2, 1, 1, 0, 2]),
                               np.array([2.0, 0.5, -0.25, 3.0, 0.0, 1.0, -2.0]))
    return out


@pytest.mark.gpu
@pytest.mark.parametrize("name", ["convdiff20", "lap3d_6", "powerlaw500", "ragged60", "dupdiag"])
@pytest.mark.parametrize("alpha,mode", [(5.0, 1), (5.0, 0), (1.5, 1), (2.5, 0)])
def test_augment_and_split_matches_reference(ref_mod, name, alpha, mode):
    from paper_2409_03095_b200.mcspai import augment_and_split
    b = _matrices()[name]
    try:
        want = ref_mod.augment_and_split(_ref_csr(ref_mod, b), alpha, mode)
    except Exception as exc:  # noqa: BLE001 — the reference rejects it: so must we, with the same message
        with pytest.raises(Exception) as got:
            augment_and_split(b, alpha, mode)
        assert str(exc).split(": ", 1)[-1] in str(got.value)
        return
    got = augment_and_split(b, alpha, mode)
    _same_csr(got.b_hat, want.b_hat)
    _same_csr(got.a, want.a)
    _same_csr(got.p, want.p)
    assert bits_equal(got.b1_diag, want.b1_diag)
    assert bits_equal(got.s_diag, want.s_diag)
    assert np.float64(got.a_norm).view(np.uint64) == np.float64(want.a_norm).view(np.uint64)


@pytest.mark.gpu
def test_augment_and_split_errors(ref_mod):
    from paper_2409_03095_b200.mcspai import CsrMatrix, SplitError, augment_and_split
    b = CsrMatrix(3, np.array([0, 2, 4, 5]), np.array([0, 1, 0, 1, 2]), np.array([1.0, -0.5, -0.5, 1.0, 1.0]))
    for alpha in (0.0, -1.0, float("nan")):
        with pytest.raises(ValueError, match="^alpha must be positive$"):
            augment_and_split(b, alpha)
    # plain mode, b_ii = -alpha * ||B||inf: degenerate diagonal at row 1 (split.cpp:67-69)
    d = CsrMatrix(3, np.array([0, 1, 2, 3]), np.array([0, 1, 2]), np.array([1.0, -2.0, 1.0]))
    with pytest.raises(SplitError, match="^degenerate diagonal after augmentation at row 1$"):
        augment_and_split(d, 1.0, 0)
    # small alpha: ||A|| >= 1 (split.cpp:94-96), the reference's std::to_string formatting
    w = CsrMatrix(2, np.array([0, 2, 4]), np.array([0, 1, 0, 1]), np.array([1.0, 3.0, 3.0, 1.0]))
    with pytest.raises(SplitError, match=r"^diagonal dominance failure: \|\|A\|\|inf = 1\.500000$") as got:
        augment_and_split(w, 0.25)
    with pytest.raises(Exception) as want:
        ref_mod.augment_and_split(_ref_csr(ref_mod, w), 0.25, 1)
    assert str(got.value) in str(want.value)


@pytest.mark.gpu
def test_transition_probabilities_any_a():
    """Rows summing to zero become empty; explicit zeros inside a non-zero row
    stay (split.cpp:102-119); checked against a sequential numpy restatement."""
    from paper_2409_03095_b200.mcspai import CsrMatrix, transition_probabilities
    rng = np.random.default_rng(4)
    n = 300
    deg = rng.integers(0, 9, size=n)
    rp = np.concatenate([[0], np.cumsum(deg)]).astype(np.int64)
    ci = rng.integers(0, n, size=rp[-1]).astype(np.int64)
    v = rng.normal(size=rp[-1]) * (rng.random(rp[-1]) < 0.8)
    for i in range(0, n, 13):
        v[rp[i]:rp[i + 1]] = 0.0  # all-zero rows
    a = CsrMatrix(n, rp, ci, v)
    got = transition_probabilities(a)
    wrp, wci, wv = [0], [], []
    for i in range(n):
        s = 0.0
        for k in range(rp[i], rp[i + 1]):
            s += abs(v[k])
        if s > 0.0:
            for k in range(rp[i], rp[i + 1]):
                wci.append(ci[k])
                wv.append(abs(v[k]) / s)
        wrp.append(len(wci))
    _same_csr(got, CsrMatrix(n, np.array(wrp), np.array(wci, np.int64), np.array(wv)))
    empty = transition_probabilities(CsrMatrix(0, np.zeros(1, np.int64), np.zeros(0, np.int64), np.zeros(0)))
    assert empty.n == 0 and empty.row_ptr.tolist() == [0]


@pytest.mark.gpu
@pytest.mark.parametrize("name,alpha,n_chains,max_len,delta",
                         [("convdiff20", 5.0, 141, 2, 0.0625), ("lap3d_6", 1.5, 500, 4, 0.01),
                          ("powerlaw500", 1.0, 64, 8, 1e-300), ("ragged60", 2.0, 33, 3, 0.1),
                          ("convdiff20", 5.0, 1, 1, 0.5)])
def test_estimate_row_matches_reference(ref_mod, name, alpha, n_chains, max_len, delta):
    from paper_2409_03095_b200.mcspai import ChainBudget, RngStream, augment_and_split, estimate_row
    b = _matrices()[name]
    sp = augment_and_split(b, alpha)
    want_sp = ref_mod.augment_and_split(_ref_csr(ref_mod, b), alpha, 1, keep_handle=True)
    try:
        for r in sorted({0, 1, b.n // 2, b.n - 1}):
            for seed in (0, 20260826):
                got = estimate_row(sp, r, ChainBudget(n_chains, max_len), delta, RngStream(seed, r))
                wc, wv = ref_mod.estimate_row(want_sp, r, n_chains, max_len, delta, seed)
                assert [c for c, _ in got] == wc.tolist(), (r, seed)
                assert bits_equal(np.array([x for _, x in got]), wv), (r, seed)
    finally:
        ref_mod.free_split(want_sp)


@pytest.mark.gpu
def test_estimate_row_rejects_other_streams():
    from paper_2409_03095_b200 import generators as G
    from paper_2409_03095_b200.mcspai import ChainBudget, RngStream, augment_and_split, estimate_row
    sp = augment_and_split(G.convection_diffusion(10), 5.0)
    with pytest.raises(ValueError, match="stream_id must equal r"):
        estimate_row(sp, 3, ChainBudget(10, 2), 0.1, RngStream(0, 4))


@pytest.mark.gpu
@pytest.mark.parametrize("name", ["convdiff20", "powerlaw500", "ragged60", "dupdiag"])
@pytest.mark.parametrize("p", [0.0, 0.1, 0.5, 0.999, 1.0])
@pytest.mark.parametrize("mode", [0, 1])
def test_drop_small_entries_matches_reference(ref_mod, name, p, mode):
    from paper_2409_03095_b200.mcspai import drop_small_entries
    b = _matrices()[name]
    _same_csr(drop_small_entries(b, p, mode), ref_mod.drop_small_entries(_ref_csr(ref_mod, b), p, mode))


@pytest.mark.gpu
def test_drop_small_entries_ties_and_errors(ref_mod):
    """Equal magnitudes (count quantile breaks ties by position) and the
    reference's range error."""
    from paper_2409_03095_b200.mcspai import CsrMatrix, drop_small_entries
    n = 40
    rng = np.random.default_rng(1)
    rp = np.arange(0, 4 * n + 1, 4)
    ci = np.array([[i, (i + 1) % n, (i + 2) % n, (i + 5) % n] for i in range(n)]).ravel()
    order = np.argsort(ci.reshape(n, 4), axis=1)
    ci = np.take_along_axis(ci.reshape(n, 4), order, axis=1).ravel()
    v = rng.choice([-0.5, 0.5, 0.25, 1.0], size=4 * n)
    b = CsrMatrix(n, rp, ci, v)
    for p in (0.2, 0.37, 0.75):
        for mode in (0, 1):
            _same_csr(drop_small_entries(b, p, mode), ref_mod.drop_small_entries(_ref_csr(ref_mod, b), p, mode))
    for bad in (-0.1, 1.1, float("nan")):
        with pytest.raises(ValueError, match=r"^drop fraction must lie in \[0,1\]$"):
            drop_small_entries(b, bad)


# ---------------------------------------------- estimate_row on a hand-built SplitSystem

def _hand_split(rng, n, density, p_mode):
    """A random SplitSystem built by hand, as the reference's tests do: A with
    random signed values (explicit zeros, empty and single-entry rows), P on A's
    pattern: transition_probabilities(A), unnormalised weights (rows summing to
    less than 1 exercise sample_transition's end-1 fallback), or zeros."""
    rows, cols, vals = [], [], []
    for i in range(n):
        k = int(rng.integers(0, max(2, int(density * n))))
        c = np.unique(rng.integers(0, n, size=k))
        rows += [i] * c.size
        cols += c.tolist()
        vals += (rng.uniform(-0.3, 0.3, size=c.size) * (rng.uniform(size=c.size) > 0.05)).tolist()
    order = np.lexsort((cols, rows))
    rows, cols, vals = np.array(rows, np.int64)[order], np.array(cols, np.int64)[order], np.array(vals)[order]
    rp = np.zeros(n + 1, np.int64)
    np.add.at(rp, rows + 1, 1)
    rp = np.cumsum(rp)
    if p_mode == "tp":
        s = np.bincount(rows, weights=np.abs(vals), minlength=n)
        s = np.where(s > 0, s, 1.0)
        p = np.abs(vals) / s[rows]
    elif p_mode == "short":
        p = rng.uniform(0.0, 1.0, size=vals.size) / np.repeat(np.maximum(np.diff(rp), 1), np.diff(rp)) * 0.9
    else:
        p = rng.uniform(0.0, 0.5, size=vals.size)
    return n, rp, cols, vals, p


@pytest.mark.gpu
@pytest.mark.parametrize("p_mode", ["tp", "short", "raw"])
@pytest.mark.parametrize("rng_seed", [1, 2, 3])
def test_estimate_rows_hand_built_split_matches_reference(ref_mod, p_mode, rng_seed):
    """mcmi_estimate_rows on split.a / split.p built by hand equals the
    reference's estimate_row on the same SplitSystem, row by row, bit for bit."""
    from paper_2409_03095_b200.mcspai import ChainBudget, CsrMatrix, SplitSystem, estimate_rows
    rng = np.random.default_rng(rng_seed)
    n, rp, ci, av, pv = _hand_split(rng, 150, 0.05, p_mode)
    a = CsrMatrix(n, rp, ci, av)
    split = SplitSystem(b_hat=a, b1_diag=np.ones(n), a=a, p=CsrMatrix(n, rp, ci, pv), s_diag=np.zeros(n), a_norm=0.5)
    want_sp = ref_mod.split_from_ap(n, rp, ci, av, pv)
    try:
        for nc, ml, delta, seed in ((200, 3, 1e-3, 5), (37, 8, 1e-9, 20261019), (1, 1, 0.5, 0)):
            got = estimate_rows(split, 0, n, ChainBudget(nc, ml), delta, seed)
            for r in range(n):
                wc, wv = ref_mod.estimate_row(want_sp, r, nc, ml, delta, seed)
                a0, a1 = got.row_ptr[r], got.row_ptr[r + 1]
                assert got.col_idx[a0:a1].tolist() == wc.tolist(), (r, nc, ml)
                assert bits_equal(got.values[a0:a1], wv), (r, nc, ml)
    finally:
        ref_mod.free_split(want_sp)


@pytest.mark.gpu
def test_estimate_row_single_transition_chain_exact():
    """test_mc_engine.cpp:112-127: A = [[0, 0.5], [0, 0]], P = transition_probabilities(A),
    (I - A)^-1 row 0 = [1, 0.5] exactly, for any seed."""
    from paper_2409_03095_b200.mcspai import (ChainBudget, CsrMatrix, RngStream, SplitSystem, estimate_row,
                                              transition_probabilities)
    a = CsrMatrix.from_triplets(2, [0], [1], [0.5])
    split = SplitSystem(b_hat=a, b1_diag=np.ones(2), a=a, p=transition_probabilities(a), s_diag=np.zeros(2),
                        a_norm=0.5)
    for seed in (1, 99, 31337):
        assert estimate_row(split, 0, ChainBudget(25, 8), 1e-6, RngStream(seed, 0)) == [(0, 1.0), (1, 0.5)]


@pytest.mark.gpu
def test_estimate_row_identity_absorbs():
    """test_mc_engine.cpp:100-110: identity input absorbs immediately -> row r = [(r, 1)]."""
    from paper_2409_03095_b200.mcspai import ChainBudget, CsrMatrix, RngStream, augment_and_split, estimate_row
    sp = augment_and_split(CsrMatrix.identity(4), 1.0)
    for r in range(4):
        assert estimate_row(sp, r, ChainBudget(50, 10), 0.01, RngStream(123, r)) == [(r, 1.0)]


# ---------------------------------------------- retain_top_k / scale_columns entry points

@pytest.mark.gpu
def test_retain_top_k_reference_cases():
    """test_mc_engine.cpp:193-213, verbatim."""
    from paper_2409_03095_b200.mcspai import retain_top_k
    row = [(0, 1.0), (3, 0.5)]
    assert retain_top_k(row, 5, 0) == row
    assert retain_top_k(row, 0, 0) == row  # 0 = unlimited
    assert retain_top_k([(1, 1.0), (3, 0.9), (5, 0.2), (7, 0.8)], 2, 1) == [(1, 1.0), (3, 0.9)]
    assert retain_top_k([(1, 0.1), (2, 5.0), (4, 5.0), (6, 5.0)], 2, 1) == [(1, 0.1), (2, 5.0)]


@pytest.mark.gpu
@pytest.mark.parametrize("seed", [0, 1, 2])
def test_retain_top_k_rows_match_reference(ref_mod, seed):
    """Every row of a random CSR (ties in |v|, signs, diagonal present or not,
    rows shorter and longer than k, k <= 0) against the reference's
    retain_top_k, row by row, bit for bit."""
    from paper_2409_03095_b200.mcspai import CsrMatrix, retain_top_k_rows
    rng = np.random.default_rng(seed)
    n = 300
    lens = rng.integers(0, 700, size=n)
    lens[:5] = [0, 1, 2, 600, 1500]
    rp = np.concatenate(([0], np.cumsum(lens))).astype(np.int64)
    ci = np.concatenate([np.sort(rng.choice(5000, size=x, replace=False)) for x in lens]).astype(np.int64)
    v = rng.choice([-0.5, 0.5, 0.25, -1e-3, 2.0], size=ci.size) * (rng.uniform(size=ci.size) < 0.5) + \
        rng.normal(size=ci.size) * (rng.uniform(size=ci.size) >= 0.5)
    diag = np.where(rng.uniform(size=n) < 0.5, np.arange(n), rng.integers(0, 5000, size=n))
    m = CsrMatrix(n, rp, ci, v)
    for k in (0, -3, 1, 7, 32, 500):
        got = retain_top_k_rows(m, k, diag)
        for r in range(n):
            wc, wv = ref_mod.retain_top_k(ci[rp[r]:rp[r + 1]], v[rp[r]:rp[r + 1]], k, int(diag[r]))
            a, b = got.row_ptr[r], got.row_ptr[r + 1]
            assert got.col_idx[a:b].tolist() == wc.tolist(), (k, r)
            assert bits_equal(got.values[a:b], wv), (k, r)


@pytest.mark.gpu
def test_scale_columns_reference_case_and_range():
    """test_mc_engine.cpp:215-220, plus the batched form and a column outside b1_diag."""
    from paper_2409_03095_b200.mcspai import CsrMatrix, scale_columns, scale_columns_rows
    row = [(0, 1.0), (1, 1.0)]
    scale_columns(row, [2.0, 4.0])
    assert row == [(0, 0.5), (1, 0.25)]
    rng = np.random.default_rng(3)
    m = CsrMatrix(3, np.array([0, 2, 2, 5]), np.array([0, 4, 1, 2, 3]), rng.normal(size=5))
    b1 = rng.uniform(0.5, 3.0, size=5)
    got = scale_columns_rows(m, b1)
    assert bits_equal(got.values, m.values / b1[m.col_idx])
    with pytest.raises(IndexError):
        scale_columns_rows(m, b1[:3])
