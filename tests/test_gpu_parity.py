"""GPU parity: the sm_100a build through the C-ABI vs the reference.

Tier 1 (bit-exact):
  * rng_mode=reference: byte-identical Matrix Market output to the UNMODIFIED
    reference on every golden case (sha256 recorded by make_goldens.py from
    oracle/_ref), plus RowMeta and the chain budget.
  * rng_mode=keyed: bit-identical to the CPU oracle's keyed restatement.
  * Full-size configs (C2, C3, C4): sampled row windows bit-identical to the
    oracle, which restates the whole split and walks only those rows.
Tier 2 (Monte Carlo tolerance, stated here): keyed vs reference stream on the
same input: ||M_K - M_R||_F / ||M_R||_F <= 0.3*eps, max |M_K - M_R| <= 0.5*eps*max|M_R|,
||I - B_hat M||_F / sqrt(n) within 10% of the reference's.
"""
import numpy as np
import pytest

from helpers import arr_sha256, bits_equal, golden_input, goldens, mm_sha256

pytestmark = pytest.mark.gpu

GOLD = goldens()


@pytest.fixture(scope="module")
def mc():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2409_03095_b200 import mcspai
    return mcspai


def _csr(mc, spec):
    n, rp, ci, v = golden_input(spec)
    return mc.CsrMatrix(n, rp, ci, v)


def _cfg(mc, d, **extra):
    d = dict(d)
    d.update(extra)
    for k in ("mode", "drop_mode", "rng_mode"):
        if k in d:
            d[k] = int(d[k])
    return mc.McConfig(**d)


@pytest.mark.parametrize("name", sorted(GOLD))
def test_reference_stream_byte_identical_to_reference(mc, name):
    case = GOLD[name]
    b = _csr(mc, case["input"])
    inv = mc.compute_preconditioner(b, _cfg(mc, case["config"]))
    assert inv.budget_echo.n_chains == case["n_chains"]
    assert inv.budget_echo.max_len == case["max_len"]
    assert inv.m.nnz() == case["nnz"]
    assert mm_sha256(b.n, inv.m.row_ptr, inv.m.col_idx, inv.m.values) == case["mm_sha256"]
    assert arr_sha256(inv.row_meta.chains_used) == case["chains_used_sha256"]
    assert arr_sha256(inv.row_meta.entries_before_retention) == case["entries_before_sha256"]


@pytest.mark.parametrize("name", sorted(GOLD))
def test_keyed_bit_identical_to_oracle(mc, oracle_mod, name):
    case = GOLD[name]
    b = _csr(mc, case["input"])
    cfg = _cfg(mc, case["config"], rng_mode=1, deg_stats=True)
    inv = mc.compute_preconditioner(b, cfg)
    want = oracle_mod.compute_preconditioner(b.n, b.row_ptr, b.col_idx, b.values, **cfg.oracle_kwargs())
    assert np.array_equal(inv.m.row_ptr, want.row_ptr)
    assert np.array_equal(inv.m.col_idx, want.col_idx)
    assert bits_equal(inv.m.values, want.values)
    assert np.array_equal(inv.row_meta.chains_used, want.chains_used)
    assert np.array_equal(inv.row_meta.entries_before_retention, want.entries_before)
    assert inv.stats["walk_steps"] == want.walk_steps
    assert inv.stats["walk_deg_sum"] == want.walk_deg_sum


@pytest.mark.parametrize("rng", [0, 1])
def test_step_counters_match_oracle(mc, oracle_mod, rng):
    b = _csr(mc, "convdiff:100:0:0")
    inv = mc.compute_preconditioner(b, mc.McConfig(rng_mode=rng, deg_stats=True))
    want = oracle_mod.compute_preconditioner(b.n, b.row_ptr, b.col_idx, b.values, rng_mode=rng)
    assert mc.compute_preconditioner(b, mc.McConfig(rng_mode=rng)).stats["walk_deg_sum"] == -1  # opt-in
    assert inv.stats["walk_steps"] == want.walk_steps
    if rng == 0:
        assert want.walk_steps == 2819436  # SURVEY.md §6 probe of the reference
    assert inv.stats["walk_deg_sum"] == want.walk_deg_sum


def test_identity_pipeline(mc):
    # test_mc_engine.cpp:222-230
    inv = mc.compute_preconditioner(mc.CsrMatrix.identity(6), mc.McConfig(alpha=1.0))
    assert inv.m.nnz() == 6
    assert all(inv.m.at(i, i) == 0.5 for i in range(6))
    assert np.all(inv.row_meta.entries_before_retention == 1)
    assert inv.budget_echo.n_chains >= 1


def test_zero_variance_equals_truncated_neumann(mc):
    # acceptance.cpp:124-162: one transition per P row -> deterministic walks
    b = mc.CsrMatrix.from_triplets(6, list(range(6)) * 2, list(range(6)) + [1, 2, 3, 4, 5, 0],
                                   [3.0, -3.0, 3.0, 3.0, -3.0, 3.0, 0.9, -0.8, 0.7, 0.6, 0.5, -0.4])
    cfg = mc.McConfig(epsilon=0.1, delta=0.02, alpha=1.5)
    ref = None
    for seed in (0, 42, 987654321):
        for rng in (0, 1):
            cfg.master_seed, cfg.rng_mode = seed, rng
            inv = mc.compute_preconditioner(b, cfg)
            assert np.all(inv.row_meta.chains_used == 1)
            if ref is None:
                ref = inv.m
            assert inv.m == ref


def test_single_transition_chain_exact(mc, ref_mod):
    # test_mc_engine.cpp:112-127 at pipeline level (the estimate_row form on a
    # hand-built SplitSystem is test_fine_grained.py::
    # test_estimate_row_single_transition_chain_exact): row 0 of B has one
    # off-diagonal entry, so its walks are deterministic, one chain runs, and
    # M equals the reference's bit for bit for any seed
    b = mc.CsrMatrix.from_triplets(2, [0, 0, 1], [0, 1, 1], [1.0, -0.5, 1.0])
    for seed in (1, 99, 31337):
        inv = mc.compute_preconditioner(b, mc.McConfig(alpha=1.0, master_seed=seed, delta=1e-6))
        assert inv.row_meta.chains_used[0] == 1
        want = ref_mod.compute_preconditioner(ref_mod.Csr(2, b.row_ptr, b.col_idx, b.values), alpha=1.0,
                                              master_seed=seed, delta=1e-6)
        assert want.chains_used[0] == 1
        assert bits_equal(inv.m.values, want.m.values) and np.array_equal(inv.m.col_idx, want.m.col_idx)


def test_empty_rows_missing_diagonal_and_n0(mc, ref_mod):
    # structurally missing diagonal (split.cpp:10-42, test_mc_split.cpp:96-102)
    b = mc.CsrMatrix.from_triplets(4, [0, 1, 3], [1, 0, 3], [0.5, 0.5, 2.0])
    for rng in (0,):
        inv = mc.compute_preconditioner(b, mc.McConfig(alpha=2.0))
        want = ref_mod.compute_preconditioner(ref_mod.Csr(4, b.row_ptr, b.col_idx, b.values), alpha=2.0)
        assert np.array_equal(inv.m.row_ptr, want.m.row_ptr)
        assert np.array_equal(inv.m.col_idx, want.m.col_idx)
        assert bits_equal(inv.m.values, want.m.values)
    inv = mc.compute_preconditioner(mc.CsrMatrix(0, np.zeros(1, np.int64)), mc.McConfig())
    assert inv.m.n == 0 and inv.m.nnz() == 0


def test_errors_match_reference(mc):
    two = mc.CsrMatrix.from_triplets(2, [0, 1], [0, 1], [-1.0, 1.0])
    with pytest.raises(mc.SplitError, match="degenerate diagonal after augmentation at row 0"):
        mc.compute_preconditioner(two, mc.McConfig(alpha=1.0, mode=mc.AugmentationMode.plain))
    dom = mc.CsrMatrix.from_triplets(2, [0, 0, 1], [0, 1, 1], [-10.0, 10.0, 1.0])
    with pytest.raises(mc.SplitError, match="diagonal dominance failure"):
        mc.compute_preconditioner(dom, mc.McConfig(alpha=1.0, mode=mc.AugmentationMode.plain))
    with pytest.raises(ValueError, match="drop fraction"):
        mc.compute_preconditioner(two, mc.McConfig(drop_fraction=1.5))
    with pytest.raises(ValueError, match="alpha must be positive"):
        mc.compute_preconditioner(two, mc.McConfig(alpha=0.0))
    bad = mc.CsrMatrix(2, np.array([0, 1, 2]), np.array([0, 7]), np.array([1.0, 1.0]))
    with pytest.raises(IndexError):
        mc.compute_preconditioner(bad, mc.McConfig())


def test_determinism_repeat(mc):
    b = _csr(mc, "brusselator:32")
    cfg = mc.McConfig(epsilon=.05, delta=.01, alpha=1.5, retain_k=32, master_seed=20260826)
    a = mc.compute_preconditioner(b, cfg)
    c = mc.compute_preconditioner(b, cfg)
    assert a.m == c.m


def test_row_shards_concatenate_to_full(mc):
    import torch
    from paper_2409_03095_b200.engine import DeviceEngine
    b = _csr(mc, "convdiff:64:20:10")
    eng = DeviceEngine(0)
    rp, ci, v = DeviceEngine.upload(b)
    for rng in (0, 1):
        cfg = mc.McConfig(master_seed=7, rng_mode=rng)
        full = eng.to_tensors(eng.build(b.n, rp, ci, v, cfg))
        parts = []
        for lo, hi in ((0, 1000), (1000, 1001), (1001, 2500), (2500, 4096)):
            parts.append(eng.to_tensors(eng.build(b.n, rp, ci, v, cfg, lo, hi)))
        cols = torch.cat([p[1] for p in parts])
        vals = torch.cat([p[2] for p in parts])
        assert torch.equal(cols, full[1]) and torch.equal(vals.view(torch.int64), full[2].view(torch.int64))
        off = 0
        rps = []
        for p in parts:
            rps.append(p[0][:-1] + off)
            off += int(p[0][-1])
        assert torch.equal(torch.cat(rps + [torch.tensor([off], device=rp.device)]), full[0])
    eng.close()


@pytest.mark.parametrize("rng", [0, 1])
def test_overflow_tier_retry(mc, oracle_mod, rng):
    # a 200-row shard (too small for the tier pilot) of rows touching up to
    # ~1700 columns: rows overflow the first shared-memory tier and are re-run
    # on larger tiers; the retried rows must still be exact
    b = _csr(mc, "broad:1024:24:1e-4:1:7")
    cfg = mc.McConfig(epsilon=.02, delta=.01, alpha=1.5, master_seed=42, rng_mode=rng)
    inv = mc.compute_preconditioner(b, cfg, rows=(0, 200))
    assert inv.stats["rows_retried"] > 0
    want = oracle_mod.compute_preconditioner(b.n, b.row_ptr, b.col_idx, b.values, row_begin=0, row_end=200,
                                             **cfg.oracle_kwargs())
    assert np.array_equal(inv.m.row_ptr, want.row_ptr)
    assert bits_equal(inv.m.values, want.values) and np.array_equal(inv.m.col_idx, want.col_idx)


@pytest.mark.parametrize("rng", [0, 1])
def test_tier_pilot_path_exact(mc, oracle_mod, rng):
    # the full 1024 rows: the pilot builds rows [0, 256) on the last tier and
    # picks the start tier for the rest; the result is tier-independent
    b = _csr(mc, "broad:1024:24:1e-4:1:7")
    cfg = mc.McConfig(epsilon=.02, delta=.01, alpha=1.5, master_seed=42, rng_mode=rng)
    inv = mc.compute_preconditioner(b, cfg)
    want = oracle_mod.compute_preconditioner(b.n, b.row_ptr, b.col_idx, b.values, **cfg.oracle_kwargs())
    assert np.array_equal(inv.m.row_ptr, want.row_ptr)
    assert bits_equal(inv.m.values, want.values) and np.array_equal(inv.m.col_idx, want.col_idx)
    assert np.array_equal(inv.row_meta.entries_before_retention, want.entries_before)


def test_keyed_within_mc_tolerance_of_reference(mc):
    import scipy.sparse as sp
    from paper_2409_03095_b200 import generators as G
    for b, cfg in ((G.convection_diffusion(100, 0.0, 0.0), mc.McConfig()),
                   (G.convection_diffusion(64), mc.McConfig(master_seed=7)),
                   (G.convection_diffusion(40, 0.0, 0.0), mc.McConfig(epsilon=.01, delta=.01))):
        cfg.rng_mode = mc.RngMode.reference
        r = mc.compute_preconditioner(b, cfg)
        cfg.rng_mode = mc.RngMode.keyed
        k = mc.compute_preconditioner(b, cfg)
        n = b.n
        MR = sp.csr_matrix((r.m.values, r.m.col_idx, r.m.row_ptr), shape=(n, n))
        MK = sp.csr_matrix((k.m.values, k.m.col_idx, k.m.row_ptr), shape=(n, n))
        B = sp.csr_matrix((b.values, b.col_idx, b.row_ptr), shape=(n, n))
        shift = cfg.alpha * abs(B).sum(axis=1).max()
        Bh = B + sp.diags(np.where(B.diagonal() < 0, -shift, shift))
        eps = cfg.epsilon
        d = MK - MR
        assert sp.linalg.norm(d) / sp.linalg.norm(MR) <= 0.3 * eps
        assert abs(d).max() <= 0.5 * eps * abs(MR).max()
        I = sp.identity(n)
        fr = lambda M: sp.linalg.norm(I - Bh @ M) / np.sqrt(n)  # noqa: E731
        assert abs(fr(MK) - fr(MR)) <= 0.1 * fr(MR)


@pytest.mark.slow
@pytest.mark.parametrize("cfgname", ["c3_lap3d_100", "c2_sym27_1p3m", "c4_convdiff_1000", "c3_lap3d_100_heavy"])
@pytest.mark.parametrize("rng", [0, 1])
def test_full_size_row_windows_bit_identical(mc, oracle_mod, cfgname, rng):
    from paper_2409_03095_b200 import generators as G
    gen, over = G.CONFIGS[cfgname]
    b = gen()
    cfg = mc.McConfig(rng_mode=rng, **over)
    inv = mc.compute_preconditioner(b, cfg)
    assert inv.m.row_ptr[-1] == inv.m.nnz()
    n = b.n
    windows = [(0, 64), (n // 2, n // 2 + 64), (n - 64, n)]
    for lo, hi in windows:
        want = oracle_mod.compute_preconditioner(n, b.row_ptr, b.col_idx, b.values, row_begin=lo, row_end=hi,
                                                 **cfg.oracle_kwargs())
        a, z = inv.m.row_ptr[lo], inv.m.row_ptr[hi]
        assert np.array_equal(inv.m.row_ptr[lo:hi + 1] - a, want.row_ptr)
        assert np.array_equal(inv.m.col_idx[a:z], want.col_idx)
        assert bits_equal(inv.m.values[a:z], want.values)
        assert np.array_equal(inv.row_meta.chains_used[lo:hi], want.chains_used)
        assert np.array_equal(inv.row_meta.entries_before_retention[lo:hi], want.entries_before)
    # size-independent properties at full size
    assert np.all(np.diff(inv.m.row_ptr) >= 1)  # diagonal always kept
    rows = np.repeat(np.arange(n), np.diff(inv.m.row_ptr))
    assert np.all(inv.m.values[inv.m.col_idx == rows] != 0.0)
    assert inv.stats["rows_retried"] >= 0


@pytest.mark.parametrize("rng", [0, 1])
@pytest.mark.parametrize("k", [0, 32, 500, 4500])
def test_global_tier_and_radix_topk(mc, oracle_mod, ref_mod, rng, k):
    # rows touching 4300-5100 distinct columns: beyond the largest shared-memory
    # tier (3072), so they run on the global-memory accumulator tier; k > 256
    # exercises the radix top-k selection, k = 0 the full column sort
    rb = ref_mod.gen_broad_spectrum(8192, 24, 1e-4, 1.0, 3)
    b = mc.CsrMatrix(rb.n, rb.row_ptr, rb.col_idx, rb.values)
    cfg = mc.McConfig(alpha=1.2, delta=1e-300, chains_override=3000, max_len_override=6, retain_k=k,
                      master_seed=11, rng_mode=rng)
    inv = mc.compute_preconditioner(b, cfg, rows=(100, 164))
    want = oracle_mod.compute_preconditioner(b.n, b.row_ptr, b.col_idx, b.values, row_begin=100, row_end=164,
                                             **cfg.oracle_kwargs())
    assert want.entries_before.max() > 3072
    assert np.array_equal(inv.m.row_ptr, want.row_ptr)
    assert np.array_equal(inv.m.col_idx, want.col_idx)
    assert bits_equal(inv.m.values, want.values)
    assert np.array_equal(inv.row_meta.entries_before_retention, want.entries_before)
    assert inv.stats["rows_retried"] > 0


@pytest.mark.parametrize("rng", [0, 1])
@pytest.mark.parametrize("k", [100, 300])
def test_radix_topk_ties_on_global_tier(mc, oracle_mod, rng, k):
    # 3D Laplacian, 10-step walks: 258-571 distinct columns per row on the
    # global-scratch tiers, whose values repeat (every step-t deposit of an
    # interior path carries the same weight), so retain_top_k cuts through ties
    # (30 of the 64 rows at k = 300) and the radix selection's column passes
    # run on the copied candidates
    from paper_2409_03095_b200 import generators as G
    g = G.laplacian3d(16)
    b = mc.CsrMatrix(g.n, g.row_ptr, g.col_idx, g.values)
    cfg = mc.McConfig(alpha=0.5, delta=1e-300, chains_override=1000, max_len_override=10, retain_k=k,
                      master_seed=3, rng_mode=rng)
    inv = mc.compute_preconditioner(b, cfg, rows=(1800, 1864))
    want = oracle_mod.compute_preconditioner(b.n, b.row_ptr, b.col_idx, b.values, row_begin=1800, row_end=1864,
                                             **cfg.oracle_kwargs())
    assert want.entries_before.max() > 256
    assert np.array_equal(inv.m.row_ptr, want.row_ptr)
    assert np.array_equal(inv.m.col_idx, want.col_idx)
    assert bits_equal(inv.m.values, want.values)
    assert np.array_equal(inv.row_meta.entries_before_retention, want.entries_before)


@pytest.mark.parametrize("rng", [0, 1])
def test_long_rows_pilot_takes_the_wave(mc, oracle_mod, ref_mod, rng):
    # N*L = 72,000 deposits per row (>= 2^15, engine.cu kLongRowDeposits): the
    # pilot sizing for long rows; 64 rows fit one wave, so the pilot launch on
    # the last tier builds them all
    rb = ref_mod.gen_broad_spectrum(8192, 24, 1e-4, 1.0, 3)
    b = mc.CsrMatrix(rb.n, rb.row_ptr, rb.col_idx, rb.values)
    cfg = mc.McConfig(alpha=1.2, delta=1e-300, chains_override=12000, max_len_override=6, retain_k=32,
                      master_seed=17, rng_mode=rng)
    inv = mc.compute_preconditioner(b, cfg, rows=(100, 164))
    want = oracle_mod.compute_preconditioner(b.n, b.row_ptr, b.col_idx, b.values, row_begin=100, row_end=164,
                                             **cfg.oracle_kwargs())
    assert np.array_equal(inv.m.row_ptr, want.row_ptr)
    assert np.array_equal(inv.m.col_idx, want.col_idx)
    assert bits_equal(inv.m.values, want.values)
    assert np.array_equal(inv.row_meta.entries_before_retention, want.entries_before)
    assert np.array_equal(inv.row_meta.chains_used, want.chains_used)


@pytest.mark.parametrize("rng", [0, 1])
def test_radix_topk_midsize_rows(mc, oracle_mod, rng):
    # 300-1700 distinct columns per row with retain_k = 32: the shared-memory
    # tiers with radix selection (rows > 256 entries)
    n, rp, ci, v = golden_input("broad:1024:24:1e-4:1:7")
    b = mc.CsrMatrix(n, rp, ci, v)
    cfg = mc.McConfig(epsilon=.02, delta=.01, alpha=1.5, retain_k=32, master_seed=42, rng_mode=rng)
    inv = mc.compute_preconditioner(b, cfg)
    want = oracle_mod.compute_preconditioner(n, rp, ci, v, **cfg.oracle_kwargs())
    assert want.entries_before.max() > 256
    assert np.array_equal(inv.m.col_idx, want.col_idx) and bits_equal(inv.m.values, want.values)


@pytest.mark.parametrize("rng", [0, 1])
def test_long_walks(mc, oracle_mod, rng):
    # max_len = 147: one chain per batch in the shared-memory log
    b = mc.CsrMatrix(500, *golden_input_tridiag(500))
    cfg = mc.McConfig(alpha=0.3, delta=1e-30, epsilon=0.3, rng_mode=rng)
    inv = mc.compute_preconditioner(b, cfg)
    want = oracle_mod.compute_preconditioner(b.n, b.row_ptr, b.col_idx, b.values, **cfg.oracle_kwargs())
    assert inv.budget_echo.max_len == want.max_len == 147
    assert np.array_equal(inv.m.col_idx, want.col_idx) and bits_equal(inv.m.values, want.values)


def golden_input_tridiag(n):
    from paper_2409_03095_b200 import generators as G
    t = G.tridiagonal(n)
    return t.row_ptr, t.col_idx, t.values


@pytest.mark.parametrize("rng", [0, 1])
@pytest.mark.parametrize("max_len", [1, 3])
def test_short_walk_lengths(mc, oracle_mod, ref_mod, rng, max_len):
    # max_len 1 (one deposit per chain) and 3 (a log stride that does not divide 32)
    b = _csr(mc, "ddm:64:0.2:11")
    cfg = mc.McConfig(epsilon=.05, delta=1e-9, alpha=1.5, max_len_override=max_len, master_seed=5, rng_mode=rng)
    inv = mc.compute_preconditioner(b, cfg)
    want = oracle_mod.compute_preconditioner(b.n, b.row_ptr, b.col_idx, b.values, **cfg.oracle_kwargs())
    assert np.array_equal(inv.m.col_idx, want.col_idx) and bits_equal(inv.m.values, want.values)
    if rng == 0:
        ref = ref_mod.compute_preconditioner(ref_mod.Csr(b.n, b.row_ptr, b.col_idx, b.values),
                                             **{k: v for k, v in cfg.oracle_kwargs().items() if k != "rng_mode"})
        assert bits_equal(inv.m.values, ref.m.values)


def test_invalid_row_ptr_rejected_without_fault(mc):
    # a decreasing row_ptr and one pointing past nnz must be rejected before any
    # column is read (the reference has undefined behaviour here)
    for rp in ([0, 2, 1, 3], [0, 1, 4, 3], [1, 1, 2, 3]):
        bad = mc.CsrMatrix(3, np.array(rp), np.array([0, 1, 2]), np.array([1.0, 1.0, 1.0]))
        with pytest.raises(ValueError, match="row_ptr"):
            mc.compute_preconditioner(bad, mc.McConfig())
    # the device is still healthy afterwards
    ok = mc.compute_preconditioner(mc.CsrMatrix.identity(4), mc.McConfig(alpha=1.0))
    assert ok.m.nnz() == 4


@pytest.mark.parametrize("rng", [0, 1])
def test_streamed_build_into_equals_handle_path(mc, rng):
    # mcmi_build_into (row chunks, D2H overlapped) == mcmi_build_rows, incl. a
    # multi-chunk build and a too-small buffer (falls back to the handle path)
    from paper_2409_03095_b200 import generators as G
    for b, cfg in ((_csr(mc, "brusselator:32"), mc.McConfig(epsilon=.05, delta=.01, alpha=1.5, retain_k=32,
                                                             master_seed=20260826, rng_mode=rng)),
                   (G.laplacian3d(64), mc.McConfig(rng_mode=rng))):
        want = mc.compute_preconditioner(b, cfg)
        for cap in (want.m.nnz() + 7, 10):
            out = {"row_ptr": np.empty(b.n + 1, np.int64), "col_idx": np.empty(cap, np.int64),
                   "values": np.empty(cap)}
            got = mc.compute_preconditioner(b, cfg, out=out)
            assert got.m == want.m
            assert np.array_equal(got.row_meta.chains_used, want.row_meta.chains_used)
            assert np.array_equal(got.row_meta.entries_before_retention, want.row_meta.entries_before_retention)
        lo, hi = b.n // 3, b.n - 5
        part = mc.compute_preconditioner(b, cfg, rows=(lo, hi))
        out = {"row_ptr": np.empty(hi - lo + 1, np.int64), "col_idx": np.empty(part.m.nnz(), np.int64),
               "values": np.empty(part.m.nnz())}
        got = mc.compute_preconditioner(b, cfg, out=out, rows=(lo, hi))
        assert got.m == part.m


@pytest.mark.parametrize("rng", [0, 1])
def test_huge_budget_cast_and_long_max_len(mc, oracle_mod, ref_mod, rng):
    # ||A|| = 1 - 1e-15: the reference's static_cast<index_t> of a 1e33 chain
    # budget is INT64_MIN on x86-64, so it runs N = 1 chain with L ~ 7.8e14;
    # the walks still stop early by delta.  The drop-in must do the same.
    # Frozen fixture (tests/golden/huge_budget_case.json, found by the fuzz generator).
    import json
    import os
    from helpers import GOLDEN
    with open(os.path.join(GOLDEN, "huge_budget_case.json")) as f:
        case = json.load(f)
    b = mc.CsrMatrix(case["n"], np.array(case["row_ptr"], np.int64), np.array(case["col_idx"], np.int64),
                     np.array([float.fromhex(x) for x in case["values_hex"]]))
    kw = dict(case["config"])
    kw.pop("rng_mode")
    cfg = mc.McConfig(**{k: (mc.AugmentationMode(v) if k == "mode" else mc.DropMode(v) if k == "drop_mode" else v)
                         for k, v in kw.items()}, rng_mode=mc.RngMode(rng))
    want = oracle_mod.compute_preconditioner(b.n, b.row_ptr, b.col_idx, b.values, **cfg.oracle_kwargs())
    assert want.n_chains == 1 and want.max_len > 10**14
    got = mc.compute_preconditioner(b, cfg)
    assert got.budget_echo.n_chains == 1 and got.budget_echo.max_len == want.max_len
    assert np.array_equal(got.m.col_idx, want.col_idx) and bits_equal(got.m.values, want.values)
    if rng == 0:
        kw = {k: v for k, v in cfg.oracle_kwargs().items() if k != "rng_mode"}
        r = ref_mod.compute_preconditioner(ref_mod.Csr(b.n, b.row_ptr, b.col_idx, b.values), **kw)
        assert r.n_chains == 1 and bits_equal(got.m.values, r.m.values)


@pytest.mark.parametrize("name", ["poisson2d_100_default_seed0", "rdb2048_acc6", "tridiag_longwalk"])
def test_reference_stream_64bit_positions(mc, name, monkeypatch):
    # budgets with N*L >= 2^32 draws per row use 64-bit draw positions; force
    # that kernel variant on the goldens (the results must not change)
    monkeypatch.setenv("MCMI_FORCE_POS64", "1")
    case = GOLD[name]
    b = _csr(mc, case["input"])
    inv = mc.compute_preconditioner(b, _cfg(mc, case["config"]))
    assert mm_sha256(b.n, inv.m.row_ptr, inv.m.col_idx, inv.m.values) == case["mm_sha256"]


@pytest.mark.parametrize("rng", [0, 1])
@pytest.mark.parametrize("max_len", [2, 3, 4, 8])
def test_walk_length_specialisations_match_generic(mc, oracle_mod, rng, max_len):
    """The compile-time L = 2 / 3 / 4 / 8 walk kernels equal the generic
    kernel (MCMI_WALK_GENERIC) and the oracle."""
    import os
    from paper_2409_03095_b200 import generators as G
    b = G.laplacian3d(24)
    cfg = mc.McConfig(chains_override=300, max_len_override=max_len, delta=1e-6, retain_k=10, master_seed=5,
                      rng_mode=rng)
    spec = mc.compute_preconditioner(b, cfg)
    os.environ["MCMI_WALK_GENERIC"] = "1"
    try:
        gen = mc.compute_preconditioner(b, cfg)
    finally:
        del os.environ["MCMI_WALK_GENERIC"]
    assert spec.m == gen.m and spec.stats["walk_steps"] == gen.stats["walk_steps"]
    want = oracle_mod.compute_preconditioner(b.n, b.row_ptr, b.col_idx, b.values, row_begin=0, row_end=300,
                                             **cfg.oracle_kwargs())
    nnz = int(spec.m.row_ptr[300])
    assert np.array_equal(spec.m.col_idx[:nnz], want.col_idx) and bits_equal(spec.m.values[:nnz], want.values)


@pytest.mark.parametrize("rng", [0, 1])
@pytest.mark.parametrize("over", [{}, {"epsilon": 0.02, "delta": 0.01}, {"retain_k": 20, "master_seed": 3},
                                  {"chains_override": 77, "max_len_override": 2, "delta": 0.2}])
@pytest.mark.parametrize("gen,cap", [("stencil27", 256), ("laplacian3d", 64), ("convdiff", 32)])
def test_neighbourhood_slot_tables_match_plain_kernel(mc, oracle_mod, rng, over, gen, cap):
    """The L = 2 / 256-slot kernel with neighbourhood slot tables (default)
    equals the plain kernel (MCMI_WALK_NB=0) bit for bit, RowMeta included, and
    the oracle on sampled rows.  stencil27 interiors use the tables (deg 26,
    125 two-hop columns); the boundary rows and delta=0.2 (chains that stop
    after one step) cover mixed and unvisited neighbourhood columns."""
    import os
    from paper_2409_03095_b200 import generators as G
    b = {"stencil27": lambda: G.stencil27(14, 13, 12, seed=4), "laplacian3d": lambda: G.laplacian3d(13),
         "convdiff": lambda: G.convection_diffusion(40)}[gen]()
    cfg = mc.McConfig(rng_mode=rng, **over)
    os.environ["MCMI_WALK_NB"] = "1"  # tables on regardless of the host's cost hint
    try:
        nbk = mc.compute_preconditioner(b, cfg)
    finally:
        del os.environ["MCMI_WALK_NB"]
    assert nbk.stats["hash_cap"] == cap and nbk.budget_echo.max_len == 2
    os.environ["MCMI_WALK_NB"] = "0"
    try:
        plain = mc.compute_preconditioner(b, cfg)
    finally:
        del os.environ["MCMI_WALK_NB"]
    assert nbk.m == plain.m and nbk.stats["walk_steps"] == plain.stats["walk_steps"]
    assert np.array_equal(nbk.row_meta.entries_before_retention, plain.row_meta.entries_before_retention)
    assert np.array_equal(nbk.row_meta.chains_used, plain.row_meta.chains_used)
    n = b.n
    for lo, hi in [(0, 40), (n // 2, n // 2 + 40)]:
        want = oracle_mod.compute_preconditioner(n, b.row_ptr, b.col_idx, b.values, row_begin=lo, row_end=hi,
                                                 **cfg.oracle_kwargs())
        a, z = nbk.m.row_ptr[lo], nbk.m.row_ptr[hi]
        assert np.array_equal(nbk.m.col_idx[a:z], want.col_idx) and bits_equal(nbk.m.values[a:z], want.values)
        assert np.array_equal(nbk.row_meta.entries_before_retention[lo:hi], want.entries_before)


@pytest.mark.parametrize("rng", [0, 1])
def test_neighbourhood_tables_zero_sum_columns(mc, oracle_mod, rng):
    """27-point stencil with off-diagonals of magnitude 1 and random signs:
    every interior transition has the same |ratio|, so 2-step deposits are
    +-R^2 and a column's sum often cancels to exactly 0.0.  Such a column was
    visited: it counts in entries_before (then is pruned from M), which the
    tables' visited marks must get right."""
    import os
    from paper_2409_03095_b200 import generators as G
    g = G.stencil27(12, 12, 12, seed=4)
    r = np.random.default_rng(7)
    v = np.where(r.random(g.values.size) < 0.5, -1.0, 1.0)
    rows = np.repeat(np.arange(g.n), np.diff(g.row_ptr))
    v[g.col_idx == rows] = 30.0
    b = mc.CsrMatrix(g.n, g.row_ptr, g.col_idx, v)
    cfg = mc.McConfig(rng_mode=rng, chains_override=3000, max_len_override=2, alpha=0.5)
    os.environ["MCMI_WALK_NB"] = "1"
    try:
        nbk = mc.compute_preconditioner(b, cfg)
    finally:
        del os.environ["MCMI_WALK_NB"]
    lo, hi = 600, 680
    want = oracle_mod.compute_preconditioner(b.n, b.row_ptr, b.col_idx, b.values, row_begin=lo, row_end=hi,
                                             **cfg.oracle_kwargs())
    assert (want.entries_before > np.diff(want.row_ptr)).any()  # zero sums pruned after counting
    a, z = nbk.m.row_ptr[lo], nbk.m.row_ptr[hi]
    assert np.array_equal(nbk.m.col_idx[a:z], want.col_idx) and bits_equal(nbk.m.values[a:z], want.values)
    assert np.array_equal(nbk.row_meta.entries_before_retention[lo:hi], want.entries_before)


def _mixed_triangle_matrix(mc, n=400, seed=3):
    """Rows with and without triangles through them: a ring (triangle-free)
    plus random chords, some closing triangles; degrees 2..8."""
    rng = np.random.default_rng(seed)
    rows, cols, vals = [], [], []
    for i in range(n):
        nb = {(i + 1) % n, (i - 1) % n}
        if rng.random() < 0.5:
            nb |= set(int(x) for x in rng.integers(0, n, size=int(rng.integers(1, 6))))
        if rng.random() < 0.3:
            nb.add((i + 2) % n)  # with i+1 -> i+2 a triangle through i
        nb.discard(i)
        for c in nb:
            rows.append(i)
            cols.append(c)
            vals.append(-rng.uniform(0.2, 1.0))
        rows.append(i)
        cols.append(i)
        vals.append(10.0)
    return mc.CsrMatrix.from_triplets(n, rows, cols, vals)


@pytest.mark.parametrize("rng", [0, 1])
@pytest.mark.parametrize("over", [{}, {"chains_override": 77, "max_len_override": 2, "delta": 0.2},
                                  {"retain_k": 4, "master_seed": 9}, {"epsilon": 0.02, "delta": 0.01}])
@pytest.mark.parametrize("gen", ["laplacian3d", "convdiff", "mixed"])
def test_split_fold_matches_plain_kernel(mc, oracle_mod, rng, over, gen, monkeypatch):
    """The L = 2 split fold (rows without a triangle through r: step-0 columns
    summed from per-transition counts) equals the plain ordered fold
    (MCMI_WALK_NO_SPLIT=1) bit for bit, RowMeta included, and the oracle."""
    from paper_2409_03095_b200 import generators as G
    b = {"laplacian3d": lambda: G.laplacian3d(12), "convdiff": lambda: G.convection_diffusion(30),
         "mixed": lambda: _mixed_triangle_matrix(mc)}[gen]()
    cfg = mc.McConfig(rng_mode=rng, **over)
    split = mc.compute_preconditioner(b, cfg)
    assert split.budget_echo.max_len == 2
    monkeypatch.setenv("MCMI_WALK_NO_SPLIT", "1")
    plain = mc.compute_preconditioner(b, cfg)
    monkeypatch.delenv("MCMI_WALK_NO_SPLIT")
    assert split.m == plain.m and split.stats["walk_steps"] == plain.stats["walk_steps"]
    assert np.array_equal(split.row_meta.entries_before_retention, plain.row_meta.entries_before_retention)
    assert np.array_equal(split.row_meta.chains_used, plain.row_meta.chains_used)
    want = oracle_mod.compute_preconditioner(b.n, b.row_ptr, b.col_idx, b.values, **cfg.oracle_kwargs())
    assert np.array_equal(split.m.row_ptr, want.row_ptr) and np.array_equal(split.m.col_idx, want.col_idx)
    assert bits_equal(split.m.values, want.values)


@pytest.mark.parametrize("cap_mode", ["estimate", "short", "none"])
def test_job_api_progressive_delivery(mc, cap_mode):
    """mcmi_build_start / mcmi_job_estimate / mcmi_job_attach / mcmi_job_finish /
    mcmi_result_copy_range (the C++ drop-in's path): chunks delivered into the
    caller's arrays during the build plus the copied tail equal the handle
    path, for an attach at the estimate, a too-short attach and none."""
    import ctypes as C
    from paper_2409_03095_b200 import _lib as L
    from paper_2409_03095_b200 import generators as G
    lib = L.load()
    b = G.laplacian3d(64)  # 262,144 rows: 4 streamed chunks, first at 10%
    cfg = mc.McConfig(master_seed=5)
    want = mc.compute_preconditioner(b, cfg)
    view = L.mcmi_csr_view(b.n, b.row_ptr.ctypes.data, b.col_idx.ctypes.data, b.values.ctypes.data)
    c = cfg.to_c()
    job = C.c_void_p()
    err = C.create_string_buffer(512)
    assert lib.mcmi_build_start(C.byref(view), C.byref(c), 0, -1, C.byref(job), err, 512) == 0
    est = C.c_int64()
    assert lib.mcmi_job_estimate(job, C.byref(est)) == 0
    nnz = want.m.nnz()
    assert est.value >= nnz * 0.9  # upper-biased extrapolation of the first chunk
    cap = {"estimate": est.value, "short": nnz // 3, "none": 0}[cap_mode]
    col = np.full(max(cap, nnz), -7, np.int64)
    val = np.full(max(cap, nnz), np.nan)
    if cap:
        assert lib.mcmi_job_attach(job, col.ctypes.data, val.ctypes.data, cap) == 0
    res = C.c_void_p()
    delivered = C.c_int64()
    assert lib.mcmi_job_finish(job, C.byref(res), C.byref(delivered), err, 512) == 0
    try:
        got_n, got_nnz = C.c_int64(), C.c_int64()
        lib.mcmi_result_sizes(res, C.byref(got_n), C.byref(got_nnz))
        assert got_nnz.value == nnz and 0 <= delivered.value <= min(cap, nnz)
        if cap_mode == "none":
            assert delivered.value == 0
        assert lib.mcmi_result_copy_range(res, delivered.value, nnz, col.ctypes.data, val.ctypes.data) == 0
        assert np.array_equal(col[:nnz], want.m.col_idx) and bits_equal(val[:nnz], want.m.values)
        assert lib.mcmi_result_copy_range(res, 5, 3, None, None) == L.MCMI_EINVAL
    finally:
        lib.mcmi_result_free(res)
