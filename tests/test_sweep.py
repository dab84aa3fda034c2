"""Sweep driver (§8f rank 3): the reference CLI's `bench` semantics
(tools/mcspai.cpp:315-515) — spec parsing, CSV format, resumption, grid order,
consolidated sorted output, failure rows.  CPU tests use an injected cell; the
GPU test runs real cells (device build + device solve)."""
import io

import numpy as np
import pytest

from paper_2409_03095_b200 import sweep as S

SPEC = """# comment
matrix = {path}
epsilons = 0.25, 0.125
drop_fractions = 0.0,0.5
retain_ks = 0 , 8
delta = 0.0625
alpha=5
reps = 2
seed = 41
solver = bicgstab
tol = 1e-8
max_iters = 500
"""


def test_spec_parse():
    s = S.parse_bench_spec_text(SPEC.format(path="/x/poisson.mtx"))
    assert s.matrix == "/x/poisson.mtx" and s.epsilons == [0.25, 0.125] and s.drop_fractions == [0.0, 0.5]
    assert s.retain_ks == [0, 8] and s.reps == 2 and s.seed == 41 and s.solver == "bicgstab"
    assert s.tol == 1e-8 and s.max_iters == 500 and s.restart == 50 and s.mode == "sign"


@pytest.mark.parametrize("text,msg", [
    ("matrix=a\nbogus\n", "spec line 2: expected key=value"),
    ("matrix=a\nfoo = 1\n", "spec line 2: unknown key 'foo'"),
    ("epsilons=1\ndrop_fractions=0\nretain_ks=0\n", "spec: 'matrix' is required"),
    ("matrix=a\nepsilons=\ndrop_fractions=0\nretain_ks=0\n", "must be non-empty"),
    ("matrix=a\nepsilons=1\ndrop_fractions=0\nretain_ks=0\nreps=0\n", "reps must be >= 1"),
])
def test_spec_errors(text, msg):
    with pytest.raises(S.SpecError, match=msg):
        S.parse_bench_spec_text(text)


def test_row_format_is_ostream_precision17():
    # expected strings from std::ostringstream with precision(17) (g++ 13)
    r = S.CsvRow("m", 10, 49, "P", 0.05, 0.0625, 5.0, 0.3, 8, 18446744073709551615, 123.456789, "gmres", 17,
                 True, 1e-6, 1.0 / 3, 1e22)
    assert r.line() == ("m,10,49,P,0.050000000000000003,0.0625,5,0.29999999999999999,8,18446744073709551615,"
                        "123.456789,gmres,17,1,9.9999999999999995e-07,0.33333333333333331,1e+22")
    assert r.key() == "m|0.050000000000000003|0.0625|5|0.29999999999999999|8|18446744073709551615|gmres|P"
    assert S.CsvRow.parse(S.split_csv_line(r.line())).line() == r.line()


def write_spec(tmp_path, mtx):
    p = tmp_path / "spec.txt"
    p.write_text(SPEC.format(path=mtx))
    return p


def make_matrix(tmp_path):
    from paper_2409_03095_b200 import generators as G
    from paper_2409_03095_b200 import matrix_market as mm
    b = G.convection_diffusion(12, 0.0, 0.0)
    path = tmp_path / "poisson12.mtx"
    mm.write_matrix_market_file(b, path)
    return path


def test_run_bench_resume_and_order(tmp_path):
    mtx = make_matrix(tmp_path)
    spec = write_spec(tmp_path, mtx)
    out = tmp_path / "out.csv"
    calls = []

    def cell(b, cfg, scfg):
        calls.append((cfg.drop_fraction, cfg.epsilon, cfg.retain_k, cfg.master_seed))
        if cfg.epsilon == 0.125 and cfg.retain_k == 8 and cfg.master_seed == 42 and cfg.drop_fraction == 0.5:
            raise RuntimeError("boom")
        return (1.5, 7, True, 1e-9, 2.5, 4.0)

    log = io.StringIO()
    assert S.run_bench(spec, out, cell, log) == 1  # one failed cell
    # grid order: drop, eps, k, rep (seed = 41 + rep)
    assert calls[:3] == [(0.0, 0.25, 0, 41), (0.0, 0.25, 0, 42), (0.0, 0.25, 8, 41)]
    assert len(calls) == 16 and log.getvalue().count("bench: ") == 16
    lines = out.read_text().splitlines()
    assert lines[0] == S.CSV_HEADER and len(lines) == 17
    rows = [S.CsvRow.parse(S.split_csv_line(x)) for x in lines[1:]]
    keys = [(r.matrix, r.drop_fraction, r.epsilon, r.retain_k, r.seed, r.solver) for r in rows]
    assert keys == sorted(keys)
    assert sum(r.method == "P-error" for r in rows) == 1
    assert all(r.matrix == "poisson12" and r.n == 144 for r in rows)
    # resumption: every key present (the failed one too) -> no cell runs
    calls.clear()
    assert S.run_bench(spec, out, cell, io.StringIO()) == 0
    assert calls == []
    assert out.read_text().splitlines() == lines


@pytest.mark.gpu
def test_gpu_sweep_end_to_end(tmp_path):
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2409_03095_b200 import matrix_market as mm
    from paper_2409_03095_b200 import solvers
    from paper_2409_03095_b200.mcspai import McConfig, compute_preconditioner
    mtx = make_matrix(tmp_path)
    spec = tmp_path / "s.txt"
    spec.write_text(f"matrix={mtx}\nepsilons=0.1\ndrop_fractions=0\nretain_ks=0,4\nreps=2\nseed=3\n"
                    "solver=bicgstab\n")
    out = tmp_path / "o.csv"
    assert S.main(["--spec", str(spec), "--out", str(out)]) == 0
    rows = [S.CsvRow.parse(S.split_csv_line(x)) for x in out.read_text().splitlines()[1:]]
    assert len(rows) == 4 and all(r.converged and r.method == "P" for r in rows)
    # each cell's iterations equal a direct device build + solve with the same config
    b = mm.read_matrix_market_file(mtx)
    for r in rows:
        m = compute_preconditioner(b, McConfig(epsilon=0.1, retain_k=r.retain_k, master_seed=r.seed)).m
        _, rep = solvers.solve(b, m, solvers.SolverConfig(method=solvers.SolverMethod.bicgstab))
        assert rep.iterations == r.iterations
        assert np.isclose(rep.final_rel_residual, r.final_rel_residual, rtol=0, atol=0)
