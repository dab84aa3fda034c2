"""Full-size reference hashes for the BASELINE.json configs (tests/golden/fullsize.json).

Run in the build container (needs oracle/_ref, the UNMODIFIED reference
library compiled in place from /root/reference by oracle/Makefile, and the
oracle restatement):

    make -C oracle ref oracle && python tests/golden/make_fullsize.py [case ...]

For each config the inputs come from paper_2409_03095_b200/generators.py,
imported by file path (pure numpy; the product library is never loaded), and
their sha256 is recorded so a drifted generator fails loudly instead of
comparing different matrices.  Then:

* ``reference``: the reference's own ``compute_preconditioner`` (all host
  threads; ``mc_engine.cpp:230-233``) builds the WHOLE matrix; we record the
  sha256 of M (``m_sha256`` below), of RowMeta, nnz and the budget.  The
  oracle restatement (rng_mode 0) rebuilds it over row ranges in parallel
  processes: its hash must be the same (the oracle pinned at full size) and
  it supplies the exact walk-step count.
* ``keyed``: the oracle restatement with the (row, chain, step) keying
  (SURVEY §8a Mode K), same hashes.

m_sha256 = sha256(row_ptr int64 || col_idx int64 || values f64 bits), little
endian, the reference's CSR layout (csr.hpp:16-21).
"""
from __future__ import annotations

import hashlib
import importlib.util
import json
import multiprocessing as mp
import os
import sys
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
REPO = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, REPO)

from oracle import oracle, ref  # noqa: E402

OUT = os.path.join(HERE, "fullsize.json")
CASES = ["c1_poisson2d_100", "c3_lap3d_100", "c4_convdiff_1000", "c2_sym27_default", "c2_sym27_1p3m",
         "c3_lap3d_100_heavy", "c5_powerlaw_4m"]


def generators():
    spec = importlib.util.spec_from_file_location(
        "mcmi_generators_standalone", os.path.join(REPO, "paper_2409_03095_b200", "generators.py"))
    mod = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(mod)
    return mod


def csr_sha256(row_ptr, col_idx, values) -> str:
    h = hashlib.sha256()
    for a in (row_ptr, col_idx, values):
        h.update(memoryview(np.ascontiguousarray(a)).cast("B"))
    return h.hexdigest()


def arr_sha256(a) -> str:
    return hashlib.sha256(memoryview(np.ascontiguousarray(a)).cast("B")).hexdigest()


_B = None  # inherited by the forked workers


def _oracle_range(job):
    lo, hi, cfg = job
    n, rp, ci, v = _B
    r = oracle.compute_preconditioner(n, rp, ci, v, row_begin=lo, row_end=hi, **cfg)
    return lo, hi, r


def oracle_hashes(b, cfg, workers):
    """The oracle restatement over row ranges in parallel, concatenated in row order."""
    global _B
    _B = (b.n, b.row_ptr, b.col_idx, b.values)
    parts = max(workers * 8, 1)
    edges = np.linspace(0, b.n, parts + 1).astype(np.int64)
    jobs = [(int(edges[i]), int(edges[i + 1]), cfg) for i in range(parts) if edges[i + 1] > edges[i]]
    rp = np.zeros(b.n + 1, np.int64)
    cols, vals, cus, ebs = [], [], [], []
    off, steps, budget = 0, 0, None
    with mp.get_context("fork").Pool(workers) as pool:
        for lo, hi, r in pool.imap(_oracle_range, jobs):
            rp[lo + 1:hi + 1] = r.row_ptr[1:] + off
            cols.append(r.col_idx)
            vals.append(r.values)
            cus.append(r.chains_used)
            ebs.append(r.entries_before)
            off += int(r.row_ptr[-1])
            steps += r.walk_steps
            budget = (r.n_chains, r.max_len)
    _B = None
    cat = lambda xs, dt: np.concatenate(xs) if xs else np.zeros(0, dt)  # noqa: E731
    ci, v = cat(cols, np.int64), cat(vals, np.float64)
    return {"n_chains": budget[0] if budget else None, "max_len": budget[1] if budget else None, "nnz": off,
            "m_sha256": csr_sha256(rp, ci, v), "chains_used_sha256": arr_sha256(cat(cus, np.int64)),
            "entries_before_sha256": arr_sha256(cat(ebs, np.int64)), "walk_steps": steps}


def run_case(name, G, workers):
    gen, over = G.CONFIGS[name]
    t0 = time.time()
    b = gen()
    entry = {"n": b.n, "nnz_B": b.nnz(), "config": over,
             "b_sha256": csr_sha256(b.row_ptr, b.col_idx, b.values)}
    print(f"[{name}] generated n={b.n} nnz={b.nnz()} in {time.time() - t0:.1f}s", flush=True)

    t0 = time.time()
    r = ref.compute_preconditioner(ref.Csr(b.n, b.row_ptr, b.col_idx, b.values), n_threads=0, **over)
    t_ref = time.time() - t0
    m = r.m
    entry["reference"] = {
        "n_chains": r.n_chains, "max_len": r.max_len, "nnz": int(m.row_ptr[-1]),
        "m_sha256": csr_sha256(m.row_ptr, m.col_idx, m.values),
        "chains_used_sha256": arr_sha256(r.chains_used), "entries_before_sha256": arr_sha256(r.entries_before),
        "ref_build_s": round(t_ref, 2), "ref_threads": ref.max_threads(),
    }
    print(f"[{name}] reference build {t_ref:.1f}s nnz={entry['reference']['nnz']}", flush=True)
    del r, m

    for mode, key in ((0, "reference"), (1, "keyed")):
        t0 = time.time()
        got = oracle_hashes(b, dict(over, rng_mode=mode), workers)
        print(f"[{name}] oracle rng_mode={mode} {time.time() - t0:.1f}s steps={got['walk_steps']}", flush=True)
        if key == "reference":
            for k in ("n_chains", "max_len", "nnz", "m_sha256", "chains_used_sha256", "entries_before_sha256"):
                if got[k] != entry["reference"][k]:
                    raise SystemExit(f"[{name}] oracle restatement differs from the reference on {k}")
            entry["reference"]["walk_steps"] = got["walk_steps"]
        else:
            entry["keyed"] = got
    return entry


def main():
    G = generators()
    names = sys.argv[1:] or CASES
    workers = os.cpu_count() or 1
    data = {}
    if os.path.exists(OUT):
        with open(OUT) as f:
            data = json.load(f)
    for name in names:
        data[name] = run_case(name, G, workers)
        with open(OUT, "w") as f:
            json.dump(data, f, indent=1, sort_keys=True)


if __name__ == "__main__":
    main()
