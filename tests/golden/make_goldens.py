"""Regenerates tests/golden/goldens.json and tests/golden/inputs.npz.

Run in the build container (needs oracle/_ref, i.e. the UNMODIFIED reference
library compiled from /root/reference by oracle/Makefile):

    make -C oracle ref && python tests/golden/make_goldens.py

For every case the reference's own compute_preconditioner_serial
(mc_engine.cpp:235-238) builds M; we record the sha256 of
write_matrix_market's output (matrix_market.cpp:155-169), nnz, the chain
budget and hashes of RowMeta.  Inputs that our numpy generators do not mirror
are frozen into inputs.npz so the GPU box needs neither /root/reference nor
oracle/_ref to check them.
"""
from __future__ import annotations

import hashlib
import json
import os
import sys
import tempfile

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))

from oracle import ref  # noqa: E402

# name -> (input spec, McConfig fields)
CASES = {
    # BASELINE.md §4 goldens
    "poisson2d_100_default_seed0": ("convdiff:100:0:0", {}),
    "rdb2048_acc6": ("brusselator:32", dict(epsilon=.05, delta=.01, alpha=1.5, retain_k=32, master_seed=20260826)),
    "convdiff_64_default_seed7": ("convdiff:64:20:10", dict(master_seed=7)),
    "broad1024_bench": ("broad:1024:24:1e-4:1:7", dict(epsilon=.02, delta=.01, alpha=1.5, retain_k=32, master_seed=42)),
    # bench_precond.cpp:47-58 corpus
    "bench_brusselator": ("brusselator:32", dict(epsilon=.02, delta=.01, alpha=1.5, retain_k=32, master_seed=42)),
    "bench_convdiff48": ("convdiff:48:20:10", dict(epsilon=.02, delta=.01, alpha=1.5, retain_k=32, master_seed=42)),
    "bench_tridiag4096": ("tridiag:4096", dict(epsilon=.02, delta=.01, alpha=1.5, retain_k=32, master_seed=42)),
    # option coverage
    "ddm64_plain_k6": ("ddm:64:0.2:11", dict(epsilon=.05, delta=.01, alpha=1.5, mode=0, retain_k=6, master_seed=3)),
    "ddm48_tests_k8": ("ddm:48:0.15:9", dict(epsilon=.1, delta=.05, alpha=1.5, retain_k=8, master_seed=777)),
    "ddm80_drop_value": ("ddm:80:0.3:5", dict(epsilon=.05, delta=.02, alpha=2.0, drop_fraction=.3, master_seed=1)),
    "ddm80_drop_quantile": ("ddm:80:0.3:5", dict(epsilon=.05, delta=.02, alpha=2.0, drop_fraction=.4, drop_mode=1, master_seed=1)),
    "broad200_quantile_k10": ("broad:200:12:1e-3:10:99", dict(epsilon=.03, delta=.005, alpha=1.2, drop_fraction=.25, drop_mode=1, retain_k=10, master_seed=5)),
    "ddm40_overrides": ("ddm:40:0.5:4", dict(delta=1e-12, alpha=2.0, chains_override=300, max_len_override=9, master_seed=12)),
    "ddm30_len0": ("ddm:30:0.4:8", dict(alpha=2.0, max_len_override=0, master_seed=2)),
    "tridiag_longwalk": ("tridiag:300", dict(epsilon=.2, delta=1e-9, alpha=1.0, master_seed=9)),
}


def make_input(spec: str) -> ref.Csr:
    kind, *a = spec.split(":")
    if kind == "convdiff":
        return ref.gen_convection_diffusion(int(a[0]), float(a[1]), float(a[2]))
    if kind == "brusselator":
        return ref.gen_brusselator(int(a[0]))
    if kind == "tridiag":
        return ref.gen_tridiagonal(int(a[0]))
    if kind == "ddm":
        return ref.gen_random_ddm(int(a[0]), float(a[1]), int(a[2]))
    if kind == "broad":
        return ref.gen_broad_spectrum(int(a[0]), int(a[1]), float(a[2]), float(a[3]), int(a[4]))
    raise ValueError(spec)


def sha(a) -> str:
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def main():
    out, arrays = {}, {}
    for name, (spec, cfg) in CASES.items():
        b = make_input(spec)
        arrays[f"{spec}/row_ptr"] = b.row_ptr
        arrays[f"{spec}/col_idx"] = b.col_idx
        arrays[f"{spec}/values"] = b.values
        with tempfile.NamedTemporaryFile(suffix=".mtx") as f:
            r = ref.compute_preconditioner(b, serial=True, mm_path=f.name, **cfg)
            mm = open(f.name, "rb").read()
        out[name] = dict(input=spec, config=cfg, mm_sha256=hashlib.sha256(mm).hexdigest(), nnz=r.m.nnz,
                         n=b.n, n_chains=r.n_chains, max_len=r.max_len,
                         chains_used_sha256=sha(r.chains_used), entries_before_sha256=sha(r.entries_before))
        print(f"{name:28s} n={b.n:6d} nnz(M)={r.m.nnz:7d} N={r.n_chains} L={r.max_len}")
    with open(os.path.join(HERE, "goldens.json"), "w") as f:
        json.dump(out, f, indent=1, sort_keys=True)
    np.savez_compressed(os.path.join(HERE, "inputs.npz"), **arrays)


if __name__ == "__main__":
    main()
