"""BASELINE.json config C5: eps/delta sweep on the power-law matrix (n = 4e6).

Grid: chains_override in {1e2, 1e3, 1e4, 1e5} x max_len_override in
{4, 8, 16, 32, 64}, delta = 1e-300 (only L truncates), alpha = 0.1,
retain_k = 32.  The full corner (1e5 x 64 x 4e6 rows =
2.6e13 steps) is infeasible, so each point builds the leading row shard whose
step count stays under --budget (mcmi_build_rows semantics: the transition
tables always cover all 4e6 states).  For every point the first --check rows
are compared bit-for-bit with the oracle.

    python tools/c5_sweep.py [--budget 4e9] [--check 4] [--rng reference]
"""
import argparse
import json
import os
import sys
import time

import numpy as np

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, REPO)


def main():
    p = argparse.ArgumentParser()
    p.add_argument("--n", type=int, default=4_000_000)
    p.add_argument("--budget", type=float, default=4e9)
    p.add_argument("--check", type=int, default=4)
    p.add_argument("--rng", default="reference", choices=["reference", "keyed"])
    p.add_argument("--chains", default="100,1000,10000,100000")
    p.add_argument("--lens", default="4,8,16,32,64")
    p.add_argument("--hash", action="store_true", help="print the sha256 (16 hex) of the timed build's M")
    a = p.parse_args()
    from paper_2409_03095_b200 import generators as G
    from paper_2409_03095_b200.engine import DeviceEngine
    from paper_2409_03095_b200.mcspai import McConfig, RngMode
    t0 = time.time()
    b = G.powerlaw(a.n)
    gen_s = time.time() - t0
    eng = DeviceEngine(0)
    rp, ci, v = DeviceEngine.upload(b)
    rng = RngMode.reference if a.rng == "reference" else RngMode.keyed
    for nc in [int(x) for x in a.chains.split(",")]:
        for ml in [int(x) for x in a.lens.split(",")]:
            rows = int(min(b.n, max(1, a.budget // (nc * ml))))
            cfg = McConfig(alpha=0.1, delta=1e-300, chains_override=nc, max_len_override=ml, retain_k=32,
                           rng_mode=rng)
            eng.build(b.n, rp, ci, v, cfg, 0, min(rows, 64))  # warm-up (tier scratch allocation)
            d = eng.build(b.n, rp, ci, v, cfg, 0, rows)
            st = d.stats
            msha = None
            if a.hash:
                import hashlib
                h = hashlib.sha256()
                for t in eng.to_tensors(d)[:3]:
                    h.update(t.cpu().numpy().tobytes())
                msha = h.hexdigest()[:16]
            ok = None
            if a.check:
                from oracle import oracle
                k = min(a.check, rows)
                want = oracle.compute_preconditioner(b.n, b.row_ptr, b.col_idx, b.values, row_begin=0, row_end=k,
                                                     **cfg.oracle_kwargs())
                grp, gci, gv, _, geb = eng.to_tensors(eng.build(b.n, rp, ci, v, cfg, 0, k))
                ok = bool(np.array_equal(gci.cpu().numpy(), want.col_idx)
                          and np.array_equal(gv.cpu().numpy().view(np.uint64), want.values.view(np.uint64))
                          and np.array_equal(geb.cpu().numpy(), want.entries_before))
            print(json.dumps({"chains": nc, "max_len": ml, "rows": rows, "steps": st["walk_steps"],
                              "ms_total": round(st["ms_total"], 3), "ms_walk_kernel": round(st["ms_walk_kernel"], 3),
                              "steps_per_s": st["walk_steps"] / (st["ms_total"] / 1e3),
                              "hash_cap": st["hash_cap"], "rows_retried": st["rows_retried"], "nnz_M": st["nnz"],
                              "exact_vs_oracle": ok, "m_sha16": msha, "rng": a.rng, "gen_s": round(gen_s, 1)}), flush=True)
    eng.close()


if __name__ == "__main__":
    main()
