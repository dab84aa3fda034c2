"""Device-resident build timings over the BASELINE.json configs (both RNG
keyings): python tools/sweep.py [config ...]  -> one JSON line per run."""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    import torch
    from paper_2409_03095_b200 import generators as G
    from paper_2409_03095_b200.engine import DeviceEngine
    from paper_2409_03095_b200.mcspai import McConfig, RngMode
    # (the C5 wide corner is built on leading rows only, by bench.py and c5_sweep.py)
    names = sys.argv[1:] or [c for c in G.CONFIGS if not c.endswith("_1e4x32")]
    eng = DeviceEngine(0)
    for name in names:
        gen, over = G.CONFIGS[name]
        t0 = time.time()
        b = gen()
        tg = time.time() - t0
        rp, ci, v = DeviceEngine.upload(b)
        for rng in (RngMode.reference, RngMode.keyed):
            cfg = McConfig(**over, rng_mode=rng)
            eng.build(b.n, rp, ci, v, cfg)  # warm-up
            runs = [eng.build(b.n, rp, ci, v, cfg).stats for _ in range(3)]
            best = min(runs, key=lambda s: s["ms_total"])
            print(json.dumps({"config": name, "rng": rng.name, "n": b.n, "nnz_B": b.nnz(), "gen_s": round(tg, 1),
                              "ms_total": round(best["ms_total"], 3), "ms_tables": round(best["ms_tables"], 3),
                              "ms_walk_kernel": round(best["ms_walk_kernel"], 3),
                              "ms_assemble": round(best["ms_assemble"], 3), "steps": best["walk_steps"],
                              "steps_per_s": best["walk_steps"] / (best["ms_total"] / 1e3),
                              "walk_steps_per_s": best["walk_steps"] / (best["ms_walk_kernel"] / 1e3),
                              "nnz_M": best["nnz"], "N": best["n_chains"], "L": best["max_len"],
                              "cap": best["hash_cap"], "retried": best["rows_retried"]}), flush=True)
        del rp, ci, v
        torch.cuda.empty_cache()
    eng.close()


if __name__ == "__main__":
    main()
