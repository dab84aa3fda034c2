"""Runs one workload twice through the device engine (warm-up + profiled
build) so `ncu -k regex:k_walk -s 1 -c 1` captures a warm walk launch.

    python tools/profile_walk.py --config c2_sym27_1p3m [--rng keyed] [--rows N]
"""
import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    p = argparse.ArgumentParser()
    p.add_argument("--config", default="c2_sym27_1p3m")
    p.add_argument("--rng", default="reference", choices=["reference", "keyed"])
    p.add_argument("--rows", type=int, default=-1, help="build only the first ROWS rows")
    p.add_argument("--repeat", type=int, default=2)
    p.add_argument("--chains", type=int, default=None, help="chains_override (C5 grid points)")
    p.add_argument("--len", type=int, default=None, help="max_len_override (C5 grid points)")
    a = p.parse_args()
    import torch
    from paper_2409_03095_b200 import generators as G
    from paper_2409_03095_b200.engine import DeviceEngine
    from paper_2409_03095_b200.mcspai import McConfig, RngMode
    gen, over = G.CONFIGS[a.config]
    b = gen()
    over = dict(over)
    if a.chains is not None:
        over["chains_override"] = a.chains
    if a.len is not None:
        over["max_len_override"] = a.len
    cfg = McConfig(**over, rng_mode=RngMode.reference if a.rng == "reference" else RngMode.keyed)
    eng = DeviceEngine(0)
    rp, ci, v = DeviceEngine.upload(b)
    for _ in range(a.repeat):
        d = eng.build(b.n, rp, ci, v, cfg, 0, a.rows)
    torch.cuda.synchronize()
    print(json.dumps(d.stats))
    eng.close()


if __name__ == "__main__":
    main()
