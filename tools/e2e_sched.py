"""Streamed host-API build (mcmi_build_into) under different chunk schedules:
wall and device ms per build.  python tools/e2e_sched.py [config]"""
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    import torch
    from paper_2409_03095_b200 import generators as G
    from paper_2409_03095_b200.mcspai import CsrMatrix, McConfig, compute_preconditioner
    name = sys.argv[1] if len(sys.argv) > 1 else "c2_sym27_1p3m"
    gen, over = G.CONFIGS[name]
    b = gen()
    cfg = McConfig(**over)
    pin = lambda a: torch.from_numpy(a).pin_memory().numpy()  # noqa: E731
    hb = CsrMatrix(b.n, pin(b.row_ptr), pin(b.col_idx), pin(b.values))
    r = compute_preconditioner(hb, cfg)
    nnz = r.m.nnz()
    out = {"row_ptr": pin(np.empty(b.n + 1, np.int64)), "col_idx": pin(np.empty(nnz, np.int64)),
           "values": pin(np.empty(nnz))}
    for chunks, ratio in [(11, 1.0), (16, 1.0), (6, 0.7), (8, 0.65), (8, 0.75), (10, 0.75), (12, 0.8), (8, 0.55)]:
        os.environ["MCMI_STREAM_CHUNKS"] = str(chunks)
        os.environ["MCMI_STREAM_RATIO"] = str(ratio)
        compute_preconditioner(hb, cfg, out=out)
        ts, dev = [], []
        for _ in range(3):
            t0 = time.perf_counter()
            g = compute_preconditioner(hb, cfg, out=out)
            ts.append(time.perf_counter() - t0)
            dev.append(g.stats["ms_total"])
        ok = g.m == r.m
        print(f"chunks {chunks:2d} ratio {ratio:.2f}: wall {1e3 * min(ts):7.1f} ms  device {min(dev):7.1f} ms  "
              f"equal={ok}", flush=True)


if __name__ == "__main__":
    main()
