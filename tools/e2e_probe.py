"""Times the host-API paths on one config: handle path (build + copy) vs the
streamed mcmi_build_into, with pinned vs pageable outputs."""
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    import torch
    from paper_2409_03095_b200 import generators as G
    from paper_2409_03095_b200.mcspai import CsrMatrix, compute_preconditioner
    name = sys.argv[1] if len(sys.argv) > 1 else "c2_sym27_1p3m"
    gen, over = G.CONFIGS[name]
    from paper_2409_03095_b200.mcspai import McConfig
    b = gen()
    cfg = McConfig(**over)
    pin = lambda a: torch.from_numpy(a).pin_memory().numpy()  # noqa: E731
    hb = CsrMatrix(b.n, pin(b.row_ptr), pin(b.col_idx), pin(b.values))
    r = compute_preconditioner(hb, cfg)
    nnz = r.m.nnz()
    print("device ms", r.stats["ms_total"], "nnz", nnz, flush=True)
    from paper_2409_03095_b200.mcspai import host_register
    reg = {"row_ptr": np.empty(b.n + 1, np.int64), "col_idx": np.empty(nnz, np.int64), "values": np.empty(nnz)}
    t0 = time.perf_counter()
    host_register(reg["row_ptr"], reg["col_idx"], reg["values"])
    hb2 = CsrMatrix(b.n, b.row_ptr.copy(), b.col_idx.copy(), b.values.copy())
    host_register(hb2.row_ptr, hb2.col_idx, hb2.values)
    print("register ms", 1e3 * (time.perf_counter() - t0), flush=True)
    for label, out in (("into-registered", reg), ("handle", None),
                       ("into-pinned", {"row_ptr": pin(np.empty(b.n + 1, np.int64)),
                                        "col_idx": pin(np.empty(nnz, np.int64)), "values": pin(np.empty(nnz))}),
                       ("into-pageable", {"row_ptr": np.empty(b.n + 1, np.int64), "col_idx": np.empty(nnz, np.int64),
                                          "values": np.empty(nnz)})):
        src = hb2 if label == "into-registered" else hb
        compute_preconditioner(src, cfg, out=out)
        ts = []
        for _ in range(3):
            t0 = time.perf_counter()
            g = compute_preconditioner(src, cfg, out=out)
            ts.append(time.perf_counter() - t0)
        ok = g.m == r.m
        print(f"{label:14s} wall {1e3 * min(ts):8.1f} ms  device {g.stats['ms_total']:8.1f} ms  equal={ok}", flush=True)


if __name__ == "__main__":
    main()
