"""Matrix Market I/O throughput: this library vs the reference (oracle/_ref).

    python tools/mm_bench.py [config] -> one JSON line
Writes and reads a generated matrix through both implementations (files under
/tmp) and checks the bytes and the parsed CSR are identical.
"""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    import numpy as np
    from oracle import ref
    from paper_2409_03095_b200 import generators as G
    from paper_2409_03095_b200 import matrix_market as mm
    name = sys.argv[1] if len(sys.argv) > 1 else "c3_lap3d_100"
    b = G.CONFIGS[name][0]()
    ours, theirs = f"/tmp/mm_ours_{os.getpid()}.mtx", f"/tmp/mm_ref_{os.getpid()}.mtx"
    out = {"config": name, "n": b.n, "nnz": b.nnz(), "threads": os.cpu_count()}
    t = time.perf_counter(); mm.write_matrix_market_file(b, ours); out["write_s"] = time.perf_counter() - t
    t = time.perf_counter(); m = mm.read_matrix_market_file(ours); out["read_s"] = time.perf_counter() - t
    rc = ref.Csr(b.n, b.row_ptr, b.col_idx, b.values)
    t = time.perf_counter(); ref.write_mm(rc, theirs); out["ref_write_s"] = time.perf_counter() - t
    t = time.perf_counter(); r = ref.read_mm(theirs); out["ref_read_s"] = time.perf_counter() - t
    with open(ours, "rb") as f1, open(theirs, "rb") as f2:
        out["bytes_identical"] = f1.read() == f2.read()
    out["csr_identical"] = bool(np.array_equal(m.col_idx, r.col_idx) and np.array_equal(m.row_ptr, r.row_ptr)
                                and np.array_equal(m.values.view(np.uint64), r.values.view(np.uint64)))
    out["mb"] = os.path.getsize(ours) / 1e6
    for k in ("write", "read"):
        out[f"{k}_speedup"] = out[f"ref_{k}_s"] / out[f"{k}_s"]
    os.remove(ours); os.remove(theirs)
    print(json.dumps({k: (round(v, 3) if isinstance(v, float) else v) for k, v in out.items()}))


if __name__ == "__main__":
    main()
