"""Recovery phase (§8f rank 4): GPU recover_inverse vs the reference's, with
its HBM traffic (16 n^2 bytes per block of 16 updates) and FP64 issue rate
(2 n^3 multiply/add operations) against the measured peaks.
    python tools/recovery_bench.py [n ...]  -> one JSON line per n"""
import json
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    import torch
    from oracle import ref
    from paper_2409_03095_b200 import recovery as R
    peaks = {}
    try:
        peaks = json.load(open(os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))),
                                            "MEASURED_PEAKS.json")))
    except OSError:
        pass
    hbm = float(peaks.get("hbm_gbs", 6544.0)) if isinstance(peaks, dict) else 6544.0
    try:  # measured by tools/fp64_peak.cu (DMUL + DADD issue rate)
        fp64 = json.load(open(os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "profiles",
                                           "fp64_peak.json")))["fp64_mul_add_ops_per_s"]
    except (OSError, KeyError, ValueError):
        fp64 = 1.85e13
    for n in [int(x) for x in sys.argv[1:]] or [1024, 2048, 4096]:
        rng = np.random.default_rng(n)
        m = rng.uniform(-1, 1, (n, n)) / n + np.eye(n)
        s = rng.uniform(-0.5, 0.5, n)
        t = torch.from_numpy(m).cuda()
        R.recover_inverse_device(t.clone(), s)  # warm-up
        torch.cuda.synchronize()
        reps = 3
        best = 1e9
        for _ in range(reps):
            u = t.clone()
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            R.recover_inverse_device(u, s)
            e1.record()
            torch.cuda.synchronize()
            best = min(best, e0.elapsed_time(e1))
        t0 = time.perf_counter()
        got = R.recover_inverse(m, s)
        host_ms = 1e3 * (time.perf_counter() - t0)
        # reference: a bounded sample of updates (the last k rows), scaled to n updates
        k = max(1, min(n, int(4e8 / (n * n))))
        sk = np.zeros(n)
        sk[n - k:] = s[n - k:]
        t0 = time.perf_counter()
        want_k = ref.recover_inverse(m, sk)
        ref_ms = 1e3 * (time.perf_counter() - t0) * n / k
        got_k = R.recover_inverse(m, sk)
        exact = bool(np.array_equal(got_k.view(np.uint64), want_k.view(np.uint64)))
        if n <= 1024:
            exact = exact and bool(np.array_equal(got.view(np.uint64), ref.recover_inverse(m, s).view(np.uint64)))
        # the kernel moves 16 n^2 bytes per block of 16 updates and issues 2 n^3
        # FP64 operations (one multiply and one add per element update, no FMA)
        gbs = 16.0 * n * n * ((n + 15) // 16) / (best / 1e3) / 1e9
        ops = 2.0 * n ** 3 / (best / 1e3)
        print(json.dumps({"n": n, "updates": n, "device_ms": round(best, 3), "host_api_ms": round(host_ms, 1),
                          "ref_ms_est": round(ref_ms, 1), "ref_sample_updates": k, "bit_exact": exact,
                          "hbm_gbs": round(gbs, 1), "frac_hbm": round(gbs / hbm, 3),
                          "fp64_ops_per_s": ops, "frac_fp64": round(ops / fp64, 3),
                          "speedup_vs_ref": round(ref_ms / best, 1)}), flush=True)


if __name__ == "__main__":
    main()
