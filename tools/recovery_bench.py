"""Recovery phase (§8f rank 4): GPU recover_inverse vs the reference's, with
the bandwidth roofline of the rank-one update (16 n^2 bytes per update).
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
        gbs = 16.0 * n * n * n / (best / 1e3) / 1e9
        print(json.dumps({"n": n, "updates": n, "device_ms": round(best, 3), "host_api_ms": round(host_ms, 1),
                          "ref_ms_est": round(ref_ms, 1), "ref_sample_updates": k, "bit_exact": exact,
                          "achieved_gbs": round(gbs, 1), "hbm_peak_gbs": hbm, "frac_hbm": round(gbs / hbm, 3),
                          "speedup_vs_ref": round(ref_ms / best, 1)}), flush=True)


if __name__ == "__main__":
    main()
