"""CPU side of SURVEY.md §8(d), timed on the GPU box's host: the unmodified
reference (oracle/_ref) `compute_preconditioner` with all host threads and
with 1 thread, and `compute_preconditioner_serial`, on the BASELINE configs
(C2 on a leading block of z-planes so one single-thread build stays ~15 s).
One warm-up, then the median of --runs.  Walk steps per build come from the
oracle restatement (same seeds, identical walks).

    python tools/cpu_reference.py [--runs 3] > profiles/r01_cpu_reference.jsonl
"""
import argparse
import json
import os
import platform
import statistics
import sys
import time

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, REPO)


def cpu_model():
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return platform.processor()


def main():
    p = argparse.ArgumentParser()
    p.add_argument("--runs", type=int, default=3)
    p.add_argument("--configs", default="c1_poisson2d_100,c3_lap3d_100,c4_convdiff_1000,c2_sym27_1p3m")
    a = p.parse_args()
    import bench
    from oracle import ref
    from paper_2409_03095_b200 import generators as G
    threads = ref.max_threads()
    for name in a.configs.split(","):
        b, cfg = bench.make_workload(name)
        kw = cfg.oracle_kwargs()
        kw.pop("rng_mode", None)
        sample = b
        note = "full matrix"
        if name.startswith("c2_"):  # single-thread C2 takes ~10 min: leading z-planes
            per = bench.plane_rows(b)
            sample = bench.principal_sample(b, per * 4)
            note = f"leading 4 of {b.n // per} z-planes ({sample.n} rows)"
        steps = bench.oracle_step_count(sample, dict(kw, rng_mode=0))
        rb = ref.Csr(sample.n, sample.row_ptr, sample.col_idx, sample.values)
        out = {"config": name, "sample": note, "rows": sample.n, "walk_steps": steps, "cpu": cpu_model(),
               "host_threads": threads}
        for label, nt, serial in (("all_threads", threads, False), ("one_thread", 1, False), ("serial", 0, True)):
            ts = []
            for i in range(a.runs + 1):
                t0 = time.perf_counter()
                ref.compute_preconditioner(rb, n_threads=nt, serial=serial, **kw)
                if i:  # first run is the warm-up
                    ts.append(time.perf_counter() - t0)
            med = statistics.median(ts)
            out[f"{label}_ms"] = round(1e3 * med, 1)
            out[f"{label}_steps_per_s"] = steps / med
        print(json.dumps(out), flush=True)
    del G


if __name__ == "__main__":
    main()
