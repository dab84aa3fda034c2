#!/usr/bin/env python
"""Benchmark of the B200 MCMCMI preconditioner build (BASELINE.json metric:
"MC walk-steps/sec & preconditioner build ms at 1/2/4/8 B200 vs CPU ref").

One step = one full build (drop -> split -> transition tables -> walks ->
accumulate/top-k/scale/prune -> CSR assembly) of the configured synthetic
matrix, B resident in HBM.  With N ranks (torchrun, one per GPU) the rows are
block-partitioned (strong scaling: the matrix is fixed) and the shards are
assembled on every rank with an NCCL all-gather.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config c2_sym27_1p3m]
    python bench.py --impl reference ...   # the reference CPU build (oracle/_ref)

Prints ONE JSON line on rank 0.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

REPO = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, REPO)

METRIC = "MC walk-steps/sec & preconditioner build ms at 1/2/4/8 B200 vs CPU ref"
UNIT = "walk-steps/s"


def parse():
    p = argparse.ArgumentParser()
    p.add_argument("--gpus", type=int, default=1)
    p.add_argument("--steps", type=int, default=10)
    p.add_argument("--warmup", type=int, default=3)
    p.add_argument("--impl", default="ours", choices=["ours", "reference"])
    p.add_argument("--config", default="c2_sym27_1p3m")
    p.add_argument("--rng", default="reference", choices=["reference", "keyed"])
    p.add_argument("--e2e-steps", type=int, default=3)
    p.add_argument("--cpu-seconds", type=float, default=12.0, help="target CPU work of the baseline sample")
    p.add_argument("--no-e2e", action="store_true")
    p.add_argument("--no-cpu", action="store_true")
    p.add_argument("--assembly", default="p2p", choices=["p2p", "nccl"],
                   help="multi-GPU assembly of M: fused peer stores (default) or NCCL all-gather-v")
    return p.parse_args()


# ------------------------------------------------------------------ inputs

def make_workload(name):
    from paper_2409_03095_b200 import generators as G
    from paper_2409_03095_b200.mcspai import McConfig
    gen, over = G.CONFIGS[name]
    return gen(), McConfig(**over)


def principal_sample(b, rows):
    """Leading principal submatrix B[:rows, :rows] (for stencils: the first z-planes)."""
    from paper_2409_03095_b200.mcspai import CsrMatrix
    rp = b.row_ptr[: rows + 1]
    ci = b.col_idx[: rp[-1]]
    v = b.values[: rp[-1]]
    keep = ci < rows
    rowid = np.repeat(np.arange(rows), np.diff(rp))
    cnt = np.bincount(rowid[keep], minlength=rows)
    nrp = np.zeros(rows + 1, np.int64)
    np.cumsum(cnt, out=nrp[1:])
    return CsrMatrix(rows, nrp, ci[keep], v[keep])


def plane_rows(b):
    """Rows per z-plane for the stencil generators (sample granularity)."""
    n = b.n
    for k in (110 * 110, 100 * 100, 1000):
        if n % k == 0 and n // k >= 2:
            return k
    return max(1, n // 100)


# ------------------------------------------------------------------ clocks

class ClockSampler:
    FIELDS = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu_index):
        self.gpu = gpu_index
        self.proc = None
        self.lines = []

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.gpu), f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits",
                 "-lms", "100"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except OSError:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def __exit__(self, *a):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except subprocess.TimeoutExpired:
                self.proc.kill()

    def summary(self):
        sm, mx, reasons = [], 0, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            f = [x.strip() for x in ln.split(",")]
            if len(f) < 9:
                continue
            try:
                sm.append(float(f[1]))
                mx = max(mx, float(f[2]))
            except ValueError:
                continue
            for nm, val in zip(names, f[5:9]):
                if val.lower() == "active":
                    reasons.add(nm)
        if not sm:
            return None
        return {"sm_mhz": statistics.median(sm), "sm_max_mhz": mx, "reasons": sorted(reasons), "samples": len(sm)}


# ------------------------------------------------------------------ reference CPU arm

def _count_steps_worker(args):
    n, rp, ci, v, lo, hi, cfg = args
    from oracle import oracle
    return oracle.compute_preconditioner(n, rp, ci, v, row_begin=lo, row_end=hi, **cfg).walk_steps


def oracle_step_count(b, cfg_kw):
    """Exact walk-step count of the reference's walks on b (oracle restatement,
    row ranges in parallel over the host cores)."""
    from concurrent.futures import ProcessPoolExecutor
    workers = max(1, min(os.cpu_count() or 1, 64))
    edges = np.linspace(0, b.n, workers + 1).astype(np.int64)
    jobs = [(b.n, b.row_ptr, b.col_idx, b.values, int(edges[i]), int(edges[i + 1]), cfg_kw)
            for i in range(workers) if edges[i + 1] > edges[i]]
    with ProcessPoolExecutor(max_workers=workers) as ex:
        return int(sum(ex.map(_count_steps_worker, jobs)))


def time_reference(sample, cfg_kw, threads):
    from oracle import ref
    rb = ref.Csr(sample.n, sample.row_ptr, sample.col_idx, sample.values)
    t0 = time.perf_counter()
    r = ref.compute_preconditioner(rb, n_threads=threads, **cfg_kw)
    return time.perf_counter() - t0, r


def choose_sample(b, cfg_kw, threads, target_s):
    """Smallest leading block of z-planes whose reference build takes ~target_s."""
    per = plane_rows(b)
    planes = 1
    t, _ = time_reference(principal_sample(b, per * planes), cfg_kw, threads)  # also the warm-up
    total_planes = b.n // per
    want = max(1, min(total_planes, int(planes * target_s / max(t, 1e-3))))
    return principal_sample(b, per * want), want, per


def run_reference_arm(args):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return  # the CPU reference runs once, on rank 0
    from oracle import ref
    b, cfg = make_workload(args.config)
    cfg_kw = cfg.oracle_kwargs()
    cfg_kw.pop("rng_mode", None)
    threads = ref.max_threads()
    per_step_s = max(1.0, min(20.0, 150.0 / max(1, args.steps + args.warmup)))
    sample, planes, per = choose_sample(b, cfg_kw, threads, per_step_s)
    steps_per_build = oracle_step_count(sample, dict(cfg_kw, rng_mode=0))
    for _ in range(args.warmup):
        time_reference(sample, cfg_kw, threads)
    times = []
    res = None
    for _ in range(args.steps):
        t, res = time_reference(sample, cfg_kw, threads)
        times.append(t)
    t_med = statistics.median(times)
    value = steps_per_build / t_med
    desc = (f"leading {planes} of {b.n // per} z-planes ({sample.n} rows, {sample.nnz()} nnz) of {args.config}; "
            f"reference compute_preconditioner, {threads} OpenMP threads; {steps_per_build} walk steps per build "
            f"(counted by the oracle restatement)")
    print(json.dumps({
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": t_med * 1e3, "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": args.config, "n": b.n, "sample_rows": sample.n, "epsilon": cfg.epsilon,
                   "delta": cfg.delta, "alpha": cfg.alpha, "nnz_M_sample": int(res.m.nnz)},
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": threads, "kind": "reference", "sample": desc},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }), flush=True)


# ------------------------------------------------------------------ our arm

def load_traffic(workload, rng):
    path = os.path.join(REPO, "profiles", "walk_traffic.json")
    try:
        with open(path) as f:
            d = json.load(f)
        e = d.get(f"{workload}/{rng}")
        return e["dram_bytes_per_launch"] if e else None
    except (OSError, ValueError, KeyError):
        return None


def run_ours(args):
    import torch
    import torch.distributed as dist

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    torch.cuda.set_device(local)
    device = torch.device("cuda", local)

    from paper_2409_03095_b200.distributed import SymmetricM, allgatherv_csr, assemble_p2p, partition_rows
    from paper_2409_03095_b200.engine import DeviceEngine
    from paper_2409_03095_b200.mcspai import McConfig, RngMode, compute_preconditioner

    b, cfg = make_workload(args.config)
    cfg.rng_mode = RngMode.reference if args.rng == "reference" else RngMode.keyed
    cfg.device = local
    lo, hi = partition_rows(b.row_ptr, world)[rank]
    eng = DeviceEngine(local)
    d_rp, d_ci, d_v = DeviceEngine.upload(b, local)
    stream = torch.cuda.current_stream(device)

    # Multi-GPU assembly of M: the fused peer-store kernel over NVLink
    # (distributed.assemble_p2p) by default; the NCCL all-gather-v is the
    # reference point.  The first warm-up step runs both and keeps p2p only if
    # every rank's M is identical.
    assembly = "none" if world == 1 else args.assembly
    sym = SymmetricM(device, dist) if world > 1 else None

    def assemble(d, mode):
        if mode == "p2p":
            return assemble_p2p(d, lo, hi, b.n, dist, sym, stream)
        rp, ci, v, _, _ = eng.to_tensors(d, stream=stream)
        return allgatherv_csr(rp, ci, v, dist)

    def step():
        d = eng.build(b.n, d_rp, d_ci, d_v, cfg, lo, hi, stream=stream)
        if world > 1:
            assemble(d, assembly)
        return d

    if world > 1 and assembly == "p2p":
        d = eng.build(b.n, d_rp, d_ci, d_v, cfg, lo, hi, stream=stream)
        ok = True
        try:
            prp, pci, pv = (t.clone() for t in assemble(d, "p2p"))
        except Exception as ex:  # noqa: BLE001 — symmetric memory unavailable: use NCCL
            print(f"p2p assembly unavailable: {ex}", file=sys.stderr)
            ok = False
        nrp, nci, nv = assemble(d, "nccl")
        if ok:
            ok = bool(torch.equal(prp, nrp) and torch.equal(pci, nci) and torch.equal(pv.view(torch.int64),
                                                                                   nv.view(torch.int64)))
        flag = torch.tensor([1 if ok else 0], device=device)
        dist.all_reduce(flag, op=dist.ReduceOp.MIN)
        if not flag.item():
            assembly = "nccl"
    for _ in range(max(args.warmup, 0)):
        step()
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    stats = []
    with ClockSampler(local) as clk:
        ev0.record(stream)
        for _ in range(args.steps):
            stats.append(step().stats)
        ev1.record(stream)
        torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    # informational: the same build with the north star's (row, chain, step)
    # keying (rng_mode keyed) — a few timed steps, not the headline
    alt = None
    if world == 1 and args.rng == "reference":
        kcfg = McConfig(**{k: getattr(cfg, k) for k in cfg.__dataclass_fields__})
        kcfg.rng_mode = RngMode.keyed
        eng.build(b.n, d_rp, d_ci, d_v, kcfg, lo, hi, stream=stream)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        ks = [eng.build(b.n, d_rp, d_ci, d_v, kcfg, lo, hi, stream=stream).stats for _ in range(3)]
        e1.record(stream)
        torch.cuda.synchronize()
        kms = e0.elapsed_time(e1) / 3
        alt = {"rng_mode": "keyed", "value": sum(x["walk_steps"] for x in ks) / 3 / (kms / 1e3), "ms_per_step": kms}
    ms_local = ev0.elapsed_time(ev1) / max(args.steps, 1)
    steps_local = sum(s["walk_steps"] for s in stats) / max(args.steps, 1)
    walk_ms_local = sum(s["ms_walk_kernel"] for s in stats) / max(args.steps, 1)
    # algorithmic bytes per build: 20*steps + 8*sum deg(s); the
    # sum of degrees comes from one extra, untimed build with MCMI_FLAG_DEG_STATS
    # (identical walks, so the count is exact for every timed build)
    dcfg = McConfig(**{k: getattr(cfg, k) for k in cfg.__dataclass_fields__})
    dcfg.deg_stats = True
    deg_sum = eng.build(b.n, d_rp, d_ci, d_v, dcfg, lo, hi, stream=stream).stats["walk_deg_sum"]
    torch.cuda.synchronize()
    alg_bytes_local = 20 * steps_local + 8 * deg_sum
    launches_local = sum(s["launches"] for s in stats) + (args.steps if assembly == "p2p" else 0)
    agg = torch.tensor([ms_local, steps_local, walk_ms_local, alg_bytes_local, launches_local],
                       dtype=torch.float64, device=device)
    if world > 1:
        mx = agg.clone()
        dist.all_reduce(mx, op=dist.ReduceOp.MAX)
        sm = agg.clone()
        dist.all_reduce(sm, op=dist.ReduceOp.SUM)
    else:
        mx = sm = agg
    ms_per_step = float(mx[0])
    total_steps = float(sm[1])
    value = total_steps / (ms_per_step / 1e3)

    # ---- end to end through the public API (host CSR in pinned memory -> host CSR)
    e2e = None
    if not args.no_e2e:
        def pinned(a):
            t = torch.from_numpy(a).pin_memory()
            return t.numpy()
        from paper_2409_03095_b200.mcspai import CsrMatrix
        hb = CsrMatrix(b.n, pinned(b.row_ptr), pinned(b.col_idx), pinned(b.values))
        nnz_out = int(stats[-1]["nnz"])
        out = {"row_ptr": pinned(np.empty(hi - lo + 1, np.int64)),
               "col_idx": pinned(np.empty(max(nnz_out, 1), np.int64)),
               "values": pinned(np.empty(max(nnz_out, 1), np.float64))}
        compute_preconditioner(hb, cfg, out=out, rows=(lo, hi))  # warm-up
        times, st = [], None
        for _ in range(max(args.e2e_steps, 1)):
            if world > 1:
                dist.barrier()
            t0 = time.perf_counter()
            r = compute_preconditioner(hb, cfg, out=out, rows=(lo, hi))
            times.append(time.perf_counter() - t0)
            st = r.stats
        t_e2e = torch.tensor([statistics.mean(times)], dtype=torch.float64, device=device)
        if world > 1:
            dist.all_reduce(t_e2e, op=dist.ReduceOp.MAX)
        h2d = b.row_ptr.nbytes + b.col_idx.nbytes + b.values.nbytes
        d2h = 8 * (hi - lo + 1) + 16 * st["nnz"] + 16 * (hi - lo)
        e2e = {"value": total_steps / float(t_e2e[0]), "unit": UNIT, "h2d_bytes_per_step": int(h2d),
               "d2h_bytes_per_step": int(d2h), "ms_per_step": float(t_e2e[0]) * 1e3}

    # ---- CPU baseline (rank 0, N=1 only): the reference on a bounded sample
    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu:
        try:
            from oracle import ref
            cfg_kw = cfg.oracle_kwargs()
            cfg_kw.pop("rng_mode", None)
            threads = ref.max_threads()
            sample, planes, per = choose_sample(b, cfg_kw, threads, args.cpu_seconds)
            t_ref, _ = time_reference(sample, cfg_kw, threads)
            from paper_2409_03095_b200.mcspai import McConfig
            scfg = McConfig(**{k: v for k, v in cfg_kw.items()}, rng_mode=RngMode.reference, device=local)
            n_steps = compute_preconditioner(sample, scfg).stats["walk_steps"]  # identical walks (tier-1 parity)
            cpu = {"value": n_steps / t_ref, "unit": UNIT, "cores": threads, "kind": "reference",
                   "sample": (f"leading {planes} of {b.n // per} z-planes ({sample.n} rows) of {args.config}, "
                              f"reference OpenMP build {t_ref * 1e3:.0f} ms, {n_steps} walk steps")}
        except Exception as exc:  # the baseline is reported, never required
            cpu = {"value": None, "unit": UNIT, "cores": 0, "kind": "reference", "sample": f"unavailable: {exc}"}

    if rank == 0:
        peaks = {}
        try:
            with open(os.path.join(REPO, "MEASURED_PEAKS.json")) as f:
                peaks = json.load(f)
        except OSError:
            pass
        peak = float(peaks.get("hbm_gbs", 6650.0))
        try:
            with open(os.path.join(REPO, "profiles", "l2_peak.json")) as f:
                l2_peak = float(json.load(f)["l2_read_gbs"])
        except (OSError, ValueError, KeyError):
            l2_peak = None
        walk_ms = float(mx[2])
        achieved = float(agg[3]) / (float(agg[2]) / 1e3) / 1e9 if float(agg[2]) > 0 else 0.0
        s0 = stats[-1]
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms_per_step, "higher_is_better": True, "scaling": "strong",
            "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"workload": args.config, "n": b.n, "nnz_B": b.nnz(), "epsilon": cfg.epsilon,
                       "delta": cfg.delta, "alpha": cfg.alpha, "rng_mode": args.rng,
                       "n_chains": s0["n_chains"], "max_len": s0["max_len"], "nnz_M": int(s0["nnz"]) if world == 1
                       else None, "parallelism": f"rows/{world}" + ({"p2p": " + fused peer-store assembly (NVLink)",
                                                                      "nccl": " + NCCL allgatherv"}.get(assembly, "")),
                       "l2": f"input B {(b.nnz() * 16) / 1e6:.0f} MB > 126 MB L2 (no flush)"},
            "phases_ms": {"tables": s0["ms_tables"], "walk": s0["ms_walk"], "assemble": s0["ms_assemble"],
                          "walk_kernel": s0["ms_walk_kernel"]},
            "roofline": {"bound": "hbm", "kernel": "k_walk", "achieved": achieved, "peak": peak, "unit": "GB/s",
                         "frac": achieved / peak, "traffic": load_traffic(args.config, args.rng),
                         "bytes_per_step": "20 + 8*deg(s)", "walk_ms": walk_ms,
                         "l2_peak": l2_peak, "frac_l2": (achieved / l2_peak) if l2_peak else None,
                         "note": "tables are L2-resident: frac_l2 is the binding roofline (L2 read peak "
                                 "measured by tools/l2_peak.cu); traffic = DRAM bytes per walk launch (ncu)"},
            "cpu_baseline": cpu, "e2e": e2e, "gpu_launches": int(sm[4]), "alt_keyed": alt,
            "clocks": clk.summary(),
        }
        print(json.dumps(line), flush=True)
    eng.close()
    if world > 1:
        dist.destroy_process_group()


def main():
    args = parse()
    if args.impl == "reference":
        run_reference_arm(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
