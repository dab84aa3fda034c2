#!/usr/bin/env python
"""Benchmark of the B200 MCMCMI preconditioner build (BASELINE.json metric:
"MC walk-steps/sec & preconditioner build ms at 1/2/4/8 B200 vs CPU ref").

One step = one full build (drop -> split -> transition tables -> walks ->
accumulate/top-k/scale/prune -> CSR assembly) of the configured synthetic
matrix, B resident in HBM.  With N ranks (torchrun, one per GPU) the rows are
block-partitioned (strong scaling: the matrix is fixed) and M is assembled on
every rank (fused NVLink peer stores).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config c2_sym27_1p3m]
    python bench.py --impl reference ...   # the reference CPU build (oracle/_ref), same config

Prints ONE JSON line on rank 0.  Both arms print ``m_sha256`` (sha256 of
row_ptr || col_idx || value bits of the built M), so the run itself shows the
two builds are byte-identical; tests/golden/fullsize.json holds the
reference's hash made in the build container (tests/golden/make_fullsize.py).
"""
from __future__ import annotations

import argparse
import hashlib
import importlib.util
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
#: north-star and parity configs timed beside the headline (device-resident build ms, max over ranks)
EXTRA_CONFIGS = ["c2_sym27_default", "c3_lap3d_100", "c3_lap3d_100_heavy", "c4_convdiff_1000",
                 "c5_powerlaw_4m_1e4x32"]
#: extra configs built on their leading rows only (the full C5 corner is 1.3e12
#: steps); single-GPU runs only
EXTRA_ROWS = {"c5_powerlaw_4m_1e4x32": 12500}


def parse():
    p = argparse.ArgumentParser()
    p.add_argument("--gpus", type=int, default=1)
    p.add_argument("--steps", type=int, default=10)
    p.add_argument("--warmup", type=int, default=3)
    p.add_argument("--impl", default="ours", choices=["ours", "reference"])
    p.add_argument("--config", default="c2_sym27_1p3m")
    p.add_argument("--rng", default="reference", choices=["reference", "keyed"])
    p.add_argument("--e2e-steps", type=int, default=3)
    p.add_argument("--cpu-runs", type=int, default=5, help="reference builds in the cpu_baseline median")
    p.add_argument("--ref-budget-s", type=float, default=float(os.environ.get("BENCH_REF_BUDGET_S", 1500)),
                   help="wall budget of --impl reference: warm-ups are dropped first, then steps (min 5)")
    p.add_argument("--no-e2e", action="store_true")
    p.add_argument("--no-cpu", action="store_true")
    p.add_argument("--no-extra", action="store_true", help="skip the extra configs (C2 defaults, C3, C4)")
    p.add_argument("--assembly", default="p2p", choices=["p2p", "nccl"],
                   help="multi-GPU assembly of M: fused peer stores (default) or NCCL all-gather-v")
    return p.parse_args()


# ------------------------------------------------------------------ inputs (no product import)

def load_generators():
    """paper_2409_03095_b200/generators.py imported by file path: pure numpy,
    so the reference arm never maps the product library."""
    name = "mcmi_generators_standalone"
    if name in sys.modules:
        return sys.modules[name]
    spec = importlib.util.spec_from_file_location(name, os.path.join(REPO, "paper_2409_03095_b200", "generators.py"))
    mod = importlib.util.module_from_spec(spec)
    sys.modules[name] = mod
    spec.loader.exec_module(mod)
    return mod


def workload(name):
    gen, over = load_generators().CONFIGS[name]
    return gen(), dict(over)


def csr_sha256(row_ptr, col_idx, values) -> str:
    """sha256(row_ptr int64 || col_idx int64 || values f64 bits): the M hash of
    tests/golden/fullsize.json."""
    h = hashlib.sha256()
    for a in (row_ptr, col_idx, values):
        h.update(memoryview(np.ascontiguousarray(a)).cast("B"))
    return h.hexdigest()


def positional_checksum(*arrays) -> str:
    """sum of word[i] * (2i+1) mod 2^64 over the 8-byte words of the arrays in
    order (tools/dropin_e2e.cpp prints the same for its M)."""
    s, i0 = np.uint64(0), 0
    with np.errstate(over="ignore"):
        for a in arrays:
            w = np.ascontiguousarray(a).view(np.uint64)
            for k in range(0, w.size, 1 << 24):
                part = w[k:k + (1 << 24)]
                idx = np.arange(i0 + k, i0 + k + part.size, dtype=np.uint64) * np.uint64(2) + np.uint64(1)
                s = np.uint64(s + np.sum(part * idx, dtype=np.uint64))
            i0 += w.size
    return f"{int(s):016x}"


def run_dropin_harness(harness, b, over, runs, steps_per_build, m_sum):
    """Times tools/dropin_e2e (the C++ drop-in, pageable vectors in and out)."""
    import shutil
    import tempfile
    d = tempfile.mkdtemp(prefix="mcmi_e2e_")
    try:
        np.array([b.n], np.int64).tofile(os.path.join(d, "n.i64"))
        b.row_ptr.astype(np.int64).tofile(os.path.join(d, "row_ptr.i64"))
        b.col_idx.astype(np.int64).tofile(os.path.join(d, "col_idx.i64"))
        b.values.astype(np.float64).tofile(os.path.join(d, "values.f64"))
        if over.get("retain_k") or over.get("chains_override") or over.get("max_len_override"):
            return {"value": None, "note": "harness takes eps/delta/alpha/seed only"}
        cmd = [harness, d, repr(over.get("epsilon", 0.0625)), repr(over.get("delta", 0.0625)),
               repr(over.get("alpha", 5.0)), str(over.get("master_seed", 0)), str(max(runs, 1))]
        r = subprocess.run(cmd, capture_output=True, text=True, timeout=900)
        if r.returncode != 0:
            return {"value": None, "note": f"harness failed: {r.stderr.strip()[-300:]}"}
        out = json.loads(r.stdout.strip().splitlines()[-1])
        t = statistics.mean(out["runs_ms"]) / 1e3
        return {"value": steps_per_build / t, "unit": UNIT, "ms_per_step": t * 1e3, "runs_ms": out["runs_ms"],
                "h2d_bytes_per_step": int(b.row_ptr.nbytes + b.col_idx.nbytes + b.values.nbytes),
                "d2h_bytes_per_step": int(8 * (b.n + 1) + 16 * out["nnz"] + 16 * b.n),
                "m_checksum_equal": out["checksum"] == m_sum,
                "api": "mcmi::compat::compute_preconditioner<ApproxInverse, SplitError>(b, cfg): the reference's "
                       "own CsrMatrix (pageable std::vector) in, ApproxInverse out (tools/dropin_e2e.cpp)"}
    finally:
        shutil.rmtree(d, ignore_errors=True)


def golden(name, b_sha):
    """The reference's full-size record for this config (same input hash), or None."""
    try:
        with open(os.path.join(REPO, "tests", "golden", "fullsize.json")) as f:
            g = json.load(f).get(name)
    except (OSError, ValueError):
        return None
    return g if g and g.get("b_sha256") == b_sha else None


def config_dict(name, b, over, n_chains, max_len, nnz_m, rng="reference"):
    """The `config` object, identical in both arms (the reference arm is the reference stream)."""
    return {"workload": name, "n": int(b.n), "nnz_B": int(b.nnz()), "epsilon": over.get("epsilon", 0.0625),
            "delta": over.get("delta", 0.0625), "alpha": over.get("alpha", 5.0), "retain_k": over.get("retain_k", 0),
            "master_seed": over.get("master_seed", 0), "rng_mode": rng, "n_chains": int(n_chains),
            "max_len": int(max_len), "nnz_M": int(nnz_m),
            "l2": f"input B {(b.nnz() * 16 + b.n * 8) / 1e6:.0f} MB > 126 MB L2 (no flush)"}


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


def oracle_step_count(b, over):
    """Exact walk-step count of the reference's walks on b (oracle restatement,
    row ranges in parallel over the host cores).  Only used when
    tests/golden/fullsize.json has no record for this input."""
    from concurrent.futures import ProcessPoolExecutor
    workers = max(1, min(os.cpu_count() or 1, 64))
    edges = np.linspace(0, b.n, workers + 1).astype(np.int64)
    cfg = dict(over, rng_mode=0)
    jobs = [(b.n, b.row_ptr, b.col_idx, b.values, int(edges[i]), int(edges[i + 1]), cfg)
            for i in range(workers) if edges[i + 1] > edges[i]]
    with ProcessPoolExecutor(max_workers=workers) as ex:
        return int(sum(ex.map(_count_steps_worker, jobs)))


def reference_runs(b, over, threads, runs, warmups=0, budget_s=None):
    """The unmodified reference (oracle/_ref) on the FULL matrix: the first
    build copies M out (hash, nnz, budget); the rest time the reference call
    alone (ref_build_timed).  Returns (first, [seconds of the timed builds], warmups done)."""
    from oracle import ref
    rb = ref.Csr(b.n, b.row_ptr, b.col_idx, b.values)
    first = ref.compute_preconditioner(rb, n_threads=threads, **over)
    est = max(first.build_s, 1e-3)
    if budget_s is not None:  # keep the whole arm inside the budget: drop warm-ups first, then runs (>= 5)
        runs = min(runs, max(5, int(budget_s / est)))
        warmups = min(warmups, max(0, int((budget_s - runs * est) / est)))
    for _ in range(warmups):
        ref.compute_preconditioner(rb, n_threads=threads, copy=False, **over)
    times = [ref.compute_preconditioner(rb, n_threads=threads, copy=False, **over).build_s for _ in range(runs)]
    return first, times, warmups


def run_reference_arm(args):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return  # the CPU reference runs once, on rank 0
    from oracle import ref
    b, over = workload(args.config)
    b_sha = csr_sha256(b.row_ptr, b.col_idx, b.values)
    threads = ref.max_threads()
    first, times, warm = reference_runs(b, over, threads, args.steps, max(args.warmup - 1, 0), args.ref_budget_s)
    m = first.m
    m_sha = csr_sha256(m.row_ptr, m.col_idx, m.values)
    g = golden(args.config, b_sha)
    steps_per_build = g["reference"]["walk_steps"] if g else oracle_step_count(b, over)
    total = sum(times)
    value = steps_per_build * len(times) / total
    t_med = statistics.median(times)
    cfg = config_dict(args.config, b, over, first.n_chains, first.max_len, int(m.row_ptr[-1]))
    desc = (f"full {args.config} ({b.n} rows, {b.nnz()} nnz): the reference's compute_preconditioner "
            f"(oracle/_ref, -O3 OpenMP) with {threads} threads, {len(times)} timed builds after "
            f"{warm + 1} warm-up(s), median {t_med * 1e3:.0f} ms; {steps_per_build} walk steps per build "
            f"({'tests/golden/fullsize.json, input sha256 matched' if g else 'counted by the oracle restatement'})")
    print(json.dumps({
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": args.gpus,
        "steps": len(times), "warmup": warm + 1, "ms_per_step": total / len(times) * 1e3, "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic", "config": cfg,
        "parallelism": f"OpenMP {threads} host threads", "m_sha256": m_sha,
        "m_sha256_matches_golden": (m_sha == g["reference"]["m_sha256"]) if g else None,
        "build_ms": {"median": t_med * 1e3, "min": min(times) * 1e3, "max": max(times) * 1e3},
        "cpu_baseline": {"value": steps_per_build / t_med, "unit": UNIT, "cores": threads, "kind": "reference",
                         "sample": desc},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }), flush=True)


# ------------------------------------------------------------------ our arm

def walk_source_sha16():
    h = hashlib.sha256()
    for f in ("walk.cu", "kernels.cuh", "common.cuh"):
        with open(os.path.join(REPO, "paper_2409_03095_b200", "csrc", f), "rb") as fh:
            h.update(fh.read())
    return h.hexdigest()[:16]


def load_ncu(workload_name, rng):
    """ncu per-launch counters of the walk kernel for this workload, only if
    they were captured on the walk kernel source being timed (profiles/walk_traffic.json)."""
    try:
        with open(os.path.join(REPO, "profiles", "walk_traffic.json")) as f:
            d = json.load(f)
    except (OSError, ValueError):
        return None
    e = d.get("entries", {}).get(f"{workload_name}/{rng}")
    if not e or e.get("walk_source_sha16") != walk_source_sha16():
        return None
    return e


def run_ours(args):
    import torch
    import torch.distributed as dist

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world > 1:
        os.environ.setdefault("NCCL_DEBUG", "INFO")
        os.environ.setdefault("NCCL_DEBUG_SUBSYS", "INIT")
        import datetime
        # a bounded store timeout: a peer that never reaches a rendezvous fails
        # the run in minutes instead of holding the node (SymmetricM / NCCL init)
        dist.init_process_group("nccl", device_id=torch.device("cuda", local),
                                timeout=datetime.timedelta(seconds=180))
    torch.cuda.set_device(local)
    device = torch.device("cuda", local)

    from paper_2409_03095_b200.distributed import SymmetricM, allgatherv_csr, assemble_p2p, partition_rows
    from paper_2409_03095_b200.engine import DeviceEngine
    from paper_2409_03095_b200.mcspai import CsrMatrix, McConfig, RngMode, compute_preconditioner

    eng = DeviceEngine(local)
    stream = torch.cuda.current_stream(device)
    assembly = "none" if world == 1 else args.assembly
    sym = SymmetricM(device, dist) if world > 1 else None

    def setup(name):
        gb, over = workload(name)
        b = CsrMatrix(gb.n, gb.row_ptr, gb.col_idx, gb.values)
        cfg = McConfig(**over)
        cfg.rng_mode = RngMode.reference if args.rng == "reference" else RngMode.keyed
        cfg.device = local
        lo, hi = partition_rows(b.row_ptr, world)[rank]
        return b, over, cfg, lo, hi, DeviceEngine.upload(b, local)

    def assemble(d, lo, hi, n, mode):
        if mode == "p2p":
            return assemble_p2p(d, lo, hi, n, dist, sym, stream)
        rp, ci, v, _, _ = eng.to_tensors(d, stream=stream)
        return allgatherv_csr(rp, ci, v, dist)

    def make_step(b, cfg, lo, hi, dv):
        def step():
            d = eng.build(b.n, *dv, cfg, lo, hi, stream=stream)
            m = assemble(d, lo, hi, b.n, assembly) if world > 1 else None
            return d, m
        return step

    def barrier():
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()

    def timed(step, k):
        """k steps between barriers, CUDA events on the launching stream; max over
        ranks.  Returns (ms per step, [stats of each step], last step's output)."""
        barrier()
        ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        st, last = [], None
        ev0.record(stream)
        for _ in range(k):
            last = step()  # only the last M is kept (an all-gathered M is the whole matrix)
            st.append(last[0].stats)
        ev1.record(stream)
        barrier()
        return ev0.elapsed_time(ev1) / max(k, 1), st, last

    def reduce(vals, op):
        t = torch.tensor(vals, dtype=torch.float64, device=device)
        if world > 1:
            dist.all_reduce(t, op=dist.ReduceOp.MAX if op == "max" else dist.ReduceOp.SUM)
        return [float(x) for x in t]

    b, over, cfg, lo, hi, dv = setup(args.config)
    step = make_step(b, cfg, lo, hi, dv)

    # Multi-GPU: the first warm-up step runs both assemblies and keeps p2p only
    # if every rank's M is identical to the NCCL all-gather-v.
    if world > 1 and assembly == "p2p":
        d = eng.build(b.n, *dv, cfg, lo, hi, stream=stream)
        ok = True
        try:
            prp, pci, pv = (t.clone() for t in assemble(d, lo, hi, b.n, "p2p"))
        except Exception as ex:  # noqa: BLE001 — symmetric memory unavailable: use NCCL
            print(f"p2p assembly unavailable: {ex}", file=sys.stderr)
            ok = False
        nrp, nci, nv = assemble(d, lo, hi, b.n, "nccl")
        if ok:
            ok = bool(torch.equal(prp, nrp) and torch.equal(pci, nci)
                      and torch.equal(pv.view(torch.int64), nv.view(torch.int64)))
        flag = torch.tensor([1 if ok else 0], device=device)
        dist.all_reduce(flag, op=dist.ReduceOp.MIN)
        if not flag.item():
            assembly = "nccl"
    for _ in range(max(args.warmup, 0)):
        step()
    with ClockSampler(local) as clk:
        ms_local, stats, last = timed(step, args.steps)
    steps_local = sum(s["walk_steps"] for s in stats) / max(args.steps, 1)
    walk_ms_local = sum(s["ms_walk_kernel"] for s in stats) / max(args.steps, 1)
    launches_local = sum(s["launches"] for s in stats) + (args.steps if assembly == "p2p" else 0)
    ms_per_step, walk_ms = reduce([ms_local, walk_ms_local], "max")
    total_steps, launches, nnz_total = reduce([steps_local, launches_local, stats[-1]["nnz"]], "sum")
    value = total_steps / (ms_per_step / 1e3)

    # the M of the last timed build, hashed on rank 0 (outside the timed region)
    d_last, m_last = last
    if world == 1:
        rp_t, ci_t, v_t, _, _ = eng.to_tensors(d_last, stream=stream)
    else:
        rp_t, ci_t, v_t = m_last
    torch.cuda.synchronize()
    m_sha = m_sum = None
    if rank == 0:
        m_host = (rp_t.cpu().numpy(), ci_t.cpu().numpy(), v_t.cpu().numpy())
        m_sha, m_sum = csr_sha256(*m_host), positional_checksum(*m_host)
        del m_host
    del last, m_last, rp_t, ci_t, v_t
    b_sha = csr_sha256(b.row_ptr, b.col_idx, b.values) if rank == 0 else None
    g = golden(args.config, b_sha) if rank == 0 else None

    # informational: the same build with the north star's (row, chain, step) keying
    alt = None
    if args.rng == "reference":
        kcfg = McConfig(**{k: getattr(cfg, k) for k in cfg.__dataclass_fields__})
        kcfg.rng_mode = RngMode.keyed
        kstep = make_step(b, kcfg, lo, hi, dv)
        kstep()
        kms, kst, _ = timed(kstep, 3)
        (kms,) = reduce([kms], "max")
        (ksteps,) = reduce([kst[-1]["walk_steps"]], "sum")
        alt = {"rng_mode": "keyed", "value": ksteps / (kms / 1e3), "ms_per_step": kms}

    # algorithmic bytes per build: 20*steps + 8*sum deg(s); the
    # sum of degrees comes from one extra, untimed build with MCMI_FLAG_DEG_STATS
    # (identical walks, so the count is exact for every timed build)
    dcfg = McConfig(**{k: getattr(cfg, k) for k in cfg.__dataclass_fields__})
    dcfg.deg_stats = True
    deg_sum = eng.build(b.n, *dv, dcfg, lo, hi, stream=stream).stats["walk_deg_sum"]
    torch.cuda.synchronize()
    alg_bytes_local = 20 * steps_local + 8 * deg_sum

    # ---- the other configs (device-resident build ms, max over ranks)
    extra = {}
    if not args.no_extra:
        for name in EXTRA_CONFIGS:
            if name == args.config or (name in EXTRA_ROWS and world > 1):
                continue
            xb, xover, xcfg, xlo, xhi, xdv = setup(name)
            if name in EXTRA_ROWS:
                xlo, xhi = 0, min(xhi, EXTRA_ROWS[name])
            xstep = make_step(xb, xcfg, xlo, xhi, xdv)
            for _ in range(2):
                xstep()
            xms, xst, _ = timed(xstep, 5)
            xs = xst[-1]
            (xms, xwalk), (xsteps,) = reduce([xms, xs["ms_walk_kernel"]], "max"), reduce([xs["walk_steps"]], "sum")
            extra[name] = {"build_ms": xms, "walk_kernel_ms": xwalk, "walk_steps": int(xsteps),
                           "value": xsteps / (xms / 1e3), "n_chains": xs["n_chains"], "max_len": xs["max_len"]}
            if name in EXTRA_ROWS:
                extra[name]["rows"] = xhi - xlo
            del xdv

    # ---- end to end through the public API: pinned host CSR in, host M out.
    # N = 1: compute_preconditioner(B) (streamed build into library-owned pinned
    # slabs, returned without a copy).  N > 1: rank 0 calls the same drop-in with
    # McConfig.n_gpus = N (one process drives all N GPUs, shards land at their
    # global offsets in one host M); the other ranks wait.  No output size is
    # known in advance.
    e2e = None
    if not args.no_e2e:
        def pinned(a):
            return torch.from_numpy(a).pin_memory().numpy()
        hb = CsrMatrix(b.n, pinned(b.row_ptr), pinned(b.col_idx), pinned(b.values))
        ecfg = McConfig(**{k: getattr(cfg, k) for k in cfg.__dataclass_fields__})
        ecfg.device, ecfg.n_gpus = 0, world
        times, st = [], None
        # ranks != 0 wait on the store, not in an NCCL barrier: a barrier kernel
        # spinning on their GPUs would share the SMs rank 0's build runs on
        store = dist.distributed_c10d._get_default_store() if world > 1 else None
        if rank == 0:
            r = compute_preconditioner(hb, ecfg)  # warm-up
            del r
            for _ in range(max(args.e2e_steps, 1)):
                t0 = time.perf_counter()
                r = compute_preconditioner(hb, ecfg)
                times.append(time.perf_counter() - t0)
                st = r.stats
                e2e_nnz = r.m.nnz()
                del r
        if world > 1:
            if rank == 0:
                store.set("mcmi_e2e_done", "1")
            else:
                import datetime
                store.wait(["mcmi_e2e_done"], datetime.timedelta(seconds=900))
            dist.barrier()
        if rank == 0:
            t_e2e = statistics.mean(times)
            h2d = b.row_ptr.nbytes + b.col_idx.nbytes + b.values.nbytes
            d2h = 8 * (b.n + 1) + 16 * e2e_nnz + 16 * b.n
            e2e = {"value": total_steps / t_e2e, "unit": UNIT, "h2d_bytes_per_step": int(h2d),
                   "d2h_bytes_per_step": int(d2h), "ms_per_step": t_e2e * 1e3,
                   "api": f"mcspai.compute_preconditioner(B pinned host CSR, McConfig(n_gpus={world}))",
                   "walk_steps": int(st["walk_steps"])}

    # ---- the C++ drop-in on the reference's own types (tools/dropin_e2e.cpp):
    # pageable std::vector B in, std::vector M out, nothing sized in advance
    e2e_cpp = None
    harness = os.path.join(REPO, "tools", "_build", "dropin_e2e")
    if rank == 0 and world == 1 and not args.no_e2e and os.path.exists(harness):
        e2e_cpp = run_dropin_harness(harness, b, over, args.e2e_steps, total_steps, m_sum)

    # ---- CPU baseline (rank 0, N=1 only): the reference on the same full matrix
    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu:
        try:
            from oracle import ref
            threads = ref.max_threads()
            first, rtimes, _ = reference_runs(b, over, threads, args.cpu_runs, 0, budget_s=240.0)
            t_med = statistics.median(rtimes)
            ref_sha = csr_sha256(first.m.row_ptr, first.m.col_idx, first.m.values)
            cpu = {"value": total_steps / t_med, "unit": UNIT, "cores": threads, "kind": "reference",
                   "sample": (f"full {args.config}: the reference's compute_preconditioner (oracle/_ref, OpenMP) "
                              f"with {threads} threads, median of {len(rtimes)} builds after one warm-up "
                              f"({t_med * 1e3:.0f} ms); walk steps counted by our build (identical walks: "
                              f"M sha256 {'equal' if ref_sha == m_sha else 'DIFFERENT'})"),
                   "build_ms_median": t_med * 1e3, "m_sha256_equal": ref_sha == m_sha}
            del first
        except Exception as exc:  # the baseline is reported, never required
            cpu = {"value": None, "unit": UNIT, "cores": 0, "kind": "reference", "sample": f"unavailable: {exc}"}

    if rank == 0:
        peaks = {}
        try:
            with open(os.path.join(REPO, "MEASURED_PEAKS.json")) as f:
                peaks = json.load(f)
        except OSError:
            pass
        hbm_peak = float(peaks.get("hbm_gbs", 6650.0))
        try:
            with open(os.path.join(REPO, "profiles", "l2_peak.json")) as f:
                l2_peak = float(json.load(f)["l2_read_gbs"])
        except (OSError, ValueError, KeyError):
            l2_peak = None
        walk_ms_rank0 = walk_ms_local
        ncu = load_ncu(args.config, args.rng)
        s0 = stats[-1]
        # This kernel's algorithmic bytes per walk step: the 32-byte state record,
        # the 32-byte {cum, ratio} pair its guide bucket points at (16 buckets
        # resolve nearly every draw there) and the 4-byte column: 68 B (a forced
        # move reads only the record).  SURVEY §8d's 20 + 8*deg(s) charges the
        # reference's linear CDF scan and is reported beside it.
        alg_bytes = 68.0 * steps_local
        t_walk = walk_ms_rank0 / 1e3 if walk_ms_rank0 > 0 else float("inf")
        achieved = alg_bytes / t_walk / 1e9
        model_gbs = alg_bytes_local / t_walk / 1e9
        roofline = {
            # The walk's tables stay L2-resident (ncu: DRAM traffic ~0.3% of the
            # L2 traffic), so L2 is the memory level it reads; it is bound below
            # that by SM instruction issue (measured.issue_active).
            "bound": "l2", "kernel": "k_walk", "achieved": achieved, "peak": l2_peak, "unit": "GB/s",
            "frac": (achieved / l2_peak) if l2_peak else None,
            "traffic": ncu["dram_bytes_per_launch"] if ncu else None,
            "peak_source": "profiles/l2_peak.json (tools/l2_peak.cu, L2-resident read kernel on a B200)",
            "bytes_per_step": "68 = 32 B state record + 32 B {cum, ratio} pair at the guide bucket + 4 B column",
            "alg_bytes_per_launch": alg_bytes, "walk_kernel_ms": walk_ms_rank0, "hbm_peak": hbm_peak,
            "model_8d": {"bytes_per_step": "20 + 8*deg(s) (SURVEY.md §8d: the reference's full CDF row)",
                         "bytes_per_launch": alg_bytes_local, "achieved": model_gbs,
                         "frac_l2": (model_gbs / l2_peak) if l2_peak else None, "frac_hbm": model_gbs / hbm_peak},
            "measured": (dict({k: ncu[k] for k in ("l2_bytes_per_launch", "dram_bytes_per_launch", "issue_active",
                                                   "ipc", "warp_instructions_per_launch", "l1_hit_rate",
                                                   "l2_hit_rate", "captured") if k in ncu},
                              l2_gbs=ncu["l2_bytes_per_launch"] / t_walk / 1e9,
                              l2_frac=(ncu["l2_bytes_per_launch"] / t_walk / 1e9 / l2_peak) if l2_peak else None,
                              dram_frac=ncu["dram_bytes_per_launch"] / t_walk / 1e9 / hbm_peak)
                         if ncu else "no ncu capture of this walk-kernel source (profiles/walk_traffic.json)"),
        }
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms_per_step, "higher_is_better": True, "scaling": "strong",
            "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": config_dict(args.config, b, over, s0["n_chains"], s0["max_len"], nnz_total, args.rng),
            "parallelism": f"rows/{world}" + ({"p2p": " + fused peer-store assembly (NVLink)",
                                              "nccl": " + NCCL allgatherv"}.get(assembly, "")),
            "m_sha256": m_sha, "m_sha256_matches_golden": (m_sha == g["reference"]["m_sha256"])
            if (g and args.rng == "reference") else None,
            "phases_ms": {"tables": s0["ms_tables"], "walk": s0["ms_walk"], "assemble": s0["ms_assemble"],
                          "walk_kernel": s0["ms_walk_kernel"]},
            "roofline": roofline, "cpu_baseline": cpu, "e2e": e2e, "e2e_cpp": e2e_cpp, "gpu_launches": int(launches),
            "alt_keyed": alt, "configs": extra, "clocks": clk.summary(),
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
