"""Resumable preconditioner sweep, mirroring the
reference CLI's `mcspai bench --spec SPEC --out CSV` (tools/mcspai.cpp:315-515)
with both halves of every cell on the B200: the preconditioner build
(mcmi_engine_build) and the left-preconditioned Krylov solve it feeds
(mcmi_solve_device, §8f rank 1).

    python -m paper_2409_03095_b200.sweep --spec SPEC --out CSV [--device D]

Same spec language (key = value lines, '#' comments; matrix, epsilons,
drop_fractions, retain_ks, delta, alpha, mode, drop_mode, seed, reps, solver,
tol, max_iters, restart), same CSV header and row format (precision 17), same
resumption (a cell whose key is already in the CSV is skipped), same grid order
(drop_fraction, epsilon, retain_k, rep; seed = spec.seed + rep), same
consolidated output sorted by (matrix, drop_fraction, epsilon, retain_k, seed,
solver), same exit status (1 if any cell failed).  Timings are wall-clock
milliseconds of the device work (synchronised), so they are not comparable
with the reference's CPU times; iterations agree with the reference solver up
to the rounding sensitivity documented in DESIGN.md §4.4.
"""
from __future__ import annotations

import argparse
import os
import sys
import time
from dataclasses import dataclass, field
from pathlib import Path
from typing import Callable

CSV_HEADER = ("matrix,n,nnz,method,epsilon,delta,alpha,drop_fraction,retain_k,seed,"
              "precond_wall_ms,solver,iterations,converged,final_rel_residual,"
              "solve_wall_ms,total_wall_ms")  # mcspai.cpp:37-40


def _g(x: float) -> str:
    """std::ostream << double with precision(17) (default floatfield): %.17g."""
    return "%.17g" % x


@dataclass
class CsvRow:  # mcspai.cpp:42-83
    matrix: str = ""
    n: int = 0
    nnz: int = 0
    method: str = ""  # "none" | "P" | "P-error"
    epsilon: float = 0.0
    delta: float = 0.0
    alpha: float = 0.0
    drop_fraction: float = 0.0
    retain_k: int = 0
    seed: int = 0
    precond_wall_ms: float = 0.0
    solver: str = ""
    iterations: int = 0
    converged: bool = False
    final_rel_residual: float = 0.0
    solve_wall_ms: float = 0.0
    total_wall_ms: float = 0.0

    def line(self) -> str:
        return ",".join([self.matrix, str(self.n), str(self.nnz), self.method, _g(self.epsilon), _g(self.delta),
                         _g(self.alpha), _g(self.drop_fraction), str(self.retain_k), str(self.seed),
                         _g(self.precond_wall_ms), self.solver, str(self.iterations),
                         "1" if self.converged else "0", _g(self.final_rel_residual), _g(self.solve_wall_ms),
                         _g(self.total_wall_ms)])

    def key(self) -> str:
        return "|".join([self.matrix, _g(self.epsilon), _g(self.delta), _g(self.alpha), _g(self.drop_fraction),
                         str(self.retain_k), str(self.seed), self.solver,
                         "none" if self.method == "none" else "P"])

    @staticmethod
    def parse(fields: list[str]) -> "CsvRow":  # mcspai.cpp:412-430
        f = fields
        return CsvRow(f[0], int(f[1]), int(f[2]), f[3], float(f[4]), float(f[5]), float(f[6]), float(f[7]),
                      int(f[8]), int(f[9]), float(f[10]), f[11], int(f[12]), f[13] == "1", float(f[14]),
                      float(f[15]), float(f[16]))


def split_csv_line(line: str) -> list[str]:
    """std::getline(ss, f, ',') splitting: a trailing empty field is dropped."""
    fields = line.split(",")
    if fields and fields[-1] == "":
        fields.pop()
    return fields


@dataclass
class BenchSpec:  # mcspai.cpp:315-330
    matrix: str = ""
    epsilons: list = field(default_factory=list)
    drop_fractions: list = field(default_factory=list)
    retain_ks: list = field(default_factory=list)
    delta: float = 0.0625
    alpha: float = 5.0
    mode: str = "sign"
    drop_mode: str = "range"
    seed: int = 0
    reps: int = 10
    solver: str = "gmres"
    tol: float = 1e-6
    max_iters: int = 30000
    restart: int = 50


class SpecError(RuntimeError):
    pass


def parse_bench_spec_text(text: str) -> BenchSpec:
    """parse_bench_spec (mcspai.cpp:332-395) over the spec text."""
    spec = BenchSpec()

    def to_list(s):
        return [t.strip(" \t") for t in s.split(",") if t.strip(" \t")]

    lines = text.split("\n")
    if lines and lines[-1] == "":
        lines.pop()
    for line_no, line in enumerate(lines, 1):
        if not line or line[0] == "#":
            continue
        if "=" not in line:
            raise SpecError(f"spec line {line_no}: expected key=value")
        key, value = line.split("=", 1)
        key, value = key.strip(" \t"), value.strip(" \t")
        if key == "matrix":
            spec.matrix = value
        elif key == "epsilons":
            spec.epsilons += [float(s) for s in to_list(value)]
        elif key == "drop_fractions":
            spec.drop_fractions += [float(s) for s in to_list(value)]
        elif key == "retain_ks":
            spec.retain_ks += [int(s) for s in to_list(value)]
        elif key == "delta":
            spec.delta = float(value)
        elif key == "alpha":
            spec.alpha = float(value)
        elif key == "mode":
            spec.mode = value
        elif key == "drop_mode":
            spec.drop_mode = value
        elif key == "seed":
            spec.seed = int(value)
        elif key == "reps":
            spec.reps = int(value)
        elif key == "solver":
            spec.solver = value
        elif key == "tol":
            spec.tol = float(value)
        elif key == "max_iters":
            spec.max_iters = int(value)
        elif key == "restart":
            spec.restart = int(value)
        else:
            raise SpecError(f"spec line {line_no}: unknown key '{key}'")
    if not spec.matrix:
        raise SpecError("spec: 'matrix' is required")
    if not spec.epsilons or not spec.drop_fractions or not spec.retain_ks:
        raise SpecError("spec: epsilons, drop_fractions and retain_ks must be non-empty")
    if spec.reps < 1:
        raise SpecError("spec: reps must be >= 1")
    return spec


def parse_bench_spec(path) -> BenchSpec:
    try:
        with open(path) as f:
            text = f.read()
    except OSError:
        raise SpecError(f"cannot open spec '{path}'") from None
    return parse_bench_spec_text(text)


def _mode(s):  # parse_mode / parse_drop_mode (mcspai.cpp:109-119)
    from .mcspai import AugmentationMode
    if s == "sign":
        return AugmentationMode.sign_aware
    if s == "plain":
        return AugmentationMode.plain
    raise SpecError("--mode must be 'sign' or 'plain'")


def _drop_mode(s):
    from .mcspai import DropMode
    if s == "range":
        return DropMode.value_range
    if s == "count":
        return DropMode.count_quantile
    raise SpecError("--drop-mode must be 'range' or 'count'")


# cell(b, cfg, solver_cfg) -> (precond_ms, iterations, converged, final_rel_residual, solve_ms, total_ms)
Cell = Callable


def gpu_cell(device: int = 0):
    """One sweep cell on the B200: device-resident build, then the GPU solve."""
    import torch

    from .engine import DeviceEngine
    from .solvers import solve_device
    eng = DeviceEngine(device)
    cache = {}

    def run(b, cfg, scfg):
        key = id(b)
        if key not in cache:
            cache.clear()
            cache[key] = DeviceEngine.upload(b, device)
        bt = cache[key]
        torch.cuda.synchronize(device)
        t0 = time.perf_counter()
        d = eng.build(b.n, *bt, cfg)
        mt = eng.to_tensors(d)[:3]
        torch.cuda.synchronize(device)
        t1 = time.perf_counter()
        _, rep = solve_device(b.n, bt, mt, None, scfg, device)
        torch.cuda.synchronize(device)
        t2 = time.perf_counter()
        return (1e3 * (t1 - t0), rep.iterations, rep.converged, rep.final_rel_residual, 1e3 * (t2 - t1),
                1e3 * (t2 - t0))

    return run


def run_bench(spec_path, out_path, cell: Cell | None = None, log=sys.stdout) -> int:
    """run_bench (mcspai.cpp:397-515).  Returns the exit status."""
    from .matrix_market import read_matrix_market_file
    from .mcspai import McConfig
    from .solvers import SolverConfig, SolverMethod
    spec = parse_bench_spec(spec_path)
    b = read_matrix_market_file(spec.matrix)
    stem = Path(spec.matrix).stem
    cell = cell or gpu_cell()

    rows: dict[str, CsvRow] = {}
    if os.path.exists(out_path):  # resumption
        with open(out_path) as f:
            f.readline()  # header
            for line in f.read().split("\n"):
                if not line:
                    continue
                fields = split_csv_line(line)
                if len(fields) < 17:
                    continue
                row = CsvRow.parse(fields)
                rows[row.key()] = row

    scfg = SolverConfig(method=SolverMethod.bicgstab if spec.solver == "bicgstab" else SolverMethod.gmres,
                        rel_tol=spec.tol, max_iters=spec.max_iters, restart=spec.restart)
    all_completed = True
    for drop in spec.drop_fractions:
        for eps in spec.epsilons:
            for k in spec.retain_ks:
                for rep in range(spec.reps):
                    cfg = McConfig(epsilon=eps, delta=spec.delta, alpha=spec.alpha, mode=_mode(spec.mode),
                                   drop_fraction=drop, drop_mode=_drop_mode(spec.drop_mode), retain_k=k,
                                   master_seed=(spec.seed + rep) % (1 << 64))
                    row = CsvRow(matrix=stem, n=b.n, nnz=b.nnz(), method="P", epsilon=eps, delta=spec.delta,
                                 alpha=spec.alpha, drop_fraction=drop, retain_k=k, seed=cfg.master_seed,
                                 solver=spec.solver)
                    if row.key() in rows:
                        continue  # resumable
                    try:
                        (row.precond_wall_ms, row.iterations, row.converged, row.final_rel_residual,
                         row.solve_wall_ms, row.total_wall_ms) = cell(b, cfg, scfg)
                    except Exception as e:  # noqa: BLE001 — a failed cell is recorded, as in the reference
                        print(f"bench cell failed: {e}", file=sys.stderr)
                        row.method = "P-error"
                        row.converged = False
                        all_completed = False
                    rows[row.key()] = row
                    print(f"bench: {row.line()}", file=log)

    ordered = sorted(rows.values(), key=lambda r: (r.matrix, r.drop_fraction, r.epsilon, r.retain_k, r.seed,
                                                   r.solver))
    try:
        with open(out_path, "w") as f:
            f.write(CSV_HEADER + "\n")
            for r in ordered:
                f.write(r.line() + "\n")
    except OSError:
        raise RuntimeError(f"cannot open '{out_path}'") from None
    return 0 if all_completed else 1


def main(argv=None) -> int:
    p = argparse.ArgumentParser(description=__doc__.split("\n\n")[0])
    p.add_argument("--spec", required=True)
    p.add_argument("--out", required=True)
    p.add_argument("--device", type=int, default=0)
    a = p.parse_args(argv)
    try:
        return run_bench(a.spec, a.out, gpu_cell(a.device))
    except (SpecError, RuntimeError, ValueError) as e:
        print(f"error: {e}", file=sys.stderr)
        return 2


if __name__ == "__main__":
    sys.exit(main())
