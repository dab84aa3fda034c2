"""Builds the sm_100a CUDA library (paper_2409_03095_b200/lib/libmcmi.so) in-tree.

nvcc cross-compiles for B200 without a GPU.  -fmad=false keeps every f64
expression un-contracted so results are bit-identical to the reference's
x86-64 build; -lineinfo maps ncu's source page back to csrc/.
"""
from __future__ import annotations

import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
REPO = os.path.dirname(HERE)
CSRC = os.path.join(HERE, "csrc")
LIB_DIR = os.path.join(HERE, "lib")
LIB = os.path.join(LIB_DIR, "libmcmi.so")
SOURCES = ["engine.cu", "tables.cu", "walk.cu", "assemble.cu", "solver.cu", "recovery.cu", "scatter.cu", "mmio.cpp"]
HEADERS = ["common.cuh", "kernels.cuh"]

NVCC_FLAGS = [
    "-gencode", "arch=compute_100a,code=sm_100a",
    "-O3", "-lineinfo", "-fmad=false", "-std=c++17",
    "-Xcompiler", "-fPIC,-O2,-pthread", "-shared",
    "-I", os.path.join(REPO, "include"),
]


def _stale() -> bool:
    if not os.path.exists(LIB):
        return True
    t = os.path.getmtime(LIB)
    deps = [os.path.join(CSRC, f) for f in SOURCES + HEADERS] + [os.path.join(REPO, "include", "mcmi.h")]
    return any(os.path.getmtime(d) > t for d in deps)


def build(force: bool = False, verbose: bool = False, out: str = LIB, defines=()) -> str:
    """Builds `out` (default: the in-tree library).  `defines` (-D macros) and a
    different `out` are for A/B kernel experiments only (tools/)."""
    if out == LIB and not defines and not force and not _stale():
        return LIB
    os.makedirs(os.path.dirname(out), exist_ok=True)
    nvcc = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
    cmd = [nvcc, *NVCC_FLAGS] + [f"-D{d}" for d in defines]
    if verbose:
        cmd += ["-Xptxas", "-v"]
    cmd += ["-o", out + ".tmp"] + [os.path.join(CSRC, f) for f in SOURCES]
    subprocess.run(cmd, check=True, cwd=CSRC)
    os.replace(out + ".tmp", out)
    return out


if __name__ == "__main__":
    args = [a for a in sys.argv[1:] if not a.startswith("-")]
    defs = [a[2:] for a in sys.argv[1:] if a.startswith("-D")]
    print(build(force="--force" in sys.argv, verbose="-v" in sys.argv, out=os.path.abspath(args[0]) if args else LIB,
                defines=defs))
