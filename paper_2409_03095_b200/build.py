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
SOURCES = ["engine.cu", "tables.cu", "walk.cu", "assemble.cu", "solver.cu", "recovery.cu", "scatter.cu", "mmio.cpp",
           "hostio.cpp", "rowops.cu"]
HEADERS = ["common.cuh", "kernels.cuh", "hostio.h"]

NVCC_FLAGS = [
    "-gencode", "arch=compute_100a,code=sm_100a",
    "-O3", "-lineinfo", "-fmad=false", "-std=c++17",
    "-Xcompiler", "-fPIC,-O2,-pthread",
    "-I", os.path.join(REPO, "include"),
]


def _deps():
    return [os.path.join(CSRC, f) for f in HEADERS] + [os.path.join(REPO, "include", "mcmi.h")]


def _stale() -> bool:
    if not os.path.exists(LIB):
        return True
    t = os.path.getmtime(LIB)
    deps = [os.path.join(CSRC, f) for f in SOURCES] + _deps()
    return any(os.path.getmtime(d) > t for d in deps)


def build(force: bool = False, verbose: bool = False, out: str = LIB, defines=()) -> str:
    """Builds `out` (default: the in-tree library): one nvcc per source file in
    parallel (objects cached next to the library, rebuilt when the source or
    any header is newer), then one link.  `defines` (-D macros) and a different
    `out` are for A/B kernel experiments only (tools/)."""
    if out == LIB and not defines and not force and not _stale():
        return LIB
    from concurrent.futures import ThreadPoolExecutor
    os.makedirs(os.path.dirname(out), exist_ok=True)
    nvcc = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
    tag = "" if (out == LIB and not defines) else "_" + str(abs(hash((out, tuple(defines)))))
    objdir = os.path.join(os.path.dirname(out), "obj" + tag)
    os.makedirs(objdir, exist_ok=True)
    hdr_t = max(os.path.getmtime(d) for d in _deps())
    extra = [f"-D{d}" for d in defines] + (["-Xptxas", "-v"] if verbose else [])

    def compile_one(src):
        obj = os.path.join(objdir, os.path.splitext(src)[0] + ".o")
        path = os.path.join(CSRC, src)
        if (not force and os.path.exists(obj) and os.path.getmtime(obj) >= max(os.path.getmtime(path), hdr_t)
                and not defines):
            return obj
        subprocess.run([nvcc, *NVCC_FLAGS, *extra, "-c", "-o", obj + ".tmp", path], check=True, cwd=CSRC)
        os.replace(obj + ".tmp", obj)
        return obj

    with ThreadPoolExecutor(max_workers=len(SOURCES)) as ex:
        objs = list(ex.map(compile_one, SOURCES))
    subprocess.run([nvcc, "-gencode", "arch=compute_100a,code=sm_100a", "-shared", "-Xcompiler", "-pthread",
                    "-o", out + ".tmp", *objs], check=True, cwd=CSRC)
    os.replace(out + ".tmp", out)
    return out


if __name__ == "__main__":
    args = [a for a in sys.argv[1:] if not a.startswith("-")]
    defs = [a[2:] for a in sys.argv[1:] if a.startswith("-D")]
    print(build(force="--force" in sys.argv, verbose="-v" in sys.argv, out=os.path.abspath(args[0]) if args else LIB,
                defines=defs))
