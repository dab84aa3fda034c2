"""A/B kernel experiments.

    python tools/ab.py build NAME [SRC_DIR] [-DMACRO ...]
        builds tools/_build/NAME/libmcmi.so from SRC_DIR (a copy of csrc/ with
        the variant's edits; default: the in-tree csrc/)
    python tools/ab.py report LOG
        tabulates the best walk-kernel time per (config, rng) and variant from
        a log of `echo "== NAME"; MCMI_LIB_PATH=... python tools/sweep.py ...`

On the GPU box:
    for v in base var base var; do export MCMI_LIB_PATH=tools/_build/$v/libmcmi.so;
        echo "== $v"; python tools/sweep.py c2_sym27_1p3m c3_lap3d_100; done > gpurun_out/ab.log
"""
import collections
import json
import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
REPO = os.path.dirname(HERE)
sys.path.insert(0, REPO)


def build(name, src=None, defines=()):
    from paper_2409_03095_b200 import build as B
    src = os.path.abspath(src or B.CSRC)
    out = os.path.join(HERE, "_build", name, "libmcmi.so")
    os.makedirs(os.path.dirname(out), exist_ok=True)
    nvcc = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
    cmd = [nvcc, *B.NVCC_FLAGS, "-shared", *[f"-D{d}" for d in defines], "-o", out]
    cmd += [os.path.join(src, f) for f in B.SOURCES if os.path.exists(os.path.join(src, f))]
    subprocess.run(cmd, check=True, cwd=src)
    print(out)


def report(log):
    res = collections.defaultdict(lambda: collections.defaultdict(list))
    v = None
    for line in open(log):
        if line.startswith("=="):
            v = line.split()[1]
            continue
        try:
            d = json.loads(line)
        except ValueError:
            continue
        res[(d["config"], d["rng"])][v].append(d["ms_walk_kernel"])
    for (cfg, rng), per in res.items():
        print(f"{cfg:22s} {rng:9s} " + "  ".join(f"{k}:{min(x):9.3f}" for k, x in per.items()))


if __name__ == "__main__":
    if sys.argv[1] == "build":
        rest = sys.argv[3:]
        src = next((a for a in rest if not a.startswith("-D")), None)
        build(sys.argv[2], src, [a[2:] for a in rest if a.startswith("-D")])
    else:
        report(sys.argv[2])
