"""Buckets an ncu source page (walk kernel) into code regions by line range:
warp instructions executed and stall samples per region.

    python tools/ncu_regions.py gpurun_out/walk.ncu-rep walk.cu:REGION=a-b ...
Without regions: the default walk.cu regions (found by marker comments).
"""
import csv
import io
import re
import subprocess
import sys


def lines(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source=cuda,sass"],
                         capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    header, fname = None, None
    res = {}
    for r in rows:
        if len(r) == 2 and r[0] == "File Path":
            fname = r[1].split("/")[-1]
            continue
        if r and r[0] == "Line No":
            header = r
            continue
        if not header or len(r) < 8 or not r[0].isdigit():
            continue
        d = dict(zip(header[4:], r[4:]))
        try:
            s = int(d.get("Warp Stall Sampling (All Samples)", "0") or 0)
            ins = int(d.get("Instructions Executed", "0") or 0)
        except ValueError:
            continue
        res[(fname, int(r[0]))] = (s, ins, r[1])
    return res


def main():
    rep = sys.argv[1]
    regions = []
    for a in sys.argv[2:]:
        m = re.match(r"(.+?):(.+?)=(\d+)-(\d+)$", a)
        regions.append((m.group(1), m.group(2), int(m.group(3)), int(m.group(4))))
    L = lines(rep)
    tot_s = sum(v[0] for v in L.values())
    tot_i = sum(v[1] for v in L.values())
    print(f"total samples {tot_s} warp-instructions {tot_i:.4e}")
    used = set()
    for f, name, a, b in regions:
        s = sum(v[0] for k, v in L.items() if k[0] == f and a <= k[1] <= b)
        i = sum(v[1] for k, v in L.items() if k[0] == f and a <= k[1] <= b)
        used |= {k for k in L if k[0] == f and a <= k[1] <= b}
        print(f"{name:28s} {100 * s / tot_s:6.1f}% samples {100 * i / tot_i:6.1f}% instr  {i:.3e}")
    rest = [k for k in L if k not in used]
    by_file = {}
    for k in rest:
        by_file.setdefault(k[0], [0, 0])
        by_file[k[0]][0] += L[k][0]
        by_file[k[0]][1] += L[k][1]
    for f, (s, i) in sorted(by_file.items(), key=lambda x: -x[1][1]):
        print(f"(other) {f:20s} {100 * s / tot_s:6.1f}% samples {100 * i / tot_i:6.1f}% instr")


if __name__ == "__main__":
    main()
