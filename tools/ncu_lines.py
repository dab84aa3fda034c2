"""Summarises an ncu report's source page per CUDA source line:
stall samples, warp instructions executed, dominant stall reasons.

    python tools/ncu_lines.py gpurun_out/walk_c2.ncu-rep [top]
"""
import csv
import io
import subprocess
import sys


def main():
    rep = sys.argv[1]
    top = int(sys.argv[2]) if len(sys.argv) > 2 else 40
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source=cuda,sass"],
                         capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    header, fname, agg = None, None, []
    tot_s = tot_i = 0
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
        stalls = {k[6:]: int(v) for k, v in d.items() if k.startswith("stall_") and "Not Issued" not in k
                  and v.isdigit() and int(v) > 0}
        top3 = sorted(stalls.items(), key=lambda kv: -kv[1])[:3]
        agg.append((s, ins, f"{fname}:{r[0]}", r[1][:70], top3))
        tot_s += s
        tot_i += ins
    agg.sort(key=lambda x: -x[0])
    print(f"total samples {tot_s}  warp-instructions {tot_i:.3e}")
    for s, ins, loc, src, t3 in agg[:top]:
        print(f"{100*s/tot_s:5.1f}% {100*ins/max(tot_i,1):5.1f}%i {loc:18s} {src:70s} {t3}")


if __name__ == "__main__":
    main()
