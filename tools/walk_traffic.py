"""Records the ncu counters of one walk-kernel launch in profiles/walk_traffic.json,
keyed by workload/rng and by the sha of the walk kernel's source, so bench.py
only reports them for the kernel it actually timed.

    python tools/walk_traffic.py REPORT.ncu-rep WORKLOAD RNG [--rows-fraction F]

REPORT: `ncu --set full -k regex:k_walk -s 2 -c 1 ...` of tools/profile_walk.py
on WORKLOAD.  --rows-fraction scales per-launch bytes to the full workload when
the capture built only a leading fraction of the rows.
"""
import argparse
import csv
import io
import json
import os
import subprocess
import sys

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, REPO)


def raw(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    h, units, v = rows[0], rows[1], rows[2]
    return {name: (v[i], units[i]) for i, name in enumerate(h)}


def num(d, key, scale_units=True):
    val, unit = d[key]
    x = float(val.replace(",", ""))
    if scale_units:
        x *= {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12, "nsecond": 1e-9, "ns": 1e-9,
              "usecond": 1e-6, "us": 1e-6, "msecond": 1e-3, "ms": 1e-3, "second": 1.0, "s": 1.0}.get(unit, 1.0)
    return x


def main():
    p = argparse.ArgumentParser()
    p.add_argument("report")
    p.add_argument("workload")
    p.add_argument("rng")
    p.add_argument("--rows-fraction", type=float, default=1.0)
    a = p.parse_args()
    import bench
    d = raw(a.report)
    f = a.rows_fraction
    dram = (num(d, "dram__bytes_read.sum") + num(d, "dram__bytes_write.sum")) / f
    l2 = num(d, "lts__t_sectors.sum", False) * 32 / f  # 32-byte sectors through L2
    t = num(d, "gpu__time_duration.sum")
    entry = {
        "walk_source_sha16": bench.walk_source_sha16(),
        "dram_bytes_per_launch": dram, "l2_bytes_per_launch": l2,
        "issue_active": num(d, "smsp__issue_active.avg.pct_of_peak_sustained_active", False) / 100.0,
        "ipc": num(d, "sm__inst_executed.avg.per_cycle_active", False),
        "warp_instructions_per_launch": num(d, "smsp__inst_executed.sum", False) / f,
        "l1_hit_rate": num(d, "l1tex__t_sector_hit_rate.pct", False) / 100.0,
        "l2_hit_rate": num(d, "lts__t_sector_hit_rate.pct", False) / 100.0,
        "kernel_ms_ncu": t * 1e3,
        "captured": os.path.basename(a.report) + (f" (rows fraction {f})" if f != 1.0 else ""),
    }
    path = os.path.join(REPO, "profiles", "walk_traffic.json")
    try:
        with open(path) as fh:
            data = json.load(fh)
    except (OSError, ValueError):
        data = {}
    if "entries" not in data:
        data = {"entries": {}}
    data["entries"][f"{a.workload}/{a.rng}"] = entry
    with open(path, "w") as fh:
        json.dump(data, fh, indent=1, sort_keys=True)
    print(json.dumps(entry, indent=1))


if __name__ == "__main__":
    main()
