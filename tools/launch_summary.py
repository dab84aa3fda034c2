"""Summarises an ncu launch list (csv from `ncu --metrics gpu__time_duration.sum,
dram__bytes_read.sum,dram__bytes_write.sum,lts__t_bytes.sum --csv`): one line
per launch (ms, DRAM MB, L2 MB) and the time share per kernel.

    python tools/launch_summary.py gpurun_out/launches.csv "header comment" > profiles/..._summary.txt
    python tools/launch_summary.py gpurun_out/launches.csv --traffic KEY  # walk_traffic.json entry
"""
import collections
import csv
import io
import json
import sys


def load(path):
    text = open(path).read()
    start = text.index('"ID"')
    rows = list(csv.DictReader(io.StringIO(text[start:])))
    launches = collections.OrderedDict()
    for r in rows:
        lid = int(r["ID"])
        name = r["Kernel Name"]
        for junk in ("void ", "mcmi::", "(anonymous namespace)::", "<unnamed>::", "unnamed>::"):
            name = name.replace(junk, "")
        d = launches.setdefault(lid, {"kernel": name})
        v = float(r["Metric Value"].replace(",", ""))
        unit = r["Metric Unit"]
        if r["Metric Name"] == "gpu__time_duration.sum":
            d["ms"] = v / 1e6 if unit in ("ns", "nsecond") else v / 1e3 if unit in ("us", "usecond") else v
        else:
            scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12, "KB": 1e3, "MB": 1e6,
                     "GB": 1e9, "TB": 1e12}.get(unit, 1)
            d[r["Metric Name"]] = v * scale
    return launches


def main():
    path = sys.argv[1]
    L = load(path)
    if len(sys.argv) > 3 and sys.argv[2] == "--traffic":
        walks = [d for d in L.values() if d["kernel"].startswith("k_walk<0, 6, 0, 0>")]
        main_walk = max(walks, key=lambda d: d["ms"])
        print(json.dumps({sys.argv[3]: {
            "dram_bytes_per_launch": main_walk["dram__bytes_read.sum"] + main_walk["dram__bytes_write.sum"],
            "lts_bytes_per_launch": main_walk["lts__t_bytes.sum"],
            "kernel_ms_cold": main_walk["ms"],
            "source": f"{path} (ncu --metrics ... bench.py --steps 2 --warmup 1), k_walk<0,6,0,0>"}}, indent=1))
        return
    if len(sys.argv) > 2:
        for line in sys.argv[2].split("\\n"):
            print("# " + line)
    print(f"{'id':>3} {'kernel':50s} {'ms':>9} {'dram MB':>9} {'L2 MB':>10}")
    share = collections.Counter()
    for lid, d in L.items():
        dram = (d.get("dram__bytes_read.sum", 0) + d.get("dram__bytes_write.sum", 0)) / 1e6
        print(f"{lid:3d} {d['kernel'][:50]:50s} {d['ms']:9.3f} {dram:9.1f} {d.get('lts__t_bytes.sum', 0) / 1e6:10.1f}")
        share[d["kernel"].split("(")[0]] += d["ms"]
    tot = sum(share.values())
    print(f"total {tot:.3f} ms; share by kernel:")
    for k, v in share.most_common():
        print(f"   {k[:30]:30s} {100 * v / tot:6.2f}%")


if __name__ == "__main__":
    main()
