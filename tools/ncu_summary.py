"""Summarise ncu launch lists (gpu__time_duration, dram bytes) into profiles/.

usage: python tools/ncu_summary.py <round-tag> gpurun_out/launches_cfg2.csv [more.csv ...]
Writes profiles/ncu_summary.json ({workload: {kernel: {...}}}, read by bench.py for
the `traffic` field) and prints a markdown table.  Workload = the csv name suffix.
"""
import csv
import json
import os
import re
import statistics
import sys

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def short(name):
    m = re.search(r"(scan2d_\w+?)(<|\()", name)
    return m.group(1) if m else name.split("(")[0][:60]


def load(path):
    per = {}
    for r in csv.DictReader(line for line in open(path) if not line.startswith("==")):
        k = short(r["Kernel Name"])
        per.setdefault(k, {}).setdefault(r["ID"], {})[r["Metric Name"]] = float(r["Metric Value"].replace(",", ""))
    out = {}
    for k, launches in per.items():
        ts = [v.get("gpu__time_duration.sum", 0.0) for v in launches.values()]
        rd = [v.get("dram__bytes_read.sum", 0.0) for v in launches.values()]
        wr = [v.get("dram__bytes_write.sum", 0.0) for v in launches.values()]
        out[k] = {"launches": len(ts), "time_ns_median": statistics.median(ts),
                  "dram_read_bytes": statistics.median(rd), "dram_write_bytes": statistics.median(wr),
                  "dram_bytes_per_launch": statistics.median([a + b for a, b in zip(rd, wr)])}
    return out


def main():
    tag, files = sys.argv[1], sys.argv[2:]
    dst = os.path.join(REPO, "profiles", "ncu_summary.json")
    try:
        summ = json.load(open(dst))
    except Exception:
        summ = {}
    for f in files:
        wl = os.path.basename(f).rsplit("_", 1)[-1].replace(".csv", "")
        summ[wl] = load(f)
        summ[wl]["_source"] = f"{tag}: ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none (cold, serialised)"
    os.makedirs(os.path.dirname(dst), exist_ok=True)
    json.dump(summ, open(dst, "w"), indent=1, sort_keys=True)
    for wl, ks in summ.items():
        print(f"\n{wl}\n| kernel | launches | median µs | DRAM read MB | DRAM write MB |\n|---|---|---|---|---|")
        for k, v in ks.items():
            if k.startswith("_"):
                continue
            print(f"| {k} | {v['launches']} | {v['time_ns_median']/1e3:.1f} | {v['dram_read_bytes']/1e6:.1f} | {v['dram_write_bytes']/1e6:.1f} |")


if __name__ == "__main__":
    main()
