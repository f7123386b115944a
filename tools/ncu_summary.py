"""Summarise an ncu --csv launch list (one row per kernel x metric) into a
per-kernel table: launches, mean / total gpu__time_duration, DRAM bytes per
launch.  Used to build the profiles/ summaries and profiles/traffic_c4.json.

    python tools/ncu_summary.py gpurun_out/launches.csv [--unknowns H=...,B=...] [--json out.json]
"""

import argparse
import csv
import json
from collections import OrderedDict, defaultdict

UNIT = {"byte": 1.0, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "ns": 1e-9, "us": 1e-6, "usecond": 1e-6,
        "msecond": 1e-3, "ms": 1e-3, "nsecond": 1e-9, "second": 1.0}


def load(path):
    rows = [r for r in csv.reader(open(path)) if len(r) > 5]
    hdr = rows[0]
    launches = OrderedDict()
    for r in rows[1:]:
        d = dict(zip(hdr, r))
        key = (d["ID"], d["Kernel Name"])
        v = float(d["Metric Value"].replace(",", "")) * UNIT.get(d.get("Metric Unit", ""), 1.0)
        launches.setdefault(key, {})[d["Metric Name"]] = v
    return launches


def short(name):
    return name.split("(")[0].replace("void ", "")


def summarise(launches):
    agg = defaultdict(lambda: {"launches": 0, "time_s": 0.0, "dram_read": 0.0, "dram_write": 0.0})
    for (_, name), m in launches.items():
        a = agg[short(name)]
        a["launches"] += 1
        a["time_s"] += m.get("gpu__time_duration.sum", 0.0)
        a["dram_read"] += m.get("dram__bytes_read.sum", 0.0)
        a["dram_write"] += m.get("dram__bytes_write.sum", 0.0)
    total = sum(a["time_s"] for a in agg.values()) or 1.0
    out = []
    for k, a in sorted(agg.items(), key=lambda kv: -kv[1]["time_s"]):
        n = a["launches"]
        out.append({"kernel": k, "launches": n, "mean_ms": 1e3 * a["time_s"] / n, "share": a["time_s"] / total,
                    "dram_bytes_per_launch": (a["dram_read"] + a["dram_write"]) / n,
                    "dram_read_per_launch": a["dram_read"] / n, "dram_write_per_launch": a["dram_write"] / n})
    return out


if __name__ == "__main__":
    ap = argparse.ArgumentParser()
    ap.add_argument("csv")
    ap.add_argument("--json")
    args = ap.parse_args()
    rows = summarise(load(args.csv))
    for r in rows:
        print(f"{r['kernel'][:70]:70s} n={r['launches']:4d} mean={r['mean_ms']:9.4f} ms share={r['share']:6.1%} "
              f"dram/launch={r['dram_bytes_per_launch'] / 1e9:8.3f} GB")
    if args.json:
        json.dump(rows, open(args.json, "w"), indent=1)
