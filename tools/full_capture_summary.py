"""Selected metrics of an ncu --set full capture of the streaming solves
(ncu -i ... --page raw --csv) -> profiles/r01_ncu_full_stream_c4.csv, and the
DRAM bytes per unknown of each -> profiles/traffic_c4.json (read by bench.py
for roofline.traffic).

    python tools/full_capture_summary.py gpurun_out/stream_full_raw.csv
"""

import csv
import json
import sys

METRICS = [
    "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
    "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
    "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
    "smsp__issue_active.avg.pct_of_peak_sustained_active", "sm__warps_active.avg.per_cycle_active",
    "launch__registers_per_thread", "launch__grid_size", "launch__block_size",
    "launch__shared_mem_per_block_dynamic", "lts__t_sector_hit_rate.pct", "smsp__inst_executed.sum",
    "smsp__average_warps_issue_stalled_wait_per_issue_active.ratio",
    "smsp__average_warps_issue_stalled_long_scoreboard_per_issue_active.ratio",
    "smsp__average_warps_issue_stalled_short_scoreboard_per_issue_active.ratio",
    "smsp__average_warps_issue_stalled_math_pipe_throttle_per_issue_active.ratio",
    "smsp__average_warps_issue_stalled_not_selected_per_issue_active.ratio",
    "smsp__average_warps_issue_stalled_dispatch_stall_per_issue_active.ratio",
]
SCALE = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12}
# unknowns per full config-4 launch (n_modes x 2048 x 1025 systems)
UNKNOWNS = {"helm": 1023 * 2048 * 1025, "bih": 1021 * 2048 * 1025}


def main(path, out_csv="profiles/r01_ncu_full_stream_c4.csv", out_json="profiles/traffic_c4.json"):
    rows = list(csv.reader(open(path)))
    hdr, units = rows[0], rows[1]
    idx = {h: i for i, h in enumerate(hdr)}
    cols = [m for m in METRICS if m in idx]
    traffic = {"config": "c4 full launches (2048 x 1025 = 2,099,200 systems; biharmonic on (m, -m) pairs)"}
    with open(out_csv, "w", newline="") as f:
        w = csv.writer(f)
        w.writerow(["kernel"] + [f"{m} [{units[idx[m]]}]" for m in cols])
        for r in rows[2:]:
            name = r[idx["Kernel Name"]]
            w.writerow([name] + [r[idx[m]] for m in cols])
            op = "helmholtz" if "helm" in name else "biharmonic"
            unk = UNKNOWNS["helm" if op == "helmholtz" else "bih"]
            rd = float(r[idx["dram__bytes_read.sum"]].replace(",", "")) * SCALE[units[idx["dram__bytes_read.sum"]]]
            wr = float(r[idx["dram__bytes_write.sum"]].replace(",", "")) * SCALE[units[idx["dram__bytes_write.sum"]]]
            traffic[op] = {"kernel": name, "dram_read_bytes": rd, "dram_write_bytes": wr, "unknowns": unk,
                           "bytes_per_unknown": (rd + wr) / unk, "read_per_unknown": rd / unk,
                           "write_per_unknown": wr / unk,
                           "time_ms": float(r[idx["gpu__time_duration.sum"]].replace(",", "")),
                           "source": "ncu --set full, " + out_csv}
    json.dump(traffic, open(out_json, "w"), indent=1)
    for op in ("helmholtz", "biharmonic"):
        if op in traffic:
            t = traffic[op]
            print(op, f"{t['bytes_per_unknown']:.2f} B/unknown, {t['time_ms']:.3f} ms")


if __name__ == "__main__":
    main(*sys.argv[1:])
