"""Summaries of the c3 `ncu --set full` capture of the wall-normal launches
(tools/profile_c3.sh step 3): details page -> {launch: {metric: value}},
raw page -> selected per-launch metrics.
  python tools/wall_capture_summary.py gpurun_out/c3_wall_full_details.csv gpurun_out/c3_wall_full_raw.csv profiles/r02"""
import csv
import json
import sys

details, raw, outdir = sys.argv[1:4]
per = {}
with open(details, newline="") as f:
    rows = [r for r in csv.reader(f) if len(r) > 5]
hdr = rows[0]
ix = {n: hdr.index(n) for n in ("ID", "Kernel Name", "Metric Name", "Metric Unit", "Metric Value")}
for r in rows[1:]:
    key = f"{r[ix['ID']]} {r[ix['Kernel Name']][:90]}"
    per.setdefault(key, {})[r[ix["Metric Name"]]] = f"{r[ix['Metric Value']]} {r[ix['Metric Unit']]}"
json.dump(per, open(f"{outdir}/c3_wall_ncu_full_details.json", "w"), indent=1)

want = ("dram__bytes_read.sum", "dram__bytes_write.sum", "gpu__time_duration.sum", "launch__registers_per_thread",
        "launch__occupancy_limit", "sm__warps_active.avg.pct_of_peak_sustained_active", "smsp__inst_executed_pipe_fp64",
        "sm__inst_executed_pipe_fp64", "sm__pipe_fp64_cycles_active", "l1tex__data_bank_conflicts_pipe_lsu",
        "smsp__average_warps_issue_stalled", "launch__shared_mem_per_block", "sm__throughput", "l1tex__throughput")
with open(raw, newline="") as f:
    rows = [r for r in csv.reader(f) if len(r) > 5]
hdr, units = rows[0], rows[1]
sel = []
for r in rows[2:]:
    d = {"kernel": r[hdr.index("Kernel Name")][:90]}
    for i, n in enumerate(hdr):
        if any(n.startswith(w) for w in want):
            d[f"{n} [{units[i]}]" if units[i] else n] = r[i]
    sel.append(d)
json.dump(sel, open(f"{outdir}/c3_wall_ncu_full_raw_selected.json", "w"), indent=1)
print(len(per), "launches (details),", len(sel), "launches (raw)")
