"""Summarise an ncu report (full set) + a launch-list CSV into profiles/ (dev tool).

usage: python tools/ncu_summary.py <report.ncu-rep> <launches.csv> <out_prefix>
writes <out_prefix>_ncu.json (key metrics of the captured kernel), <out_prefix>_launches.csv
(per-launch durations) and <out_prefix>_top_lines.txt (stall samples per source line).
"""
import csv
import json
import subprocess
import sys

rep, launches, prefix = sys.argv[1], sys.argv[2], sys.argv[3]
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(raw.splitlines()))
hdr, units, vals = rows[0], rows[1], rows[2]
want = ["Kernel Name", "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "dram__throughput.avg.pct_of_peak_sustained_elapsed", "lts__t_sector_hit_rate.pct",
        "l1tex__t_sector_hit_rate.pct", "sm__warps_active.avg.pct_of_peak_sustained_active",
        "smsp__issue_active.avg.pct_of_peak_sustained_active", "smsp__inst_executed.sum",
        "launch__registers_per_thread", "launch__grid_size", "launch__block_size",
        "launch__shared_mem_per_block_dynamic", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
        "lts__t_sectors_op_read.sum", "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum",
        "smsp__average_warps_issue_stalled_long_scoreboard_per_issue_active.ratio",
        "smsp__average_warps_issue_stalled_no_instruction_per_issue_active.ratio",
        "smsp__average_warps_issue_stalled_wait_per_issue_active.ratio",
        "smsp__average_warps_issue_stalled_short_scoreboard_per_issue_active.ratio"]
out = {}
for w in want:
    if w in hdr:
        i = hdr.index(w)
        out[w] = {"value": vals[i], "unit": units[i]}
json.dump(out, open(prefix + "_ncu.json", "w"), indent=1)
# launch list: keep kernel name + duration
lines = [l for l in open(launches).read().splitlines() if not l.startswith("==")]
r = list(csv.reader(lines))
h = r[0]
ki, mi, vi = h.index("Kernel Name"), h.index("Metric Name"), h.index("Metric Value")
with open(prefix + "_launches.csv", "w", newline="") as f:
    wcsv = csv.writer(f)
    wcsv.writerow(["launch", "kernel", "gpu__time_duration"])
    for n, x in enumerate(r[1:]):
        if x[mi] == "gpu__time_duration.sum":
            wcsv.writerow([n, x[ki].split("(")[0], x[vi]])
top = subprocess.run([sys.executable, "tools/ncu_lines.py", rep, "40"], capture_output=True, text=True).stdout
open(prefix + "_top_lines.txt", "w").write(top)
print(json.dumps(out, indent=1))
