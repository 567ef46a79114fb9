"""Selected metrics of every launch in an `ncu -i X.ncu-rep --page raw --csv` dump
(one line per launch), for the summaries kept under profiles/.

usage: python scripts/ncu_raw_summary.py gpurun_out/NAME.raw.csv [more.csv ...]"""
import csv
import sys

KEYS = ["gpu__time_duration.sum", "launch__grid_size", "launch__block_size", "launch__registers_per_thread",
        "launch__occupancy_limit_registers", "launch__occupancy_limit_shared_mem",
        "sm__warps_active.avg.pct_of_peak_sustained_active", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
        "sm__pipe_tensor_subpipe_dmma_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active",
        "smsp__issue_active.avg.pct_of_peak_sustained_active",
        "dram__bytes_read.sum", "dram__bytes_write.sum", "dram__throughput.avg.pct_of_peak_sustained_elapsed",
        "lts__t_sector_hit_rate.pct", "l1tex__t_sector_hit_rate.pct",
        "smsp__average_warps_issue_stalled_barrier_per_issue_active.ratio",
        "smsp__average_warps_issue_stalled_long_scoreboard_per_issue_active.ratio",
        "smsp__average_warps_issue_stalled_membar_per_issue_active.ratio",
        "smsp__average_warps_issue_stalled_sleeping_per_issue_active.ratio"]
for path in sys.argv[1:]:
    rows = list(csv.reader(open(path)))
    hdr = next(r for r in rows if r and r[0] == "ID")
    units = rows[rows.index(hdr) + 1]
    idx = {h: i for i, h in enumerate(hdr)}
    print("#", path)
    for r in rows[rows.index(hdr) + 2:]:
        if len(r) != len(hdr):
            continue
        name = r[idx["Kernel Name"]].split("(")[0].replace("h2g::", "")
        vals = ["%s=%s%s" % (k, r[idx[k]], (" " + units[idx[k]]) if units[idx[k]] else "") for k in KEYS if k in idx]
        print(name, "|", ", ".join(vals))
