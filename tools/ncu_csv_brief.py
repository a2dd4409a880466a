#!/usr/bin/env python
"""Key counters + top stall reasons of every kernel in a `--page raw --csv` export."""
import csv
import sys

KEYS = ["gpu__time_duration.sum", "smsp__thread_inst_executed_per_inst_executed.ratio",
        "sm__warps_active.avg.pct_of_peak_sustained_active", "smsp__issue_active.avg.pct_of_peak_sustained_active",
        "smsp__inst_executed.sum", "l1tex__t_sector_hit_rate.pct", "lts__t_sector_hit_rate.pct",
        "dram__bytes_read.sum", "dram__bytes_write.sum", "launch__registers_per_thread",
        "launch__occupancy_limit_registers", "launch__occupancy_limit_shared_mem", "launch__grid_size",
        "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum", "smsp__warps_eligible.avg.per_cycle_active",
        "smsp__average_warp_latency_per_inst_issued.ratio"]
for path in sys.argv[1:]:
    rows = list(csv.reader(open(path)))
    hdr, units = rows[0], rows[1]
    for r in rows[2:]:
        d = dict(zip(hdr, r))
        print(d["Kernel Name"][:90])
        for k in KEYS:
            if k in d:
                print("   %-58s %s %s" % (k, d[k], units[hdr.index(k)]))
        st = [(float(d[k]), k) for k in hdr if k.startswith("smsp__average_warps_issue_stalled")
              and k.endswith("per_issue_active.ratio") and d[k]]
        print("   stalls/issue:", ", ".join("%s %.2f" % (k.split("stalled_")[1].split("_per")[0], v)
                                         for v, k in sorted(st)[-9:][::-1]))
