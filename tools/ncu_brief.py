#!/usr/bin/env python
"""Key counters + top stall reasons of every kernel in an ncu report."""
import csv, io, subprocess, sys
out = subprocess.run(["ncu", "-i", sys.argv[1], "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
hdr, units = rows[0], rows[1]
for r in rows[2:]:
    d = dict(zip(hdr, r))
    print(d["Kernel Name"][:70])
    for k in ["gpu__time_duration.sum", "smsp__thread_inst_executed_per_inst_executed.ratio",
              "sm__warps_active.avg.pct_of_peak_sustained_active", "smsp__issue_active.avg.pct_of_peak_sustained_active",
              "smsp__inst_executed.sum", "l1tex__t_sector_hit_rate.pct", "lts__t_sector_hit_rate.pct",
              "dram__bytes_read.sum", "launch__grid_size", "launch__registers_per_thread",
              "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum", "l1tex__t_requests_pipe_lsu_mem_global_op_ld.sum",
              "l1tex__t_sectors_pipe_lsu_mem_global_op_ld.sum"]:
        if k in d:
            print("   %-58s %s %s" % (k, d[k], units[hdr.index(k)]))
    st = [(float(d[k]), k) for k in hdr if k.startswith("smsp__average_warps_issue_stalled")
          and k.endswith("per_issue_active.ratio") and d[k]]
    print("   stalls/issue:", ", ".join("%s %.2f" % (k.split("stalled_")[1].split("_per")[0], v) for v, k in sorted(st)[-8:][::-1]))
