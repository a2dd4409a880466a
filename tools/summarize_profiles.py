#!/usr/bin/env python
"""Summarise a GPU session's ncu captures + launch lists + bench lines into profiles/.

    python tools/summarize_profiles.py TAG [CONFIG ...]

Reads gpurun_out/{launches_C_TAG.csv, prof_C_TAG.ncu-rep, bench_C_TAG.json} and writes
profiles/TAG_C.md (launch shares, key ncu counters of the top kernel) and copies the
bench JSON line to profiles/bench_C_TAG.json.
"""
import collections
import csv
import io
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
OUT = os.path.join(ROOT, "gpurun_out")
PROF = os.path.join(ROOT, "profiles")

KEYS = [
    ("gpu__time_duration.sum", "duration"),
    ("dram__bytes_read.sum", "DRAM read"),
    ("dram__bytes_write.sum", "DRAM write"),
    ("dram__throughput.avg.pct_of_peak_sustained_elapsed", "DRAM throughput % of peak"),
    ("lts__t_sector_hit_rate.pct", "L2 hit rate"),
    ("lts__throughput.avg.pct_of_peak_sustained_elapsed", "L2 throughput % of peak"),
    ("l1tex__t_sector_hit_rate.pct", "L1 hit rate"),
    ("smsp__thread_inst_executed_per_inst_executed.ratio", "warp execution efficiency (threads/inst, ideal 32)"),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "achieved occupancy"),
    ("launch__registers_per_thread", "registers/thread"),
    ("launch__grid_size", "grid"),
    ("launch__block_size", "block"),
    ("smsp__issue_active.avg.pct_of_peak_sustained_active", "issue slots busy"),
    ("sm__throughput.avg.pct_of_peak_sustained_elapsed", "SM throughput % of peak"),
    ("smsp__inst_executed.sum", "warp instructions executed"),
    ("smsp__average_warps_issue_stalled_long_scoreboard_per_issue_active.ratio", "stall long_scoreboard / issue"),
    ("smsp__average_warps_issue_stalled_wait_per_issue_active.ratio", "stall wait / issue"),
    ("smsp__average_warps_issue_stalled_short_scoreboard_per_issue_active.ratio", "stall short_scoreboard / issue"),
    ("smsp__average_warps_issue_stalled_sleeping_per_issue_active.ratio", "stall sleeping / issue"),
    ("smsp__average_warps_issue_stalled_branch_resolving_per_issue_active.ratio", "stall branch_resolving / issue"),
]


def launches(path):
    rows = [r for r in csv.reader(open(path)) if len(r) > 10]
    hdr = rows[0]
    ki, vi, ui = hdr.index("Kernel Name"), hdr.index("Metric Value"), hdr.index("Metric Unit")
    agg = collections.OrderedDict()
    for r in rows[1:]:
        v = float(r[vi].replace(",", ""))
        v *= {"ns": 1e-6, "us": 1e-3, "usecond": 1e-3, "ms": 1.0, "msecond": 1.0}.get(r[ui], 1e-6)
        agg.setdefault(r[ki], []).append(v)
    return agg


def ncu_raw(rep):
    if rep.endswith(".csv"):  # exported on the box (`ncu -i … --page raw --csv`) when the report was too big
        out = open(rep).read()
    else:
        out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    if len(rows) < 3:
        return []
    hdr, units = rows[0], rows[1]
    return [(dict(zip(hdr, r)), dict(zip(hdr, units))) for r in rows[2:]]


def main():
    tag = sys.argv[1]
    cfgs = sys.argv[2:] or ["C1", "C2", "C3"]
    os.makedirs(PROF, exist_ok=True)
    for c in cfgs:
        lines = ["# %s %s — ncu evidence" % (tag, c), ""]
        bj = os.path.join(OUT, "bench_%s_%s.json" % (c, tag))
        if os.path.exists(bj):
            txt = [x for x in open(bj).read().splitlines() if x.strip().startswith("{")]
            if txt:
                d = json.loads(txt[-1])
                with open(os.path.join(PROF, "bench_%s_%s.json" % (c, tag)), "w") as f:
                    f.write(txt[-1] + "\n")
                r = d["roofline"]
                lines += ["## bench line (CUDA events, not under ncu)", "",
                          "- value: %.4g %s, ms_per_step %.4f, co-mining pass %.4f ms (form %s), window_end_kernel %s ms" % (
                              d["value"], d["unit"], d["ms_per_step"], r["kernel_ms"], r.get("kernel_form"),
                              r.get("window_end_kernel_ms")),
                          "- roofline: B_alg %.4g B/launch (%.1f B/root) → %.1f GB/s = %.4f of %.1f GB/s (%s)" % (
                              r["bytes_alg_per_launch"], r["bytes_alg_per_root"], r["achieved"], r["frac"],
                              r["peak"], r["peak_source"]),
                          "- parity vs oracle: %s; co-mined == independent: %s" % (
                              d.get("parity_vs_oracle"), (d.get("independent_gpu") or {}).get("counts_equal")),
                          "- independent per-motif GPU: %s ms → co-mining speedup %s" % (
                              (d.get("independent_gpu") or {}).get("ms_per_step"),
                              (d.get("independent_gpu") or {}).get("speedup_comine")),
                          "- e2e: %s" % json.dumps(d.get("e2e")),
                          "- cpu_baseline: %s" % json.dumps(d.get("cpu_baseline")),
                          "- clocks: %s" % json.dumps(d.get("clocks")), ""]
        lp = os.path.join(OUT, "launches_%s_%s.csv" % (c, tag))
        if os.path.exists(lp):
            agg = launches(lp)
            tot = sum(sum(v) for v in agg.values())
            lines += ["## launch list (ncu gpu__time_duration.sum, --clock-control none; cold-cache, serialised)", "",
                      "| kernel | launches | mean ms | share |", "|---|---|---|---|"]
            for k, v in agg.items():
                lines.append("| `%s` | %d | %.4f | %.1f%% |" % (k[:90], len(v), sum(v) / len(v), 100 * sum(v) / tot))
            lines.append("")
        rp = os.path.join(OUT, "prof_%s_%s.ncu-rep" % (c, tag))
        if not os.path.exists(rp):
            rp = os.path.join(OUT, "prof_%s_%s_raw.csv" % (c, tag))
        if os.path.exists(rp):
            for d, u in ncu_raw(rp):
                lines += ["## `ncu --set full` of `%s`" % d.get("Kernel Name", "?")[:100], "",
                          "| counter | value |", "|---|---|"]
                for k, name in KEYS:
                    if k in d:
                        lines.append("| %s (`%s`) | %s %s |" % (name, k, d[k], u.get(k, "")))
                lines.append("")
            # DRAM traffic of one co-mining pass for bench.py: the kernels bench.py's achieved
            # bandwidth covers (the events after mid_event: window_end_kernel excluded)
            def traffic(path):
                tot, names = 0.0, []
                for d, u in ncu_raw(path):
                    if "window_end_kernel" in d.get("Kernel Name", ""):
                        continue
                    for k in ("dram__bytes_read.sum", "dram__bytes_write.sum"):
                        v = float(d.get(k, "0").replace(",", "") or 0)
                        tot += v * {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(u.get(k, "byte"), 1)
                    names.append(d.get("Kernel Name", "?")[:80])
                return tot, names
            tot, names = traffic(rp)
            if names:
                tj = os.path.join(PROF, "ncu_traffic.json")
                allt = json.load(open(tj)) if os.path.exists(tj) else {}
                allt[c] = {"dram_bytes_per_launch": tot, "kernels": names, "tag": tag,
                           "note": "dram__bytes_read.sum + dram__bytes_write.sum summed over the co-mining kernels "
                                   "of one pass (window_end_kernel excluded, as in bench.py's achieved), "
                                   "ncu --set full, default --cache-control all (caches flushed before each replay)"}
                wp = os.path.join(OUT, "prof_%s_%s_warm_raw.csv" % (c, tag))
                if os.path.exists(wp):
                    allt[c]["dram_bytes_per_launch_warm"] = traffic(wp)[0]
                    allt[c]["note_warm"] = "the same capture with --cache-control none (caches kept across replays)"
                json.dump(allt, open(tj, "w"), indent=1)
        with open(os.path.join(PROF, "%s_%s.md" % (tag, c)), "w") as f:
            f.write("\n".join(lines) + "\n")
        print("wrote profiles/%s_%s.md" % (tag, c))


if __name__ == "__main__":
    main()
