#!/usr/bin/env python
"""Round / occupancy counters of the warp-synchronous depth-first kernel (wdfs.cuh) on a config:
MAYURA_WDFS_STATS=1 routes mayura_comine_stats through the instrumented wdfs kernel; with
MAYURA_KERNEL=warp (no breadth-first level) every counter is the warp kernel's own.

    MAYURA_KERNEL=warp python tools/wdfs_stats.py C4
"""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
os.environ["MAYURA_WDFS_STATS"] = "1"
os.environ.setdefault("MAYURA_KERNEL", "warp")
import synth  # noqa: E402
import paper_2507_14813_b200 as M  # noqa: E402

cfg = synth.CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "C4"]
src, dst, t, V = cfg.graph()
g = M.Graph(src, dst, t, V, device=0)
tree = M.MGTree(cfg.group(), cfg.delta)
st = M.comine_stats(g, tree)
names = {"roots": "items taken", "nodes": "inner hits (child partial matches)", "windows": "pieces pushed",
         "entries": "valid window entries", "probes": "lanes given an entry (sum T)", "batches": "rounds",
         "matches": "completions", "offloads": "spills", "contexts": "reloads"}
out = {names.get(k, k): v for k, v in st.items() if k != "bytes_alg"}
r = max(1, st["batches"])
out["lanes per round"] = st["probes"] / r
out["valid entries per round"] = st["entries"] / r
out["kernel_form"] = M.mayura_kernel_form(g.handle)
out["counts_equal_comine"] = st["matches"] == sum(M.comine(g, tree))
print(json.dumps({"config": cfg.name, "wdfs_stats": out}))
