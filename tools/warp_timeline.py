#!/usr/bin/env python
"""Per-warp timeline of the instrumented lane kernel (debug aid; GPU needed).

    python tools/warp_timeline.py C2 [out.npy]
"""
import os
import sys
import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import synth  # noqa: E402
import paper_2507_14813_b200 as M  # noqa: E402

cfg = synth.CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "C2"]
path = "/tmp/mayura_warps.bin"
os.environ["MAYURA_DEBUG_WARPS"] = path
src, dst, t, V = cfg.graph()
g = M.Graph(src, dst, t, V, device=0)
tree = M.MGTree(cfg.group(), cfg.delta)
for _ in range(2):
    st = M.comine_stats(g, tree)
rec = np.fromfile(path, dtype=np.uint64).reshape(-1, 8)
rec = rec[rec[:, 1] > 0].astype(np.int64)
t0 = rec[:, 0].min()
start, end, iters, helps, roots, rdone, sm = (rec[:, 0] - t0, rec[:, 1] - t0, rec[:, 2], rec[:, 3], rec[:, 4],
                                              np.where(rec[:, 5] > 0, rec[:, 5] - t0, -1), rec[:, 6])
dur = end - start
print(cfg.name, "warps", len(rec), "kernel span us %.1f" % (end.max() / 1e3))
print("warp end us: p10 %.1f p50 %.1f p90 %.1f p99 %.1f max %.1f" % tuple(np.percentile(end, [10, 50, 90, 99, 100]) / 1e3))
print("roots-exhausted seen at us: min %.1f p50 %.1f max %.1f" % tuple(np.percentile(rdone[rdone >= 0], [0, 50, 100]) / 1e3))
print("iterations/warp: p50 %d p90 %d max %d; help batches p50 %d max %d; roots/warp p50 %d max %d" % (
    np.median(iters), np.percentile(iters, 90), iters.max(), np.median(helps), helps.max(), np.median(roots), roots.max()))
o = np.argsort(-end)[:12]
print("slowest warps: end_us iters helps roots roots_done_us sm  ns/iter")
for i in o:
    print("  %8.1f %7d %6d %5d %8.1f %4d %7.0f" % (end[i] / 1e3, iters[i], helps[i], roots[i], rdone[i] / 1e3, sm[i],
                                                 dur[i] / max(iters[i], 1)))
print("ns/iter overall median %.0f" % np.median(dur / np.maximum(iters, 1)))
if len(sys.argv) > 2:
    np.save(sys.argv[2], rec)
