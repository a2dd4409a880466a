#!/usr/bin/env python
"""e2e steps with a second graph resident (as in bench.py): per-phase times."""
import os, sys, time
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch
import synth
import paper_2507_14813_b200 as M
name = sys.argv[1] if len(sys.argv) > 1 else "C1"
cfg = synth.CONFIGS[name]
src, dst, t, V = cfg.graph()
g = M.Graph(src, dst, t, V, device=0)
tree = M.MGTree(cfg.group(), cfg.delta)
flush = torch.empty(512 << 18, dtype=torch.int32, device="cuda")
for i in range(3):
    M.comine(g, tree)
st = M.comine_stats(g, tree)
ps, pd, pt = (torch.from_numpy(a).pin_memory().numpy() for a in (src, dst, t))
for rep in range(5):
    torch.cuda.synchronize()
    t0 = time.perf_counter(); g2 = M.Graph(ps, pd, pt, V, device=0); t1 = time.perf_counter()
    c = M.comine(g2, tree); t2 = time.perf_counter()
    g2.close(); t3 = time.perf_counter()
    print("%s rep%d load %.2f ms  comine %.2f ms  free %.2f ms" % (name, rep, 1e3 * (t1 - t0), 1e3 * (t2 - t1), 1e3 * (t3 - t2)), flush=True)
