#!/usr/bin/env python
"""Break down the e2e path (load_graph on GPU, first comine, steady comine, free) per config."""
import os, sys, time
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch
import synth
import paper_2507_14813_b200 as M
for name in sys.argv[1:] or ["C1", "C2"]:
    cfg = synth.CONFIGS[name]
    src, dst, t, V = cfg.graph()
    ps, pd, pt = (torch.from_numpy(a).pin_memory().numpy() for a in (src, dst, t))
    tree = M.MGTree(cfg.group(), cfg.delta)
    for rep in range(3):
        torch.cuda.synchronize()
        t0 = time.perf_counter(); g = M.Graph(ps, pd, pt, V, device=0); t1 = time.perf_counter()
        c = M.comine(g, tree); t2 = time.perf_counter()
        c = M.comine(g, tree); t3 = time.perf_counter()
        g.close(); t4 = time.perf_counter()
        print("%s rep%d load %.2f ms  comine#1 %.2f ms  comine#2 %.2f ms  free %.2f ms" % (
            name, rep, 1e3 * (t1 - t0), 1e3 * (t2 - t1), 1e3 * (t3 - t2), 1e3 * (t4 - t3)))
