#!/usr/bin/env python
"""One C5 co-mining pass for an ncu capture (500 M edges, 8 motifs, the default warp form):
    ncu --set full -k regex:wdfs_kernel -s 1 -c 1 -o prof_c5 python tools/prof_c5.py
The first pass is the warm-up (skipped by -s 1), the second is captured."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import paper_2507_14813_b200 as M  # noqa: E402
import synth  # noqa: E402

cfg = synth.CONFIGS["C5"]
src, dst, t, V = cfg.graph()
g = M.Graph(src, dst, t, V, device=0)
tree = M.MGTree(cfg.group(), cfg.delta)
for _ in range(2):
    c = M.comine(g, tree)
torch.cuda.synchronize()
print("C5 counts", dict(zip(cfg.motifs, c)), M.mayura_kernel_form(g.handle))
