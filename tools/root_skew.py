#!/usr/bin/env python
"""Work skew across root edges: instrumented-kernel stats per chunk of roots (GPU)."""
import os, sys
import numpy as np
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import synth
import paper_2507_14813_b200 as M
cfg = synth.CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "C2"]
chunk = int(sys.argv[2]) if len(sys.argv) > 2 else 256
src, dst, t, V = cfg.graph()
g = M.Graph(src, dst, t, V, device=0)
tree = M.MGTree(cfg.group(), cfg.delta)
E = g.n_edges
ent, nod = [], []
for a in range(0, E, chunk):
    st = M.comine_stats(g, tree, (a, min(E, a + chunk)))
    ent.append(st["entries"]); nod.append(st["nodes"])
ent = np.array(ent, float); nod = np.array(nod, float)
print(cfg.name, "chunks", len(ent), "chunk", chunk)
print("entries/chunk: mean %.0f p50 %.0f p99 %.0f max %.0f  (max/mean %.1f)" % (ent.mean(), np.median(ent), np.percentile(ent, 99), ent.max(), ent.max() / ent.mean()))
print("nodes/chunk: mean %.0f max %.0f" % (nod.mean(), nod.max()))
o = np.argsort(-ent)[:10]
print("top chunks (start, entries, nodes):", [(int(i) * chunk, int(ent[i]), int(nod[i])) for i in o])
# single-root resolution inside the heaviest chunk
a = int(o[0]) * chunk
per = []
for r in range(a, min(E, a + chunk)):
    per.append(M.comine_stats(g, tree, (r, r + 1))["entries"])
per = np.array(per)
print("heaviest chunk roots: max entries %d, top5 %s, sum %d" % (per.max(), sorted(per)[-5:], per.sum()))
