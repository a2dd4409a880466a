#!/usr/bin/env python
"""Per-rank device time of an 8-way root partition (order shuffled), and of equal-count splits."""
import os, sys, time
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch
import synth
import paper_2507_14813_b200 as M
cfg = synth.CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "C3"]
src, dst, t, V = cfg.graph()
g = M.Graph(src, dst, t, V, device=0)
tree = M.MGTree(cfg.group(), cfg.delta)
E = g.n_edges
counts = torch.zeros(tree.n_motifs, dtype=torch.int64, device="cuda")
sp = torch.cuda.current_stream().cuda_stream
def tm(a, b, reps=3):
    M.mayura_comine(g.handle, tree.handle, a, b, sp, counts)
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(reps)]
    for x, y in ev:
        x.record(); M.mayura_comine(g.handle, tree.handle, a, b, sp, counts); y.record()
    torch.cuda.synchronize()
    return sorted(x.elapsed_time(y) for x, y in ev)[reps // 2]
b = g.partition(cfg.delta, 8)
print("bounds", b)
for order in (list(range(8)), list(range(7, -1, -1))):
    print("partition order", order, ["%.2f" % tm(b[r], b[r + 1]) for r in order])
eq = [E * r // 8 for r in range(9)]
print("equal-count", ["%.2f" % tm(eq[r], eq[r + 1]) for r in range(8)])
st = [M.comine_stats(g, tree, (b[r], b[r + 1]))["entries"] for r in range(8)]
print("entries per rank", st)
for r in range(8):
    print("rank", r, M.comine_stats(g, tree, (b[r], b[r + 1])))
