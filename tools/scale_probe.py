#!/usr/bin/env python
"""Per-rank device time of the bench's N-way work-balanced root split, rank by rank on one GPU
(L2 flushed before each), for N = 1, 2, 4, 8: the kernel part of a strong-scaling run."""
import os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch
import synth
import paper_2507_14813_b200 as M
cfg = synth.CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "C2"]
src, dst, t, V = cfg.graph()
g = M.Graph(src, dst, t, V, device=0)
tree = M.MGTree(cfg.group(), cfg.delta)
counts = torch.zeros(tree.n_motifs, dtype=torch.int64, device="cuda")
s = torch.cuda.current_stream()
flush = torch.empty(128 << 20, dtype=torch.int32, device="cuda")
def tm(a, b, reps=5):
    out = []
    for i in range(reps + 2):
        flush.fill_(i)
        x, y = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        x.record(s); M.mayura_comine(g.handle, tree.handle, a, b, s.cuda_stream, counts); y.record(s)
        torch.cuda.synchronize()
        if i >= 2:
            out.append(x.elapsed_time(y))
    return sorted(out)[len(out) // 2]
base = None
for n in (1, 2, 4, 8):
    b = g.partition(cfg.delta, n)
    ts = [tm(b[r], b[r + 1]) for r in range(n)]
    base = base or max(ts)
    print("N=%d per-rank ms max %.4f min %.4f  speedup %.2f  eff %.2f" % (n, max(ts), min(ts), base / max(ts), base / max(ts) / n), flush=True)
