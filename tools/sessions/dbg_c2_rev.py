import os, sys
sys.path.insert(0, os.getcwd())
import numpy as np, synth
import paper_2507_14813_b200 as M
cfg = synth.CONFIGS["C2"]
src, dst, t, V = cfg.graph()
def tr(ms): return [[(v, u) for u, v in m] for m in ms]
def rv(ms): return [list(reversed(m)) for m in ms]
for name, (s, d, tt, mot) in {"base": (src, dst, t, cfg.group()), "time": (src, dst, -t, rv(cfg.group())),
                              "dir": (dst, src, t, tr(cfg.group()))}.items():
    g = M.Graph(s, d, tt, V, device=0); tree = M.MGTree(mot, cfg.delta)
    try:
        print(name, os.environ.get("MAYURA_KERNEL"), os.environ.get("MAYURA_DFS"), M.comine(g, tree), flush=True)
    except Exception as e:
        print(name, "ERR", e, flush=True); raise
