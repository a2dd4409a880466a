import os, sys
sys.path.insert(0, os.getcwd())
import synth, oracle, numpy as np
import paper_2507_14813_b200 as M
os.environ["MAYURA_KERNEL"] = "warp"
for seed in range(4):
    src, dst, t, V = synth.random_graph(90 + seed, 6, 6000, 3000, 0.01)
    motifs = synth.group(synth.GROUP_C4)
    g = M.Graph(src, dst, t, V, device=0); tree = M.MGTree(motifs, 40)
    got = M.comine(g, tree); exp = oracle.backtrack(src, dst, t, V, motifs, 40)
    print(seed, got == exp, flush=True)
