"""Per-phase wall times of the e2e path's graph build (MAYURA_TRACE=1: the library synchronises the
device after each phase and prints the time since the previous one) on one config, pinned host
arrays as bench.py's e2e leg passes them.  usage: MAYURA_TRACE=1 python tools/trace_build.py [C4] [reps]"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
os.environ.setdefault("MAYURA_TRACE", "1")
import torch  # noqa: E402

import paper_2507_14813_b200 as M  # noqa: E402
import synth  # noqa: E402

cfg = synth.CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "C4"]
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 3
src, dst, t, V = cfg.graph()
pin = [torch.from_numpy(a).pin_memory().numpy() for a in (src, dst, t)]
tree = M.MGTree(cfg.group(), cfg.delta)
for i in range(reps):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    g = M.Graph(*pin, V, device=0)
    t1 = time.perf_counter()
    c = M.comine(g, tree)
    t2 = time.perf_counter()
    g.close()
    print(f"rep {i}: load {1e3 * (t1 - t0):.2f} ms  comine {1e3 * (t2 - t1):.2f} ms  total {sum(c)}", file=sys.stderr,
          flush=True)
