#!/usr/bin/env python
"""C5 (AML transaction-shaped, 10 M vertices / 500 M edges, 8 motifs) on one B200.

C5 is BASELINE.json's 8xB200 configuration.  With one GPU available, this runs the whole
graph on one GPU and, separately, each of the 8 work-balanced root ranges an 8-rank job
would give its ranks (`mayura_partition_roots`), so the per-rank device time of the 8-GPU
job (max over ranks; the all-reduce of 64 bytes is negligible) is measured rank by rank.
Parity: exact on sampled root ranges vs the oracle; sum over the 8 ranges == whole graph;
planted-pattern lower bounds (P7).

    python tools/run_c5.py [out.json] [--no-oracle]
"""
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import oracle  # noqa: E402
import paper_2507_14813_b200 as M  # noqa: E402
import synth  # noqa: E402
from tests.test_oracle_pins import _planted_lower_bounds  # noqa: E402


def timed(fn, reps):
    s = torch.cuda.current_stream()
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(reps)]
    out = None
    for a, b in ev:
        a.record(s)
        out = fn()
        b.record(s)
    torch.cuda.synchronize()
    return sorted(a.elapsed_time(b) for a, b in ev)[reps // 2], out


def main():
    args = [a for a in sys.argv[1:] if not a.startswith("--")]
    no_oracle = "--no-oracle" in sys.argv
    out_path = args[0] if args else "gpurun_out/c5.json"
    cfg = synth.CONFIGS["C5"]
    rec = {"config": cfg.name, "title": cfg.title}
    t0 = time.time()
    src, dst, t, V, planted = cfg.graph_planted()
    rec["gen_s"] = time.time() - t0
    t0 = time.time()
    g = M.Graph(src, dst, t, V, device=0)
    torch.cuda.synchronize()
    rec["load_s"] = time.time() - t0
    rec["device_bytes"] = g.device_bytes
    tree = M.MGTree(cfg.group(), cfg.delta)
    k = tree.n_motifs
    dev = torch.device("cuda", 0)
    counts = torch.zeros(k, dtype=torch.int64, device=dev)
    sp = torch.cuda.current_stream().cuda_stream
    E = g.n_edges

    def run(rb, re_, indep=False):
        fn = M.mayura_mine_independent if indep else M.mayura_comine
        return fn(g.handle, tree.handle, rb, re_, sp, counts)

    run(0, E)
    ms, _ = timed(lambda: run(0, E), 3)
    full = counts.cpu().tolist()
    rec["comine_ms_1gpu"] = ms
    rec["roots_per_s_1gpu"] = E / (ms * 1e-3)
    rec["counts"] = dict(zip(cfg.motifs, full))
    ims, _ = timed(lambda: run(0, E, True), 1)
    rec["independent_ms_1gpu"] = ims
    rec["independent_equal"] = counts.cpu().tolist() == full
    # the 8-rank job, rank by rank
    bounds = g.partition(cfg.delta, 8)
    per, tot = [], [0] * k
    for r in range(8):
        run(bounds[r], bounds[r + 1])
        m, _ = timed(lambda: run(bounds[r], bounds[r + 1]), 3)
        per.append(m)
        tot = [a + b for a, b in zip(tot, counts.cpu().tolist())]
    rec["rank_ms_8gpu"] = per
    rec["job_ms_8gpu"] = max(per)
    rec["roots_per_s_8gpu"] = E / (max(per) * 1e-3)
    rec["rank_balance_max_over_mean"] = max(per) / (sum(per) / 8)
    rec["ranks_sum_equals_full"] = tot == full
    # the hybrid form (breadth-first level + warp kernel) on the whole graph, for the form choice
    os.environ["MAYURA_KERNEL"] = "hybrid"
    run(0, E)
    hms, _ = timed(lambda: run(0, E), 3)
    rec["hybrid_ms_1gpu"] = hms
    rec["hybrid_equal"] = counts.cpu().tolist() == full
    del os.environ["MAYURA_KERNEL"]
    rec["kernel_form"] = M.mayura_kernel_form(g.handle)
    # parity on 8 evenly spaced 2,000-root ranges, one oracle graph build
    samples = []
    if not no_oracle:
        rngs = [(i * (E // 8) + E // 16, i * (E // 8) + E // 16 + 2000) for i in range(8)]
        per_o, build_s, mine_s = oracle.backtrack_ranges(src, dst, t, V, cfg.group(), cfg.delta, rngs)
        for rng, exp in zip(rngs, per_o):
            run(*rng)
            samples.append({"range": rng, "exact": counts.cpu().tolist() == exp})
        rec["oracle_build_s"] = build_s
        rec["oracle_roots_per_s"] = 16000 / mine_s
    rec["sampled_parity"] = samples
    lb = _planted_lower_bounds(planted)
    rec["planted_lower_bounds_hold"] = all(rec["counts"][n] >= lb[n] for n in lb)
    rec["planted"] = {kk: {str(a): b for a, b in v.items()} for kk, v in planted.items()}
    st = M.comine_stats(g, tree)
    rec["search_stats"] = st
    b_alg = 16 * E + 8 * (st["entries"] + st["windows"])  # SURVEY.md:540
    rec["bytes_alg_per_root"] = b_alg / E
    peak = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))["hbm_gbs"] if os.path.exists(
        os.path.join(ROOT, "MEASURED_PEAKS.json")) else 6650.0
    rec["roofline_frac_1gpu"] = b_alg / (ms * 1e-3) / 1e9 / peak
    print(json.dumps(rec))
    os.makedirs(os.path.dirname(out_path) or ".", exist_ok=True)
    with open(out_path, "w") as f:
        f.write(json.dumps(rec) + "\n")


if __name__ == "__main__":
    main()
