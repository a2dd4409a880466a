"""GPU parity: the CUDA co-mining path (through the C ABI) vs the CPU oracle, bit-exact.

Integer counts -> the bar is exact equality.  Covered: hand-worked
examples, >= 200 random groups of 2-6 motifs on tie-heavy fuzz graphs,
closed forms at 10^5-10^6 edges, the full 3-edge family (87 motifs; every anchor kind
including the all-edges candidate path), the C1/C2/C3 workloads in full, sampled
root ranges, co-mined == independent, range additivity, edge cases."""
import json
import os

import numpy as np
import pytest

import synth
from tests import _pins
from tests._sample import oracle_on_time_windows

pytestmark = pytest.mark.gpu

GOLDEN = os.path.join(os.path.dirname(__file__), "golden", "hand_examples.json")


@pytest.fixture(scope="module")
def M():
    import torch
    if not torch.cuda.is_available():
        pytest.fail("GPU tests need a CUDA device")
    import paper_2507_14813_b200 as M
    return M


def gpu_counts(M, src, dst, t, V, motifs, delta, root_range=None, independent=False):
    g = M.Graph(src, dst, t, V, device=0)
    tree = M.MGTree(motifs, delta)
    fn = M.mine_independent if independent else M.comine
    out = fn(g, tree, root_range)
    g.close()
    tree.close()
    return out


def test_hand_examples(M):
    cases = json.load(open(GOLDEN))["cases"]
    for c in cases:
        e = np.array(c["edges"], dtype=np.int64).reshape(-1, 3)
        V = int(e[:, :2].max()) + 1
        got = gpu_counts(M, e[:, 0], e[:, 1], e[:, 2], V, [[tuple(x) for x in c["motif"]]], c["delta"])
        assert got == [c["expected"]], c["name"]


def test_fuzz_groups_vs_oracle(M, oracle_mod):
    """>= 200 random groups of 2-6 motifs (<= 4 edges, some prefix-disconnected) on
    random tie-heavy multigraphs with self-loops."""
    nz = 0
    for seed in range(220):
        rng = np.random.default_rng(seed)
        V = int(rng.integers(3, 30))
        E = int(rng.integers(1, 300))
        src, dst, t, V = synth.random_graph(seed, V, E, int(rng.integers(5, 200)))
        k = int(rng.integers(2, 7))
        motifs = [synth.random_motif(seed * 101 + j, int(rng.integers(1, 5)), int(rng.integers(2, 6)))
                  for j in range(k)]
        delta = int(rng.integers(0, 80))
        exp = oracle_mod.backtrack(src, dst, t, V, motifs, delta)
        got = gpu_counts(M, src, dst, t, V, motifs, delta)
        assert got == exp, (seed, motifs, delta)
        ind = gpu_counts(M, src, dst, t, V, motifs, delta, independent=True)
        assert ind == exp, (seed, motifs, delta)
        nz += sum(1 for x in exp if x)
    assert nz > 300


def test_hub_lists_longer_than_a_warp(M, oracle_mod):
    """Few vertices, many edges: adjacency lists of 10^3-10^4 entries exercise the
    32-ary window search and multi-batch windows."""
    for seed in range(6):
        src, dst, t, V = synth.random_graph(70 + seed, 5 + seed, 20_000, 4_000 + 3000 * seed, 0.01)
        motifs = synth.group(synth.GROUP_C2) + [synth.MOTIFS["recip2"], synth.MOTIFS["repeat2"]]
        delta = 10 + 7 * seed
        assert gpu_counts(M, src, dst, t, V, motifs, delta) == \
            oracle_mod.backtrack(src, dst, t, V, motifs, delta)


def test_closed_forms_at_scale(M):
    n = 200_000
    src, dst, t, V = synth.out_star(n)
    got = gpu_counts(M, src, dst, t, V, [synth.MOTIFS["star_out3"], synth.MOTIFS["star_out4"],
                                         synth.MOTIFS["edge1"]], 40)
    assert got == [_pins.star_fanout_count(n, 3, 40), _pins.star_fanout_count(n, 4, 40), n]
    n = 1_000_001
    src, dst, t, V = synth.alternating_pair(n)
    got = gpu_counts(M, src, dst, t, V, [synth.MOTIFS["recip2"], synth.MOTIFS["repeat2"],
                                         synth.MOTIFS["pingpong3"]], 9)
    assert got == [_pins.alt_reciprocal(n, 9), _pins.alt_repeat(n, 9), _pins.alt_pingpong(n, 9)]
    L, n = 4, 400_000
    src, dst, t, V = synth.cycle_graph(L, n)
    cyc = [(i, (i + 1) % L) for i in range(L)]
    got = gpu_counts(M, src, dst, t, V, [cyc, [(0, 1), (1, 2), (2, 3)]], 23)
    assert got == [_pins.cycle_graph_path(L, n, L, 23), _pins.cycle_graph_path(L, n, 3, 23)]


@pytest.mark.parametrize("m", [2, 3])
def test_full_family_identity(M, m):
    fam = _pins.canonical_motifs(m)
    for seed in range(3):
        src, dst, t, V = synth.random_graph(600 + seed, 9, 400, 300, self_loop_frac=0.05)
        got = gpu_counts(M, src, dst, t, V, fam, 25)
        assert sum(got) == _pins.family_total(src, dst, t, m, 25)


def test_full_family_vs_oracle(M, oracle_mod):
    fam = _pins.canonical_motifs(3)
    src, dst, t, V = synth.random_graph(4321, 7, 300, 120, self_loop_frac=0.05)
    assert gpu_counts(M, src, dst, t, V, fam, 15) == oracle_mod.backtrack(src, dst, t, V, fam, 15)


@pytest.mark.parametrize("name", ["C1", "C2"])
def test_config_full_parity(M, oracle_mod, name):
    cfg = synth.CONFIGS[name]
    src, dst, t, V = cfg.graph()
    exp = oracle_mod.backtrack(src, dst, t, V, cfg.group(), cfg.delta)
    assert gpu_counts(M, src, dst, t, V, cfg.group(), cfg.delta) == exp
    assert gpu_counts(M, src, dst, t, V, cfg.group(), cfg.delta, independent=True) == exp


@pytest.mark.slow
def test_config_c3_full_parity(M, oracle_mod):
    cfg = synth.CONFIGS["C3"]
    src, dst, t, V = cfg.graph()
    exp = oracle_mod.backtrack(src, dst, t, V, cfg.group(), cfg.delta)
    assert gpu_counts(M, src, dst, t, V, cfg.group(), cfg.delta) == exp


def test_range_additivity_and_sampled_ranges(M, oracle_mod):
    cfg = synth.CONFIGS["C2"]
    src, dst, t, V = cfg.graph()
    g = M.Graph(src, dst, t, V, device=0)
    tree = M.MGTree(cfg.group(), cfg.delta)
    full = M.comine(g, tree)
    cuts = [0, 1, 31, 33, 100_000, 250_007, g.n_edges]
    parts = [M.comine(g, tree, (a, b)) for a, b in zip(cuts[:-1], cuts[1:])]
    assert [sum(x) for x in zip(*parts)] == full
    for a, b in [(0, 4096), (165_000, 169_096), (g.n_edges - 4096, g.n_edges)]:
        assert M.comine(g, tree, (a, b)) == oracle_mod.backtrack(src, dst, t, V, cfg.group(), cfg.delta,
                                                                 root_range=(a, b))
    assert M.comine(g, tree, (5, 5)) == [0] * tree.n_motifs


def test_edge_cases(M, oracle_mod):
    tri = [synth.MOTIFS["tri_cycle"], synth.MOTIFS["edge1"]]
    assert gpu_counts(M, [], [], [], 3, tri, 10) == [0, 0]                 # empty graph
    assert gpu_counts(M, [1, 2, 2], [1, 2, 2], [1, 2, 3], 3, tri, 10) == [0, 0]   # all self-loops
    s, d, t = [0, 1, 2], [1, 2, 0], [5, 5, 5]
    assert gpu_counts(M, s, d, t, 3, tri, 100) == [0, 3]                    # all tied
    src, dst, t, V = synth.random_graph(9, 10, 500, 100)
    assert gpu_counts(M, src, dst, t, V, synth.group(synth.GROUP_C2), 0) == \
        oracle_mod.backtrack(src, dst, t, V, synth.group(synth.GROUP_C2), 0)   # delta = 0
    big = 2 ** 62   # t_r + delta = 2^63 would wrap: compared with the (saturating) oracle
    rm = [synth.MOTIFS["recip2"]]
    assert gpu_counts(M, [0, 1], [1, 0], [big, big + 5], 2, rm, 2 ** 62) == \
        oracle_mod.backtrack([0, 1], [1, 0], [big, big + 5], 2, rm, 2 ** 62) == \
        [oracle_mod.python_bruteforce([0, 1], [1, 0], [big, big + 5], rm[0], 2 ** 62)]


def test_disconnected_prefix_motifs(M, oracle_mod):
    """(0->1, 2->3, ...) motifs use the all-edges (GLOBAL) candidate path (reading R6)."""
    motifs = [[(0, 1), (2, 3)], [(0, 1), (2, 3), (3, 0)], [(0, 1), (2, 3), (1, 2)], [(0, 1), (2, 3), (4, 5)]]
    for seed in range(5):
        src, dst, t, V = synth.random_graph(50 + seed, 12, 250, 150)
        assert gpu_counts(M, src, dst, t, V, motifs, 20) == oracle_mod.backtrack(src, dst, t, V, motifs, 20)


def test_counts_on_device_and_stream(M, oracle_mod):
    import torch
    cfg = synth.CONFIGS["C1"]
    src, dst, t, V = cfg.graph()
    g = M.Graph(src, dst, t, V, device=0)
    tree = M.MGTree(cfg.group(), cfg.delta)
    out = torch.full((tree.n_motifs,), -1, dtype=torch.int64, device="cuda:0")
    s = torch.cuda.Stream()
    M.comine(g, tree, None, stream=s.cuda_stream, counts_out=out)
    s.synchronize()
    assert out.cpu().tolist() == oracle_mod.backtrack(src, dst, t, V, cfg.group(), cfg.delta)


def test_stats_kernel_counts_and_work(M):
    cfg = synth.CONFIGS["C1"]
    src, dst, t, V = cfg.graph()
    g = M.Graph(src, dst, t, V, device=0)
    tree = M.MGTree(cfg.group(), cfg.delta)
    st = M.comine_stats(g, tree)
    si = M.comine_stats(g, tree, independent=True)
    assert st["matches"] == sum(M.comine(g, tree))
    assert st["roots"] == int((src != dst).sum())
    assert st["entries"] < si["entries"] and st["bytes_alg"] < si["bytes_alg"]  # co-mining removes work


def test_heavy_hub_roots_offload(M):
    """One hub with a dense burst: per-root search trees of 10^5-10^6 nodes.  The dynamic
    context offload (idle warps) must split them and counts must stay exact."""
    n, delta = 4000, 1000
    src, dst, t, V = synth.out_star(n)
    g = M.Graph(src, dst, t, V, device=0)
    tree = M.MGTree([synth.MOTIFS["star_out3"], [(0, 1), (0, 2)]], delta)
    assert M.comine(g, tree) == [_pins.star_fanout_count(n, 3, delta), _pins.star_fanout_count(n, 2, delta)]
    st = M.comine_stats(g, tree)
    assert st["offloads"] > 0          # long hub windows were split off (warp pass / handed out)
    assert st["matches"] == _pins.star_fanout_count(n, 3, delta) + _pins.star_fanout_count(n, 2, delta)
    # mixed: the hub burst plus random background, vs the oracle
    import oracle
    s2, d2, t2, V2 = synth.random_graph(5, 50, 20_000, 20_000)
    src = np.concatenate([src, s2 + V]); dst = np.concatenate([dst, d2 + V]); t = np.concatenate([t, t2])
    motifs = synth.group(synth.GROUP_C2)
    assert gpu_counts(M, src, dst, t, V + V2, motifs, 300) == oracle.backtrack(src, dst, t, V + V2, motifs, 300)


def test_bfs_overflow_fallbacks(M, oracle_mod, monkeypatch):
    """Tiny frontier segments and long-item capacity: every overflowing partial match is
    mined depth-first in place and long windows are scanned in place -- counts stay exact."""
    monkeypatch.setenv("MAYURA_BFS_SEG_CAP", "3")
    monkeypatch.setenv("MAYURA_BFS_LONG_CAP", "5")
    cfg = synth.CONFIGS["C1"]
    src, dst, t, V = cfg.graph()
    motifs = synth.group(synth.GROUP_C2) + [[(0, 1), (2, 3), (3, 0)]]
    g = M.Graph(src, dst, t, V, device=0)
    tree = M.MGTree(motifs, cfg.delta)
    exp = oracle_mod.backtrack(src, dst, t, V, motifs, cfg.delta)
    assert M.comine(g, tree) == exp
    st = M.comine_stats(g, tree)
    assert st["matches"] == sum(exp)
    if os.environ.get("MAYURA_KERNEL", "bfs") == "bfs":
        assert st["contexts"] > 0      # the depth-first fallback ran


def test_gpu_graph_build_matches_host_builder(M):
    """Step a0 on the GPU (CUB radix sorts + binary searches) produces exactly the arrays of
    the host builder: edge order, time ranks, CSR offsets/entries/sentinels, successor pointers."""
    cases = [synth.CONFIGS["C1"].graph(), synth.random_graph(11, 40, 5000, 300, self_loop_frac=0.05),
             synth.out_star(1000), synth.random_graph(12, 3, 1, 5), ([], [], [], 4)]
    big = synth.random_graph(13, 20, 2000, 50)
    cases.append((big[0], big[1], big[2] + (1 << 40), big[3]))           # large timestamps
    cases.append((big[0], big[1], big[2] - (1 << 40), big[3]))           # negative timestamps
    for src, dst, t, V in cases:
        eh = M.Graph(src, dst, t, V, device=-1).export()
        ed = M.Graph(src, dst, t, V, device=0).export()
        assert set(eh) == set(ed)
        for key in eh:
            assert np.array_equal(eh[key], ed[key]), key


def test_gpu_graph_build_errors(M):
    with pytest.raises(M.MayuraError):
        M.Graph([0, 1], [1, 7], [0, 1], 3, device=0)     # vertex id >= n_vertices


def _heaviest_roots(src, dst, t, delta, k, hubs=64):
    """The k roots with the most edges inside their root-node windows: out(src) and in(dst)
    entries with t_r < t <= t_r + delta (the hub bursts of the workload; the partition proxy of
    mayura_partition_roots grows with the same window sizes), searched among the roots incident
    to the `hubs` highest-degree vertices.  Vectorised with (vertex, t) keys."""
    import numpy as np
    deg = np.bincount(src, minlength=int(max(src.max(), dst.max())) + 1) + \
        np.bincount(dst, minlength=int(max(src.max(), dst.max())) + 1)
    hub = np.zeros(deg.size, bool)
    hub[np.argsort(-deg, kind="stable")[:hubs]] = True
    cand = np.nonzero(hub[src] | hub[dst])[0]
    tt = t - t.min()
    span = int(tt.max()) + int(delta) + 2
    def window_sizes(v):
        keys = np.sort(v.astype(np.int64) * span + tt)
        q = v[cand].astype(np.int64) * span + tt[cand]
        return np.searchsorted(keys, q + delta, side="right") - np.searchsorted(keys, q, side="right")
    w = window_sizes(src) + window_sizes(dst)
    top = cand[np.argsort(-w, kind="stable")[:k]]
    order = np.argsort(t, kind="stable")   # edge id = position in the stable time order (R1)
    rank_t = np.empty_like(order)
    rank_t[order] = np.arange(t.size)
    return sorted(int(rank_t[i]) for i in top), sorted((int(x) for x in np.sort(w)[::-1][:k]), reverse=True)


@pytest.mark.slow
def test_config_c4_sampled_parity(M, oracle_mod):
    """C4 (63.5 M edges, delta = 1 day, 16 motifs up to 5 edges): the whole graph is mined on
    the GPU; exact parity per motif on 32 evenly spaced 64-root chunks and on the 8 roots with
    the largest root-node windows (hub bursts), all from one oracle graph build (the oracle
    cannot finish C4 in full); co-mined == independent on a sample; range
    additivity at full size; the default (warp) form and the hybrid form agree."""
    cfg = synth.CONFIGS["C4"]
    src, dst, t, V = cfg.graph()
    g = M.Graph(src, dst, t, V, device=0)
    tree = M.MGTree(cfg.group(), cfg.delta)
    E = g.n_edges
    full = M.comine(g, tree)
    assert all(x >= 0 for x in full) and sum(full) > 0
    stride = E // 32
    ranges = [(i * stride + stride // 2, i * stride + stride // 2 + 64) for i in range(32)]
    heavy, sizes = _heaviest_roots(src, dst, t, cfg.delta, 8)
    assert min(sizes) > 50                                   # they are hub roots
    ranges += [(r, r + 1) for r in heavy]
    # the oracle's ids are its own (t, input rank) sort; the GPU's are the same order (R1)
    per, _, _ = oracle_mod.backtrack_ranges(src, dst, t, V, cfg.group(), cfg.delta, ranges)
    for rg, exp in zip(ranges, per):
        assert M.comine(g, tree, rg) == exp, rg
    assert sum(sum(x) for x in per[32:]) > 0                 # the heavy roots have matches
    assert M.mine_independent(g, tree, ranges[5]) == per[5]
    cut = E // 2
    halves = [M.comine(g, tree, (0, cut)), M.comine(g, tree, (cut, E))]
    assert [x + y for x, y in zip(*halves)] == full
    os.environ["MAYURA_KERNEL"] = "hybrid"
    try:
        assert M.comine(g, tree) == full
    finally:
        del os.environ["MAYURA_KERNEL"]


@pytest.mark.slow
def test_config_c5_sampled_parity_full_size(M, oracle_mod):
    """C5 at full size (500 M edges, 10 M vertices, planted AML patterns, 8 motifs): the whole
    graph on the GPU (one replica, ~50 GB), exact per-motif parity on 4 evenly spaced 2,000-root
    ranges against the oracle, and the planted lower bounds."""
    cfg = synth.CONFIGS["C5"]
    src, dst, t, V = cfg.graph()
    g = M.Graph(src, dst, t, V, device=0)
    tree = M.MGTree(cfg.group(), cfg.delta)
    E = g.n_edges
    full = M.comine(g, tree)
    ranges = [(i * (E // 4) + E // 8, i * (E // 4) + E // 8 + 2000) for i in range(4)]
    per = oracle_on_time_windows(oracle_mod, src, dst, t, V, cfg.group(), cfg.delta, ranges)
    for rg, exp in zip(ranges, per):
        assert M.comine(g, tree, rg) == exp, rg
    # planted patterns: every planted instance is a match (lower bounds; the background adds more)
    planted_fan_out = sum(v for k, v in synth.plant_aml(cfg.planted, cfg.n_vertices, cfg.span, cfg.delta,
                                                           cfg.seed)[3]["fan_out"].items())
    assert full[cfg.motifs.index("fan_out3")] >= planted_fan_out


def test_config_c5s_full_parity(M, oracle_mod):
    """C5's AML recipe at test size (2 M edges with planted fan-in/fan-out/cycle/scatter-gather
    patterns): exact parity in full, co-mined == independent."""
    cfg = synth.CONFIGS["C5s"]
    src, dst, t, V = cfg.graph()
    exp = oracle_mod.backtrack(src, dst, t, V, cfg.group(), cfg.delta)
    assert gpu_counts(M, src, dst, t, V, cfg.group(), cfg.delta) == exp
    assert gpu_counts(M, src, dst, t, V, cfg.group(), cfg.delta, independent=True) == exp


def test_partition_device_equals_host(M):
    """mayura_partition_roots on a device-built graph (proxy + prefix sum + cuts on the GPU)
    returns exactly the host-graph bounds."""
    cases = [(synth.CONFIGS["C2"].graph(), 3600), (synth.CONFIGS["C1"].graph(), 600),
             (synth.random_graph(5, 30, 3000, 200, self_loop_frac=0.05), 17), (([], [], [], 3), 5)]
    for (src, dst, t, V), delta in cases:
        gh = M.Graph(src, dst, t, V, device=-1)
        gd = M.Graph(src, dst, t, V, device=0)
        for parts in (1, 2, 3, 8, 64):
            assert gd.partition(delta, parts) == gh.partition(delta, parts), (parts, delta)
