"""GPU parity of each kernel form vs the oracle, forced with MAYURA_KERNEL: "flat" (level-
synchronous, entry-parallel; csrc/flat.cuh; the default for graphs that fit in L2),
"hybrid" (one breadth-first level + the warp-synchronous depth-first kernel, wdfs.cuh; the
default for larger graphs), "warp" (the warp kernel straight from the roots), "lane" (the
per-lane depth-first kernel) and "mixed".  Random groups, hub lists, the C1 workload, the
87-motif 3-edge family (every anchor kind incl. GLOBAL), and forced overflow of the
window-piece and frontier buffers (the depth-first fallback must keep counts exact)."""
import os

import numpy as np
import pytest

import synth

pytestmark = pytest.mark.gpu


@pytest.fixture(params=["flat", "hybrid", "lane", "mixed", "warp"])
def M(monkeypatch, request):
    import torch
    if not torch.cuda.is_available():
        pytest.fail("GPU tests need a CUDA device")
    monkeypatch.setenv("MAYURA_KERNEL", request.param)
    import paper_2507_14813_b200 as M
    return M


def run(M, src, dst, t, V, motifs, delta):
    g = M.Graph(src, dst, t, V, device=0)
    tree = M.MGTree(motifs, delta)
    out = M.comine(g, tree)
    g.close()
    tree.close()
    return out


def test_form_fuzz(M, oracle_mod):
    for seed in range(80):
        rng = np.random.default_rng(3000 + seed)
        V = int(rng.integers(3, 30))
        src, dst, t, V = synth.random_graph(3000 + seed, V, int(rng.integers(1, 300)), int(rng.integers(5, 200)))
        motifs = [synth.random_motif(seed * 13 + j, int(rng.integers(1, 5)), int(rng.integers(2, 6)))
                  for j in range(int(rng.integers(1, 7)))]
        delta = int(rng.integers(0, 80))
        assert run(M, src, dst, t, V, motifs, delta) == oracle_mod.backtrack(src, dst, t, V, motifs, delta), seed


def test_form_hubs_and_c1(M, oracle_mod):
    for seed in range(3):
        src, dst, t, V = synth.random_graph(70 + seed, 5 + seed, 20_000, 4_000 + 3000 * seed, 0.01)
        motifs = synth.group(synth.GROUP_C2) + [synth.MOTIFS["recip2"], synth.MOTIFS["repeat2"]]
        assert run(M, src, dst, t, V, motifs, 10 + 7 * seed) == oracle_mod.backtrack(src, dst, t, V, motifs, 10 + 7 * seed)
    cfg = synth.CONFIGS["C1"]
    src, dst, t, V = cfg.graph()
    assert run(M, src, dst, t, V, cfg.group(), cfg.delta) == oracle_mod.backtrack(src, dst, t, V, cfg.group(), cfg.delta)


def test_form_family_m3(M, oracle_mod):
    from tests import _pins
    fam = _pins.canonical_motifs(3)
    assert len(fam) == 87
    src, dst, t, V = synth.random_graph(17, 12, 1500, 400, 0.02)
    assert run(M, src, dst, t, V, fam, 40) == oracle_mod.backtrack(src, dst, t, V, fam, 40)


def test_form_overflow_fallbacks(M, oracle_mod, monkeypatch):
    monkeypatch.setenv("MAYURA_FLAT_WIN_CAP", "7")
    monkeypatch.setenv("MAYURA_BFS_SEG_CAP", "3")
    cfg = synth.CONFIGS["C1"]
    src, dst, t, V = cfg.graph()
    motifs = synth.group(synth.GROUP_C2) + [[(0, 1), (2, 3), (3, 0)]]
    assert run(M, src, dst, t, V, motifs, cfg.delta) == oracle_mod.backtrack(src, dst, t, V, motifs, cfg.delta)


def test_form_edge_cases(M, oracle_mod):
    """Empty graph, all self-loops, all tied timestamps, delta = 0, 2^62 timestamps, a
    1-edge-only group (no MG-Tree level below the root) -- in every kernel form."""
    tri = [synth.MOTIFS["tri_cycle"], synth.MOTIFS["edge1"]]
    assert run(M, [], [], [], 3, tri, 10) == [0, 0]
    assert run(M, [1, 2, 2], [1, 2, 2], [1, 2, 3], 3, tri, 10) == [0, 0]
    assert run(M, [0, 1, 2], [1, 2, 0], [5, 5, 5], 3, tri, 100) == [0, 3]
    src, dst, t, V = synth.random_graph(9, 10, 500, 100)
    g2 = synth.group(synth.GROUP_C2)
    assert run(M, src, dst, t, V, g2, 0) == oracle_mod.backtrack(src, dst, t, V, g2, 0)
    big = 2 ** 62   # t_r + delta = 2^63 would wrap: compared with the (saturating) oracle
    rm = [synth.MOTIFS["recip2"]]
    assert run(M, [0, 1], [1, 0], [big, big + 5], 2, rm, 2 ** 62) == \
        oracle_mod.backtrack([0, 1], [1, 0], [big, big + 5], 2, rm, 2 ** 62) == \
        [oracle_mod.python_bruteforce([0, 1], [1, 0], [big, big + 5], rm[0], 2 ** 62)]
    assert run(M, src, dst, t, V, [synth.MOTIFS["edge1"]], 10) == \
        oracle_mod.backtrack(src, dst, t, V, [synth.MOTIFS["edge1"]], 10)


def test_form_maximum_motif_size(M, oracle_mod):
    """MAYURA_MAX_EDGES = 8 edges per motif and up to 16 motif vertices (the largest register
    class of m2g), 7 MG-Tree levels below the root: an 8-edge fan-out against its closed form
    at 3,000 edges, and 8-edge path / cycle / fan-in / mixed motifs plus 8 disjoint edges
    (16 vertices, every window from the edge array) against the oracle on a small graph."""
    from tests import _pins
    src, dst, t, V = synth.out_star(3000)
    star8 = [(0, i) for i in range(1, 9)]
    assert run(M, src, dst, t, V, [star8], 12) == [_pins.star_fanout_count(3000, 8, 12)]
    src, dst, t, V = synth.random_graph(31, 9, 500, 50, 0.0)
    path8 = [(i, i + 1) for i in range(8)]
    cyc8 = [(i, (i + 1) % 8) for i in range(8)]
    fanin8 = [(i, 0) for i in range(1, 9)]
    mixed = [(0, 1), (1, 2), (2, 0), (0, 3), (3, 1), (1, 0), (2, 3), (3, 0)]
    group = [path8, cyc8, fanin8, mixed]
    exp = oracle_mod.backtrack(src, dst, t, V, group, 20)
    assert all(exp) and run(M, src, dst, t, V, group, 20) == exp
    src, dst, t, V = synth.random_graph(32, 40, 60, 30, 0.0)
    disj = [[(2 * i, 2 * i + 1) for i in range(8)]]
    assert run(M, src, dst, t, V, disj, 9) == oracle_mod.backtrack(src, dst, t, V, disj, 9)


def test_form_family_m4(M, oracle_mod):
    """The full 4-edge family: 1,657 canonical motifs, 1,752 trie rows -- more completion slots
    than per-thread shared-memory counters can hold, so the breadth-first / flat passes count
    with block-shared atomics (bfs::thread_cnt).  Exact vs the oracle, and the family identity
    (P4: the sum over the family = all increasing windowed 4-tuples of non-self-loop edges)."""
    from tests import _pins
    fam = _pins.canonical_motifs(4)
    assert len(fam) == 1657
    src, dst, t, V = synth.random_graph(23, 7, 220, 90, 0.03)
    got = run(M, src, dst, t, V, fam, 30)
    assert got == oracle_mod.backtrack(src, dst, t, V, fam, 30)
    assert sum(got) == _pins.family_total(src, dst, t, 4, 30)


@pytest.mark.parametrize("hook", ["MAYURA_WDFS_SMALL=1", "MAYURA_WDFS_SMALL=1 MAYURA_WDFS_SPILL_CAP=0",
                                  "MAYURA_WDFS_SMALL=1 MAYURA_WDFS_SPILL_CAP=40"])
def test_form_small_warp_stacks(M, oracle_mod, monkeypatch, hook):
    """The warp kernel's piece stack at 64 entries: full stacks spill their bottom half to the
    per-warp global spill area and reload it when they run empty; with no (or a 40-piece) spill
    area the pushes past the capacity are mined depth-first by the lane (bfs::dfs) -- exact."""
    for kv in hook.split():
        k, v = kv.split("=")
        monkeypatch.setenv(k, v)
    for seed in range(2):
        src, dst, t, V = synth.random_graph(90 + seed, 6, 6000, 3000, 0.01)
        motifs = synth.group(synth.GROUP_C4)
        assert run(M, src, dst, t, V, motifs, 40) == oracle_mod.backtrack(src, dst, t, V, motifs, 40)


def test_form_many_single_entry_windows(M, oracle_mod):
    """Sparse graphs whose windows mostly hold one entry: the warp kernel's rounds then take 64
    one-entry pieces whole (the case where no piece is split), and hub-free roots dominate."""
    for seed in range(3):
        src, dst, t, V = synth.random_graph(400 + seed, 3000, 60_000, 200_000, 0.002)
        motifs = synth.group(synth.GROUP_C2) + [synth.MOTIFS["recip2"], synth.MOTIFS["path2"]]
        assert run(M, src, dst, t, V, motifs, 400) == oracle_mod.backtrack(src, dst, t, V, motifs, 400)


def test_warp_form_fresh_process_fallback(oracle_mod):
    """The warp form's serial fallback (full stack, no spill area) in a process that never ran
    another form: its graph has no breadth-first scratch, so the kernel's diagnostic fallback
    counter must not be dereferenced (it was, through a null control-word pointer, before r2)."""
    import subprocess
    import sys
    code = (
        "import os, sys; sys.path.insert(0, %r)\n"
        "os.environ.update(MAYURA_KERNEL='warp', MAYURA_WDFS_SMALL='1', MAYURA_WDFS_SPILL_CAP='0')\n"
        "import synth, oracle, paper_2507_14813_b200 as M\n"
        "src, dst, t, V = synth.random_graph(90, 6, 6000, 3000, 0.01)\n"
        "mo = synth.group(synth.GROUP_C4)\n"
        "g = M.Graph(src, dst, t, V, device=0); tree = M.MGTree(mo, 40)\n"
        "assert M.comine(g, tree) == oracle.backtrack(src, dst, t, V, mo, 40)\n"
        "print('ok')\n" % os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    out = subprocess.run([sys.executable, "-c", code], capture_output=True, text=True, timeout=600)
    assert out.returncode == 0 and "ok" in out.stdout, out.stderr[-2000:]


def test_warp_stats_instance(oracle_mod, monkeypatch):
    """MAYURA_WDFS_STATS=1: the instrumented warp kernel (tools/wdfs_stats.py) counts exactly the
    oracle's matches; every round gives at most 64 candidates and every valid entry is a lane."""
    import paper_2507_14813_b200 as M
    monkeypatch.setenv("MAYURA_KERNEL", "warp")
    monkeypatch.setenv("MAYURA_WDFS_STATS", "1")
    src, dst, t, V = synth.random_graph(77, 40, 5000, 2000, 0.01)
    motifs = synth.group(synth.GROUP_C2)
    g = M.Graph(src, dst, t, V, device=0)
    tree = M.MGTree(motifs, 60)
    st = M.comine_stats(g, tree)
    exp = oracle_mod.backtrack(src, dst, t, V, motifs, 60)
    assert st["matches"] == sum(exp) and M.comine(g, tree) == exp
    assert st["batches"] > 0 and st["probes"] <= 64 * st["batches"] and st["entries"] <= st["probes"]
