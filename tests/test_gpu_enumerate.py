"""GPU parity of enumeration (mayura_enumerate, NEXT-3): the
CUDA path's match lists vs the oracle's (oracle.enumerate_matches, pinned in
test_enumerate_oracle.py).  Tuples are input edge indices in motif edge order; the
order of the matches is unspecified, so each motif's list is compared as a sorted
array (exact, every word), and the counts must equal mayura_comine's."""
import numpy as np
import pytest

import synth

pytestmark = pytest.mark.gpu


@pytest.fixture(params=["flat", "lane", "flat-overflow"])
def M(request, monkeypatch):
    """Small graphs enumerate in the flat form by default; MAYURA_ENUM_LANE=1 forces the
    depth-first form; tiny piece / frontier capacities make the flat attempt overflow and
    fall back to the depth-first form."""
    import torch
    if not torch.cuda.is_available():
        pytest.fail("GPU tests need a CUDA device")
    if request.param == "lane":
        monkeypatch.setenv("MAYURA_ENUM_LANE", "1")
    if request.param == "flat-overflow":
        monkeypatch.setenv("MAYURA_FLAT_WIN_CAP", "70")
        monkeypatch.setenv("MAYURA_BFS_SEG_CAP", "2")
    import paper_2507_14813_b200 as M
    return M


def _sorted_rows(a):
    a = np.asarray(a, dtype=np.int64)
    if a.size == 0:
        return a.reshape(0, a.shape[1] if a.ndim == 2 else 0)
    return a[np.lexsort(a.T[::-1])]


def check(M, oracle_mod, src, dst, t, V, motifs, delta, root_range=None):
    g = M.Graph(src, dst, t, V, device=0)
    tree = M.MGTree(motifs, delta)
    counts, lists = M.enumerate_matches(g, tree, root_range)
    assert counts == M.comine(g, tree, root_range)
    for q, mo in enumerate(motifs):
        exp = oracle_mod.enumerate_matches(src, dst, t, V, mo, delta, root_range)
        got = lists[q]
        assert got.shape == exp.shape, (q, mo, got.shape, exp.shape)
        assert np.array_equal(_sorted_rows(got), _sorted_rows(exp)), (q, mo)
    g.close()
    tree.close()
    return counts


def test_enumerate_fuzz_groups(M, oracle_mod):
    """Random groups of 1-5 motifs (<= 4 edges, some prefix-disconnected: GLOBAL anchor)
    on tie-heavy multigraphs with self-loops."""
    nz = 0
    for seed in range(60):
        rng = np.random.default_rng(500 + seed)
        V = int(rng.integers(3, 25))
        src, dst, t, V = synth.random_graph(500 + seed, V, int(rng.integers(1, 250)), int(rng.integers(5, 150)))
        motifs = [synth.random_motif(seed * 31 + j, int(rng.integers(1, 5)), int(rng.integers(2, 6)))
                  for j in range(int(rng.integers(1, 6)))]
        nz += sum(1 for c in check(M, oracle_mod, src, dst, t, V, motifs, int(rng.integers(0, 60))) if c)
    assert nz > 60


def test_enumerate_hubs_warp_help_and_donation(M, oracle_mod):
    """Adjacency lists of 10^3-10^4 entries: long leaf windows are scanned by the whole
    warp (tuples written by the helping lanes) and long searches are split into tasks
    (their prefixes travel with the task)."""
    for seed in range(3):
        src, dst, t, V = synth.random_graph(90 + seed, 5 + seed, 6_000, 2_000 + 1000 * seed, 0.01)
        motifs = synth.group(synth.GROUP_C2) + [synth.MOTIFS["recip2"], synth.MOTIFS["repeat2"]]
        check(M, oracle_mod, src, dst, t, V, motifs, 8 + 4 * seed)


def test_enumerate_c1_full_and_ranges(M, oracle_mod):
    cfg = synth.CONFIGS["C1"]
    src, dst, t, V = cfg.graph()
    counts = check(M, oracle_mod, src, dst, t, V, cfg.group(), cfg.delta)
    assert all(c > 0 for c in counts)
    E = len(src)
    check(M, oracle_mod, src, dst, t, V, cfg.group(), cfg.delta, (E // 3, E // 3 + 2500))


def test_enumerate_duplicates_one_edge_and_prefix_motifs(M, oracle_mod):
    """Duplicate motifs (reading R10) get identical lists; a 1-edge motif lists every
    non-self-loop edge; a motif that is a prefix of another (an inner completion node)."""
    src, dst, t, V = synth.random_graph(7, 12, 800, 300, 0.05)
    motifs = [[(0, 1), (1, 2), (2, 0)], [(5, 6), (6, 9), (9, 5)], [(0, 1)], [(0, 1), (1, 2)],
              [(0, 1), (1, 2), (2, 3)], [(0, 1), (2, 3)]]
    check(M, oracle_mod, src, dst, t, V, motifs, 40)


def test_enumerate_device_output_and_capacity(M, oracle_mod):
    import torch
    cfg = synth.CONFIGS["C1"]
    src, dst, t, V = cfg.graph()
    g = M.Graph(src, dst, t, V, device=0)
    tree = M.MGTree(cfg.group(), cfg.delta)
    host_counts, words = M.mayura_enumerate(g.handle, tree.handle, 0, g.n_edges)
    need = len(words)
    buf = torch.zeros(need, dtype=torch.int32, device="cuda:0")
    dev_counts, need2 = M.mayura_enumerate(g.handle, tree.handle, 0, g.n_edges, None, buf, need)
    assert dev_counts == host_counts and need2 == need
    dev = buf.cpu().numpy().view(np.uint32)
    for a, b in zip(M.split_tuples(host_counts, tree.lens, words), M.split_tuples(dev_counts, tree.lens, dev)):
        assert np.array_equal(_sorted_rows(a), _sorted_rows(b))
    small = torch.zeros(max(need - 1, 1), dtype=torch.int32, device="cuda:0")
    with pytest.raises(M.MayuraError):
        M.mayura_enumerate(g.handle, tree.handle, 0, g.n_edges, None, small, need - 1)
    g.close()
    tree.close()


def test_enumerate_edge_cases(M, oracle_mod):
    """Empty graph, all self-loops, delta = 0: zero tuples (size query and host output)."""
    for src, dst, t, V, delta in (([], [], [], 3, 10), ([1, 2, 2], [1, 2, 2], [1, 2, 3], 3, 10),
                                  ([0, 1, 2], [1, 2, 0], [1, 2, 3], 3, 0)):
        g = M.Graph(src, dst, t, V, device=0)
        tree = M.MGTree([synth.MOTIFS["tri_cycle"], synth.MOTIFS["recip2"]], delta)
        counts, lists = M.enumerate_matches(g, tree)
        assert counts == [0, 0] and all(len(x) == 0 for x in lists)
        assert M.mayura.mayura_enumerate_size(g.handle, tree.handle, 0, g.n_edges)[1] == 0
        g.close()
        tree.close()


def test_enumerate_maximum_motif_size(M, oracle_mod):
    """8-edge motifs (prefixes of up to 7 edges travel with tasks and frames), up to 16 motif
    vertices (8 disjoint edges: every window from the edge array)."""
    src, dst, t, V = synth.random_graph(31, 9, 500, 50, 0.0)
    group = [[(i, i + 1) for i in range(8)], [(i, (i + 1) % 8) for i in range(8)],
             [(0, 1), (1, 2), (2, 0), (0, 3), (3, 1), (1, 0), (2, 3), (3, 0)]]
    assert all(check(M, oracle_mod, src, dst, t, V, group, 20))
    src, dst, t, V = synth.random_graph(32, 40, 60, 30, 0.0)
    assert check(M, oracle_mod, src, dst, t, V, [[(2 * i, 2 * i + 1) for i in range(8)]], 9)[0] > 0


def test_enum_form_reports_the_form_that_ran(M, request):
    """mayura_enum_form names the form the last enumeration took: flat by default, depth-first
    when forced or when a flat buffer overflowed (C1: the tiny capacities overflow)."""
    cfg = synth.CONFIGS["C1"]
    src, dst, t, V = cfg.graph()
    g = M.Graph(src, dst, t, V, device=0)
    tree = M.MGTree(cfg.group(), cfg.delta)
    assert M.mayura_enum_form(g.handle) == "none"
    M.enumerate_matches(g, tree)
    want = {"flat": "flat", "lane": "depth-first", "flat-overflow": "depth-first"}[request.node.callspec.params["M"]]
    assert M.mayura_enum_form(g.handle) == want
    g.close()
    tree.close()


def test_enumerate_repeated_on_one_graph(M, oracle_mod):
    """The input ranks behind list positions are computed on the first enumeration of a graph
    (in place over the edge ids the build leaves there); later enumerations of the same graph,
    with other groups and root ranges, and counting in between, must read the same ranks."""
    src, dst, t, V = synth.random_graph(41, 30, 3_000, 900, 0.02)
    g = M.Graph(src, dst, t, V, device=0)
    groups = [synth.group(synth.GROUP_C2), [[(0, 1), (1, 2)], [(0, 1), (1, 0)]], synth.group(synth.GROUP_C2)]
    E = len(src)
    for i, motifs in enumerate(groups):
        tree = M.MGTree(motifs, 25)
        rr = None if i != 1 else (E // 4, E // 2)
        M.comine(g, tree)
        counts, lists = M.enumerate_matches(g, tree, rr)
        assert counts == M.comine(g, tree, rr)
        for q, mo in enumerate(motifs):
            exp = oracle_mod.enumerate_matches(src, dst, t, V, mo, 25, rr)
            assert np.array_equal(_sorted_rows(lists[q]), _sorted_rows(exp)), (i, q)
        tree.close()
    g.close()
