"""CPU-only tests of the C-ABI library: it loads, exports every symbol declared in
include/mayura.h, and its host-side logic (graph builder, MG-Tree compiler,
root partitioning) is right.  No compute call is made (no GPU here)."""
import ctypes
import os
import re
from fractions import Fraction

import numpy as np
import pytest

import synth

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def M():
    import __graft_entry__
    __graft_entry__.build()
    import paper_2507_14813_b200 as M
    return M


def test_exports_every_header_symbol(M):
    hdr = open(os.path.join(ROOT, "include", "mayura.h")).read()
    declared = sorted(set(re.findall(r"\b(mayura_[a-z_]+)\s*\(", hdr)) - {"mayura_status"})
    assert len(declared) >= 14
    lib = ctypes.CDLL(M.mayura.LIB_PATH)
    for name in declared:
        assert hasattr(lib, name), name
    assert set(declared) == set(M.mayura.SIGNATURES)


def test_host_graph_builder_matches_definition(M):
    src, dst, t, V = synth.random_graph(3, 40, 3000, 500, self_loop_frac=0.02)
    g = M.Graph(src, dst, t, V, device=-1)
    ex = g.export()
    order = np.argsort(t, kind="stable")          # (t, input rank)
    assert np.array_equal(ex["perm"].astype(np.int64), order)
    assert np.array_equal(ex["src"], src[order]) and np.array_equal(ex["dst"], dst[order])
    ts = t[order]
    assert np.array_equal(ex["t"], ts)
    assert np.array_equal(ex["tr"], np.searchsorted(ts, ts, side="left"))
    lists = {}
    for direction, key, nbr in (("out", ex["src"], ex["dst"]), ("in", ex["dst"], ex["src"])):
        off, ent = ex[direction + "_off"], ex[direction + "_ent"].reshape(-1, 2)
        assert off[0] == 0 and off[-1] == len(src) + V
        for x in range(V):
            ids = np.nonzero(key == x)[0]       # edge ids of x, increasing = time order
            sl = ent[off[x]:off[x + 1] - 1]
            assert np.array_equal(sl[:, 0], ex["tr"][ids]) and np.array_equal(sl[:, 1], nbr[ids])
            assert tuple(ent[off[x + 1] - 1]) == (0xFFFFFFFF, 0xFFFFFFFF)   # sentinel
        lists[direction] = (off, ent)
    # successor pointers: first position after t_e in out(a), in(b), out(b), in(a)
    for e in range(0, len(src), 7):
        a, b, tre = ex["src"][e], ex["dst"][e], ex["tr"][e]
        for j, (d, x) in enumerate((("out", a), ("in", b), ("out", b), ("in", a))):
            off, ent = lists[d]
            seg = ent[off[x]:off[x + 1] - 1, 0]
            assert ex["eptr"][e, j] == off[x] + np.searchsorted(seg, tre, side="right")
    g.close()


def test_graph_builder_matches_oracle_edge_ids(M, oracle_mod):
    src, dst, t, V = synth.CONFIGS["C1"].graph()
    g = M.Graph(src, dst, t, V, device=-1)
    assert np.array_equal(g.export()["perm"].astype(np.int64), oracle_mod.sorted_order(t))


def test_graph_errors(M):
    with pytest.raises(M.MayuraError, match="INVALID"):
        M.Graph([0, 5], [1, 1], [0, 1], 3, device=-1)
    g = M.Graph([], [], [], 4, device=-1)
    assert (g.n_edges, g.n_vertices) == (0, 4)
    assert g.partition(10, 3) == [0, 0, 0, 0]


def _sm(motifs):
    import paper_2507_14813_b200 as M
    return M.MGTree(motifs, 10).info["sm"]


def test_mgtree_fig5_fig6_shape(M):
    """PAPER.md:487-499 (Figs. 5/6): [M3,M4,M5] -> I1(a>b>c){M3, I2(..>d){M4,M5}}."""
    m3 = [(0, 1), (1, 2), (2, 0)]
    m4 = [(0, 1), (1, 2), (2, 3), (3, 0)]
    m5 = [(0, 1), (1, 2), (2, 3), (3, 1)]
    t = M.MGTree([m3, m4, m5], 100)
    assert t.dump().splitlines() == [
        "I C=(0>1,1>2)",
        "  Q=0 C=(0>1,1>2,2>0)",
        "  I C=(0>1,1>2,2>3)",
        "    Q=1 C=(0>1,1>2,2>3,3>0)",
        "    Q=2 C=(0>1,1>2,2>3,3>1)",
    ]
    assert t.info["n_mg_nodes"] == 5
    assert abs(t.info["sm"] - 5 / 11) < 1e-12
    assert abs(_sm([m3, m4]) - 2 / 7) < 1e-12


def test_mgtree_labels_are_canonicalised(M):
    a = M.MGTree([[(7, 3), (3, 9), (9, 7)]], 5).dump()
    b = M.MGTree([[(0, 1), (1, 2), (2, 0)]], 5).dump()
    assert a == b == "Q=0 C=(0>1,1>2,2>0)\n"           # single motif: root is the leaf


def test_mgtree_prefix_motif_and_duplicates(M):
    t = M.MGTree([[(0, 1), (1, 2)], [(0, 1), (1, 2), (2, 0)]], 5)
    assert t.dump().splitlines() == ["Q=0 C=(0>1,1>2)", "  Q=1 C=(0>1,1>2,2>0)"]
    d = M.MGTree([[(0, 1), (1, 0)], [(5, 6), (6, 5)]], 5)           # duplicates share a node
    assert d.dump().splitlines() == ["Q=0,1 C=(0>1,1>0)"]


@pytest.mark.parametrize("cfg,expected", [("C1", Fraction(1, 3)), ("C2", Fraction(1, 2)),
                                          ("C3", Fraction(23, 38)), ("C4", Fraction(2, 3)),
                                          ("C5", Fraction(1, 2))])
def test_config_group_similarity_metric(M, cfg, expected):
    """SM of our config groups, SURVEY.md §8(c) P6."""
    assert abs(_sm(synth.CONFIGS[cfg].group()) - float(expected)) < 1e-12


def test_trie_node_counts(M):
    counts = [M.MGTree(synth.CONFIGS[c].group(), 1).info["n_trie_nodes"] for c in ("C1", "C2", "C3", "C4", "C5")]
    assert counts == [8, 13, 15, 19, 15]


def test_family_tree_paranjape(M):
    """The 36 connected 3-edge <=3-vertex motifs: 43 MG-Tree nodes, SM 65/108."""
    from tests._pins import canonical_motifs
    fam = [m for m in canonical_motifs(3) if max(max(e) for e in m) <= 2]
    assert len(fam) == 36
    t = M.MGTree(fam, 1)
    assert t.info["n_mg_nodes"] == 43
    assert abs(t.info["sm"] - 65 / 108) < 1e-12


def test_mgtree_errors(M):
    with pytest.raises(M.MayuraError, match="INVALID"):
        M.MGTree([[(0, 0)]], 1)
    with pytest.raises(M.MayuraError, match="INVALID"):
        M.MGTree([], 1)
    with pytest.raises(M.MayuraError, match="INVALID"):
        M.MGTree([[(0, 1)]], -1)
    with pytest.raises(M.MayuraError, match="LIMIT"):
        M.MGTree([[(i, i + 1) for i in range(9)]], 1)
    # 8 disjoint edges = 16 vertices is the largest motif accepted
    assert M.MGTree([[(2 * i, 2 * i + 1) for i in range(8)]], 1).info["max_vertices"] == 16


def _partition_reference(ex, delta, parts):
    """mayura_partition_roots' documented rule, re-derived in numpy from the exported arrays:
    p(r) = 1 + min(s_r, 65535)^2, s_r = entries with t_r < t <= t_r + delta in out(src),
    in(dst), out(dst), in(src); cuts at the first prefix reaching floor(total * p / P)."""
    t, tr = ex["t"], ex["tr"].astype(np.int64)
    E = t.size
    H = np.searchsorted(t, t + delta, side="right") - 1          # last id with t <= t_r + delta
    lists = [(ex["out_off"], ex["out_ent"], ex["src"]), (ex["in_off"], ex["in_ent"], ex["dst"]),
             (ex["out_off"], ex["out_ent"], ex["dst"]), (ex["in_off"], ex["in_ent"], ex["src"])]
    s = np.zeros(E, np.int64)
    for k, (off, ent, who) in enumerate(lists):
        keys = ent[0::2].astype(np.int64)
        for r in range(E):
            x = int(who[r])
            lo, hi = int(ex["eptr"][r, k]), int(off[x + 1]) - 1
            s[r] += int(np.searchsorted(keys[lo:hi], H[r], side="right"))
    proxy = 1 + np.minimum(s, 65535) ** 2
    pref = np.concatenate([[0], np.cumsum(proxy)])
    total = int(pref[-1])
    b = [0]
    for q in range(1, parts):
        target = (total // parts) * q + ((total % parts) * q) // parts
        b.append(max(min(int(np.searchsorted(pref, target, side="left")), E), b[-1]))
    return b + [E], proxy


def test_partition_roots(M):
    src, dst, t, V = synth.CONFIGS["C1"].graph()
    g = M.Graph(src, dst, t, V, device=-1)
    for parts in (1, 2, 3, 8):
        b = g.partition(600, parts)
        assert b[0] == 0 and b[-1] == g.n_edges and all(x <= y for x, y in zip(b, b[1:]))
    ex = g.export()
    for parts in (2, 4, 7):
        ref, proxy = _partition_reference(ex, 600, parts)
        b = g.partition(600, parts)
        assert b == ref
        per = [int(proxy[a:c].sum()) for a, c in zip(b, b[1:])]
        assert max(per) <= sum(per) / parts + proxy.max()         # balanced up to one root


def test_kernel_form_host_only_graph(M):
    """mayura_kernel_form: 'none' for host-only graphs and NULL (no CUDA call is made)."""
    g = M.Graph(np.array([0, 1], np.uint32), np.array([1, 2], np.uint32), np.array([1, 2], np.int64), 3, device=-1)
    assert M.mayura_kernel_form(g.handle) == "none"
    assert M.mayura_kernel_form(None) == "none"
    assert M.mayura_enum_form(g.handle) == "none"
    assert M.mayura_enum_form(None) == "none"


def test_partition_roots_shifted_timestamps(M):
    """The window end t_r + delta saturates instead of wrapping: a partition of
    timestamps shifted to negative values equals the numpy rule on the shifted graph and the
    partition of the unshifted graph (it depends on differences only)."""
    src, dst, t, V = synth.random_graph(3, 30, 3000, 5000)
    g0 = M.Graph(src, dst, t, V, device=-1)
    for shift in (-(1 << 40), -(1 << 62)):
        g = M.Graph(src, dst, t + np.int64(shift), V, device=-1)
        ex = g.export()
        for parts in (2, 4):
            ref, _ = _partition_reference(ex, 600, parts)
            assert g.partition(600, parts) == ref == g0.partition(600, parts)
    # timestamps next to INT64_MAX with a huge delta: every later edge is in every window
    top = np.iinfo(np.int64).max - 5000 + t
    g = M.Graph(src, dst, top, V, device=-1)
    big = g.partition(np.iinfo(np.int64).max, 4)
    assert big[0] == 0 and big[-1] == 3000 and all(a <= b for a, b in zip(big, big[1:]))
