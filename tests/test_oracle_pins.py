"""Pins for the CPU oracle (O1 brute force, O2 Algorithm-1 backtracking) against
things other than itself: hand-worked examples (tests/golden), closed forms on
structured graphs, the full-family identity, time/direction-reversal invariants,
delta-monotonicity and an independent pure-Python brute force.
SURVEY.md §8(c) pins P1-P5; DESIGN.md §4."""
import json
import os

import numpy as np
import pytest

import synth
from tests import _pins
from tests._sample import oracle_on_time_windows

GOLDEN = os.path.join(os.path.dirname(__file__), "golden", "hand_examples.json")


def _cases():
    with open(GOLDEN) as f:
        return json.load(f)["cases"]


@pytest.mark.parametrize("case", _cases(), ids=lambda c: c["name"])
def test_hand_examples(oracle_mod, case):
    e = np.array(case["edges"], dtype=np.int64).reshape(-1, 3)
    src, dst, t = e[:, 0], e[:, 1], e[:, 2]
    V = int(e[:, :2].max()) + 1
    motif = [tuple(x) for x in case["motif"]]
    exp = case["expected"]
    assert oracle_mod.python_bruteforce(src, dst, t, motif, case["delta"]) == exp
    assert oracle_mod.bruteforce(src, dst, t, V, motif, case["delta"]) == exp
    assert oracle_mod.backtrack(src, dst, t, V, [motif], case["delta"], threads=1) == [exp]


def test_o1_o2_python_agree_fuzz(oracle_mod):
    """P1: >= 500 seeds, <= 30 vertices, motifs <= 4 edges, ties and self-loops."""
    nonzero = 0
    for seed in range(520):
        rng = np.random.default_rng(seed)
        V = int(rng.integers(2, 8))
        E = int(rng.integers(0, 24))
        src, dst, t, V = synth.random_graph(seed, V, E, int(rng.integers(1, 20)))
        m = int(rng.integers(1, 5))
        motif = synth.random_motif(seed + 7919, m, max_vertices=int(rng.integers(2, 6)))
        delta = int(rng.integers(0, 15))
        a = oracle_mod.python_bruteforce(src, dst, t, motif, delta) if E <= 20 or m <= 2 else None
        b = oracle_mod.bruteforce(src, dst, t, V, motif, delta)
        c = oracle_mod.backtrack(src, dst, t, V, [motif], delta, threads=2)[0]
        if a is not None:
            assert a == b, (seed, motif, delta)
        assert b == c, (seed, motif, delta)
        nonzero += b > 0
    assert nonzero > 150  # the fuzz is not vacuous


def test_o1_o2_agree_larger(oracle_mod):
    """P1 at the SPEC's upper bound: <= 30 vertices, <= 200 edges, random delta."""
    for seed in range(60):
        rng = np.random.default_rng(10_000 + seed)
        src, dst, t, V = synth.random_graph(10_000 + seed, int(rng.integers(3, 31)),
                                            int(rng.integers(50, 201)), int(rng.integers(20, 400)))
        motifs = [synth.random_motif(seed * 13 + j, int(rng.integers(1, 5)), 4) for j in range(3)]
        delta = int(rng.integers(0, 60))
        o2 = oracle_mod.backtrack(src, dst, t, V, motifs, delta)
        o1 = [oracle_mod.bruteforce(src, dst, t, V, m, delta) for m in motifs]
        assert o1 == o2, (seed, motifs, delta)


@pytest.mark.parametrize("n,delta", [(40, 5), (40, 100), (200, 17), (1, 3)])
def test_closed_form_out_star(oracle_mod, n, delta):
    src, dst, t, V = synth.out_star(n)
    motifs = [synth.MOTIFS[x] for x in ("edge1", "repeat2", "path2", "star_out3", "star_out4",
                                        "star_in3")]
    got = oracle_mod.backtrack(src, dst, t, V, motifs, delta)
    assert got == [n, 0, 0, _pins.star_fanout_count(n, 3, delta),
                   _pins.star_fanout_count(n, 4, delta), 0]
    # star_out2 == (0->1, 0->2)
    assert oracle_mod.backtrack(src, dst, t, V, [[(0, 1), (0, 2)]], delta) == \
        [_pins.star_fanout_count(n, 2, delta)]


@pytest.mark.parametrize("n,delta", [(30, 4), (31, 7), (200, 25), (2, 0)])
def test_closed_form_alternating_pair(oracle_mod, n, delta):
    src, dst, t, V = synth.alternating_pair(n)
    motifs = [synth.MOTIFS[x] for x in ("recip2", "repeat2", "pingpong3", "path2", "tri_cycle")]
    got = oracle_mod.backtrack(src, dst, t, V, motifs, delta)
    assert got == [_pins.alt_reciprocal(n, delta), _pins.alt_repeat(n, delta),
                   _pins.alt_pingpong(n, delta), 0, 0]
    for m, exp in zip(motifs[:3], got[:3]):
        assert oracle_mod.bruteforce(src, dst, t, V, m, delta) == exp


@pytest.mark.parametrize("L,n,delta", [(3, 40, 10), (4, 60, 20), (5, 80, 31), (3, 30, 1), (4, 50, 3)])
def test_closed_form_cycle_graph(oracle_mod, L, n, delta):
    src, dst, t, V = synth.cycle_graph(L, n)
    cyc = [(i, (i + 1) % L) for i in range(L)]
    paths = [[(i, i + 1) for i in range(j)] for j in range(1, L)]
    got = oracle_mod.backtrack(src, dst, t, V, [cyc] + paths, delta)
    assert got[0] == _pins.cycle_graph_path(L, n, L, delta)
    for j, g in zip(range(1, L), got[1:]):
        assert g == _pins.cycle_graph_path(L, n, j, delta)
    # a path longer than the cycle allows repeats a vertex -> 0
    long_path = [(i, i + 1) for i in range(L)]
    assert oracle_mod.backtrack(src, dst, t, V, [long_path], delta) == [0]


@pytest.mark.parametrize("m", [1, 2, 3])
def test_full_family_identity(oracle_mod, m):
    """P4: sum over all canonical m-edge motifs == number of windowed strictly increasing
    m-tuples of non-self-loop edges (exercises every candidate path and injectivity)."""
    fam = _pins.canonical_motifs(m)
    for seed in range(6):
        src, dst, t, V = synth.random_graph(500 + seed, 6 + seed, 60, 40, self_loop_frac=0.1)
        delta = 6 + 2 * seed
        got = oracle_mod.backtrack(src, dst, t, V, fam, delta)
        assert sum(got) == _pins.family_total(src, dst, t, m, delta)


def test_full_family_identity_m4(oracle_mod):
    fam = _pins.canonical_motifs(4)
    src, dst, t, V = synth.random_graph(77, 7, 45, 30, self_loop_frac=0.1)
    got = oracle_mod.backtrack(src, dst, t, V, fam, 9)
    assert sum(got) == _pins.family_total(src, dst, t, 4, 9)


def _canon(motif):
    lab = {}
    out = []
    for u, v in motif:
        for x in (u, v):
            if x not in lab:
                lab[x] = len(lab)
        out.append((lab[u], lab[v]))
    return out


def test_time_and_direction_reversal(oracle_mod):
    """P5: count(M,G) == count(reverse-order M, G with -t) == count(M^T, G^T)."""
    for seed in range(40):
        src, dst, t, V = synth.random_graph(900 + seed, 8, 80, 50)
        motif = synth.random_motif(seed, 1 + seed % 4, 4, relabel=False)
        delta = 5 + seed % 11
        base = oracle_mod.backtrack(src, dst, t, V, [motif], delta)[0]
        rev = _canon(list(reversed(motif)))
        assert oracle_mod.backtrack(src, dst, -t, V, [rev], delta)[0] == base
        tr = _canon([(v, u) for u, v in motif])
        assert oracle_mod.backtrack(dst, src, t, V, [tr], delta)[0] == base


def test_delta_monotone_and_relabel(oracle_mod):
    src, dst, t, V = synth.random_graph(4242, 10, 150, 100)
    motifs = synth.group(synth.GROUP_C2)
    prev = None
    for delta in (0, 3, 10, 30, 100):
        cur = oracle_mod.backtrack(src, dst, t, V, motifs, delta)
        if prev is not None:
            assert all(c >= p for c, p in zip(cur, prev))
        prev = cur
    # vertex relabelling of the graph leaves counts unchanged
    perm = np.random.default_rng(1).permutation(V).astype(np.uint32)
    assert oracle_mod.backtrack(perm[src], perm[dst], t, V, motifs, 30) == \
        oracle_mod.backtrack(src, dst, t, V, motifs, 30)


def test_root_range_additivity(oracle_mod):
    src, dst, t, V = synth.random_graph(31337, 12, 300, 200)
    motifs = synth.group(synth.GROUP_C2)
    full = oracle_mod.backtrack(src, dst, t, V, motifs, 25)
    cuts = [0, 37, 150, 151, 300]
    parts = [oracle_mod.backtrack(src, dst, t, V, motifs, 25, root_range=(a, b))
             for a, b in zip(cuts[:-1], cuts[1:])]
    assert [sum(x) for x in zip(*parts)] == full
    assert oracle_mod.bruteforce(src, dst, t, V, motifs[4], 25, root_range=(37, 150)) == parts[1][4]


def test_oracle_rejects_bad_input(oracle_mod):
    with pytest.raises(oracle_mod.OracleError):
        oracle_mod.backtrack([0], [1], [0], 2, [[(0, 0)]], 1)  # motif self-loop
    with pytest.raises(oracle_mod.OracleError):
        oracle_mod.backtrack([0], [5], [0], 2, [[(0, 1)]], 1)  # vertex id >= V
    with pytest.raises(oracle_mod.OracleError):
        oracle_mod.bruteforce(np.zeros(10), np.ones(10), np.arange(10), 2, [(0, 1)], 1, guard=5)


def test_synthetic_config_c1_nontrivial(oracle_mod):
    """The C1 workload has non-trivial counts for every motif of its group."""
    cfg = synth.CONFIGS["C1"]
    src, dst, t, V = cfg.graph()
    assert src.size == cfg.n_edges
    counts = oracle_mod.backtrack(src, dst, t, V, cfg.group(), cfg.delta)
    assert all(c > 0 for c in counts), counts


def _planted_lower_bounds(planted):
    """Matches every planted AML pattern contributes by construction (P7): a fan-out (fan-in)
    of k edges with increasing times holds C(k, 3) / C(k, 4) fan-out3/4 (fan-in3/4) tuples;
    each planted L-cycle is one L-cycle match rooted at its first edge; each scatter-gather is
    one (0->1, 0->2, 1->3, 2->3) match."""
    from math import comb
    lb = {"fan_out3": 0, "fan_out4": 0, "fan_in3": 0, "fan_in4": 0, "cycle3": 0, "cycle4": 0, "cycle5": 0,
          "scatter_gather": planted["scatter_gather"].get(2, 0)}
    for k, n in planted["fan_out"].items():
        lb["fan_out3"] += n * comb(k, 3)
        lb["fan_out4"] += n * comb(k, 4)
    for k, n in planted["fan_in"].items():
        lb["fan_in3"] += n * comb(k, 3)
        lb["fan_in4"] += n * comb(k, 4)
    for L, n in planted["cycle"].items():
        lb["cycle%d" % L] += n
    return lb


def test_planted_aml_patterns(oracle_mod):
    """The AML planting (C5 recipe) on its own: each pattern is found exactly as constructed
    (no background edges), pinning both the generator and the oracle on these motifs."""
    ps, pd, pt, planted = synth.plant_aml(60, 10_000, 10 * 86400, 3600, seed=3)
    V = 10_000
    motifs = synth.group(synth.GROUP_C5)
    got = dict(zip(synth.GROUP_C5, oracle_mod.backtrack(ps, pd, pt, V, motifs, 3600)))
    lb = _planted_lower_bounds(planted)
    for name in synth.GROUP_C5:
        assert got[name] >= lb[name], name
    # isolated patterns on random vertices of a 10k-vertex graph rarely touch: equal counts
    assert sum(got.values()) <= sum(lb.values()) + 5
    assert lb["cycle3"] + lb["cycle4"] + lb["cycle5"] == sum(planted["cycle"].values())


def test_c5s_planted_lower_bounds(oracle_mod):
    """P7 on the C5 recipe (test-sized twin C5s): every planted pattern is counted."""
    cfg = synth.CONFIGS["C5s"]
    src, dst, t, V, planted = cfg.graph_planted()
    assert src.size == cfg.n_edges
    got = dict(zip(cfg.motifs, oracle_mod.backtrack(src, dst, t, V, cfg.group(), cfg.delta)))
    for name, lb in _planted_lower_bounds(planted).items():
        assert got[name] >= lb, name


# ---------------------------------------------------------------- int64 extremes
I64 = np.iinfo(np.int64)


def _extreme_cases():
    """(edges, motif, delta, expected) at the ends of the int64 timestamp domain.  Expected
    values follow from the definition t_m - t_1 <= delta computed with Python's
    exact integers (python_bruteforce), so neither t_1 + delta nor t_m - t_1 may wrap."""
    big = 2 ** 62
    recip = [(0, 1), (1, 0)]
    return [
        ([(0, 1, big), (1, 0, big + 5)], recip, big, 1),                  # t_1 + delta = 2^63 (wraps)
        ([(0, 1, 5), (1, 0, 9)], recip, I64.max, 1),                       # delta = INT64_MAX
        ([(0, 1, -big), (1, 0, big - 1)], recip, I64.max, 1),              # t_m - t_1 = 2^63 - 1
        ([(0, 1, -big), (1, 0, big)], recip, I64.max, 0),                  # t_m - t_1 = 2^63 > delta
        ([(0, 1, I64.min), (1, 0, I64.max)], recip, I64.max, 0),           # span 2^64 - 1
        ([(0, 1, I64.min), (1, 0, -1)], recip, I64.max, 1),                # span 2^63 - 1
        ([(0, 1, -7), (1, 2, -3), (2, 0, -1)], [(0, 1), (1, 2), (2, 0)], 6, 1),   # negative times
        ([(0, 1, -7), (1, 2, -3), (2, 0, -1)], [(0, 1), (1, 2), (2, 0)], 5, 0),
        ([(0, 1, I64.max - 2), (1, 2, I64.max - 1), (2, 0, I64.max)], [(0, 1), (1, 2), (2, 0)], 2, 1),
    ]


@pytest.mark.parametrize("case", range(9))
def test_int64_extremes(oracle_mod, case):
    edges, motif, delta, exp = _extreme_cases()[case]
    e = np.array(edges, dtype=object)
    src = np.array([x[0] for x in edges], np.uint32)
    dst = np.array([x[1] for x in edges], np.uint32)
    t = np.array([x[2] for x in edges], np.int64)
    V = int(max(src.max(), dst.max())) + 1
    assert oracle_mod.python_bruteforce(src, dst, t, motif, delta) == exp
    assert oracle_mod.bruteforce(src, dst, t, V, motif, delta) == exp
    assert oracle_mod.backtrack(src, dst, t, V, [motif], delta, threads=1) == [exp]
    del e


def test_time_translation_invariance(oracle_mod):
    """P5: counts depend on timestamp differences only, so shifting every
    timestamp by a constant -- to negative times, or next to INT64_MAX -- changes nothing."""
    motifs = synth.group(synth.GROUP_C2)
    for seed in range(12):
        src, dst, t, V = synth.random_graph(5100 + seed, 9, 120, 60)
        delta = 3 + seed % 9
        base = oracle_mod.backtrack(src, dst, t, V, motifs, delta)
        for shift in (-(1 << 40), -(1 << 62), (1 << 62), int(I64.max) - 60):
            ts = t + np.int64(shift)
            assert oracle_mod.backtrack(src, dst, ts, V, motifs, delta) == base, (seed, shift)
        assert [oracle_mod.bruteforce(src, dst, t - np.int64(1 << 62), V, mo, delta) for mo in motifs[:4]] == base[:4]


def test_backtrack_ranges_equals_single_ranges(oracle_mod):
    """oracle_backtrack_ranges (one graph build, many root ranges) == oracle_backtrack per range."""
    src, dst, t, V = synth.random_graph(777, 15, 400, 150)
    motifs = synth.group(synth.GROUP_C2)
    ranges = [(0, 37), (37, 37), (100, 180), (350, 400)]
    per, build_s, mine_s = oracle_mod.backtrack_ranges(src, dst, t, V, motifs, 20, ranges, threads=3)
    assert per == [oracle_mod.backtrack(src, dst, t, V, motifs, 20, root_range=r) for r in ranges]
    assert build_s >= 0 and mine_s >= 0


def test_time_window_subgraph_oracle(oracle_mod):
    """The time-window reduction used by the full-size C5 test equals the oracle on the whole graph
    (tie-heavy random graph, ranges starting inside tie groups)."""
    src, dst, t, V = synth.random_graph(4242, 30, 3000, 400)
    motifs = synth.group(synth.GROUP_C2)
    ranges = [(0, 50), (700, 913), (1500, 1501), (2950, 3000)]
    assert oracle_on_time_windows(oracle_mod, src, dst, t, V, motifs, 25, ranges) == \
        [oracle_mod.backtrack(src, dst, t, V, motifs, 25, root_range=r) for r in ranges]
