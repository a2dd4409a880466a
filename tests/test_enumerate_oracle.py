"""Pins of the oracle's enumeration form (oracle.enumerate_matches; "a
comprehensive list of all matching motifs (enumeration)", Algo 1 l.201).

The enumeration is pinned without re-running its own code: every listed tuple is checked
against the plain definition (§2.1) by an independent checker written
here, the tuples are distinct, and their number equals the count that O1/O2 and the pure
Python brute force agree on (test_oracle_pins.py).  A set of `count` distinct valid
matches IS the set of all matches."""
import itertools
import json
import os

import numpy as np
import pytest

import synth

GOLDEN = os.path.join(os.path.dirname(__file__), "golden", "hand_examples.json")


def is_match(src, dst, t, motif, delta, tup):
    """The definition, written out: strictly increasing times, t_m - t_1 <= delta, and an
    injective phi with phi(u_j) = src(e_j), phi(v_j) = dst(e_j)."""
    ts = [int(t[e]) for e in tup]
    if any(ts[i] >= ts[i + 1] for i in range(len(ts) - 1)) or ts[-1] - ts[0] > delta:
        return False
    phi = {}
    for (a, b), e in zip(motif, tup):
        for mv, gv in ((a, int(src[e])), (b, int(dst[e]))):
            if phi.setdefault(mv, gv) != gv:
                return False
    return len(set(phi.values())) == len(phi)


def test_hand_example_three_cycle(oracle_mod):
    """SPEC.md:344 / golden: {A->B@1, B->C@2, C->A@3}, delta = 30: exactly one 3-cycle,
    the tuple of all three edges in time order (input order here is scrambled)."""
    src, dst, t = [2, 0, 1], [0, 1, 2], [3, 1, 2]   # C->A@3, A->B@1, B->C@2
    rows = oracle_mod.enumerate_matches(src, dst, t, 3, [(0, 1), (1, 2), (2, 0)], 30)
    assert rows.tolist() == [[1, 2, 0]]
    assert oracle_mod.enumerate_matches(src, dst, t, 3, [(0, 1), (1, 2), (2, 0)], 1).shape == (0, 3)


def test_golden_cases_enumerated(oracle_mod):
    for c in json.load(open(GOLDEN))["cases"]:
        e = np.array(c["edges"], dtype=np.int64).reshape(-1, 3)
        V = int(e[:, :2].max()) + 1
        motif = [tuple(x) for x in c["motif"]]
        rows = oracle_mod.enumerate_matches(e[:, 0], e[:, 1], e[:, 2], V, motif, c["delta"])
        assert len(rows) == c["expected"], c["name"]
        assert len({tuple(r) for r in rows.tolist()}) == len(rows), c["name"]
        for r in rows.tolist():
            assert is_match(e[:, 0], e[:, 1], e[:, 2], motif, c["delta"], r), c["name"]


def test_enumeration_is_the_match_set_fuzz(oracle_mod):
    """Random tie-heavy multigraphs with self-loops: every row valid, rows distinct, row
    count == O1 count == pure-Python brute force (tiny) == O2 count."""
    for seed in range(120):
        rng = np.random.default_rng(1000 + seed)
        V = int(rng.integers(3, 12))
        E = int(rng.integers(1, 60))
        src, dst, t, V = synth.random_graph(1000 + seed, V, E, int(rng.integers(3, 40)))
        m = int(rng.integers(1, 5))
        motif = synth.random_motif(seed, m, int(rng.integers(2, 6)))
        delta = int(rng.integers(0, 30))
        rows = oracle_mod.enumerate_matches(src, dst, t, V, motif, delta)
        n = oracle_mod.bruteforce(src, dst, t, V, motif, delta)
        assert len(rows) == n == oracle_mod.backtrack(src, dst, t, V, [motif], delta, threads=1)[0]
        if E <= 18:
            assert n == oracle_mod.python_bruteforce(src, dst, t, motif, delta)
        assert len({tuple(r) for r in rows.tolist()}) == n
        for r in rows.tolist():
            assert is_match(src, dst, t, motif, delta, r), (seed, motif, r)


def test_enumeration_brute_force_set_equality_tiny(oracle_mod):
    """On tiny graphs compare the SET itself with an itertools enumeration of the definition."""
    for seed in range(40):
        src, dst, t, V = synth.random_graph(2000 + seed, 5, 14, 12)
        motif = synth.random_motif(seed + 7, 1 + seed % 3, 4)
        delta = 3 + seed % 9
        exp = set()
        for combo in itertools.permutations(range(len(src)), len(motif)):
            if is_match(src, dst, t, motif, delta, combo):
                exp.add(tuple(combo))
        got = {tuple(r) for r in oracle_mod.enumerate_matches(src, dst, t, V, motif, delta).tolist()}
        assert got == exp, (seed, motif, delta)


def test_enumeration_root_ranges_partition(oracle_mod):
    """Reading R16: a match belongs to the range holding its first edge (sorted edge ids);
    the ranges' lists are disjoint and their union is the whole list."""
    src, dst, t, V = synth.random_graph(77, 10, 400, 150)
    motif = [(0, 1), (1, 2), (2, 0)]
    whole = {tuple(r) for r in oracle_mod.enumerate_matches(src, dst, t, V, motif, 60).tolist()}
    parts = set()
    for a, b in ((0, 100), (100, 250), (250, 400)):
        rows = {tuple(r) for r in oracle_mod.enumerate_matches(src, dst, t, V, motif, 60, (a, b)).tolist()}
        assert not (rows & parts)
        parts |= rows
    assert parts == whole and len(whole) > 0
