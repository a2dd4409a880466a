"""NEXT-4 host logic: the paper's co-mining heuristic (§6): co-mine
if the graph is bipartite or the group's Similarity Metric is >= 0.44 (reading R18).
Bipartiteness is checked against an independent BFS 2-colouring written here."""
from collections import deque

import numpy as np
import pytest

import synth


@pytest.fixture(scope="module")
def M():
    import __graft_entry__
    __graft_entry__.build()
    import paper_2507_14813_b200 as M
    return M


def bfs_bipartite(src, dst, V):
    adj = [[] for _ in range(V)]
    for a, b in zip(src, dst):
        if a == b:
            return False
        adj[a].append(b)
        adj[b].append(a)
    col = [-1] * V
    for s in range(V):
        if col[s] >= 0:
            continue
        col[s] = 0
        q = deque([s])
        while q:
            x = q.popleft()
            for y in adj[x]:
                if col[y] < 0:
                    col[y] = col[x] ^ 1
                    q.append(y)
                elif col[y] == col[x]:
                    return False
    return True


def heur(M, src, dst, V, motifs, delta=10):
    t = np.arange(len(src), dtype=np.int64)
    g = M.Graph(np.asarray(src, np.uint32), np.asarray(dst, np.uint32), t, V, device=-1)
    tree = M.MGTree(motifs, delta)
    return M.mayura_comine_heuristic(g.handle, tree.handle)


TRI = [[(0, 1), (1, 2), (2, 0)], [(0, 1), (1, 2), (0, 2)], [(0, 1), (0, 2), (0, 3)], [(0, 1), (2, 1), (3, 1)]]


def test_known_graphs(M):
    even = ([0, 1, 2, 3], [1, 2, 3, 0])          # 4-cycle: bipartite
    odd = ([0, 1, 2], [1, 2, 0])                 # 3-cycle: not
    loop = ([0, 1], [1, 1])                      # self-loop: odd cycle
    star = ([0, 0, 0, 4], [1, 2, 3, 0])          # a tree
    assert heur(M, *even, 4, TRI)["bipartite"] is True
    assert heur(M, *odd, 3, TRI)["bipartite"] is False
    assert heur(M, *loop, 2, TRI)["bipartite"] is False
    assert heur(M, *star, 5, TRI)["bipartite"] is True


def test_random_graphs_vs_bfs(M):
    for seed in range(60):
        rng = np.random.default_rng(seed)
        V = int(rng.integers(2, 40))
        if seed % 2:  # planted bipartite: edges only across a random split (either direction)
            side = rng.integers(0, 2, V)
            a_set, b_set = np.flatnonzero(side == 0), np.flatnonzero(side == 1)
            if len(a_set) == 0 or len(b_set) == 0:
                continue
            E = int(rng.integers(1, 80))
            a = rng.choice(a_set, E)
            b = rng.choice(b_set, E)
            flip = rng.integers(0, 2, E).astype(bool)
            src, dst = np.where(flip, b, a), np.where(flip, a, b)
            if seed % 4 == 1:  # one edge inside a side breaks it (unless it closes no odd cycle)
                src = np.append(src, a_set[0])
                dst = np.append(dst, a_set[-1] if len(a_set) > 1 else a_set[0])
        else:
            E = int(rng.integers(1, 3 * V))
            src, dst = rng.integers(0, V, E), rng.integers(0, V, E)
        assert heur(M, src, dst, V, TRI)["bipartite"] == bfs_bipartite(list(src), list(dst), V), seed


def test_rule(M):
    """co-mine iff bipartite or SM >= 0.44; C1's group has SM 1/3, C2's 1/2 (P6)."""
    odd = ([0, 1, 2], [1, 2, 0])
    even = ([0, 1, 2, 3], [1, 2, 3, 0])
    c1, c2 = synth.group(synth.GROUP_C1), synth.group(synth.GROUP_C2)
    h = heur(M, *odd, 3, c1)
    assert abs(h["sm"] - 1 / 3) < 1e-12 and h["use_comine"] is False
    assert heur(M, *odd, 3, c2)["use_comine"] is True
    assert heur(M, *even, 4, c1)["use_comine"] is True
