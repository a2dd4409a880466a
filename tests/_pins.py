"""Independent pins for the oracle: closed forms, motif-family enumeration and the
family identity.  Nothing here matches motifs; each quantity follows from the
definition by counting arguments written out in the
docstrings (derivations in DESIGN.md §4)."""
from __future__ import annotations

from math import comb
from typing import List, Tuple

import numpy as np

Motif = List[Tuple[int, int]]


def canonical_motifs(m: int) -> List[Motif]:
    """All motifs with m edges, no self-loop edges, in canonical first-appearance
    labelling (u before v).  Every edge sequence is isomorphic to exactly one."""
    out: List[Motif] = []

    def rec(prefix: Motif, nv: int):
        if len(prefix) == m:
            out.append(list(prefix))
            return
        # endpoint choices: an existing label, or the next fresh label
        for u in range(nv + 1):
            nv_u = max(nv, u + 1)
            for v in range(nv_u + 1):
                if v == u:
                    continue
                prefix.append((u, v))
                rec(prefix, max(nv_u, v + 1))
                prefix.pop()

    rec([], 0)
    # the first edge must be (0,1) in canonical form
    return [mm for mm in out if mm[0] == (0, 1)]


def family_total(src, dst, t, m: int, delta: int) -> int:
    """Number of m-tuples of non-self-loop edges with strictly increasing timestamps and
    t_m - t_1 <= delta.  Every such tuple matches exactly one canonical m-edge motif
    (its own pattern), so this equals the sum of counts over canonical_motifs(m).
    Computed per root r as e_{m-1} of the tie-group sizes of the later non-self-loop
    edges with t in (t_r, t_r + delta]."""
    src = np.asarray(src); dst = np.asarray(dst); t = np.asarray(t, np.int64)
    keep = src != dst
    ts = np.sort(t[keep])
    total = 0
    for tr in ts:
        later = ts[(ts > tr) & (ts <= tr + delta)]
        _, sizes = np.unique(later, return_counts=True)
        # elementary symmetric polynomial e_{m-1}(sizes)
        e = [1] + [0] * (m - 1)
        for s in sizes:
            for j in range(m - 1, 0, -1):
                e[j] += e[j - 1] * int(s)
        total += e[m - 1]
    return total


def star_fanout_count(n: int, k: int, delta: int) -> int:
    """out_star(n): edges 0->i at t=i.  Motif 0->1,0->2,...,0->k: the root i picks any
    k-1 of the min(delta, n-i) later edges (all destinations distinct)."""
    return sum(comb(min(delta, n - i), k - 1) for i in range(1, n + 1))


def alt_reciprocal(n: int, delta: int) -> int:
    """alternating_pair(n): the reply must have the opposite parity offset (odd)."""
    return sum(-(-min(delta, n - i) // 2) for i in range(1, n + 1))


def alt_repeat(n: int, delta: int) -> int:
    """same direction again: even positive offsets."""
    return sum(min(delta, n - i) // 2 for i in range(1, n + 1))


def alt_pingpong(n: int, delta: int) -> int:
    """0->1,1->0,0->1: odd offset a then even offset b > a, b <= w; sum_{s} (q - s)
    over odd a = 2s+1 gives C(q+1, 2) with q = floor(w/2)."""
    return sum(comb(min(delta, n - i) // 2 + 1, 2) for i in range(1, n + 1))


def cycle_graph_path(L: int, n: int, j: int, delta: int) -> int:
    """cycle_graph(L, n): edge k = (k mod L)->(k+1 mod L) at t=k.  A j-edge path/cycle
    starting at edge k1 continues with gaps 1 + L*s_i (s_i >= 0), span (j-1) + L*S,
    S = sum s_i; needs span <= delta and k1 + span <= n-1.  Number of (j-1)-vectors
    with sum <= S_max is C(S_max + j - 1, j - 1).  Valid (injective) for the j-edge
    path when j + 1 <= L, and for the L-cycle when j == L."""
    if delta < j - 1:
        return 0
    total = 0
    for k1 in range(0, n - j + 1):
        smax = min((delta - j + 1) // L, (n - j - k1) // L)
        total += comb(smax + j - 1, j - 1)
    return total
