"""Sampling helpers for the full-size parity tests (test infrastructure: calls only oracle/)."""


def oracle_on_time_windows(oracle_mod, src, dst, t, V, motifs, delta, ranges):
    """Oracle counts of root ranges [a, b) of the (t, input rank) order, each from the sub-graph of
    the edges with t_a <= t <= t_(b-1) + delta: every match of a root r uses only edges with
    t_r < t <= t_r + delta, so the counts are those of the whole graph.  The sub-graph
    keeps the input order, so its own (t, input rank) order is the global one restricted, and root a
    sits at position a - #{t < t_a}.  O(E) numpy per range instead of a 500 M-edge oracle build."""
    import numpy as np
    out = []
    for a, b in ranges:
        ta = np.partition(t, a)[a]
        tb = np.partition(t, b - 1)[b - 1]
        keep = (t >= ta) & (t <= tb + delta)
        c = int(np.count_nonzero(t < ta))
        out.append(oracle_mod.backtrack(src[keep], dst[keep], t[keep], V, motifs, delta, root_range=(a - c, b - c)))
    return out
