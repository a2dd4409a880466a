"""Enumeration parity at scale: the C3 workload (7.8 M edges, 12 motifs; DRAM-resident, so
the counts come from the hybrid form and the tuples from the flat enumeration passes) on a
sampled root range, every tuple compared with oracle_enumerate (sorted per motif)."""
import numpy as np
import pytest

import synth

pytestmark = pytest.mark.gpu


def _sorted_rows(a):
    a = np.asarray(a, dtype=np.int64)
    return a[np.lexsort(a.T[::-1])] if a.size else a


def test_enumerate_c3_sampled_range(oracle_mod):
    import torch
    if not torch.cuda.is_available():
        pytest.fail("GPU tests need a CUDA device")
    import paper_2507_14813_b200 as M
    cfg = synth.CONFIGS["C3"]
    src, dst, t, V = cfg.graph()
    g = M.Graph(src, dst, t, V, device=0)
    tree = M.MGTree(cfg.group(), cfg.delta)
    E = g.n_edges
    rng = (E // 2, E // 2 + 1500)
    counts, lists = M.enumerate_matches(g, tree, rng)
    assert counts == M.comine(g, tree, rng) and sum(counts) > 0
    for q, mo in enumerate(cfg.group()):
        exp = oracle_mod.enumerate_matches(src, dst, t, V, mo, cfg.delta, rng)
        assert lists[q].shape == exp.shape, (q, lists[q].shape, exp.shape)
        assert np.array_equal(_sorted_rows(lists[q]), _sorted_rows(exp)), q
    g.close()
    tree.close()
