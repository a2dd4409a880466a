"""GPU invariants and int64 timestamp extremes, every kernel form, through the C ABI.

The definition (§2.1) fixes three symmetries that any correct path must
respect at any size:
  * time translation  -- count(M, G, delta) depends on timestamp differences only, so
                         shifting every t (to negative times, next to INT64_MAX) changes nothing;
  * time reversal     -- count(M, G, delta) = count(reverse-order M, {(u, v, -t)}, delta);
  * direction reversal -- count(M, G, delta) = count(M^T, G^T, delta) (swaps out- and in-CSR).
At C2 scale every side is also compared with the oracle element by element; at C3 scale the
GPU is compared with itself under the transformation (the oracle takes ~1 min there and runs
in full in test_gpu_parity's slow C3 test).  The int64 cases take their expected values from
O1 and the pure-Python brute force (Python integers: no wraparound), never from literals."""
import numpy as np
import pytest

import synth

pytestmark = pytest.mark.gpu

FORMS = ["flat", "hybrid", "lane", "mixed", "bfs", "warp"]
I64 = np.iinfo(np.int64)


@pytest.fixture(params=FORMS)
def M(monkeypatch, request):
    import torch
    if not torch.cuda.is_available():
        pytest.fail("GPU tests need a CUDA device")
    monkeypatch.setenv("MAYURA_KERNEL", request.param)
    import paper_2507_14813_b200 as M
    return M


@pytest.fixture(scope="module")
def c2():
    return synth.CONFIGS["C2"].graph()


@pytest.fixture(scope="module")
def c3():
    return synth.CONFIGS["C3"].graph()


def run(M, src, dst, t, V, motifs, delta, root_range=None):
    g = M.Graph(src, dst, t, V, device=0)
    tree = M.MGTree(motifs, delta)
    out = M.comine(g, tree, root_range)
    g.close()
    tree.close()
    return out


def reverse_time(motifs):
    return [list(reversed(m)) for m in motifs]


def transpose(motifs):
    return [[(v, u) for u, v in m] for m in motifs]


@pytest.mark.parametrize("shift", [-(1 << 40), -(1 << 62)])
def test_shifted_timestamps_c2_vs_oracle(M, oracle_mod, c2, shift):
    """C2 with every timestamp shifted to negative values: GPU == oracle on the shifted graph ==
    GPU on the unshifted graph (the window end t_r + delta must not wrap for t_r < 0)."""
    cfg = synth.CONFIGS["C2"]
    src, dst, t, V = c2
    ts = t + np.int64(shift)
    exp = oracle_mod.backtrack(src, dst, ts, V, cfg.group(), cfg.delta)
    assert run(M, src, dst, ts, V, cfg.group(), cfg.delta) == exp
    assert run(M, src, dst, t, V, cfg.group(), cfg.delta) == exp


def test_time_and_direction_reversal_c2_vs_oracle(M, oracle_mod, c2):
    cfg = synth.CONFIGS["C2"]
    src, dst, t, V = c2
    exp = oracle_mod.backtrack(src, dst, t, V, cfg.group(), cfg.delta)
    assert run(M, src, dst, -t, V, reverse_time(cfg.group()), cfg.delta) == exp
    assert oracle_mod.backtrack(src, dst, -t, V, [_canon(m) for m in reverse_time(cfg.group())], cfg.delta) == exp
    assert run(M, dst, src, t, V, transpose(cfg.group()), cfg.delta) == exp


@pytest.mark.parametrize("kind", ["translate", "time", "direction"])
def test_invariants_c3_scale(M, c3, kind):
    """C3 (7.8 M edges, 12 motifs): the GPU under each transformation equals the GPU on the
    original graph, on the full graph."""
    cfg = synth.CONFIGS["C3"]
    src, dst, t, V = c3
    base = run(M, src, dst, t, V, cfg.group(), cfg.delta)
    assert sum(base) > 0
    if kind == "translate":
        got = run(M, src, dst, t - np.int64(1 << 50), V, cfg.group(), cfg.delta)
    elif kind == "time":
        got = run(M, src, dst, -t, V, reverse_time(cfg.group()), cfg.delta)
    else:
        got = run(M, dst, src, t, V, transpose(cfg.group()), cfg.delta)
    assert got == base


def _canon(m):
    lab, out = {}, []
    for u, v in m:
        for x in (u, v):
            if x not in lab:
                lab[x] = len(lab)
        out.append((lab[u], lab[v]))
    return out


def _extreme_graphs():
    """Small graphs at the ends of the int64 domain, with deltas that make t_r + delta wrap."""
    big = 2 ** 62
    recip, tri = [(0, 1), (1, 0)], [(0, 1), (1, 2), (2, 0)]
    out = [
        ([0, 1], [1, 0], [big, big + 5], [recip], big),
        ([0, 1], [1, 0], [5, 9], [recip], int(I64.max)),
        ([0, 1], [1, 0], [-big, big - 1], [recip], int(I64.max)),
        ([0, 1], [1, 0], [-big, big], [recip], int(I64.max)),
        ([0, 1], [1, 0], [int(I64.min), int(I64.max)], [recip], int(I64.max)),
        ([0, 1, 2], [1, 2, 0], [-7, -3, -1], [tri, recip], 6),
        ([0, 1, 2], [1, 2, 0], [int(I64.max) - 2, int(I64.max) - 1, int(I64.max)], [tri], 2),
    ]
    # random tie-heavy graphs pushed next to INT64_MAX / INT64_MIN with huge deltas
    for seed, (base, delta) in enumerate([(int(I64.max) - 40, int(I64.max)), (int(I64.min), int(I64.max)),
                                          (int(I64.max) - 40, 2 ** 62), (-(2 ** 62), 2 ** 62 + 3)]):
        s, d, t, V = synth.random_graph(700 + seed, 6, 26, 40)
        out.append((s, d, (t + np.int64(base)) if base > 0 else (t.astype(object) + base).astype(np.int64),
                    synth.group(["recip2", "path2", "tri_cycle", "star_out3"]), delta))
    return out


@pytest.mark.parametrize("case", range(11))
def test_int64_extremes_vs_o1(M, oracle_mod, case):
    src, dst, t, motifs, delta = _extreme_graphs()[case]
    src = np.asarray(src, np.uint32)
    dst = np.asarray(dst, np.uint32)
    t = np.asarray(t, np.int64)
    V = int(max(src.max(), dst.max())) + 1
    exp = [oracle_mod.bruteforce(src, dst, t, V, m, delta) for m in motifs]
    assert exp == [oracle_mod.python_bruteforce(src, dst, t, m, delta) for m in motifs]
    assert exp == oracle_mod.backtrack(src, dst, t, V, motifs, delta)
    assert run(M, src, dst, t, V, motifs, delta) == exp
