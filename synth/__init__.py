"""Seeded synthetic inputs shared by the oracle tests, the CUDA-path tests and bench.py.

This module holds NONE of the method's arithmetic (no matching, no windows, no
MG-Tree logic, no counting).  It only draws graphs and motif groups:

* ``random_graph`` / ``random_motif``  -- tiny fuzz instances (ties, self-loops,
  multi-edges) for the brute-force pins.
* ``out_star`` / ``alternating_pair`` / ``cycle_graph`` -- exact structured
  graphs with no RNG, whose counts have closed forms.
* ``cascade_zipf`` -- the "cascade-Zipf" temporal generator of SURVEY.md §8(d):
  power-law (Chung-Lu / Zipf) out/in activity, uniform + bursty background
  events, each spawning a sub-critical Galton-Watson reply/forward cascade with
  1 + Exp(tau) second delays, integer timestamps (hence ties), 0.1 % self-loops.
  It mimics the SNAP email / message / Q&A graphs of PAPER.md Table 1
  (§6 "Five Datasets").
* ``CONFIGS`` -- BASELINE.json ``configs`` C1..C5 made concrete (generator
  parameters, motif group, delta, seed), the recipe stated in DESIGN.md.

Every graph is returned as ``(src u32[E], dst u32[E], t i64[E], n_vertices)`` in
*input order* (not time-sorted): sorting is part of the path under test.
Motifs are lists of (u, v) motif-vertex pairs in temporal order (PAPER.md:123,
"ordered sequence of m edges").
"""
from __future__ import annotations

import dataclasses
from typing import Dict, List, Sequence, Tuple

import numpy as np

Motif = List[Tuple[int, int]]

# --------------------------------------------------------------------------
# Motif library (canonical first-appearance labels; names are ours -- the
# paper's M1..M14 survive only in the lost Fig. 12).
# --------------------------------------------------------------------------
MOTIFS: Dict[str, Motif] = {
    "edge1": [(0, 1)],
    "recip2": [(0, 1), (1, 0)],
    "path2": [(0, 1), (1, 2)],
    "repeat2": [(0, 1), (0, 1)],
    "tri_cycle": [(0, 1), (1, 2), (2, 0)],
    "tri_ff": [(0, 1), (1, 2), (0, 2)],
    "star_out3": [(0, 1), (0, 2), (0, 3)],
    "star_in3": [(0, 1), (2, 1), (3, 1)],
    "path3": [(0, 1), (1, 2), (2, 3)],
    "cycle4": [(0, 1), (1, 2), (2, 3), (3, 0)],
    "path3_back": [(0, 1), (1, 2), (2, 3), (3, 1)],
    "pingpong3": [(0, 1), (1, 0), (0, 1)],
    "star_out4": [(0, 1), (0, 2), (0, 3), (0, 4)],
    "path4": [(0, 1), (1, 2), (2, 3), (3, 4)],
    "cycle5": [(0, 1), (1, 2), (2, 3), (3, 4), (4, 0)],
    "star_in4": [(0, 1), (2, 1), (3, 1), (4, 1)],
    "cycle4_repeat": [(0, 1), (1, 2), (2, 3), (3, 0), (0, 1)],
    "path5": [(0, 1), (1, 2), (2, 3), (3, 4), (4, 5)],
    # AML-style patterns (C5)
    "fan_out3": [(0, 1), (0, 2), (0, 3)],
    "fan_out4": [(0, 1), (0, 2), (0, 3), (0, 4)],
    "fan_in3": [(0, 1), (2, 1), (3, 1)],
    "fan_in4": [(0, 1), (2, 1), (3, 1), (4, 1)],
    "cycle3": [(0, 1), (1, 2), (2, 0)],
    "scatter_gather": [(0, 1), (0, 2), (1, 3), (2, 3)],
}

GROUP_C1 = ["tri_cycle", "tri_ff", "star_out3", "star_in3"]
GROUP_C2 = GROUP_C1 + ["path3", "cycle4", "path3_back", "pingpong3"]
GROUP_C3 = GROUP_C2 + ["recip2", "path2", "star_out4", "path4"]
GROUP_C4 = GROUP_C3 + ["cycle5", "star_in4", "cycle4_repeat", "path5"]
GROUP_C5 = ["fan_out3", "fan_out4", "fan_in3", "fan_in4", "cycle3", "cycle4", "cycle5",
            "scatter_gather"]


def group(names: Sequence[str]) -> List[Motif]:
    return [list(MOTIFS[n]) for n in names]


# --------------------------------------------------------------------------
# Tiny fuzz instances
# --------------------------------------------------------------------------
def random_graph(seed: int, n_vertices: int, n_edges: int, t_max: int,
                 self_loop_frac: float = 0.05):
    """Uniform random multigraph with integer timestamps in [0, t_max] (ties when
    t_max is small), a few self-loops and parallel edges."""
    rng = np.random.default_rng(seed)
    src = rng.integers(0, n_vertices, n_edges, dtype=np.int64)
    dst = rng.integers(0, n_vertices, n_edges, dtype=np.int64)
    loops = rng.random(n_edges) < self_loop_frac
    dst = np.where(loops, src, dst)
    t = rng.integers(0, t_max + 1, n_edges, dtype=np.int64)
    return src.astype(np.uint32), dst.astype(np.uint32), t.astype(np.int64), int(n_vertices)


def random_motif(seed: int, m: int, max_vertices: int = 4, relabel: bool = True) -> Motif:
    """Random motif with m edges, no motif self-loops, connected in temporal order is
    NOT required (prefix-disconnected motifs exercise the all-edges candidate path).
    With relabel=True the vertex labels are a random (non-canonical) permutation."""
    rng = np.random.default_rng(seed)
    edges: Motif = []
    for _ in range(m):
        while True:
            u = int(rng.integers(0, max_vertices))
            v = int(rng.integers(0, max_vertices))
            if u != v:
                break
        edges.append((u, v))
    if relabel:
        perm = rng.permutation(max_vertices + 3) + 2  # labels need not be dense
        edges = [(int(perm[u]), int(perm[v])) for u, v in edges]
    return edges


# --------------------------------------------------------------------------
# Closed-form structured graphs (no RNG)
# --------------------------------------------------------------------------
def out_star(n: int):
    """Edges 0 -> i at t = i for i = 1..n."""
    i = np.arange(1, n + 1, dtype=np.int64)
    return (np.zeros(n, np.uint32), i.astype(np.uint32), i.copy(), n + 1)


def alternating_pair(n: int):
    """A=0 -> B=1 at odd t, B -> A at even t, t = 1..n."""
    t = np.arange(1, n + 1, dtype=np.int64)
    odd = (t % 2) == 1
    src = np.where(odd, 0, 1).astype(np.uint32)
    dst = np.where(odd, 1, 0).astype(np.uint32)
    return src, dst, t, 2


def cycle_graph(L: int, n: int):
    """Edge k = (k mod L) -> ((k+1) mod L) at t = k, k = 0..n-1."""
    k = np.arange(n, dtype=np.int64)
    return ((k % L).astype(np.uint32), ((k + 1) % L).astype(np.uint32), k.copy(), L)


# --------------------------------------------------------------------------
# cascade-Zipf temporal generator
# --------------------------------------------------------------------------
def _zipf_weights(n: int, alpha: float) -> np.ndarray:
    # Chung-Lu weights (i+1)^(-1/(alpha-1)) give a power-law degree tail of exponent alpha.
    w = (np.arange(n, dtype=np.float64) + 1.0) ** (-1.0 / (alpha - 1.0))
    return w / w.sum()


def _hash_u64(x: np.ndarray) -> np.ndarray:
    """SplitMix64 finaliser (counter-based, used only to pick stable 'contacts')."""
    z = (x.astype(np.uint64) + np.uint64(0x9E3779B97F4A7C15))
    z = (z ^ (z >> np.uint64(30))) * np.uint64(0xBF58476D1CE4E5B9)
    z = (z ^ (z >> np.uint64(27))) * np.uint64(0x94D049BB133111EB)
    return z ^ (z >> np.uint64(31))


def cascade_zipf(n_vertices: int, n_edges: int, span: int, alpha: float, p: float,
                 tau: float, seed: int, burst_frac: float = 0.0, burst_width: float = 600.0,
                 n_bursts: int = 0, self_loop_frac: float = 0.001, n_contacts: int = 4):
    """Power-law, bursty temporal graph with reply/forward cascades.

    * out-activity and in-activity of vertex i ~ Zipf weights under two independent
      random permutations (power-law out/in degrees);
    * background events: t ~ U[0, span) (a fraction ``burst_frac`` instead drawn
      around ``n_bursts`` burst centres with N(0, burst_width) jitter);
    * each event spawns j children with P(>= j) = p^j, j <= 4 (mean < 1: sub-critical);
      a child is sent by the parent's destination after 1 + Exp(tau) seconds to
      the parent's source (reply, 40 %), to one of ``n_contacts`` stable contacts
      of the sender (30 %), or to a Zipf-random vertex (30 %);
    * timestamps are integer seconds (ties); 0.1 % of edges are made self-loops.
    Exactly ``n_edges`` edges are returned, in a shuffled input order.
    """
    rng = np.random.default_rng(seed)
    w_out = _zipf_weights(n_vertices, alpha)
    w_in = _zipf_weights(n_vertices, alpha)
    perm_out = rng.permutation(n_vertices)
    perm_in = rng.permutation(n_vertices)
    cdf_out = np.cumsum(w_out)
    cdf_in = np.cumsum(w_in)

    def zipf_out(k):
        return perm_out[np.minimum(np.searchsorted(cdf_out, rng.random(k)), n_vertices - 1)]

    def zipf_in(k):
        return perm_in[np.minimum(np.searchsorted(cdf_in, rng.random(k)), n_vertices - 1)]

    mean_children = sum(p ** j for j in range(1, 5))
    n_bg = max(1, int(n_edges * (1.0 - mean_children) * 1.02))
    centres = rng.random(max(n_bursts, 1)) * span

    out_s, out_d, out_t = [], [], []
    total = 0
    while total < n_edges:
        # background events
        bs = zipf_out(n_bg)
        bd = zipf_in(n_bg)
        same = bs == bd
        while same.any():
            bd[same] = zipf_in(int(same.sum()))
            same = bs == bd
        bt = rng.random(n_bg) * span
        if burst_frac > 0 and n_bursts > 0:
            inb = rng.random(n_bg) < burst_frac
            c = centres[rng.integers(0, n_bursts, int(inb.sum()))]
            bt[inb] = np.clip(c + rng.normal(0.0, burst_width, int(inb.sum())), 0, span - 1)
        lvl_s, lvl_d, lvl_t = bs, bd, np.floor(bt)
        while lvl_s.size and total < n_edges:
            out_s.append(lvl_s); out_d.append(lvl_d); out_t.append(lvl_t)
            total += lvl_s.size
            # children per event: P(>= j) = p^j, capped at 4
            u = rng.random(lvl_s.size)
            nchild = np.zeros(lvl_s.size, np.int64)
            for j in range(1, 5):
                nchild += (u < p ** j)
            par = np.repeat(np.arange(lvl_s.size), nchild)
            if par.size == 0:
                break
            ps, pd, pt = lvl_s[par], lvl_d[par], lvl_t[par]
            cs = pd.copy()
            kind = rng.random(par.size)
            cd = np.empty_like(cs)
            rep = kind < 0.4
            con = (kind >= 0.4) & (kind < 0.7)
            rnd = kind >= 0.7
            cd[rep] = ps[rep]
            j = rng.integers(0, n_contacts, int(con.sum()))
            h = _hash_u64(cs[con].astype(np.uint64) * np.uint64(64) + j.astype(np.uint64) +
                          np.uint64(seed) * np.uint64(1_000_003))
            # stable contact = Zipf-distributed pick driven by the hash
            hu = (h >> np.uint64(11)).astype(np.float64) / float(1 << 53)
            cd[con] = perm_in[np.minimum(np.searchsorted(cdf_in, hu), n_vertices - 1)]
            cd[rnd] = zipf_in(int(rnd.sum()))
            fix = cd == cs
            if fix.any():
                cd[fix] = ps[fix]
            ct = np.floor(pt + 1.0 + rng.exponential(tau, par.size))
            keep = ct < span
            lvl_s, lvl_d, lvl_t = cs[keep], cd[keep], ct[keep]
    src = np.concatenate(out_s)[:n_edges].astype(np.uint32)
    dst = np.concatenate(out_d)[:n_edges].astype(np.uint32)
    t = np.concatenate(out_t)[:n_edges].astype(np.int64)
    n_loops = int(round(self_loop_frac * n_edges))
    if n_loops:
        idx = rng.choice(n_edges, n_loops, replace=False)
        dst[idx] = src[idx]
    order = rng.permutation(n_edges)
    return src[order], dst[order], t[order], int(n_vertices)


# --------------------------------------------------------------------------
# Planted AML patterns (C5; "fan-out/fan-in k = 3-6 within delta/2,
# cycles 3-5 within delta, scatter-gather"; the pattern names follow the AML work the paper
# cites)
# --------------------------------------------------------------------------
PLANT_KINDS = ("fan_out", "fan_in", "cycle", "scatter_gather")


def plant_aml(n_patterns: int, n_vertices: int, span: int, delta: int, seed: int):
    """n_patterns laundering-style patterns, kinds in rotation, each on fresh random vertices
    (distinct within a pattern) with strictly increasing timestamps:
      fan_out k (k = 3..6): s -> d_1..d_k inside delta/2;   fan_in k: s_1..s_k -> d inside delta/2;
      cycle L (L = 3..5): v_0 -> v_1 -> ... -> v_{L-1} -> v_0 inside delta;
      scatter_gather: s -> m_1, s -> m_2, then m_1 -> d, m_2 -> d inside delta.
    Returns (src, dst, t, planted) with planted[kind][size] = number of instances."""
    rng = np.random.default_rng(seed + 7_777_777)
    out_s, out_d, out_t = [], [], []
    planted = {k: {} for k in PLANT_KINDS}
    for i in range(n_patterns):
        kind = PLANT_KINDS[i % len(PLANT_KINDS)]
        t0 = int(rng.integers(0, max(1, span - delta)))
        if kind in ("fan_out", "fan_in"):
            k = int(rng.integers(3, 7))
            vs = rng.choice(n_vertices, k + 1, replace=False)
            ts = t0 + np.sort(rng.choice(max(k, delta // 2), k, replace=False))
            hub, others = int(vs[0]), vs[1:]
            for v, tt in zip(others, ts):
                out_s.append(hub if kind == "fan_out" else int(v))
                out_d.append(int(v) if kind == "fan_out" else hub)
                out_t.append(int(tt))
            planted[kind][k] = planted[kind].get(k, 0) + 1
        elif kind == "cycle":
            L = int(rng.integers(3, 6))
            vs = rng.choice(n_vertices, L, replace=False)
            ts = t0 + np.sort(rng.choice(max(L, delta), L, replace=False))
            for j in range(L):
                out_s.append(int(vs[j])); out_d.append(int(vs[(j + 1) % L])); out_t.append(int(ts[j]))
            planted[kind][L] = planted[kind].get(L, 0) + 1
        else:
            vs = rng.choice(n_vertices, 4, replace=False)
            ts = t0 + np.sort(rng.choice(max(4, delta), 4, replace=False))
            s_, m1, m2, d_ = (int(x) for x in vs)
            for (a, b), tt in zip(((s_, m1), (s_, m2), (m1, d_), (m2, d_)), ts):
                out_s.append(a); out_d.append(b); out_t.append(int(tt))
            planted[kind][2] = planted[kind].get(2, 0) + 1
    return (np.array(out_s, np.uint32), np.array(out_d, np.uint32), np.array(out_t, np.int64), planted)


# --------------------------------------------------------------------------
# Workload configs (BASELINE.json "configs", made concrete)
# --------------------------------------------------------------------------
DAY = 86400


@dataclasses.dataclass(frozen=True)
class Config:
    name: str
    title: str
    n_vertices: int
    n_edges: int
    span: int
    delta: int
    motifs: Tuple[str, ...]
    alpha: float
    p: float
    tau: float
    seed: int
    burst_frac: float = 0.0
    burst_width: float = 600.0
    n_bursts: int = 0
    planted: int = 0          # AML patterns planted on top of the background (C5)

    def graph(self, cache: bool = True):
        """(src, dst, t, V) in input order.  Workloads of >= 1 M edges go through the versioned
        binary cache (synth/cache.py): the first process on a machine generates and writes it,
        the others (N bench ranks, the second bench arm, later test modules) load it."""
        if cache and self.n_edges >= 1_000_000:
            from . import cache as _cache
            return _cache.cached(self)
        return self.generate()

    def generate(self):
        if not self.planted:
            return cascade_zipf(self.n_vertices, self.n_edges, self.span, self.alpha, self.p,
                                self.tau, self.seed, self.burst_frac, self.burst_width,
                                self.n_bursts)
        return self.graph_planted()[:4]

    def graph_planted(self):
        """(src, dst, t, V, planted): background cascade-Zipf edges plus planted AML
        patterns, n_edges in total, shuffled together."""
        ps, pd, pt, planted = plant_aml(self.planted, self.n_vertices, self.span, self.delta, self.seed)
        bs, bd, bt, V = cascade_zipf(self.n_vertices, self.n_edges - ps.size, self.span, self.alpha, self.p,
                                     self.tau, self.seed, self.burst_frac, self.burst_width, self.n_bursts)
        order = np.random.default_rng(self.seed + 1).permutation(self.n_edges)
        return (np.concatenate([bs, ps])[order], np.concatenate([bd, pd])[order],
                np.concatenate([bt, pt])[order], V, planted)

    def group(self) -> List[Motif]:
        return group(self.motifs)


CONFIGS: Dict[str, Config] = {
    "C1": Config("C1", "synthetic 1k nodes / 20k edges, delta=600s, 4 three-edge motifs",
                 1_000, 20_000, 1 * DAY, 600, tuple(GROUP_C1), 2.2, 0.45, 60.0, 1),
    "C2": Config("C2", "email-Eu-core-temporal-shaped 1k nodes / 330k edges, delta=3600s, 8 motifs",
                 1_000, 330_000, 803 * DAY, 3600, tuple(GROUP_C2), 2.0, 0.45, 120.0, 2,
                 burst_frac=0.3, burst_width=1800.0, n_bursts=2000),
    "C3": Config("C3", "wiki-talk-temporal-shaped 1.14M nodes / 7.83M edges, delta=3600s, 12 motifs",
                 1_140_149, 7_833_140, int(6.24 * 365 * DAY), 3600, tuple(GROUP_C3), 2.1, 0.45,
                 120.0, 3, burst_frac=0.2, burst_width=1800.0, n_bursts=20000),
    # alpha calibrated (SURVEY.md §8(d) calibration rule: tune the generator, not delta): at
    # alpha = 2.1 the top vertex takes ~2.4 % of all edges (~550 per day), and 4-edge stars
    # at delta = 1 day give ~1e6 matches per root; alpha = 2.5 gives a top vertex of ~31 edges
    # per day (the SNAP stackoverflow-temporal order of magnitude) and ~60 matches per root.
    "C4": Config("C4", "stackoverflow-temporal-shaped 2.6M nodes / 63.5M edges, delta=86400s, 16 motifs",
                 2_601_977, 63_497_050, int(7.6 * 365 * DAY), 86400, tuple(GROUP_C4), 2.5, 0.40,
                 600.0, 4),
    # alpha calibrated as for C4 (at 2.0 the top vertex takes ~6 % of 500 M edges, ~1,000 per
    # hour, and fan-out-4 at delta = 1 h explodes); 2.5 keeps hubs at ~25 edges per hour.
    "C5": Config("C5", "transaction-graph-shaped (AML) 10M nodes / 500M edges, delta=3600s, 8 motifs",
                 10_000_000, 500_000_000, int(3.58 * 365 * DAY), 3600, tuple(GROUP_C5), 2.5, 0.40,
                 120.0, 5, planted=200_000),
    # C5's recipe at 1/250 scale (same span density per vertex is NOT preserved: a test-sized
    # instance the oracle finishes in full, for exact parity and the planted lower bounds)
    "C5s": Config("C5s", "AML-shaped test instance 40k nodes / 2M edges, delta=3600s, 8 motifs",
                  40_000, 2_000_000, 60 * DAY, 3600, tuple(GROUP_C5), 2.5, 0.40, 120.0, 55,
                  planted=4_000),
}
