"""CPU oracle for MG-Tree temporal motif co-mining -- TEST INFRASTRUCTURE ONLY.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s ``cpu_baseline`` /
``--impl reference`` legs may import this package.  The product path
(``paper_2507_14813_b200``) never imports it and shares no code with it.

* ``bruteforce``  (O1) -- the plain definition of a delta-temporal motif match
  (§2.1), tuple enumeration; guarded to small graphs.
* ``backtrack``   (O2) -- Algorithm 1 "Temporal Motif Mining",
  every motif mined independently, threaded over root edges.
* ``enumerate_matches`` -- O2 in enumeration form (Algo 1 l.201): one row of
  input edge indices per match, single-threaded.
* ``python_bruteforce`` -- a second, independent brute force in pure Python
  (itertools), for tiny inputs only.

Readings of the paper (ties, window closure, injectivity ...) are listed in
DESIGN.md §3.  Pins: tests/test_oracle_pins.py.
"""
from __future__ import annotations

import ctypes
import itertools
import os
import subprocess
from typing import List, Optional, Sequence, Tuple

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "mayura_oracle.c")
_LIB = os.path.join(_HERE, "liboracle.so")
_lib = None


def build(force: bool = False) -> str:
    """Compile the C oracle (plain gcc, -O2, pthreads)."""
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        tmp = _LIB + ".tmp%d" % os.getpid()
        subprocess.check_call(["gcc", "-O2", "-std=c11", "-Wall", "-Wextra", "-shared", "-fPIC",
                               "-pthread", _SRC, "-o", tmp])
        os.replace(tmp, _LIB)
    return _LIB


def _load():
    global _lib
    if _lib is None:
        build()
        lib = ctypes.CDLL(_LIB)
        P = ctypes.c_void_p
        u64, u32, i64, i32 = ctypes.c_uint64, ctypes.c_uint32, ctypes.c_int64, ctypes.c_int
        lib.oracle_bruteforce.argtypes = [P, P, P, u64, u32, P, u32, i64, u64, u64, u64, P]
        lib.oracle_bruteforce.restype = i32
        lib.oracle_backtrack.argtypes = [P, P, P, u64, u32, P, P, u32, i64, u64, u64, i32, P]
        lib.oracle_backtrack.restype = i32
        lib.oracle_backtrack_ranges.argtypes = [P, P, P, u64, u32, P, P, u32, i64, P, u32, i32, P, P,
                                                ctypes.c_double, P]
        lib.oracle_backtrack_ranges.restype = i32
        lib.oracle_enumerate.argtypes = [P, P, P, u64, u32, P, u32, i64, u64, u64, P, u64, P]
        lib.oracle_enumerate.restype = i32
        lib.oracle_sorted_order.argtypes = [P, u64, P]
        lib.oracle_sorted_order.restype = i32
        _lib = lib
    return _lib


def _arr(a, dtype):
    return np.ascontiguousarray(np.asarray(a, dtype=dtype))


def _ptr(a: np.ndarray):
    return a.ctypes.data_as(ctypes.c_void_p)


class OracleError(RuntimeError):
    pass


def bruteforce(src, dst, t, n_vertices: int, motif: Sequence[Tuple[int, int]], delta: int,
               root_range: Optional[Tuple[int, int]] = None, guard: int = 5000) -> int:
    """O1: count of one motif by enumerating time-increasing edge tuples."""
    lib = _load()
    s, d, tt = _arr(src, np.uint32), _arr(dst, np.uint32), _arr(t, np.int64)
    E = s.size
    rb, re_ = root_range if root_range is not None else (0, E)
    me = _arr([x for e in motif for x in e], np.uint32)
    out = np.zeros(1, np.uint64)
    rc = lib.oracle_bruteforce(_ptr(s), _ptr(d), _ptr(tt), E, n_vertices, _ptr(me), len(motif),
                               int(delta), rb, re_, guard, _ptr(out))
    if rc != 0:
        raise OracleError("oracle_bruteforce failed rc=%d" % rc)
    return int(out[0])


def backtrack(src, dst, t, n_vertices: int, motifs: Sequence[Sequence[Tuple[int, int]]],
              delta: int, root_range: Optional[Tuple[int, int]] = None,
              threads: Optional[int] = None) -> List[int]:
    """O2: per-motif counts, each motif mined independently by Algorithm 1."""
    lib = _load()
    s, d, tt = _arr(src, np.uint32), _arr(dst, np.uint32), _arr(t, np.int64)
    E = s.size
    rb, re_ = root_range if root_range is not None else (0, E)
    me = _arr([x for m in motifs for e in m for x in e], np.uint32)
    ml = _arr([len(m) for m in motifs], np.uint32)
    out = np.zeros(len(motifs), np.uint64)
    nt = threads if threads is not None else (os.cpu_count() or 1)
    rc = lib.oracle_backtrack(_ptr(s), _ptr(d), _ptr(tt), E, n_vertices, _ptr(me), _ptr(ml),
                              len(motifs), int(delta), rb, re_, nt, _ptr(out))
    if rc != 0:
        raise OracleError("oracle_backtrack failed rc=%d" % rc)
    return [int(x) for x in out]


def backtrack_ranges(src, dst, t, n_vertices: int, motifs: Sequence[Sequence[Tuple[int, int]]],
                     delta: int, ranges: Sequence[Tuple[int, int]], threads: Optional[int] = None,
                     budget_s: float = 0.0):
    """O2 over several root ranges of one graph build: ([[count per motif] per mined range],
    build seconds, mining seconds).  budget_s > 0: ranges are started only while less than
    budget_s seconds of mining have elapsed, so the result covers a prefix of `ranges`."""
    lib = _load()
    s, d, tt = _arr(src, np.uint32), _arr(dst, np.uint32), _arr(t, np.int64)
    E = s.size
    me = _arr([x for m in motifs for e in m for x in e], np.uint32)
    ml = _arr([len(m) for m in motifs], np.uint32)
    rg = _arr([x for r in ranges for x in r], np.uint64)
    out = np.zeros(len(ranges) * len(motifs), np.uint64)
    secs = np.zeros(2, np.float64)
    done = np.zeros(1, np.uint32)
    nt = threads if threads is not None else (os.cpu_count() or 1)
    rc = lib.oracle_backtrack_ranges(_ptr(s), _ptr(d), _ptr(tt), E, n_vertices, _ptr(me), _ptr(ml),
                                     len(motifs), int(delta), _ptr(rg), len(ranges), nt, _ptr(out), _ptr(secs),
                                     float(budget_s), _ptr(done))
    if rc != 0:
        raise OracleError("oracle_backtrack_ranges failed rc=%d" % rc)
    k = len(motifs)
    return ([[int(x) for x in out[i * k:(i + 1) * k]] for i in range(int(done[0]))],
            float(secs[0]), float(secs[1]))


def enumerate_matches(src, dst, t, n_vertices: int, motif: Sequence[Tuple[int, int]], delta: int,
                      root_range: Optional[Tuple[int, int]] = None) -> np.ndarray:
    """O2 in enumeration form (Algo 1 l.201): a (count, m) array of input edge indices,
    one row per match of `motif`, edges in motif order."""
    lib = _load()
    s, d, tt = _arr(src, np.uint32), _arr(dst, np.uint32), _arr(t, np.int64)
    E = s.size
    rb, re_ = root_range if root_range is not None else (0, E)
    me = _arr([x for e in motif for x in e], np.uint32)
    m = len(motif)
    cnt = np.zeros(1, np.uint64)
    rc = lib.oracle_enumerate(_ptr(s), _ptr(d), _ptr(tt), E, n_vertices, _ptr(me), m, int(delta), rb, re_,
                              None, 0, _ptr(cnt))
    if rc not in (0, -2):
        raise OracleError("oracle_enumerate failed rc=%d" % rc)
    n = int(cnt[0])
    out = np.zeros(max(n * m, 1), np.uint32)
    rc = lib.oracle_enumerate(_ptr(s), _ptr(d), _ptr(tt), E, n_vertices, _ptr(me), m, int(delta), rb, re_,
                              _ptr(out), n, _ptr(cnt))
    if rc != 0:
        raise OracleError("oracle_enumerate failed rc=%d" % rc)
    return out[:n * m].reshape(n, m)


def sorted_order(t) -> np.ndarray:
    """Input ranks in (t, input rank) order -- the oracle's edge-id assignment."""
    lib = _load()
    tt = _arr(t, np.int64)
    perm = np.zeros(tt.size, np.uint64)
    rc = lib.oracle_sorted_order(_ptr(tt), tt.size, _ptr(perm))
    if rc != 0:
        raise OracleError("oracle_sorted_order failed")
    return perm.astype(np.int64)


def python_bruteforce(src, dst, t, motif: Sequence[Tuple[int, int]], delta: int) -> int:
    """Independent twin of O1 in pure Python: all m-subsets of edges, ordered by time,
    checked against the definition.  Exponential -- tiny inputs only (<= ~25 edges)."""
    edges = list(zip([int(x) for x in src], [int(x) for x in dst], [int(x) for x in t]))
    m = len(motif)
    n = 0
    for combo in itertools.combinations(range(len(edges)), m):
        tup = sorted((edges[i] for i in combo), key=lambda e: e[2])
        ts = [e[2] for e in tup]
        if any(ts[i] >= ts[i + 1] for i in range(m - 1)):
            continue
        if ts[-1] - ts[0] > delta:
            continue
        phi = {}
        ok = True
        for (a, b), (gs, gd, _) in zip(motif, tup):
            for mv, gv in ((a, gs), (b, gd)):
                if phi.setdefault(mv, gv) != gv:
                    ok = False
        if ok and len(set(phi.values())) == len(phi):
            n += 1
    return n
