"""Thin ctypes binding of libmayura.so (include/mayura.h) -- argument marshalling only.

Every function of the C ABI is exposed under the same name; every step of the
co-mining path runs in the library's CUDA kernels.  There is no CPU fallback:
if the shared library is missing this module raises at import time.

Convenience wrappers ``Graph`` / ``MGTree`` own the opaque handles and free them.
Arrays are numpy (host) or, for ``counts_on_device=True``, any object exposing a
CUDA device pointer via ``data_ptr()`` (a torch tensor of dtype int64/uint64).
"""
from __future__ import annotations

import ctypes
import os
from typing import List, Optional, Sequence, Tuple

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("MAYURA_LIB_PATH") or os.path.join(_HERE, "lib", "libmayura.so")  # override: A/B builds

if not os.path.exists(LIB_PATH):
    raise ImportError("libmayura.so not built (%s); run `python -m paper_2507_14813_b200.build` "
                      "or __graft_entry__.build()" % LIB_PATH)

_lib = ctypes.CDLL(LIB_PATH)

_P = ctypes.c_void_p
_u64, _u32, _i64, _int, _dbl, _sz = (ctypes.c_uint64, ctypes.c_uint32, ctypes.c_int64, ctypes.c_int,
                                      ctypes.c_double, ctypes.c_size_t)
_PP = ctypes.POINTER(ctypes.c_void_p)

SIGNATURES = {
    "mayura_load_graph": ([_P, _P, _P, _u64, _u32, _int, _PP], _int),
    "mayura_graph_info": ([_P, _P, _P, _P], _int),
    "mayura_graph_export": ([_P, _P, _P, _P, _P, _P, _P, _P, _P, _P], _int),
    "mayura_graph_export_succ": ([_P, _P], _int),
    "mayura_free_graph": ([_P], None),
    "mayura_build_mgtree": ([_P, _P, _u32, _i64, _PP], _int),
    "mayura_mgtree_info": ([_P, _P, _P, _P, _P, _P, _P], _int),
    "mayura_mgtree_dump": ([_P, _P, _sz, _P], _int),
    "mayura_free_mgtree": ([_P], None),
    "mayura_comine": ([_P, _P, _u64, _u64, _P, _P, _int], _int),
    "mayura_mine_independent": ([_P, _P, _u64, _u64, _P, _P, _int], _int),
    "mayura_comine_ex": ([_P, _P, _u64, _u64, _P, _P, _int, _int, _P], _int),
    "mayura_comine_stats": ([_P, _P, _u64, _u64, _int, _P], _int),
    "mayura_partition_roots": ([_P, _i64, _u32, _P], _int),
    "mayura_enumerate": ([_P, _P, _u64, _u64, _P, _P, _u64, _int, _P, _P], _int),
    "mayura_comine_heuristic": ([_P, _P, _P, _P, _P], _int),
    "mayura_last_error": ([], ctypes.c_char_p),
    "mayura_kernel_form": ([_P], ctypes.c_char_p),
    "mayura_enum_form": ([_P], ctypes.c_char_p),
    "mayura_version": ([], ctypes.c_char_p),
    "mayura_launch_count": ([], _u64),
}
for _name, (_args, _res) in SIGNATURES.items():
    _f = getattr(_lib, _name)
    _f.argtypes = _args
    _f.restype = _res

STATUS = {0: "MAYURA_OK", -1: "MAYURA_E_INVALID", -2: "MAYURA_E_LIMIT", -3: "MAYURA_E_OOM",
          -4: "MAYURA_E_CUDA", -5: "MAYURA_E_STATE"}
STATS_FIELDS = ("roots", "nodes", "windows", "entries", "probes", "batches", "bytes_alg", "matches",
                "offloads", "contexts")


class MayuraError(RuntimeError):
    def __init__(self, status: int, msg: str):
        super().__init__("%s: %s" % (STATUS.get(status, status), msg))
        self.status = status


def _check(rc: int):
    if rc != 0:
        raise MayuraError(rc, mayura_last_error())


def _np(a, dtype):
    return np.ascontiguousarray(np.asarray(a, dtype=dtype))


def _ptr(a: Optional[np.ndarray]):
    return None if a is None else a.ctypes.data_as(ctypes.c_void_p)


# ------------------------------------------------------------ raw ABI names --
def mayura_last_error() -> str:
    return (_lib.mayura_last_error() or b"").decode()


def mayura_version() -> str:
    return _lib.mayura_version().decode()


def mayura_kernel_form(g: int) -> str:
    return _lib.mayura_kernel_form(g).decode()


def mayura_enum_form(g: int) -> str:
    return _lib.mayura_enum_form(g).decode()


def mayura_launch_count() -> int:
    """The library's own kernel launches enqueued so far in this process."""
    return int(_lib.mayura_launch_count())


def mayura_load_graph(src, dst, t, n_vertices: int, device: int = 0) -> int:
    s, d, tt = _np(src, np.uint32), _np(dst, np.uint32), _np(t, np.int64)
    if not (s.size == d.size == tt.size):
        raise ValueError("src, dst, t must have the same length")
    h = ctypes.c_void_p()
    _check(_lib.mayura_load_graph(_ptr(s), _ptr(d), _ptr(tt), s.size, int(n_vertices), int(device),
                                  ctypes.byref(h)))
    return h.value


def mayura_graph_info(g: int) -> Tuple[int, int, int]:
    e, v, b = ctypes.c_uint64(), ctypes.c_uint32(), ctypes.c_uint64()
    _check(_lib.mayura_graph_info(g, ctypes.byref(e), ctypes.byref(v), ctypes.byref(b)))
    return e.value, v.value, b.value


def mayura_graph_export(g: int) -> dict:
    E, V, _ = mayura_graph_info(g)
    out = dict(src=np.empty(E, np.uint32), dst=np.empty(E, np.uint32), t=np.empty(E, np.int64),
               tr=np.empty(E, np.uint32), perm=np.empty(E, np.uint64),
               out_off=np.empty(V + 1, np.uint32), out_ent=np.empty(2 * (E + V), np.uint32),
               in_off=np.empty(V + 1, np.uint32), in_ent=np.empty(2 * (E + V), np.uint32))
    _check(_lib.mayura_graph_export(g, *[_ptr(out[k]) for k in ("src", "dst", "t", "tr", "perm", "out_off",
                                                                 "out_ent", "in_off", "in_ent")]))
    return out


def mayura_graph_export_succ(g: int) -> np.ndarray:
    E, _, _ = mayura_graph_info(g)
    out = np.empty(4 * E, np.uint32)
    _check(_lib.mayura_graph_export_succ(g, _ptr(out)))
    return out.reshape(E, 4)


def mayura_free_graph(g: int) -> None:
    _lib.mayura_free_graph(g)


def _motif_arrays(motifs: Sequence[Sequence[Tuple[int, int]]]):
    edges = _np([x for m in motifs for e in m for x in e], np.uint32)
    lens = _np([len(m) for m in motifs], np.uint32)
    return edges, lens


def mayura_build_mgtree(motifs: Sequence[Sequence[Tuple[int, int]]], delta: int) -> int:
    edges, lens = _motif_arrays(motifs)
    h = ctypes.c_void_p()
    _check(_lib.mayura_build_mgtree(_ptr(edges) if edges.size else None, _ptr(lens) if lens.size else None,
                                    len(motifs), int(delta), ctypes.byref(h)))
    return h.value


def mayura_mgtree_info(m: int) -> dict:
    v = [ctypes.c_uint32() for _ in range(5)]
    sm = ctypes.c_double()
    _check(_lib.mayura_mgtree_info(m, *[ctypes.byref(x) for x in v], ctypes.byref(sm)))
    return dict(n_motifs=v[0].value, n_trie_nodes=v[1].value, n_mg_nodes=v[2].value,
                max_vertices=v[3].value, max_edges=v[4].value, sm=sm.value)


def mayura_mgtree_dump(m: int) -> str:
    need = ctypes.c_size_t()
    _check(_lib.mayura_mgtree_dump(m, None, 0, ctypes.byref(need)))
    buf = ctypes.create_string_buffer(need.value)
    _check(_lib.mayura_mgtree_dump(m, buf, need.value, ctypes.byref(need)))
    return buf.value.decode()


def mayura_free_mgtree(m: int) -> None:
    _lib.mayura_free_mgtree(m)


def _counts_call(fn, g, m, root_begin, root_end, stream, counts_out):
    k = mayura_mgtree_info(m)["n_motifs"]
    if counts_out is None:
        host = np.zeros(k, np.uint64)
        _check(fn(g, m, root_begin, root_end, stream, _ptr(host), 0))
        return [int(x) for x in host]
    _check(fn(g, m, root_begin, root_end, stream, ctypes.c_void_p(counts_out.data_ptr()), 1))
    return counts_out


def mayura_comine(g: int, m: int, root_begin: int, root_end: int, stream: Optional[int] = None,
                  counts_out=None):
    """Co-mine roots [root_begin, root_end).  counts_out=None -> host list of ints (synchronous);
    counts_out=<device tensor of k int64> -> enqueued on `stream`, returns the tensor."""
    return _counts_call(_lib.mayura_comine, g, m, root_begin, root_end, stream, counts_out)


def mayura_mine_independent(g: int, m: int, root_begin: int, root_end: int,
                            stream: Optional[int] = None, counts_out=None):
    return _counts_call(_lib.mayura_mine_independent, g, m, root_begin, root_end, stream, counts_out)


def mayura_comine_ex(g: int, m: int, root_begin: int, root_end: int, stream: Optional[int],
                     counts_out, independent: bool = False, mid_event: Optional[int] = None):
    """Device-output co-mining (or independent) call that records the cudaEvent_t
    `mid_event` between the window-end kernel and the co-mining kernel(s)."""
    _check(_lib.mayura_comine_ex(g, m, root_begin, root_end, stream, ctypes.c_void_p(counts_out.data_ptr()), 1,
                                 int(independent), mid_event))
    return counts_out


def mayura_comine_stats(g: int, m: int, root_begin: int, root_end: int, independent: bool = False) -> dict:
    out = np.zeros(len(STATS_FIELDS), np.uint64)
    _check(_lib.mayura_comine_stats(g, m, root_begin, root_end, int(independent), _ptr(out)))
    return dict(zip(STATS_FIELDS, (int(x) for x in out)))


def mayura_enumerate(g: int, m: int, root_begin: int, root_end: int, stream: Optional[int] = None,
                     tuples_out=None, capacity_words: int = 0):
    """Enumerate the matches of roots [root_begin, root_end).

    tuples_out=None: the library writes into a host buffer sized by a first (size-query)
    call; returns (counts, words) with words a uint32 numpy array.  tuples_out=<device
    tensor of >= capacity_words int32/uint32>: written in place on the device; returns
    (counts, words_needed).  Layout: include/mayura.h (motif q's tuples at W_q, len_q input
    edge indices each)."""
    k = mayura_mgtree_info(m)["n_motifs"]
    counts = np.zeros(k, np.uint64)
    need = ctypes.c_uint64(0)
    if tuples_out is not None:
        _check(_lib.mayura_enumerate(g, m, root_begin, root_end, stream, ctypes.c_void_p(tuples_out.data_ptr()),
                                     int(capacity_words), 1, _ptr(counts), ctypes.byref(need)))
        return [int(x) for x in counts], int(need.value)
    _check(_lib.mayura_enumerate(g, m, root_begin, root_end, stream, None, 0, 0, _ptr(counts), ctypes.byref(need)))
    words = np.zeros(max(int(need.value), 1), np.uint32)
    _check(_lib.mayura_enumerate(g, m, root_begin, root_end, stream, _ptr(words), int(need.value), 0, _ptr(counts),
                                 ctypes.byref(need)))
    return [int(x) for x in counts], words[:int(need.value)]


def mayura_enumerate_size(g: int, m: int, root_begin: int, root_end: int, stream: Optional[int] = None):
    """Size query of mayura_enumerate (tuples_out = NULL): (counts, words needed)."""
    k = mayura_mgtree_info(m)["n_motifs"]
    counts = np.zeros(k, np.uint64)
    need = ctypes.c_uint64(0)
    _check(_lib.mayura_enumerate(g, m, root_begin, root_end, stream, None, 0, 0, _ptr(counts), ctypes.byref(need)))
    return [int(x) for x in counts], int(need.value)


def split_tuples(counts: Sequence[int], lens: Sequence[int], words: np.ndarray) -> List[np.ndarray]:
    """The enumeration buffer split per motif: a (count_q, len_q) array of input edge indices."""
    out, w = [], 0
    for c, L in zip(counts, lens):
        out.append(np.asarray(words[w:w + c * L]).reshape(c, L))
        w += c * L
    return out


def mayura_comine_heuristic(g: int, m: int) -> dict:
    """The paper's co-mining heuristic: {use_comine, bipartite, sm}."""
    use, bip, sm = ctypes.c_int(0), ctypes.c_int(0), ctypes.c_double(0.0)
    _check(_lib.mayura_comine_heuristic(g, m, ctypes.byref(use), ctypes.byref(bip), ctypes.byref(sm)))
    return {"use_comine": bool(use.value), "bipartite": bool(bip.value), "sm": sm.value}


def mayura_partition_roots(g: int, delta: int, n_parts: int) -> List[int]:
    out = np.zeros(n_parts + 1, np.uint64)
    _check(_lib.mayura_partition_roots(g, int(delta), int(n_parts), _ptr(out)))
    return [int(x) for x in out]


# -------------------------------------------------------------- wrappers --
class Graph:
    """Owns a mayura_graph handle.  device=-1: host-only (inspection / partitioning)."""

    def __init__(self, src, dst, t, n_vertices: int, device: int = 0):
        self.handle = mayura_load_graph(src, dst, t, n_vertices, device)
        self.device = device
        self.n_edges, self.n_vertices, self.device_bytes = mayura_graph_info(self.handle)

    def export(self) -> dict:
        d = mayura_graph_export(self.handle)
        d["eptr"] = mayura_graph_export_succ(self.handle)
        return d

    def partition(self, delta: int, n_parts: int) -> List[int]:
        return mayura_partition_roots(self.handle, delta, n_parts)

    def close(self):
        if self.handle:
            mayura_free_graph(self.handle)
            self.handle = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


class MGTree:
    """Owns a mayura_mgtree handle (compiled motif group + delta)."""

    def __init__(self, motifs: Sequence[Sequence[Tuple[int, int]]], delta: int):
        self.handle = mayura_build_mgtree(motifs, delta)
        self.info = mayura_mgtree_info(self.handle)
        self.n_motifs = self.info["n_motifs"]
        self.delta = delta
        self.lens = [len(mo) for mo in motifs]

    def dump(self) -> str:
        return mayura_mgtree_dump(self.handle)

    def close(self):
        if self.handle:
            mayura_free_mgtree(self.handle)
            self.handle = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def comine(graph: Graph, tree: MGTree, root_range: Optional[Tuple[int, int]] = None,
           stream: Optional[int] = None, counts_out=None):
    rb, re_ = root_range if root_range is not None else (0, graph.n_edges)
    return mayura_comine(graph.handle, tree.handle, rb, re_, stream, counts_out)


def mine_independent(graph: Graph, tree: MGTree, root_range: Optional[Tuple[int, int]] = None,
                     stream: Optional[int] = None, counts_out=None):
    rb, re_ = root_range if root_range is not None else (0, graph.n_edges)
    return mayura_mine_independent(graph.handle, tree.handle, rb, re_, stream, counts_out)


def comine_stats(graph: Graph, tree: MGTree, root_range=None, independent: bool = False) -> dict:
    rb, re_ = root_range if root_range is not None else (0, graph.n_edges)
    return mayura_comine_stats(graph.handle, tree.handle, rb, re_, independent)


def enumerate_matches(graph: Graph, tree: MGTree, root_range=None, stream: Optional[int] = None):
    """Host enumeration: (counts, [per-motif (count, len) arrays of input edge indices])."""
    rb, re_ = root_range if root_range is not None else (0, graph.n_edges)
    counts, words = mayura_enumerate(graph.handle, tree.handle, rb, re_, stream)
    return counts, split_tuples(counts, tree.lens, words)
