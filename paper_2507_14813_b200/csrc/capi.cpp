// capi.cpp -- host-only entry points of the C ABI (include/mayura.h): errors,
// graph inspection, MG-Tree build/inspection, multi-GPU root partitioning.
#include <algorithm>
#include <cstring>
#include <new>

#include "internal.h"

namespace mayura {
static thread_local std::string g_last_error;

mayura_status fail(mayura_status s, const std::string &msg) {
    g_last_error = msg;
    return s;
}
void clear_error() { g_last_error.clear(); }
}  // namespace mayura

using namespace mayura;

extern "C" const char *mayura_last_error(void) { return g_last_error.c_str(); }

extern "C" const char *mayura_version(void) { return "mayura-b200 0.3 sm_100a"; }

namespace mayura {
uint64_t launch_count();
}
extern "C" uint64_t mayura_launch_count(void) { return mayura::launch_count(); }

extern "C" mayura_status mayura_graph_info(mayura_graph g, uint64_t *n_edges, uint32_t *n_vertices,
                                           uint64_t *device_bytes) {
    clear_error();
    if (!g) return fail(MAYURA_E_INVALID, "mayura_graph_info: NULL handle");
    if (n_edges) *n_edges = g->E;
    if (n_vertices) *n_vertices = g->V;
    if (device_bytes) *device_bytes = g->device_bytes;
    return MAYURA_OK;
}

extern "C" mayura_status mayura_graph_export(mayura_graph g, uint32_t *src, uint32_t *dst, int64_t *t,
                                             uint32_t *tr, uint64_t *perm, uint32_t *out_off,
                                             uint32_t *out_ent, uint32_t *in_off, uint32_t *in_ent) {
    clear_error();
    if (!g) return fail(MAYURA_E_INVALID, "mayura_graph_export: NULL handle");
    if (mayura_status s = ensure_host(g)) return s;  // device-built graph: download once
    const size_t E = (size_t)g->E, V1 = (size_t)g->V + 1;
    if (src) std::memcpy(src, g->src.data(), 4 * E);
    if (dst) std::memcpy(dst, g->dst.data(), 4 * E);
    if (t) std::memcpy(t, g->t.data(), 8 * E);
    if (tr) std::memcpy(tr, g->tr.data(), 4 * E);
    if (perm) std::memcpy(perm, g->perm.data(), 8 * E);
    if (out_off) std::memcpy(out_off, g->out_off.data(), 4 * V1);
    if (in_off) std::memcpy(in_off, g->in_off.data(), 4 * V1);
    if (out_ent) std::memcpy(out_ent, g->out_ent.data(), 4 * g->out_ent.size());
    if (in_ent) std::memcpy(in_ent, g->in_ent.data(), 4 * g->in_ent.size());
    return MAYURA_OK;
}

extern "C" mayura_status mayura_graph_export_succ(mayura_graph g, uint32_t *eptr) {
    clear_error();
    if (!g || !eptr) return fail(MAYURA_E_INVALID, "mayura_graph_export_succ: NULL argument");
    if (mayura_status s = ensure_host(g)) return s;
    std::memcpy(eptr, g->eptr.data(), 4 * g->eptr.size());
    return MAYURA_OK;
}

extern "C" mayura_status mayura_build_mgtree(const uint32_t *motif_edges, const uint32_t *motif_len,
                                             uint32_t n_motifs, int64_t delta, mayura_mgtree *out) {
    clear_error();
    if (!out) return fail(MAYURA_E_INVALID, "mayura_build_mgtree: out is NULL");
    mayura_mgtree_s *m = new (std::nothrow) mayura_mgtree_s();
    if (!m) return fail(MAYURA_E_OOM, "mayura_build_mgtree: out of host memory");
    mayura_status s;
    try {
        s = compile_tree(motif_edges, motif_len, n_motifs, delta, m);
    } catch (const std::bad_alloc &) {
        s = fail(MAYURA_E_OOM, "mayura_build_mgtree: out of host memory");
    }
    if (s != MAYURA_OK) {
        delete m;
        return s;
    }
    *out = m;
    return MAYURA_OK;
}

extern "C" mayura_status mayura_mgtree_info(mayura_mgtree m, uint32_t *n_motifs, uint32_t *n_trie_nodes,
                                            uint32_t *n_mg_nodes, uint32_t *max_vertices, uint32_t *max_edges,
                                            double *sm) {
    clear_error();
    if (!m) return fail(MAYURA_E_INVALID, "mayura_mgtree_info: NULL handle");
    if (n_motifs) *n_motifs = m->n_motifs;
    if (n_trie_nodes) *n_trie_nodes = (uint32_t)m->group.nodes.size();
    if (n_mg_nodes) *n_mg_nodes = m->n_mg_nodes;
    if (max_vertices) *max_vertices = m->group.max_vertices;
    if (max_edges) *max_edges = m->group.max_edges;
    if (sm) *sm = m->sm;
    return MAYURA_OK;
}

extern "C" mayura_status mayura_mgtree_dump(mayura_mgtree m, char *buf, size_t cap, size_t *needed) {
    clear_error();
    if (!m) return fail(MAYURA_E_INVALID, "mayura_mgtree_dump: NULL handle");
    if (needed) *needed = m->dump.size() + 1;
    if (buf && cap > 0) {
        size_t n = std::min(cap - 1, m->dump.size());
        std::memcpy(buf, m->dump.data(), n);
        buf[n] = 0;
    }
    return MAYURA_OK;
}

extern "C" void mayura_free_mgtree(mayura_mgtree m) {
    if (!m) return;
    free_mgtree_device(m);
    delete m;
}

// Work-balanced contiguous split of the root ids.  Proxy work of root r:
//   p(r) = 1 + min(s_r, 65535)^2,  s_r = entries of the four adjacency lists at the root's
//   endpoints (out(src), in(dst), out(dst), in(src)) with t_r < t <= t_r + delta
// (the root's level-1 window sizes; squared because the search below a root grows with
// products of window sizes).  Cut points at equal shares of the prefix sum:
//   bounds[p] = first r with prefix(r) >= floor(total * p / P)  (non-decreasing).
// Host graphs compute it here; device-built graphs on the GPU (graph_gpu.cu, same
// integer arithmetic, same bounds).
namespace mayura {
uint64_t proxy_host(const mayura_graph_s *g, uint64_t r, uint32_t H) {
    const uint32_t a = g->src[r], b = g->dst[r];
    const uint32_t xs[4] = {a, b, b, a};
    const std::vector<uint32_t> *offs[4] = {&g->out_off, &g->in_off, &g->out_off, &g->in_off};
    const std::vector<uint32_t> *ents[4] = {&g->out_ent, &g->in_ent, &g->out_ent, &g->in_ent};
    uint64_t s = 0;
    for (int k = 0; k < 4; k++) {
        uint32_t lo = g->eptr[4 * r + k], hi = (*offs[k])[xs[k] + 1] - 1;  // sentinel at hi
        const uint32_t start = lo;
        while (lo < hi) {  // first position with time rank > H
            const uint32_t m = lo + (hi - lo) / 2;
            if ((*ents[k])[2 * (size_t)m] > H) hi = m;
            else lo = m + 1;
        }
        s += lo - start;
    }
    s = std::min<uint64_t>(s, 65535);
    return 1 + s * s;
}
}  // namespace mayura

extern "C" mayura_status mayura_partition_roots(mayura_graph g, int64_t delta, uint32_t n_parts,
                                                uint64_t *bounds_out) {
    clear_error();
    if (!g || !bounds_out || n_parts == 0) return fail(MAYURA_E_INVALID, "mayura_partition_roots: bad argument");
    if (delta < 0) return fail(MAYURA_E_INVALID, "mayura_partition_roots: delta < 0");
    const uint64_t E = g->E;
    std::vector<uint64_t> cut(n_parts + 1, 0);  // raw first-index for each share
    if (!g->host_built) {
        if (mayura_status s = partition_device(g, delta, n_parts, cut.data())) return s;
    } else {
        const std::vector<int64_t> &t = g->t;
        std::vector<uint64_t> pref(E + 1, 0);
        uint64_t k = 0;  // first index with t > t_r + delta
        for (uint64_t r = 0; r < E; r++) {
            const int64_t lim = (t[r] > INT64_MAX - delta) ? INT64_MAX : t[r] + delta;  // delta >= 0: no overflow
            if (k < r + 1) k = r + 1;
            while (k < E && t[k] <= lim) k++;
            pref[r + 1] = pref[r] + proxy_host(g, r, (uint32_t)(k - 1));
        }
        const uint64_t total = pref[E];
        for (uint32_t p = 1; p < n_parts; p++) {
            const uint64_t target = (total / n_parts) * p + ((total % n_parts) * p) / n_parts;
            cut[p] = (uint64_t)(std::lower_bound(pref.begin(), pref.end(), target) - pref.begin());
        }
    }
    bounds_out[0] = 0;
    for (uint32_t p = 1; p < n_parts; p++) bounds_out[p] = std::max(std::min<uint64_t>(cut[p], E), bounds_out[p - 1]);
    bounds_out[n_parts] = E;
    return MAYURA_OK;
}

// NEXT-4: the paper's co-mining heuristic (§6 "Heuristic for Co-Mining";
// its Listing "heuristic.py" is figure-only, reading R18): co-mining always paid off on
// bipartite graphs, and otherwise needs a Similarity Metric of at least 0.44.
// Bipartiteness of the underlying undirected graph: union-find with parity over the edges
// (an edge joins opposite colours; a self-loop is an odd cycle).
namespace mayura {
namespace {
bool graph_bipartite(const std::vector<uint32_t> &src, const std::vector<uint32_t> &dst, uint32_t V) {
    std::vector<uint32_t> parent(V), par(V, 0);  // par: colour relative to the parent
    for (uint32_t v = 0; v < V; v++) parent[v] = v;
    auto find = [&](uint32_t x, uint32_t &colour) {
        uint32_t c = 0, r = x;
        while (parent[r] != r) {
            c ^= par[r];
            r = parent[r];
        }
        // path compression: point x's chain at the root with its colour relative to it
        uint32_t cx = c;
        while (parent[x] != r && parent[x] != x) {
            const uint32_t nx = parent[x], px = par[x];
            parent[x] = r;
            par[x] = cx;
            cx ^= px;
            x = nx;
        }
        colour = c;
        return r;
    };
    for (size_t i = 0; i < src.size(); i++) {
        const uint32_t a = src[i], b = dst[i];
        if (a == b) return false;
        uint32_t ca = 0, cb = 0;
        const uint32_t ra = find(a, ca), rb = find(b, cb);
        if (ra == rb) {
            if (ca == cb) return false;
        } else {
            parent[ra] = rb;
            par[ra] = ca ^ cb ^ 1u;  // colour(a) != colour(b)
        }
    }
    return true;
}
}  // namespace
}  // namespace mayura

extern "C" mayura_status mayura_comine_heuristic(mayura_graph g, mayura_mgtree m, int *use_comine, int *bipartite,
                                                 double *sm) {
    clear_error();
    if (!g || !m) return fail(MAYURA_E_INVALID, "mayura_comine_heuristic: NULL handle");
    if (mayura_status s = ensure_host(g)) return s;
    bool bip;
    try {
        bip = graph_bipartite(g->src, g->dst, g->V);
    } catch (const std::bad_alloc &) {
        return fail(MAYURA_E_OOM, "mayura_comine_heuristic: out of host memory");
    }
    if (bipartite) *bipartite = bip ? 1 : 0;
    if (sm) *sm = m->sm;
    if (use_comine) *use_comine = (bip || m->sm >= 0.44) ? 1 : 0;
    return MAYURA_OK;
}
