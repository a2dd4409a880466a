// graph_build.cpp -- host graph builder (step a0).
//
// "Data-Loading" of PAPER.md:415,420 (§4.2): the edge list is turned into
// time-ordered edge arrays and per-vertex adjacency "with edges sorted in
// ascending order of timestamps".  B200-first layout:
//   src/dst/tr u32 [E], t i64 [E]  in edge-id order, ids = stable (t, input rank) order
//   tr[e] = id of the first edge whose timestamp equals t[e]  (time rank: tr_a < tr_b
//           <=> t_a < t_b, so the strict order test is one u32 compare, reading R1)
//   out_off/in_off u32 [V+1], out_ent/in_ent (tr, nbr) u32 pairs [E]
// Every stage is a parallel, stable LSD radix sort or a parallel scan.
#include <algorithm>
#include <atomic>
#include <cstring>
#include <functional>
#include <thread>

#include "internal.h"

namespace mayura {

int host_threads() {
    unsigned n = std::thread::hardware_concurrency();
    return n == 0 ? 1 : (int)std::min(n, 128u);
}

static void parallel_chunks(size_t n, int T, const std::function<void(size_t, size_t, int)> &fn) {
    if (n < 65536 || T <= 1) {
        fn(0, n, 0);
        return;
    }
    std::vector<std::thread> th;
    size_t per = (n + T - 1) / T;
    for (int i = 0; i < T; i++) {
        size_t lo = std::min(n, per * i), hi = std::min(n, per * (i + 1));
        th.emplace_back(fn, lo, hi, i);
    }
    for (auto &x : th) x.join();
}

// Stable LSD radix sort of (key, value) pairs on the low `bits` bits of key.
template <typename K>
static void radix_sort_kv(std::vector<K> &k, std::vector<uint32_t> &v, int bits, int T) {
    const size_t n = k.size();
    if (n < 2 || bits <= 0) return;
    std::vector<K> k2(n);
    std::vector<uint32_t> v2(n);
    const int D = 8, B = 1 << D;
    int Tn = (n < 65536) ? 1 : T;
    size_t per = (n + Tn - 1) / Tn;
    std::vector<size_t> hist((size_t)Tn * B);
    for (int shift = 0; shift < bits; shift += D) {
        std::fill(hist.begin(), hist.end(), 0);
        parallel_chunks(n, Tn, [&](size_t lo, size_t hi, int tid) {
            size_t *h = &hist[(size_t)tid * B];
            for (size_t i = lo; i < hi; i++) h[(k[i] >> shift) & (B - 1)]++;
        });
        size_t sum = 0;
        for (int d = 0; d < B; d++)
            for (int t = 0; t < Tn; t++) {
                size_t c = hist[(size_t)t * B + d];
                hist[(size_t)t * B + d] = sum;
                sum += c;
            }
        (void)per;
        parallel_chunks(n, Tn, [&](size_t lo, size_t hi, int tid) {
            size_t *h = &hist[(size_t)tid * B];
            for (size_t i = lo; i < hi; i++) {
                size_t pos = h[(k[i] >> shift) & (B - 1)]++;
                k2[pos] = k[i];
                v2[pos] = v[i];
            }
        });
        k.swap(k2);
        v.swap(v2);
    }
}

static int bits_for(uint64_t maxval) {
    int b = 0;
    while (b < 64 && (maxval >> b) != 0) b++;
    return b;
}

// Build one CSR direction: key[e] = vertex owning edge e in this direction, nbr[e] = other end.
// Each list is followed by a sentinel entry (tr = nbr = 0xFFFFFFFF) so a window scan can stop
// on "time rank > window end" alone; off[x] = start of list x, off[x+1] - 1 = its sentinel.
static void build_csr(const std::vector<uint32_t> &key, const std::vector<uint32_t> &nbr,
                      const std::vector<uint32_t> &tr, uint32_t V, int T,
                      std::vector<uint32_t> &off, std::vector<uint32_t> &ent, std::vector<uint32_t> &ids_out) {
    const size_t E = key.size();
    std::vector<uint32_t> k(key);
    std::vector<uint32_t> ids(E);
    parallel_chunks(E, T, [&](size_t lo, size_t hi, int) {
        for (size_t i = lo; i < hi; i++) ids[i] = (uint32_t)i;
    });
    radix_sort_kv(k, ids, bits_for(V ? V - 1 : 0), T);  // stable: ids ascending within a vertex
    off.assign((size_t)V + 1, 0);
    parallel_chunks((size_t)V + 1, T, [&](size_t lo, size_t hi, int) {
        for (size_t x = lo; x < hi; x++)  // + x: one sentinel slot per earlier list
            off[x] = (uint32_t)(std::lower_bound(k.begin(), k.end(), (uint32_t)x) - k.begin() + x);
    });
    const size_t N = E + V;
    ent.assign(2 * N, 0xFFFFFFFFu);
    ids_out.assign(N, 0xFFFFFFFFu);
    parallel_chunks(E, T, [&](size_t lo, size_t hi, int) {
        for (size_t i = lo; i < hi; i++) {
            const uint32_t e = ids[i];
            const size_t pos = i + k[i];  // sorted position + number of sentinels before it
            ent[2 * pos] = tr[e];
            ent[2 * pos + 1] = nbr[e];
            ids_out[pos] = e;
        }
    });
}

// P(e): first position with time rank > tr[e] in the four lists an edge's endpoints own.
static void build_succ(mayura_graph_s *g, const std::vector<uint32_t> &out_ids,
                       const std::vector<uint32_t> &in_ids, int T) {
    const size_t E = g->E, N = E + g->V;
    g->eptr.assign(4 * E, 0);
    auto first_after = [&](const std::vector<uint32_t> &off, const std::vector<uint32_t> &ent, uint32_t x,
                           uint32_t key) -> uint32_t {
        uint32_t lo = off[x], hi = off[x + 1] - 1;  // [lo, hi) excludes the sentinel
        while (lo < hi) {
            uint32_t mid = lo + (hi - lo) / 2;
            if (ent[2 * (size_t)mid] > key) hi = mid;
            else lo = mid + 1;
        }
        return lo;
    };
    parallel_chunks(E, T, [&](size_t lo, size_t hi, int) {
        for (size_t e = lo; e < hi; e++) {
            const uint32_t a = g->src[e], b = g->dst[e], key = g->tr[e];
            g->eptr[4 * e + 0] = first_after(g->out_off, g->out_ent, a, key);
            g->eptr[4 * e + 1] = first_after(g->in_off, g->in_ent, b, key);
            g->eptr[4 * e + 2] = first_after(g->out_off, g->out_ent, b, key);
            g->eptr[4 * e + 3] = first_after(g->in_off, g->in_ent, a, key);
        }
    });
    g->out_ptr.assign(4 * N, 0);
    g->in_ptr.assign(4 * N, 0);
    parallel_chunks(N, T, [&](size_t lo, size_t hi, int) {
        for (size_t i = lo; i < hi; i++) {
            if (out_ids[i] != 0xFFFFFFFFu)
                for (int j = 0; j < 4; j++) g->out_ptr[4 * i + j] = g->eptr[4 * (size_t)out_ids[i] + j];
            if (in_ids[i] != 0xFFFFFFFFu)
                for (int j = 0; j < 4; j++) g->in_ptr[4 * i + j] = g->eptr[4 * (size_t)in_ids[i] + j];
        }
    });
}

mayura_status build_graph_host(const uint32_t *src, const uint32_t *dst, const int64_t *t,
                               uint64_t E, uint32_t V, mayura_graph_s *g) {
    const int T = host_threads();
    g->E = E;
    g->V = V;
    // validate vertex ids
    std::atomic<bool> bad{false};
    parallel_chunks(E, T, [&](size_t lo, size_t hi, int) {
        for (size_t i = lo; i < hi; i++)
            if (src[i] >= V || dst[i] >= V) {
                bad = true;
                return;
            }
    });
    if (bad) return fail(MAYURA_E_INVALID, "mayura_load_graph: vertex id >= n_vertices");

    // 1. stable sort by (t, input rank): radix on t - t_min, values = input rank
    int64_t tmin = 0, tmax = 0;
    if (E) {
        tmin = tmax = t[0];
        for (uint64_t i = 1; i < E; i++) {
            tmin = std::min(tmin, t[i]);
            tmax = std::max(tmax, t[i]);
        }
    }
    std::vector<uint64_t> key(E);
    std::vector<uint32_t> rank(E);
    parallel_chunks(E, T, [&](size_t lo, size_t hi, int) {
        for (size_t i = lo; i < hi; i++) {
            key[i] = (uint64_t)t[i] - (uint64_t)tmin;
            rank[i] = (uint32_t)i;
        }
    });
    radix_sort_kv(key, rank, bits_for((uint64_t)tmax - (uint64_t)tmin), T);
    key.clear();
    key.shrink_to_fit();

    g->src.resize(E);
    g->dst.resize(E);
    g->t.resize(E);
    g->tr.resize(E);
    g->perm.resize(E);
    parallel_chunks(E, T, [&](size_t lo, size_t hi, int) {
        for (size_t i = lo; i < hi; i++) {
            uint32_t r = rank[i];
            g->src[i] = src[r];
            g->dst[i] = dst[r];
            g->t[i] = t[r];
            g->perm[i] = r;
        }
    });
    // 2. time rank: tr[e] = first id with the same timestamp
    parallel_chunks(E, T, [&](size_t lo, size_t hi, int) {
        if (lo >= hi) return;
        uint32_t cur = (uint32_t)(std::lower_bound(g->t.begin(), g->t.begin() + lo, g->t[lo]) -
                                  g->t.begin());
        g->tr[lo] = cur;
        for (size_t i = lo + 1; i < hi; i++) {
            if (g->t[i] != g->t[i - 1]) cur = (uint32_t)i;
            g->tr[i] = cur;
        }
    });
    // 3. out/in adjacency, each list in increasing edge id (= timestamp) order
    if (E + (uint64_t)V + 64 > 0xFFFFFFFFull)
        return fail(MAYURA_E_LIMIT, "mayura_load_graph: n_edges + n_vertices exceeds 32-bit list positions");
    std::vector<uint32_t> out_ids, in_ids;
    build_csr(g->src, g->dst, g->tr, V, T, g->out_off, g->out_ent, out_ids);
    build_csr(g->dst, g->src, g->tr, V, T, g->in_off, g->in_ent, in_ids);
    // 4. successor pointers
    build_succ(g, out_ids, in_ids, T);
    return MAYURA_OK;
}

}  // namespace mayura
