// bfs.cuh -- level-synchronous co-mining (kernel v4, the default), included by comine.cu.
//
// Algorithm 3 "Co-Mining" expands, for every root edge, a search
// tree whose level-k vertices are partial matches of the MG-Tree node at depth k.  The
// depth-first walk of one root per warp (v2) or per lane (v3) is a chain of dependent
// loads: profiles (profiles/r01_*.md, tools/warp_timeline.py) showed a few dozen
// warp-iterations per warp at 2-8 us each.  Here the search trees of ALL roots advance
// one MG-Tree level per pass, so every pass is a wide, independent stream:
//
//   pass k, thread per partial match x of depth k (the frontier F_k, 16-byte records):
//     for each anchor group of node(x): locate the window (successor pointers P of x's
//     last edge, the root's R, a binary search, or the edge array -- Algo 1 l.210-214),
//     scan it (time test, class of the neighbour against m2g, at most one child per
//     class -- Algo 1 l.219 + full injectivity R4):
//       completion child  -> count[Q_N]++                          (Algo 3 l.661)
//       pre-leaf child    -> its (short) leaf windows are counted inline
//       other inner child -> a record appended to F_{k+1}           (Algo 3 l.665-669)
//     windows of >= kLong entries are deferred to a warp-per-window pass (coalesced
//     32-entry batches, one ballot per child).
//   Appends go to one of kStripes segments (warp-aggregated atomics on 64 counters).
//   A full segment never loses work: the thread mines that subtree depth-first itself
//   (`dfs`, local-memory frames) -- correct by construction, rare by sizing.
// Counts are u32 per thread in shared memory (flushed before overflow), reduced per
// block and added to the per-motif u64 counts with one atomic per block and motif.

namespace bfs {

constexpr int kTB = 256;            // threads per block (expand pass)
constexpr int kStripes = 64;        // output segments per level
constexpr uint32_t kLong = 16;      // windows of >= kLong entries go to the warp pass
constexpr int kTile = 4;            // entries loaded together at a window's start
constexpr int kMaxLevels = MAYURA_MAX_EDGES;
constexpr uint8_t NODE_PRELEAF = 8; // LNode flag: has children, all of them leaves

template <int MAXV>
struct Rec {  // words per frontier record: node|nv<<16, root, tr_prev, h, P(4), m2g(MAXV)
    static constexpr int W = (8 + MAXV + 3) & ~3;
};

struct Front {
    uint32_t *data;  // kStripes segments x seg_cap records
    uint32_t *cnt;   // kStripes counters (records appended; may exceed seg_cap)
    uint32_t seg_cap;
};

struct BParams {
    const uint32_t *src, *dst, *tr, *hi;
    const int64_t *T;        // flat form: timestamps, so its level-0 pass computes hi (else null)
    int64_t delta;
    uint32_t E;
    uint32_t *hi_w;          // hi, writable (the flat level-0 pass stores what it computed)
    const uint4 *eptr;
    const uint32_t *out_off, *in_off;
    const uint2 *out_ent, *in_ent;
    const uint4 *out_ptr, *in_ptr;
    const lane::LNode *nodes;
    const DGroup *groups;
    const uint32_t *motif_node;
    uint32_t n_nodes, n_groups, n_motifs, n_slots;
    uint32_t r0, n_roots;
    Front in, out;
    uint32_t *long_items;  // 3 words per item: frontier index, group, window start
    uint32_t *long_cnt;    // [0] items appended
    uint32_t long_cap;
    uint32_t *fallback;    // [0] subtrees mined depth-first because a segment was full
    uint32_t inline_preleaf;  // 1: count short pre-leaf windows inline (v4); 0: emit every inner child
    uint32_t heavy_min;       // level 0 of the hybrid: a root is split breadth-first only if one of its
                              // windows has >= heavy_min entries; lighter roots are handed to the
                              // depth-first kernel whole, as a root record (0: split every root)
    uint32_t *light;          // heavy_min > 0: the light roots, listed for the depth-first kernel (warp-
    uint32_t *light_cnt;      //   aggregated appends; [0] = entries), so it needs no heavy test of its own
    unsigned long long *counts;
    unsigned long long *stats;
};

// ------------------------------------------------------------------ state
template <int MAXV>
struct PM {  // one partial match (a vertex of the search tree)
    uint32_t node, nv, root, tr_prev, h;
    uint4 P;            // successor pointers of the partial match's last edge
    uint32_t m2g[MAXV]; // kNone beyond nv
};

struct Ctx {  // per-thread counters + stats
    uint32_t *cnt;      // this thread's counters: slot s at cnt[s * stride]
    uint32_t stride;
    unsigned long long *tot;
    unsigned long long st[ST_N];
    uint32_t em_next, em_end;  // this thread's reserved run of output slots (chunked appends)
};
constexpr uint32_t kChunk = 8;     // output slots a thread reserves at once (expand pass)
constexpr uint32_t kHole = 0xFFFFu; // node id of an unused reserved slot (skipped by readers)

__device__ __forceinline__ void count_add(Ctx &c, uint32_t slot, uint32_t n) {
    if (!c.cnt) {  // groups with many completion slots: block-shared u64 counters (thread_cnt)
        atomicAdd(&c.tot[slot], (unsigned long long)n);
        return;
    }
    uint32_t *q = c.cnt + slot * c.stride;
    uint32_t v = *q + n;
    if (v >= 0x80000000u) {
        atomicAdd(&c.tot[slot], (unsigned long long)v);
        v = 0;
    }
    *q = v;
}

template <int MAXV, bool STATS>
__device__ __forceinline__ uint32_t window_start(const BParams &p, const DGroup &G, const PM<MAXV> &x,
                                                 uint32_t &lim, Ctx &c) {
    lim = kNone;
    if (G.start < START_R0) return lane::pick4(x.P, G.start);
    if (G.start < START_SEARCH) {
        const uint4 R = __ldg(p.eptr + x.root);
        return lane::pick4(R, G.start - START_R0);
    }
    if (G.start == START_SEARCH) {
        const uint32_t v = lane::m2g_get<MAXV>(x.m2g, G.anchor);
        const uint32_t *off = (G.kind == ANCHOR_OUT) ? p.out_off : p.in_off;
        const uint2 *ent = (G.kind == ANCHOR_OUT) ? p.out_ent : p.in_ent;
        uint32_t lo = __ldg(off + v), hi2 = __ldg(off + v + 1) - 1;
        while (lo < hi2) {
            const uint32_t mid = lo + ((hi2 - lo) >> 1);
            if (__ldg(&ent[mid].x) > x.tr_prev) hi2 = mid;
            else lo = mid + 1;
            if (STATS) c.st[ST_PROBES]++;
        }
        if (STATS) c.st[ST_BYTES] += 8;
        return lo;
    }
    // GLOBAL: edge ids after the tie group of the last edge, up to hi(root) (reading R6)
    uint32_t lo = x.tr_prev, hi2 = x.h + 1;
    while (lo < hi2) {
        const uint32_t mid = lo + ((hi2 - lo) >> 1);
        if (__ldg(p.tr + mid) > x.tr_prev) hi2 = mid;
        else lo = mid + 1;
        if (STATS) c.st[ST_PROBES]++;
    }
    lim = x.h + 1;
    return lo;
}

// entry `pos` of group G's list: time rank, neighbour (lists) or (src, dst) (edge array)
__device__ __forceinline__ void load_entry(const BParams &p, const DGroup &G, uint32_t pos, uint32_t lim,
                                           uint32_t &etr, uint32_t &e1, uint32_t &e2) {
    if (G.kind == ANCHOR_GLOBAL) {
        if (pos < lim) {
            etr = __ldg(p.tr + pos);
            e1 = __ldg(p.src + pos);
            e2 = __ldg(p.dst + pos);
        } else {
            etr = kNone; e1 = e2 = 0;
        }
    } else {
        const uint2 e = __ldg((G.kind == ANCHOR_OUT ? p.out_ent : p.in_ent) + pos);
        etr = e.x; e1 = e.y; e2 = 0;
    }
}

template <int MAXV>
__device__ __forceinline__ uint32_t entry_class(const DGroup &G, const uint32_t (&m)[MAXV], uint32_t e1,
                                                uint32_t e2) {
    if (G.kind == ANCHOR_GLOBAL)
        return (e1 != e2 && lane::classify<MAXV>(m, e1) == CLS_NEW && lane::classify<MAXV>(m, e2) == CLS_NEW)
                   ? CLS_NEW : 0xFEu;
    return lane::classify<MAXV>(m, e1);
}

__device__ __forceinline__ uint32_t find_child(const lane::LNode *nodes, const DGroup &G, uint32_t cls) {
    for (uint32_t c = G.child_begin; c < G.child_end; ++c)
        if (nodes[c].want == cls) return c;
    return kNone;
}

// the child partial match created by matching entry (etr, e1, e2) at position pos
template <int MAXV>
__device__ __forceinline__ void make_child(const BParams &p, const DGroup &G, const lane::LNode &dn, uint32_t c,
                                           const PM<MAXV> &x, uint32_t pos, uint32_t etr, uint32_t e1, uint32_t e2,
                                           PM<MAXV> &y) {
#pragma unroll
    for (int k = 0; k < MAXV; k++) y.m2g[k] = x.m2g[k];
    if (dn.n_new >= 1) lane::m2g_set<MAXV>(y.m2g, x.nv, e1);
    if (dn.n_new == 2) lane::m2g_set<MAXV>(y.m2g, x.nv + 1, e2);
    y.nv = dn.nv;
    y.node = c;
    y.root = x.root;
    y.h = x.h;
    y.tr_prev = etr;
    y.P = (G.kind == ANCHOR_GLOBAL) ? __ldg(p.eptr + pos)
                                    : __ldg((G.kind == ANCHOR_OUT ? p.out_ptr : p.in_ptr) + pos);
}

// Depth-first mining of the subtree below partial match x (the rare fallback when the
// next frontier is full): one thread, frames in local memory.
template <int MAXV, bool STATS>
__device__ __noinline__ void dfs(const BParams &p, const lane::LNode *nodes, const DGroup *groups, PM<MAXV> x,
                                 Ctx &c, uint32_t g_first = kNone) {  // g_first: start at this group of x
    struct Fr {
        uint32_t node, nv, g, pos, lim, tr_prev;
        uint4 P;
        uint32_t m2g[MAXV];
    } fr[kMaxLevels];
    int d = 0;
    uint32_t g = g_first != kNone ? g_first : nodes[x.node].group_begin, pos = 0, lim = kNone;
    bool scan = false;
    for (;;) {
        const lane::LNode xn = nodes[x.node];
        if (!scan) {
            if (g == xn.group_end) {
                if (d == 0) return;
                --d;
                x.node = fr[d].node; x.nv = fr[d].nv; x.tr_prev = fr[d].tr_prev; x.P = fr[d].P;
#pragma unroll
                for (int k = 0; k < MAXV; k++) x.m2g[k] = fr[d].m2g[k];
                g = fr[d].g; pos = fr[d].pos; lim = fr[d].lim;
                scan = true;
                continue;
            }
            pos = window_start<MAXV, STATS>(p, groups[g], x, lim, c);
            if (STATS) c.st[ST_WINDOWS]++;
            scan = true;
        }
        const DGroup G = groups[g];
        uint32_t etr, e1, e2;
        load_entry(p, G, pos, lim, etr, e1, e2);
        if (etr > x.h || pos >= lim) {
            ++g;
            scan = false;
            continue;
        }
        ++pos;
        if (etr <= x.tr_prev) continue;
        if (STATS) { c.st[ST_ENTRIES]++; c.st[ST_BYTES] += G.kind == ANCHOR_GLOBAL ? 12 : 8; }
        const uint32_t ch = find_child(nodes, G, entry_class<MAXV>(G, x.m2g, e1, e2));
        if (ch == kNone) continue;
        const lane::LNode dn = nodes[ch];
        if (dn.flags & NODE_COMPLETION) {
            count_add(c, dn.slot, 1);
            if (STATS) c.st[ST_MATCHES]++;
        }
        if (dn.flags & NODE_INNER) {
            fr[d].node = x.node; fr[d].nv = x.nv; fr[d].tr_prev = x.tr_prev; fr[d].P = x.P;
#pragma unroll
            for (int k = 0; k < MAXV; k++) fr[d].m2g[k] = x.m2g[k];
            fr[d].g = g; fr[d].pos = pos; fr[d].lim = lim;
            ++d;
            PM<MAXV> y;
            make_child<MAXV>(p, G, dn, ch, x, pos - 1, etr, e1, e2, y);
            x = y;
            g = dn.group_begin;
            scan = false;
            if (STATS) { c.st[ST_NODES]++; c.st[ST_BYTES] += 16; }
        }
    }
}

__device__ __forceinline__ uint32_t out_seg() {
    return ((blockIdx.x * (blockDim.x >> 5)) + (threadIdx.x >> 5)) % kStripes;
}

// Append y to the next frontier, else mine it here.  CHUNK (thread-per-item passes): the
// thread reserves kChunk slots per atomic -- lanes reach this point divergently, so a
// per-call warp-aggregated atomic would serialise one global round trip per lane; leftover
// slots become holes (node kHole) written by close_chunk.  !CHUNK (warp passes, converged
// lanes): one aggregated atomic per call.
template <int MAXV, bool STATS, bool CHUNK = false>
__device__ __forceinline__ void emit(const BParams &p, const lane::LNode *nodes, const DGroup *groups,
                                     const PM<MAXV> &y, Ctx &c) {
    constexpr int W = Rec<MAXV>::W;
    const uint32_t seg = out_seg();
    uint32_t idx;
    if (CHUNK) {
        if (c.em_next == c.em_end) {
            c.em_next = atomicAdd(p.out.cnt + seg, kChunk);
            c.em_end = c.em_next + kChunk;
        }
        idx = c.em_next++;
    } else {
        const unsigned am = __activemask();
        const int lane_id = threadIdx.x & 31;
        const int leader = __ffs(am) - 1;
        uint32_t base = 0;
        if (lane_id == leader) base = atomicAdd(p.out.cnt + seg, (uint32_t)__popc(am));
        base = __shfl_sync(am, base, leader);
        idx = base + __popc(am & ((1u << lane_id) - 1u));
    }
    if (idx < p.out.seg_cap) {
        uint4 *r = reinterpret_cast<uint4 *>(p.out.data + ((size_t)seg * p.out.seg_cap + idx) * W);
        r[0] = make_uint4(y.node | (y.nv << 16), y.root, y.tr_prev, y.h);
        r[1] = y.P;
#pragma unroll
        for (int q = 0; q < W / 4 - 2; q++) {
            uint32_t w[4];
#pragma unroll
            for (int k = 0; k < 4; k++) w[k] = (4 * q + k < MAXV) ? y.m2g[4 * q + k] : 0u;
            r[2 + q] = make_uint4(w[0], w[1], w[2], w[3]);
        }
        if (STATS) c.st[ST_BYTES] += 0;  // frontier traffic is not algorithmic
    } else {
        if (STATS) c.st[ST_CONTEXTS]++;
        if (p.fallback) atomicAdd(p.fallback, 1u);
        dfs<MAXV, STATS>(p, nodes, groups, y, c);
    }
}

// Mark the unused rest of this thread's reserved run as holes.
template <int MAXV>
__device__ __forceinline__ void close_chunk(const BParams &p, Ctx &c) {
    constexpr int W = Rec<MAXV>::W;
    const uint32_t seg = out_seg();
    for (uint32_t i = c.em_next; i < c.em_end && i < p.out.seg_cap; i++)
        p.out.data[((size_t)seg * p.out.seg_cap + i) * W] = kHole;
    c.em_next = c.em_end = 0;
}

// A matched inner child: count a pre-leaf child's leaf windows inline when they are
// short, else hand the child to the next level.
template <int MAXV, bool STATS, bool CHUNK>
__device__ __forceinline__ void child(const BParams &p, const lane::LNode *nodes, const DGroup *groups,
                                      const DGroup &G, const lane::LNode &dn, uint32_t ch, const PM<MAXV> &x,
                                      uint32_t pos, uint32_t etr, uint32_t e1, uint32_t e2, Ctx &c) {
    PM<MAXV> y;
    make_child<MAXV>(p, G, dn, ch, x, pos, etr, e1, e2, y);
    if (STATS) { c.st[ST_NODES]++; c.st[ST_BYTES] += 16; }
    if (p.inline_preleaf && (dn.flags & NODE_PRELEAF)) {
        // all windows short? (a window of >= kLong entries is left to the warp pass)
        bool short_ok = true;
        uint32_t starts[4], lims[4];
        const uint32_t ng = dn.group_end - dn.group_begin;
        if (ng <= 4) {
            for (uint32_t i = 0; i < ng && short_ok; i++) {
                const DGroup G2 = groups[dn.group_begin + i];
                starts[i] = window_start<MAXV, STATS>(p, G2, y, lims[i], c);
                if (G2.kind == ANCHOR_GLOBAL) {
                    short_ok = starts[i] + kLong > y.h + 1;
                } else {
                    const uint2 *ent = (G2.kind == ANCHOR_OUT) ? p.out_ent : p.in_ent;
                    const uint32_t *off = (G2.kind == ANCHOR_OUT) ? p.out_off : p.in_off;
                    short_ok = !lane::window_has(ent, off, lane::m2g_get<MAXV>(y.m2g, G2.anchor), starts[i], kLong, y.h);
                }
            }
        } else {
            short_ok = false;
        }
        if (short_ok) {
            for (uint32_t i = 0; i < ng; i++) {
                const DGroup G2 = groups[dn.group_begin + i];
                if (STATS) c.st[ST_WINDOWS]++;
                for (uint32_t q = starts[i];; ++q) {
                    uint32_t t2, a2, b2;
                    load_entry(p, G2, q, lims[i], t2, a2, b2);
                    if (t2 > y.h || q >= lims[i]) break;
                    if (t2 <= y.tr_prev) continue;
                    if (STATS) { c.st[ST_ENTRIES]++; c.st[ST_BYTES] += G2.kind == ANCHOR_GLOBAL ? 12 : 8; }
                    const uint32_t c2 = find_child(nodes, G2, entry_class<MAXV>(G2, y.m2g, a2, b2));
                    if (c2 != kNone) {
                        count_add(c, nodes[c2].slot, 1);
                        if (STATS) c.st[ST_MATCHES]++;
                    }
                }
                if (STATS) c.st[ST_BYTES] += G2.kind == ANCHOR_GLOBAL ? 12 : 8;
            }
            return;
        }
    }
    emit<MAXV, STATS, CHUNK>(p, nodes, groups, y, c);
}

// Read frontier record `item` (global index over the input segments, prefix in smem).
template <int MAXV>
__device__ __forceinline__ bool load_rec(const BParams &p, const uint32_t *s_pref, uint32_t item, PM<MAXV> &x) {
    constexpr int W = Rec<MAXV>::W;
    int lo = 0, hi = kStripes - 1;  // segment s with s_pref[s] <= item < s_pref[s+1]
    while (lo < hi) {
        const int mid = (lo + hi + 1) >> 1;
        if (s_pref[mid] <= item) lo = mid;
        else hi = mid - 1;
    }
    const uint32_t idx = item - s_pref[lo];
    const uint4 *r = reinterpret_cast<const uint4 *>(p.in.data + ((size_t)lo * p.in.seg_cap + idx) * W);
    const uint4 a = __ldcs(r), b = __ldcs(r + 1);
    x.node = a.x & 0xffffu;
    x.nv = a.x >> 16;
    x.root = a.y;
    x.tr_prev = a.z;
    x.h = a.w;
    x.P = b;
#pragma unroll
    for (int q = 0; q < W / 4 - 2; q++) {
        const uint4 w = __ldcs(r + 2 + q);
        if (4 * q + 0 < MAXV) x.m2g[(4 * q + 0) % MAXV] = w.x;
        if (4 * q + 1 < MAXV) x.m2g[(4 * q + 1) % MAXV] = w.y;
        if (4 * q + 2 < MAXV) x.m2g[(4 * q + 2) % MAXV] = w.z;
        if (4 * q + 3 < MAXV) x.m2g[(4 * q + 3) % MAXV] = w.w;
    }
    return true;
}

// root r as a partial match of the MG-Tree root (canonical edge 0->1); false for a
// self-loop (never matches, reading R7)
template <int MAXV>
__device__ __forceinline__ bool load_root(const BParams &p, uint32_t r, PM<MAXV> &x) {
    const uint32_t rs = __ldg(p.src + r), rd = __ldg(p.dst + r);
    if (rs == rd) return false;
#pragma unroll
    for (int k = 0; k < MAXV; k++) x.m2g[k] = kNone;
    x.m2g[0] = rs;
    x.m2g[1] = rd;
    x.node = 0;
    x.nv = 2;
    x.root = r;
    x.tr_prev = __ldg(p.tr + r);
    x.h = __ldg(p.hi + r);
    x.P = __ldg(p.eptr + r);
    return true;
}

// Per-thread u32 counters (one per completion slot) while they take <= kThreadCntSmem bytes of
// shared memory; groups with more completion slots (e.g. the 1,657-motif 4-edge family) count
// with shared-memory u64 atomics on the block totals instead, so any group within the ABI
// limits launches (the node and group tables alone stay under 120 KB).
constexpr size_t kThreadCntSmem = 64 * 1024;
__host__ __device__ inline bool thread_cnt(uint32_t ns, int threads) {
    return (size_t)ns * threads * 4 <= kThreadCntSmem;
}
// shared memory: nodes | groups | slot totals | per-thread u32 counters (thread_cnt) | stripe prefix
__host__ __device__ inline size_t smem_bytes(uint32_t nn, uint32_t ng, uint32_t ns, int threads) {
    return lane::align16((size_t)nn * sizeof(lane::LNode)) + lane::align16((size_t)ng * sizeof(DGroup)) +
           lane::align16((size_t)ns * 8) + (thread_cnt(ns, threads) ? (size_t)ns * threads * 4 : 0) +
           (kStripes + 1) * 4;
}

struct Smem {
    lane::LNode *nodes;
    DGroup *groups;
    unsigned long long *tot;
    uint32_t *cnt;      // per-thread counters, or null (!thread_cnt: atomics on tot)
    uint32_t *pref;
};

__device__ __forceinline__ Smem smem_setup(const BParams &p, unsigned char *smem, bool level0) {
    Smem s;
    size_t o = 0;
    s.nodes = reinterpret_cast<lane::LNode *>(smem + o);
    o += lane::align16((size_t)p.n_nodes * sizeof(lane::LNode));
    s.groups = reinterpret_cast<DGroup *>(smem + o);
    o += lane::align16((size_t)p.n_groups * sizeof(DGroup));
    s.tot = reinterpret_cast<unsigned long long *>(smem + o);
    o += lane::align16((size_t)p.n_slots * 8);
    const bool tc = thread_cnt(p.n_slots, blockDim.x);
    s.cnt = tc ? reinterpret_cast<uint32_t *>(smem + o) : nullptr;
    o += tc ? (size_t)p.n_slots * blockDim.x * 4 : 0;
    s.pref = reinterpret_cast<uint32_t *>(smem + o);
    for (uint32_t i = threadIdx.x; i < p.n_nodes; i += blockDim.x) s.nodes[i] = p.nodes[i];
    for (uint32_t i = threadIdx.x; i < p.n_groups; i += blockDim.x) s.groups[i] = p.groups[i];
    for (uint32_t i = threadIdx.x; i < p.n_slots; i += blockDim.x) s.tot[i] = 0;
    if (tc)
        for (uint32_t i = 0; i < p.n_slots; i++) s.cnt[i * blockDim.x + threadIdx.x] = 0;
    if (!level0 && threadIdx.x == 0) {
        uint32_t acc = 0;
        for (int i = 0; i < kStripes; i++) {
            s.pref[i] = acc;
            acc += min(p.in.cnt[i], p.in.seg_cap);
        }
        s.pref[kStripes] = acc;
    }
    __syncthreads();
    return s;
}

template <bool STATS>
__device__ __forceinline__ void flush(const BParams &p, const Smem &s, Ctx &c) {
    __syncthreads();
    const int lane_id = threadIdx.x & 31, nw = blockDim.x >> 5;
    for (uint32_t sl = threadIdx.x >> 5; s.cnt && sl < p.n_slots; sl += nw) {
        unsigned long long v = 0;
        for (uint32_t i = lane_id; i < blockDim.x; i += 32) v += s.cnt[sl * blockDim.x + i];
#pragma unroll
        for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(kFull, v, o);
        if (lane_id == 0) s.tot[sl] += v;
    }
    __syncthreads();
    for (uint32_t i = threadIdx.x; i < p.n_motifs; i += blockDim.x) {
        const unsigned long long v = s.tot[s.nodes[p.motif_node[i]].slot];
        if (v) atomicAdd(p.counts + i, v);
    }
    if (STATS) {
#pragma unroll
        for (int i = 0; i < ST_N; i++) {
            unsigned long long v = c.st[i];
#pragma unroll
            for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(kFull, v, o);
            if (lane_id == 0 && v) atomicAdd(p.stats + i, v);
        }
    }
}

// ------------------------------------------------------------------ expand pass
template <int MAXV, bool LEVEL0, bool STATS>
__global__ void __launch_bounds__(kTB) expand_kernel(const __grid_constant__ BParams p) {
    pdl_begin();
    extern __shared__ __align__(16) unsigned char smem[];
    const Smem s = smem_setup(p, smem, LEVEL0);
    Ctx c;
    c.cnt = s.cnt ? s.cnt + threadIdx.x : nullptr;
    c.stride = blockDim.x;
    c.tot = s.tot;
#pragma unroll
    for (int i = 0; i < ST_N; i++) c.st[i] = 0;
    c.em_next = c.em_end = 0;
    const uint32_t n_items = LEVEL0 ? p.n_roots : s.pref[kStripes];
    const lane::LNode root = s.nodes[0];
    const uint32_t lane_id = threadIdx.x & 31;
    // warp-uniform trip count: each warp takes 32 consecutive items per iteration, so the
    // light-root list can be appended with one ballot and one atomic per warp
    for (uint32_t base = blockIdx.x * blockDim.x + (threadIdx.x & ~31u); base < n_items; base += gridDim.x * blockDim.x) {
        const uint32_t item = base + lane_id;
        PM<MAXV> x;
        bool go = item < n_items;  // this thread expands x breadth-first
        if (LEVEL0) {
            bool light = false;
            const uint32_t r = p.r0 + item;
            if (go && !load_root<MAXV>(p, r, x)) {
                if (STATS) c.st[ST_BYTES] += 16;
                go = false;
            }
            if (go) {
                if (root.flags & NODE_COMPLETION) count_add(c, root.slot, 1);
                if (STATS) {
                    c.st[ST_ROOTS]++;
                    c.st[ST_BYTES] += 16 + ((root.flags & NODE_INNER) ? 16 : 0);
                    c.st[ST_MATCHES] += (root.flags & NODE_COMPLETION) ? 1 : 0;
                    if (root.flags & NODE_INNER) c.st[ST_NODES]++;
                }
                if (!(root.flags & NODE_INNER)) go = false;
                else if (p.heavy_min && !lane::heavy_root<MAXV>(s.nodes, s.groups, root, x.P, x.h, x.m2g[0], x.m2g[1],
                                                                p.out_off, p.out_ent, p.in_off, p.in_ent, p.heavy_min)) {
                    light = true;  // the depth-first kernel mines it whole
                    go = false;
                }
            }
            if (p.light) {
                const unsigned lm = __ballot_sync(kFull, light);
                if (lm) {
                    uint32_t b = 0;
                    if (lane_id == 0) b = atomicAdd(p.light_cnt, (uint32_t)__popc(lm));
                    b = __shfl_sync(kFull, b, 0);
                    if (light) p.light[b + __popc(lm & ((1u << lane_id) - 1u))] = r;
                }
            }
        } else if (go) {
            load_rec<MAXV>(p, s.pref, item, x);
            go = x.node != kHole;
        }
        if (!go) continue;
        const lane::LNode xn = s.nodes[x.node];
        for (uint32_t g = xn.group_begin; g < xn.group_end; ++g) {
            const DGroup G = s.groups[g];
            uint32_t lim;
            const uint32_t start = window_start<MAXV, STATS>(p, G, x, lim, c);
            if (STATS) { c.st[ST_WINDOWS]++; c.st[ST_BYTES] += G.kind == ANCHOR_GLOBAL ? 12 : 8; }
            // one round trip: the window's first kTile entries and the long-window probe
            const bool glob = G.kind == ANCHOR_GLOBAL;
            uint32_t etr[kTile], e1[kTile], e2[kTile];
#pragma unroll
            for (int k = 0; k < kTile; k++) load_entry(p, G, start + k, lim, etr[k], e1[k], e2[k]);
            bool is_long;
            if (glob) {
                is_long = start + kLong <= x.h + 1;
            } else {
                const uint2 *ent = (G.kind == ANCHOR_OUT) ? p.out_ent : p.in_ent;
                const uint32_t *off = (G.kind == ANCHOR_OUT) ? p.out_off : p.in_off;
                is_long = lane::window_has(ent, off, lane::m2g_get<MAXV>(x.m2g, G.anchor), start, kLong, x.h);
            }
            if (is_long) {  // long window -> warp pass
                const uint32_t li = atomicAdd(p.long_cnt, 1u);
                if (li < p.long_cap) {
                    p.long_items[3 * (size_t)li + 0] = LEVEL0 ? x.root : item;
                    p.long_items[3 * (size_t)li + 1] = g;
                    p.long_items[3 * (size_t)li + 2] = start;
                    if (STATS) c.st[ST_OFFLOADS]++;
                    continue;
                }
                // no room: scan it here
            }
            // the tile, unrolled: completions counted in place, inner matches collected
            bool open = true;
            unsigned inner = 0;
            uint32_t ich[kTile];
#pragma unroll
            for (int k = 0; k < kTile; k++) {
                open = open && !(etr[k] > x.h || start + k >= lim);
                ich[k] = kNone;
                if (open && etr[k] > x.tr_prev) {
                    if (STATS) { c.st[ST_ENTRIES]++; c.st[ST_BYTES] += glob ? 12 : 8; }
                    const uint32_t ch = find_child(s.nodes, G, entry_class<MAXV>(G, x.m2g, e1[k], e2[k]));
                    if (ch != kNone) {
                        const lane::LNode dn = s.nodes[ch];
                        if (dn.flags & NODE_COMPLETION) {
                            count_add(c, dn.slot, 1);
                            if (STATS) c.st[ST_MATCHES]++;
                        }
                        if (dn.flags & NODE_INNER) {
                            inner |= 1u << k;
                            ich[k] = ch;
                        }
                    }
                }
            }
            while (inner) {
                const int k = __ffs(inner) - 1;
                inner &= inner - 1;
                uint32_t t_ = etr[0], a_ = e1[0], b_ = e2[0], ch = ich[0];
#pragma unroll
                for (int q = 1; q < kTile; q++)
                    if (q == k) { t_ = etr[q]; a_ = e1[q]; b_ = e2[q]; ch = ich[q]; }
                child<MAXV, STATS, true>(p, s.nodes, s.groups, G, s.nodes[ch], ch, x, start + k, t_, a_, b_, c);
            }
            if (!open) continue;
            for (uint32_t pos = start + kTile;; ++pos) {  // windows longer than the tile
                uint32_t etr, e1, e2;
                load_entry(p, G, pos, lim, etr, e1, e2);
                if (etr > x.h || pos >= lim) break;
                if (etr <= x.tr_prev) continue;
                if (STATS) { c.st[ST_ENTRIES]++; c.st[ST_BYTES] += G.kind == ANCHOR_GLOBAL ? 12 : 8; }
                const uint32_t ch = find_child(s.nodes, G, entry_class<MAXV>(G, x.m2g, e1, e2));
                if (ch == kNone) continue;
                const lane::LNode dn = s.nodes[ch];
                if (dn.flags & NODE_COMPLETION) {
                    count_add(c, dn.slot, 1);
                    if (STATS) c.st[ST_MATCHES]++;
                }
                if (dn.flags & NODE_INNER) child<MAXV, STATS, true>(p, s.nodes, s.groups, G, dn, ch, x, pos, etr, e1, e2, c);
            }
        }
    }
    close_chunk<MAXV>(p, c);
    flush<STATS>(p, s, c);
}

// ------------------------------------------------------------------ long-window pass
// warp per deferred window: 32 entries per step; completion children by ballot/popc,
// inner children handled by the lane that holds the matching entry.
template <int MAXV, bool LEVEL0, bool STATS>
__global__ void __launch_bounds__(kTB) long_kernel(const __grid_constant__ BParams p) {
    pdl_begin();
    extern __shared__ __align__(16) unsigned char smem[];
    const Smem s = smem_setup(p, smem, LEVEL0);
    Ctx c;
    c.cnt = s.cnt ? s.cnt + threadIdx.x : nullptr;
    c.stride = blockDim.x;
    c.tot = s.tot;
#pragma unroll
    for (int i = 0; i < ST_N; i++) c.st[i] = 0;
    c.em_next = c.em_end = 0;
    const int lane_id = threadIdx.x & 31;
    const uint32_t n_items = min(*(volatile uint32_t *)p.long_cnt, p.long_cap);
    const uint32_t wid = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, nwarps = (gridDim.x * blockDim.x) >> 5;
    for (uint32_t it = wid; it < n_items; it += nwarps) {
        const uint32_t idx = __ldg(p.long_items + 3 * (size_t)it + 0);
        const uint32_t g = __ldg(p.long_items + 3 * (size_t)it + 1);
        const uint32_t start = __ldg(p.long_items + 3 * (size_t)it + 2);
        PM<MAXV> x;
        if (LEVEL0) load_root<MAXV>(p, idx, x);
        else load_rec<MAXV>(p, s.pref, idx, x);
        const DGroup G = s.groups[g];
        const uint32_t lim = G.kind == ANCHOR_GLOBAL ? x.h + 1 : kNone;
        for (uint32_t b = start;; b += 32) {
            const uint32_t pos = b + lane_id;
            uint32_t etr, e1, e2;
            load_entry(p, G, pos, lim, etr, e1, e2);
            const unsigned fm = __ballot_sync(kFull, etr > x.h || pos >= lim);
            const unsigned inmask = fm ? ((1u << (__ffs(fm) - 1)) - 1u) : kFull;
            const bool w = ((inmask >> lane_id) & 1u) && etr > x.tr_prev;
            const uint32_t cls = entry_class<MAXV>(G, x.m2g, e1, e2);
            for (uint32_t ch = G.child_begin; ch < G.child_end; ++ch) {
                const lane::LNode dn = s.nodes[ch];
                const bool hit = w && cls == dn.want;
                const unsigned mc = __ballot_sync(kFull, hit);
                if (!mc) continue;
                if ((dn.flags & NODE_COMPLETION) && lane_id == 0) {
                    count_add(c, dn.slot, __popc(mc));
                    if (STATS) c.st[ST_MATCHES] += __popc(mc);
                }
                if ((dn.flags & NODE_INNER) && hit)
                    child<MAXV, STATS, false>(p, s.nodes, s.groups, G, dn, ch, x, pos, etr, e1, e2, c);
            }
            if (STATS) {
                const uint32_t we = __popc(__ballot_sync(kFull, w));
                if (lane_id == 0) {
                    c.st[ST_ENTRIES] += we;
                    c.st[ST_BYTES] += (G.kind == ANCHOR_GLOBAL ? 12ull : 8ull) * we;
                    c.st[ST_BATCHES]++;
                }
            }
            if (fm) break;
        }
    }
    flush<STATS>(p, s, c);
}

}  // namespace bfs
