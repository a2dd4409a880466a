// tile.cuh -- co-mining as waves of fixed-size window tiles (kernel v6, the default);
// included by comine.cu after wave.cuh (whose striped lists it reuses).
//
// Algorithm 3 "Co-Mining": from every root edge, the search tree
// grows one MG-Tree level per wave; expanding a partial match x means scanning one
// candidate window per anchor group of its node (Algo 1 l.210-222).  Unit of work: a
// TASK = one window of one partial match {node, group, start, root, tr_prev, h, m2g}.
//
//   wave k, kernel A (thread per task): load the first kTile entries of the window with
//     independent loads and process them FULLY UNROLLED -- every lane executes the same
//     predicated instructions whatever its window looks like (windows average ~2
//     entries):  time test (t_prev < t <= t_root + delta), class of the neighbour against
//     m2g (which mapped motif vertex, or NEW: full injectivity, reading R4), the child
//     that wants that class (packed wants, one SIMD byte compare):
//        completion child -> count[Q_N]++                                (Algo 3 l.661)
//        inner child      -> one task per anchor group of the child, wave k+1
//                                                                       (Algo 3 l.665-669)
//     a window that continues past the tile becomes a long task of the SAME wave;
//   wave k, kernel B (warp per long task): 32 entries per step, same per-entry logic.
//
// Appends go to wave::kStripes segments (warp-aggregated atomics); a full segment never
// loses work -- the window or subtree is mined in place, depth-first (bfs::dfs).
namespace tile {

using bfs::Ctx;
using bfs::PM;

constexpr int kTB = 256;
constexpr int kTile = 4;  // entries per task tile
#ifndef TILE_MIN_BLOCKS
#define TILE_MIN_BLOCKS 4
#endif
constexpr int kMinBlocks = TILE_MIN_BLOCKS;  // resident blocks per SM the register budget must allow

template <int MAXV>
struct Task {  // words per task: node|g<<16, start, root, tr_prev, h, m2g[MAXV] (16-byte padded)
    static constexpr int W = (5 + MAXV + 3) & ~3;
};

struct TParams {
    const uint32_t *src, *dst, *tr, *hi;
    const uint4 *eptr;
    const uint32_t *out_off, *in_off;
    const uint2 *out_ent, *in_ent;
    const uint4 *out_ptr, *in_ptr;
    const lane::LNode *nodes;
    const DGroup *groups;
    const uint32_t *gwant;      // per group: wants of its first 4 children (bytes), 0xFD pad
    const uint32_t *motif_node;
    uint32_t n_nodes, n_groups, n_motifs, n_slots;
    uint32_t r0, n_roots;
    wave::List in_tasks;        // this kernel's input (normal or long list of this wave)
    wave::List out_norm;        // next wave's tasks
    wave::List out_long;        // this wave's long tasks (written by kernel A / root kernel)
    uint32_t *fallback;
    unsigned long long *counts;
    unsigned long long *stats;
};

__device__ __forceinline__ bfs::BParams gp(const TParams &w) {
    bfs::BParams b;
    b.src = w.src; b.dst = w.dst; b.tr = w.tr; b.hi = w.hi; b.eptr = w.eptr;
    b.out_off = w.out_off; b.in_off = w.in_off; b.out_ent = w.out_ent; b.in_ent = w.in_ent;
    b.out_ptr = w.out_ptr; b.in_ptr = w.in_ptr;
    b.nodes = w.nodes; b.groups = w.groups; b.motif_node = w.motif_node;
    b.n_nodes = w.n_nodes; b.n_groups = w.n_groups; b.n_motifs = w.n_motifs; b.n_slots = w.n_slots;
    b.r0 = w.r0; b.n_roots = w.n_roots;
    b.counts = w.counts; b.stats = w.stats;
    return b;
}

struct Sm {
    lane::LNode *nodes;
    DGroup *groups;
    uint32_t *gwant;
    unsigned long long *tot;
    uint32_t *cnt;
    uint32_t *pref;
};

__host__ __device__ inline size_t smem_bytes(uint32_t nn, uint32_t ng, uint32_t ns) {
    return lane::align16((size_t)nn * sizeof(lane::LNode)) + lane::align16((size_t)ng * sizeof(DGroup)) +
           lane::align16((size_t)ng * 4) + lane::align16((size_t)ns * 8) + (size_t)ns * kTB * 4 +
           (wave::kStripes + 1) * 4;
}

__device__ __forceinline__ Sm setup(const TParams &w, unsigned char *smem, bool prefix) {
    Sm s;
    size_t o = 0;
    s.nodes = reinterpret_cast<lane::LNode *>(smem + o);
    o += lane::align16((size_t)w.n_nodes * sizeof(lane::LNode));
    s.groups = reinterpret_cast<DGroup *>(smem + o);
    o += lane::align16((size_t)w.n_groups * sizeof(DGroup));
    s.gwant = reinterpret_cast<uint32_t *>(smem + o);
    o += lane::align16((size_t)w.n_groups * 4);
    s.tot = reinterpret_cast<unsigned long long *>(smem + o);
    o += lane::align16((size_t)w.n_slots * 8);
    s.cnt = reinterpret_cast<uint32_t *>(smem + o);
    o += (size_t)w.n_slots * kTB * 4;
    s.pref = reinterpret_cast<uint32_t *>(smem + o);
    for (uint32_t i = threadIdx.x; i < w.n_nodes; i += kTB) s.nodes[i] = w.nodes[i];
    for (uint32_t i = threadIdx.x; i < w.n_groups; i += kTB) {
        s.groups[i] = w.groups[i];
        s.gwant[i] = w.gwant[i];
    }
    for (uint32_t i = threadIdx.x; i < w.n_slots; i += kTB) s.tot[i] = 0;
    for (uint32_t i = 0; i < w.n_slots; i++) s.cnt[i * kTB + threadIdx.x] = 0;
    if (prefix && threadIdx.x == 0) {
        uint32_t acc = 0;
        for (int i = 0; i < wave::kStripes; i++) {
            s.pref[i] = acc;
            acc += min(*(volatile uint32_t *)(w.in_tasks.cnt + i), w.in_tasks.seg_cap);
        }
        s.pref[wave::kStripes] = acc;
    }
    __syncthreads();
    return s;
}

__device__ __forceinline__ void flush_counts(const TParams &w, const Sm &s, Ctx &c, bool stats) {
    __syncthreads();
    const int lane_id = threadIdx.x & 31;
    for (uint32_t sl = threadIdx.x >> 5; sl < w.n_slots; sl += kTB / 32) {
        unsigned long long v = 0;
        for (uint32_t i = lane_id; i < kTB; i += 32) v += s.cnt[sl * kTB + i];
#pragma unroll
        for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(kFull, v, o);
        if (lane_id == 0) s.tot[sl] += v;
    }
    __syncthreads();
    for (uint32_t i = threadIdx.x; i < w.n_motifs; i += kTB) {
        const unsigned long long v = s.tot[s.nodes[w.motif_node[i]].slot];
        if (v) atomicAdd(w.counts + i, v);
    }
    if (stats) {
#pragma unroll
        for (int i = 0; i < ST_N; i++) {
            unsigned long long v = c.st[i];
#pragma unroll
            for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(kFull, v, o);
            if (lane_id == 0 && v) atomicAdd(w.stats + i, v);
        }
    }
}

// child row wanting class `cls` in group g (kNone if none): SIMD byte compare of the
// group's packed wants; groups of more than 4 children fall back to a scan
__device__ __forceinline__ uint32_t lookup(const Sm &s, const DGroup &G, uint32_t g, uint32_t cls) {
    const uint32_t nch = G.child_end - G.child_begin;
    if (nch <= 4) {
        const uint32_t eq = __vcmpeq4(s.gwant[g], cls * 0x01010101u);
        return eq ? G.child_begin + ((__ffs(eq) - 1) >> 3) : kNone;
    }
    for (uint32_t c = G.child_begin; c < G.child_end; ++c)
        if (s.nodes[c].want == cls) return c;
    return kNone;
}

template <int MAXV>
__device__ __forceinline__ void store_task(uint32_t *t, uint32_t node, uint32_t g, uint32_t start,
                                           const PM<MAXV> &x) {
    constexpr int W = Task<MAXV>::W;
    uint32_t v[W];
    v[0] = node | (g << 16);
    v[1] = start;
    v[2] = x.root;
    v[3] = x.tr_prev;
    v[4] = x.h;
#pragma unroll
    for (int k = 0; k < MAXV; k++) v[5 + k] = x.m2g[k];
#pragma unroll
    for (int k = 5 + MAXV; k < W; k++) v[k] = 0;
    uint4 *r = reinterpret_cast<uint4 *>(t);
#pragma unroll
    for (int q = 0; q < W / 4; q++) r[q] = make_uint4(v[4 * q], v[4 * q + 1], v[4 * q + 2], v[4 * q + 3]);
}

template <int MAXV>
__device__ __forceinline__ void load_task(const uint32_t *t, const Sm &s, PM<MAXV> &x, uint32_t &g,
                                          uint32_t &start) {
    constexpr int W = Task<MAXV>::W;
    const uint4 *r = reinterpret_cast<const uint4 *>(t);
    uint32_t v[W];
#pragma unroll
    for (int q = 0; q < W / 4; q++) {
        const uint4 a = __ldcs(r + q);
        v[4 * q] = a.x; v[4 * q + 1] = a.y; v[4 * q + 2] = a.z; v[4 * q + 3] = a.w;
    }
    x.node = v[0] & 0xffffu;
    g = v[0] >> 16;
    start = v[1];
    x.root = v[2];
    x.tr_prev = v[3];
    x.h = v[4];
#pragma unroll
    for (int k = 0; k < MAXV; k++) x.m2g[k] = v[5 + k];
    x.nv = s.nodes[x.node].nv;
}

// Append one task to list L (warp-aggregated); false if the segment is full.
template <int MAXV>
__device__ __forceinline__ bool push(const wave::List &L, uint32_t node, uint32_t g, uint32_t start,
                                     const PM<MAXV> &x) {
    const uint32_t seg = wave::my_seg();
    const uint32_t idx = wave::append(L.cnt, seg);
    if (idx >= L.seg_cap) return false;
    store_task<MAXV>(L.data + ((size_t)seg * L.seg_cap + idx) * Task<MAXV>::W, node, g, start, x);
    return true;
}

// Inner child y matched: one next-wave task per anchor group of y's node.
template <int MAXV, bool STATS>
__device__ __noinline__ void spawn(const TParams &w, const Sm &s, const PM<MAXV> &y, Ctx &c) {
    const bfs::BParams bp = gp(w);
    const lane::LNode dn = s.nodes[y.node];
    for (uint32_t g2 = dn.group_begin; g2 < dn.group_end; ++g2) {
        uint32_t lim;
        const uint32_t start = bfs::window_start<MAXV, STATS>(bp, s.groups[g2], y, lim, c);
        if (!push<MAXV>(w.out_norm, y.node, g2, start, y)) {
            // no room: mine this window (and anything below it) right here
            if (STATS) c.st[ST_CONTEXTS]++;
            atomicAdd(w.fallback, 1u);
            const DGroup G = s.groups[g2];
            for (uint32_t pos = start;; ++pos) {
                uint32_t etr, e1, e2;
                bfs::load_entry(bp, G, pos, lim, etr, e1, e2);
                if (etr > y.h || pos >= lim) break;
                if (etr <= y.tr_prev) continue;
                const uint32_t ch = lookup(s, G, g2, bfs::entry_class<MAXV>(G, y.m2g, e1, e2));
                if (ch == kNone) continue;
                const lane::LNode cn = s.nodes[ch];
                if (cn.flags & NODE_COMPLETION) {
                    bfs::count_add(c, cn.slot, 1);
                    if (STATS) c.st[ST_MATCHES]++;
                }
                if (cn.flags & NODE_INNER) {
                    PM<MAXV> z;
                    bfs::make_child<MAXV>(bp, G, cn, ch, y, pos, etr, e1, e2, z);
                    bfs::dfs<MAXV, STATS>(bp, s.nodes, s.groups, z, c);
                }
            }
        }
    }
}

// Process the first kTile entries of window (x, g) from `start`, fully unrolled; returns
// true if the window continues past the tile.
template <int MAXV, bool STATS>
__device__ __forceinline__ bool tile4(const TParams &w, const Sm &s, const PM<MAXV> &x, uint32_t g, uint32_t start,
                                      Ctx &c) {
    const DGroup G = s.groups[g];
    const bool glob = G.kind == ANCHOR_GLOBAL;
    const uint32_t lim = glob ? x.h + 1 : kNone;
    uint32_t etr[kTile], e1[kTile], e2[kTile];
    if (glob) {
#pragma unroll
        for (int k = 0; k < kTile; k++) {
            const uint32_t pos = start + k;
            const bool ok = pos < lim;
            etr[k] = ok ? __ldg(w.tr + pos) : kNone;
            e1[k] = ok ? __ldg(w.src + pos) : 0u;
            e2[k] = ok ? __ldg(w.dst + pos) : 0u;
        }
    } else {
        const uint2 *ent = (G.kind == ANCHOR_OUT ? w.out_ent : w.in_ent) + start;
#pragma unroll
        for (int k = 0; k < kTile; k++) {
            const uint2 e = __ldg(ent + k);
            etr[k] = e.x;
            e1[k] = e.y;
            e2[k] = 0;
        }
    }
    if (STATS) { c.st[ST_WINDOWS]++; c.st[ST_BATCHES]++; }
    bool open = true;
    unsigned inner = 0;  // entries whose child has children of its own
    uint32_t ich[kTile];
#pragma unroll
    for (int k = 0; k < kTile; k++) {
        open = open && etr[k] <= x.h;
        ich[k] = kNone;
        if (open && etr[k] > x.tr_prev) {
            const uint32_t cls = glob ? ((e1[k] != e2[k] && lane::classify<MAXV>(x.m2g, e1[k]) == CLS_NEW &&
                                          lane::classify<MAXV>(x.m2g, e2[k]) == CLS_NEW) ? CLS_NEW : 0xFEu)
                                      : lane::classify<MAXV>(x.m2g, e1[k]);
            const uint32_t ch = lookup(s, G, g, cls);
            if (STATS) { c.st[ST_ENTRIES]++; c.st[ST_BYTES] += glob ? 12 : 8; }
            if (ch != kNone) {
                const lane::LNode dn = s.nodes[ch];
                if (dn.flags & NODE_COMPLETION) {
                    bfs::count_add(c, dn.slot, 1);
                    if (STATS) c.st[ST_MATCHES]++;
                }
                if (dn.flags & NODE_INNER) {
                    inner |= 1u << k;
                    ich[k] = ch;
                }
            }
        }
    }
    if (STATS && !open) c.st[ST_BYTES] += glob ? 12 : 8;  // the terminating entry
    if (inner) {
        const bfs::BParams bp = gp(w);
        while (inner) {
            const int k = __ffs(inner) - 1;
            inner &= inner - 1;
            uint32_t t_ = etr[0], a_ = e1[0], b_ = e2[0], ch = ich[0];
#pragma unroll
            for (int q = 1; q < kTile; q++)
                if (q == k) { t_ = etr[q]; a_ = e1[q]; b_ = e2[q]; ch = ich[q]; }
            const lane::LNode dn = s.nodes[ch];
            PM<MAXV> y;
            bfs::make_child<MAXV>(bp, G, dn, ch, x, start + k, t_, a_, b_, y);
            if (STATS) { c.st[ST_NODES]++; c.st[ST_BYTES] += 16; }
            spawn<MAXV, STATS>(w, s, y, c);
        }
    }
    return open;
}

// ---------------------------------------------------------------- kernel A, wave 0: roots
template <int MAXV, bool STATS>
__global__ void __launch_bounds__(kTB, kMinBlocks) root_kernel(const __grid_constant__ TParams w) {
    extern __shared__ __align__(16) unsigned char smem[];
    const Sm s = setup(w, smem, false);
    Ctx c;
    c.cnt = s.cnt + threadIdx.x;
    c.stride = kTB;
    c.tot = s.tot;
#pragma unroll
    for (int i = 0; i < ST_N; i++) c.st[i] = 0;
    const bfs::BParams bp = gp(w);
    const lane::LNode root = s.nodes[0];
    for (uint32_t i = blockIdx.x * kTB + threadIdx.x; i < w.n_roots; i += gridDim.x * kTB) {
        PM<MAXV> x;
        if (!bfs::load_root<MAXV>(bp, w.r0 + i, x)) {  // self-loops never match 0->1 (R7)
            if (STATS) c.st[ST_BYTES] += 16;
            continue;
        }
        if (root.flags & NODE_COMPLETION) bfs::count_add(c, root.slot, 1);
        if (STATS) {
            c.st[ST_ROOTS]++;
            c.st[ST_BYTES] += 16 + ((root.flags & NODE_INNER) ? 16 : 0);
            c.st[ST_MATCHES] += (root.flags & NODE_COMPLETION) ? 1 : 0;
            if (root.flags & NODE_INNER) c.st[ST_NODES]++;
        }
        for (uint32_t g = root.group_begin; g < root.group_end; ++g) {
            uint32_t lim;
            const uint32_t start = bfs::window_start<MAXV, STATS>(bp, s.groups[g], x, lim, c);
            if (tile4<MAXV, STATS>(w, s, x, g, start, c)) {
                if (!push<MAXV>(w.out_long, 0, g, start + kTile, x)) {
                    if (STATS) c.st[ST_CONTEXTS]++;
                    atomicAdd(w.fallback, 1u);
                    PM<MAXV> y = x;  // scan the rest here: reuse spawn's in-place path on a copy
                    // mine the remaining window serially (inner children depth-first)
                    const DGroup G = s.groups[g];
                    for (uint32_t pos = start + kTile;; ++pos) {
                        uint32_t etr, e1, e2;
                        bfs::load_entry(bp, G, pos, lim, etr, e1, e2);
                        if (etr > y.h || pos >= lim) break;
                        if (etr <= y.tr_prev) continue;
                        const uint32_t ch = lookup(s, G, g, bfs::entry_class<MAXV>(G, y.m2g, e1, e2));
                        if (ch == kNone) continue;
                        const lane::LNode cn = s.nodes[ch];
                        if (cn.flags & NODE_COMPLETION) bfs::count_add(c, cn.slot, 1);
                        if (cn.flags & NODE_INNER) {
                            PM<MAXV> z;
                            bfs::make_child<MAXV>(bp, G, cn, ch, y, pos, etr, e1, e2, z);
                            bfs::dfs<MAXV, STATS>(bp, s.nodes, s.groups, z, c);
                        }
                    }
                } else if (STATS) {
                    c.st[ST_OFFLOADS]++;
                }
            }
        }
    }
    flush_counts(w, s, c, STATS);
}

// ---------------------------------------------------------------- kernel A: window tiles
template <int MAXV, bool STATS>
__global__ void __launch_bounds__(kTB, kMinBlocks) tile_kernel(const __grid_constant__ TParams w) {
    constexpr int W = Task<MAXV>::W;
    extern __shared__ __align__(16) unsigned char smem[];
    const Sm s = setup(w, smem, true);
    Ctx c;
    c.cnt = s.cnt + threadIdx.x;
    c.stride = kTB;
    c.tot = s.tot;
#pragma unroll
    for (int i = 0; i < ST_N; i++) c.st[i] = 0;
    const uint32_t n = s.pref[wave::kStripes];
    for (uint32_t t = blockIdx.x * kTB + threadIdx.x; t < n; t += gridDim.x * kTB) {
        int lo = 0, hi = wave::kStripes - 1;
        while (lo < hi) {
            const int mid = (lo + hi + 1) >> 1;
            if (s.pref[mid] <= t) lo = mid;
            else hi = mid - 1;
        }
        PM<MAXV> x;
        uint32_t g, start;
        load_task<MAXV>(w.in_tasks.data + ((size_t)lo * w.in_tasks.seg_cap + (t - s.pref[lo])) * W, s, x, g, start);
        if (tile4<MAXV, STATS>(w, s, x, g, start, c)) {
            if (!push<MAXV>(w.out_long, x.node, g, start + kTile, x)) {
                if (STATS) c.st[ST_CONTEXTS]++;
                atomicAdd(w.fallback, 1u);
                const bfs::BParams bp = gp(w);
                const DGroup G = s.groups[g];
                const uint32_t lim = G.kind == ANCHOR_GLOBAL ? x.h + 1 : kNone;
                for (uint32_t pos = start + kTile;; ++pos) {
                    uint32_t etr, e1, e2;
                    bfs::load_entry(bp, G, pos, lim, etr, e1, e2);
                    if (etr > x.h || pos >= lim) break;
                    if (etr <= x.tr_prev) continue;
                    const uint32_t ch = lookup(s, G, g, bfs::entry_class<MAXV>(G, x.m2g, e1, e2));
                    if (ch == kNone) continue;
                    const lane::LNode cn = s.nodes[ch];
                    if (cn.flags & NODE_COMPLETION) bfs::count_add(c, cn.slot, 1);
                    if (cn.flags & NODE_INNER) {
                        PM<MAXV> z;
                        bfs::make_child<MAXV>(bp, G, cn, ch, x, pos, etr, e1, e2, z);
                        bfs::dfs<MAXV, STATS>(bp, s.nodes, s.groups, z, c);
                    }
                }
            } else if (STATS) {
                c.st[ST_OFFLOADS]++;
            }
        }
    }
    flush_counts(w, s, c, STATS);
}

// ---------------------------------------------------------------- kernel B: long windows
// warp per task, 32 entries per step from the continuation point; the group agrees on
// the window end by ballot (entries past a list's sentinel belong to the next vertex).
template <int MAXV, bool STATS>
__global__ void __launch_bounds__(kTB, kMinBlocks) long_kernel(const __grid_constant__ TParams w) {
    constexpr int W = Task<MAXV>::W;
    extern __shared__ __align__(16) unsigned char smem[];
    const Sm s = setup(w, smem, true);
    Ctx c;
    c.cnt = s.cnt + threadIdx.x;
    c.stride = kTB;
    c.tot = s.tot;
#pragma unroll
    for (int i = 0; i < ST_N; i++) c.st[i] = 0;
    const bfs::BParams bp = gp(w);
    const int lane_id = threadIdx.x & 31;
    const uint32_t n = s.pref[wave::kStripes];
    const uint32_t wid = (blockIdx.x * kTB + threadIdx.x) >> 5, nw = (gridDim.x * kTB) >> 5;
    for (uint32_t t = wid; t < n; t += nw) {
        int lo = 0, hi = wave::kStripes - 1;
        while (lo < hi) {
            const int mid = (lo + hi + 1) >> 1;
            if (s.pref[mid] <= t) lo = mid;
            else hi = mid - 1;
        }
        PM<MAXV> x;
        uint32_t g, start;
        load_task<MAXV>(w.in_tasks.data + ((size_t)lo * w.in_tasks.seg_cap + (t - s.pref[lo])) * W, s, x, g, start);
        const DGroup G = s.groups[g];
        const bool glob = G.kind == ANCHOR_GLOBAL;
        const uint32_t lim = glob ? x.h + 1 : kNone;
        for (uint32_t b = start;; b += 32) {
            const uint32_t pos = b + lane_id;
            uint32_t etr, e1, e2;
            bfs::load_entry(bp, G, pos, lim, etr, e1, e2);
            const unsigned fm = __ballot_sync(kFull, etr > x.h || pos >= lim);
            const bool valid = (fm == 0 || lane_id < __ffs(fm) - 1) && etr > x.tr_prev;
            if (STATS && lane_id == 0) c.st[ST_BATCHES]++;
            if (valid) {
                if (STATS) { c.st[ST_ENTRIES]++; c.st[ST_BYTES] += glob ? 12 : 8; }
                const uint32_t ch = lookup(s, G, g, bfs::entry_class<MAXV>(G, x.m2g, e1, e2));
                if (ch != kNone) {
                    const lane::LNode dn = s.nodes[ch];
                    if (dn.flags & NODE_COMPLETION) {
                        bfs::count_add(c, dn.slot, 1);
                        if (STATS) c.st[ST_MATCHES]++;
                    }
                    if (dn.flags & NODE_INNER) {
                        PM<MAXV> y;
                        bfs::make_child<MAXV>(bp, G, dn, ch, x, pos, etr, e1, e2, y);
                        if (STATS) { c.st[ST_NODES]++; c.st[ST_BYTES] += 16; }
                        spawn<MAXV, STATS>(w, s, y, c);
                    }
                }
            }
            if (fm) break;
        }
    }
    flush_counts(w, s, c, STATS);
}

}  // namespace tile
