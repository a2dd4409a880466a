// wave.cuh -- co-mining as waves of window tasks (kernel v5, the default); included by
// comine.cu after bfs.cuh (whose partial-match helpers it reuses).
//
// Algorithm 3 "Co-Mining" grows, from every root edge, a search tree
// whose depth-k vertices are partial matches of the MG-Tree nodes at depth k; expanding a
// vertex means scanning one candidate window per anchor group of its node (Algo 1
// l.210-222).  Here the unit of GPU work is that WINDOW, not the root or the vertex:
//
//   wave 0:  thread per root edge -> its root-node windows become tasks {root, group, start}
//   wave k:  every window task of depth k is scanned by a small lane group (kSub lanes,
//            entry start+j, start+j+kSub, ...; a whole warp for windows of >= kLongMin
//            entries).  Per entry: time test, class of the neighbour against m2g, the one
//            child that wants that class (full injectivity, reading R4):
//              completion child -> count[Q_N]++ (lane-private shared counter)
//              inner child      -> the child's partial-match record + one task per anchor
//                                  group of the child, for wave k+1
//
// so every wave is a wide, uniform stream of short, independent scans -- no per-thread
// loops over nested windows (the divergence that capped v4 at ~4.5 active lanes per
// instruction) and no dependent chain longer than one window.  Appends go to kStripes
// segments (warp-aggregated atomics).  A full segment never loses work: that window or
// subtree is mined in place, depth-first (bfs::dfs), so counts are exact by construction.
namespace wave {

using bfs::Ctx;
using bfs::PM;

constexpr int kTB = 256;
constexpr int kStripes = 64;
constexpr int kSub = 4;              // lanes per normal window task
constexpr uint32_t kLongMin = 16;    // windows of >= kLongMin entries are warp tasks
constexpr int kTaskWords = 3;        // {partial match ref, group, window start}

struct List {             // kStripes segments of fixed-size items
    uint32_t *data;
    uint32_t *cnt;        // per segment: items appended (may exceed seg_cap: overflow)
    uint32_t seg_cap;
};

struct WParams {
    const uint32_t *src, *dst, *tr, *hi;
    const uint4 *eptr;
    const uint32_t *out_off, *in_off;
    const uint2 *out_ent, *in_ent;
    const uint4 *out_ptr, *in_ptr;
    const lane::LNode *nodes;
    const DGroup *groups;
    const uint32_t *motif_node;
    uint32_t n_nodes, n_groups, n_motifs, n_slots;
    uint32_t r0, n_roots;
    const uint32_t *in_pm;      // this wave's partial-match records (slot-addressed)
    List in_tasks;              // this wave's tasks (normal or long list)
    uint32_t *out_pm;           // next wave's records: kStripes segments of pm_seg_cap
    uint32_t *out_pm_cnt;
    uint32_t pm_seg_cap;
    List out_norm, out_long;    // next wave's tasks
    uint32_t *fallback;         // [0] windows/subtrees mined in place (a segment was full)
    unsigned long long *counts;
    unsigned long long *stats;
};

template <int MAXV>
__device__ __forceinline__ void store_pm(uint32_t *rec, const PM<MAXV> &y) {
    constexpr int W = bfs::Rec<MAXV>::W;
    uint4 *r = reinterpret_cast<uint4 *>(rec);
    r[0] = make_uint4(y.node | (y.nv << 16), y.root, y.tr_prev, y.h);
    r[1] = y.P;
#pragma unroll
    for (int q = 0; q < W / 4 - 2; q++) {
        uint32_t w[4];
#pragma unroll
        for (int k = 0; k < 4; k++) w[k] = (4 * q + k < MAXV) ? y.m2g[4 * q + k] : 0u;
        r[2 + q] = make_uint4(w[0], w[1], w[2], w[3]);
    }
}

template <int MAXV>
__device__ __forceinline__ void load_pm(const uint32_t *rec, PM<MAXV> &x) {
    constexpr int W = bfs::Rec<MAXV>::W;
    const uint4 *r = reinterpret_cast<const uint4 *>(rec);
    const uint4 a = __ldg(r), b = __ldg(r + 1);
    x.node = a.x & 0xffffu;
    x.nv = a.x >> 16;
    x.root = a.y;
    x.tr_prev = a.z;
    x.h = a.w;
    x.P = b;
#pragma unroll
    for (int q = 0; q < W / 4 - 2; q++) {
        const uint4 w = __ldg(r + 2 + q);
        if (4 * q + 0 < MAXV) x.m2g[(4 * q + 0) % MAXV] = w.x;
        if (4 * q + 1 < MAXV) x.m2g[(4 * q + 1) % MAXV] = w.y;
        if (4 * q + 2 < MAXV) x.m2g[(4 * q + 2) % MAXV] = w.z;
        if (4 * q + 3 < MAXV) x.m2g[(4 * q + 3) % MAXV] = w.w;
    }
}

// Warp-aggregated append of one item per active lane to segment `seg`; returns the index
// within the segment (>= cap: no room).
__device__ __forceinline__ uint32_t append(uint32_t *cnt, uint32_t seg) {
    const unsigned am = __activemask();
    const int ln = threadIdx.x & 31;
    // converged lanes may target different lists: aggregate per target counter
    const unsigned grp = __match_any_sync(am, (unsigned long long)(cnt + seg));
    const int leader = __ffs(grp) - 1;
    uint32_t base = 0;
    if (ln == leader) base = atomicAdd(cnt + seg, (uint32_t)__popc(grp));
    base = __shfl_sync(grp, base, leader);
    return base + __popc(grp & ((1u << ln) - 1u));
}

__device__ __forceinline__ uint32_t my_seg() {
    return ((blockIdx.x * (blockDim.x >> 5)) + (threadIdx.x >> 5)) % kStripes;
}

template <int MAXV, bool STATS>
__device__ __noinline__ void scan_serial(const WParams &w, const bfs::BParams &bp, const lane::LNode *nodes,
                                         const DGroup *groups, const PM<MAXV> &x, uint32_t g, uint32_t start,
                                         uint32_t lim, Ctx &c);

// Queue the windows of child partial match y (already a record at `slot`) for the next wave.
template <int MAXV, bool STATS>
__device__ __forceinline__ void queue_windows(const WParams &w, const bfs::BParams &bp, const lane::LNode *nodes,
                                              const DGroup *groups, const lane::LNode &dn, const PM<MAXV> &y,
                                              uint32_t slot, Ctx &c) {
    for (uint32_t g2 = dn.group_begin; g2 < dn.group_end; ++g2) {
        const DGroup G2 = groups[g2];
        uint32_t lim;
        uint32_t start = bfs::window_start<MAXV, STATS>(bp, G2, y, lim, c);
        if (G2.start >= START_R0 && G2.start < START_SEARCH) {
            // the root's successor pointer is only a lower bound: gallop to the first entry
            // after the partial match's last edge, so the window (and its length) is exact
            const uint2 *ent = (G2.kind == ANCHOR_OUT) ? w.out_ent : w.in_ent;
            if (__ldg(&ent[start].x) <= y.tr_prev) {
                // the anchor's list ends with its sentinel (time rank kNone) at off[v+1]-1
                const uint32_t v = lane::m2g_get<MAXV>(y.m2g, G2.anchor);
                const uint32_t last = __ldg(((G2.kind == ANCHOR_OUT) ? w.out_off : w.in_off) + v + 1) - 1;
                uint32_t lo = start + 1, step = 1, hi2 = last;  // invariant: ent[lo-1] <= tr_prev
                for (;;) {
                    const uint32_t probe = min(lo + step - 1, last);
                    if (STATS) c.st[ST_PROBES]++;
                    if (__ldg(&ent[probe].x) > y.tr_prev) {
                        hi2 = probe;
                        break;
                    }
                    lo = probe + 1;
                    step <<= 1;
                }
                while (lo < hi2) {
                    const uint32_t mid = lo + ((hi2 - lo) >> 1);
                    if (STATS) c.st[ST_PROBES]++;
                    if (__ldg(&ent[mid].x) > y.tr_prev) hi2 = mid;
                    else lo = mid + 1;
                }
                start = lo;
            }
        }
        bool is_long;
        if (G2.kind == ANCHOR_GLOBAL) {
            is_long = start + kLongMin <= y.h + 1;
        } else {
            const uint2 *ent = (G2.kind == ANCHOR_OUT) ? w.out_ent : w.in_ent;
            is_long = __ldg(&ent[start + kLongMin - 1].x) <= y.h;
        }
        const List &L = is_long ? w.out_long : w.out_norm;
        const uint32_t seg = my_seg();
        const uint32_t idx = append(L.cnt, seg);
        if (idx < L.seg_cap) {
            uint32_t *t = L.data + ((size_t)seg * L.seg_cap + idx) * kTaskWords;
            t[0] = slot;
            t[1] = g2;
            t[2] = start;
            if (STATS && is_long) c.st[ST_OFFLOADS]++;
        } else {
            if (STATS) c.st[ST_CONTEXTS]++;
            atomicAdd(w.fallback, 1u);
            scan_serial<MAXV, STATS>(w, bp, nodes, groups, y, g2, start, lim, c);
        }
    }
}

// One matched inner child: record + window tasks for the next wave (or mined in place).
template <int MAXV, bool STATS>
__device__ __forceinline__ void spawn(const WParams &w, const bfs::BParams &bp, const lane::LNode *nodes,
                                     const DGroup *groups, const DGroup &G, const lane::LNode &dn, uint32_t ch,
                                     const PM<MAXV> &x, uint32_t pos, uint32_t etr, uint32_t e1, uint32_t e2,
                                     Ctx &c) {
    constexpr int W = bfs::Rec<MAXV>::W;
    PM<MAXV> y;
    bfs::make_child<MAXV>(bp, G, dn, ch, x, pos, etr, e1, e2, y);
    if (STATS) { c.st[ST_NODES]++; c.st[ST_BYTES] += 16; }
    const uint32_t seg = my_seg();
    const uint32_t idx = append(w.out_pm_cnt, seg);
    if (idx >= w.pm_seg_cap) {
        if (STATS) c.st[ST_CONTEXTS]++;
        atomicAdd(w.fallback, 1u);
        bfs::dfs<MAXV, STATS>(bp, nodes, groups, y, c);
        return;
    }
    const uint32_t slot = seg * w.pm_seg_cap + idx;
    store_pm<MAXV>(w.out_pm + (size_t)slot * W, y);
    queue_windows<MAXV, STATS>(w, bp, nodes, groups, dn, y, slot, c);
}

// Scan one window serially (fallback path): inner children are mined depth-first.
template <int MAXV, bool STATS>
__device__ __noinline__ void scan_serial(const WParams &w, const bfs::BParams &bp, const lane::LNode *nodes,
                                         const DGroup *groups, const PM<MAXV> &x, uint32_t g, uint32_t start,
                                         uint32_t lim, Ctx &c) {
    const DGroup G = groups[g];
    for (uint32_t pos = start;; ++pos) {
        uint32_t etr, e1, e2;
        bfs::load_entry(bp, G, pos, lim, etr, e1, e2);
        if (etr > x.h || pos >= lim) break;
        if (etr <= x.tr_prev) continue;
        const uint32_t ch = bfs::find_child(nodes, G, bfs::entry_class<MAXV>(G, x.m2g, e1, e2));
        if (ch == kNone) continue;
        const lane::LNode dn = nodes[ch];
        if (dn.flags & NODE_COMPLETION) {
            bfs::count_add(c, dn.slot, 1);
            if (STATS) c.st[ST_MATCHES]++;
        }
        if (dn.flags & NODE_INNER) {
            PM<MAXV> y;
            bfs::make_child<MAXV>(bp, G, dn, ch, x, pos, etr, e1, e2, y);
            bfs::dfs<MAXV, STATS>(bp, nodes, groups, y, c);
        }
    }
}

__device__ __forceinline__ bfs::BParams graph_params(const WParams &w) {
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

// shared memory: nodes | groups | slot totals | per-thread counters | task-list prefix
__host__ __device__ inline size_t smem_bytes(uint32_t nn, uint32_t ng, uint32_t ns) {
    return bfs::smem_bytes(nn, ng, ns, kTB);
}

__device__ __forceinline__ bfs::Smem setup(const WParams &w, const bfs::BParams &bp, unsigned char *smem,
                                           bool prefix) {
    bfs::Smem s;
    size_t o = 0;
    s.nodes = reinterpret_cast<lane::LNode *>(smem + o);
    o += lane::align16((size_t)w.n_nodes * sizeof(lane::LNode));
    s.groups = reinterpret_cast<DGroup *>(smem + o);
    o += lane::align16((size_t)w.n_groups * sizeof(DGroup));
    s.tot = reinterpret_cast<unsigned long long *>(smem + o);
    o += lane::align16((size_t)w.n_slots * 8);
    s.cnt = reinterpret_cast<uint32_t *>(smem + o);
    o += (size_t)w.n_slots * blockDim.x * 4;
    s.pref = reinterpret_cast<uint32_t *>(smem + o);
    for (uint32_t i = threadIdx.x; i < w.n_nodes; i += blockDim.x) s.nodes[i] = w.nodes[i];
    for (uint32_t i = threadIdx.x; i < w.n_groups; i += blockDim.x) s.groups[i] = w.groups[i];
    for (uint32_t i = threadIdx.x; i < w.n_slots; i += blockDim.x) s.tot[i] = 0;
    for (uint32_t i = 0; i < w.n_slots; i++) s.cnt[i * blockDim.x + threadIdx.x] = 0;
    if (prefix && threadIdx.x == 0) {
        uint32_t acc = 0;
        for (int i = 0; i < kStripes; i++) {
            s.pref[i] = acc;
            acc += min(w.in_tasks.cnt[i], w.in_tasks.seg_cap);
        }
        s.pref[kStripes] = acc;
    }
    (void)bp;
    __syncthreads();
    return s;
}

// ---------------------------------------------------------------- wave 0: root tasks
template <int MAXV, bool STATS>
__global__ void __launch_bounds__(kTB) root_kernel(const __grid_constant__ WParams w) {
    extern __shared__ __align__(16) unsigned char smem[];
    const bfs::BParams bp = graph_params(w);
    const bfs::Smem s = setup(w, bp, smem, false);
    Ctx c;
    c.cnt = s.cnt + threadIdx.x;
    c.stride = blockDim.x;
    c.tot = s.tot;
#pragma unroll
    for (int i = 0; i < ST_N; i++) c.st[i] = 0;
    const lane::LNode root = s.nodes[0];
    for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < w.n_roots; i += gridDim.x * blockDim.x) {
        const uint32_t r = w.r0 + i;
        PM<MAXV> x;
        if (!bfs::load_root<MAXV>(bp, r, x)) {  // a self-loop never matches 0->1 (reading R7)
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
        if (root.flags & NODE_INNER) queue_windows<MAXV, STATS>(w, bp, s.nodes, s.groups, root, x, r, c);
    }
    bfs::flush<STATS>(bp, s, c);
}

// ---------------------------------------------------------------- wave k: scan window tasks
// SUB lanes per task (kSub, or 32 for long windows); lane j takes entries start+j, +SUB, ...
template <int MAXV, int SUB, bool L0, bool STATS>
__global__ void __launch_bounds__(kTB) scan_kernel(const __grid_constant__ WParams w) {
    constexpr int W = bfs::Rec<MAXV>::W;
    extern __shared__ __align__(16) unsigned char smem[];
    const bfs::BParams bp = graph_params(w);
    const bfs::Smem s = setup(w, bp, smem, true);
    Ctx c;
    c.cnt = s.cnt + threadIdx.x;
    c.stride = blockDim.x;
    c.tot = s.tot;
#pragma unroll
    for (int i = 0; i < ST_N; i++) c.st[i] = 0;
    const uint32_t n_tasks = s.pref[kStripes];
    const uint32_t gtid = blockIdx.x * blockDim.x + threadIdx.x;
    const uint32_t j = gtid % SUB;
    const uint32_t gshift = (threadIdx.x & 31) & ~(uint32_t)(SUB - 1);
    const unsigned gmask = (SUB == 32) ? kFull : (((1u << SUB) - 1u) << gshift);
    for (uint32_t t = gtid / SUB; t < n_tasks; t += (gridDim.x * blockDim.x) / SUB) {
        int lo = 0, hi = kStripes - 1;  // segment of task t
        while (lo < hi) {
            const int mid = (lo + hi + 1) >> 1;
            if (s.pref[mid] <= t) lo = mid;
            else hi = mid - 1;
        }
        const uint32_t *tk = w.in_tasks.data + ((size_t)lo * w.in_tasks.seg_cap + (t - s.pref[lo])) * kTaskWords;
        const uint32_t ref = __ldg(tk), g = __ldg(tk + 1), start = __ldg(tk + 2);
        PM<MAXV> x;
        if (L0) bfs::load_root<MAXV>(bp, ref, x);
        else load_pm<MAXV>(w.in_pm + (size_t)ref * W, x);
        const DGroup G = s.groups[g];
        const uint32_t lim = G.kind == ANCHOR_GLOBAL ? x.h + 1 : kNone;
        if (STATS && j == 0) { c.st[ST_WINDOWS]++; c.st[ST_BYTES] += G.kind == ANCHOR_GLOBAL ? 12 : 8; }
        // the window ends at the FIRST entry past hi(root): entries after a list's sentinel
        // belong to the next vertex, so the lane group agrees on the end per batch
        for (uint32_t b = start;; b += SUB) {
            const uint32_t pos = b + j;
            uint32_t etr, e1, e2;
            bfs::load_entry(bp, G, pos, lim, etr, e1, e2);
            if (STATS) c.st[ST_BATCHES]++;
            const bool out = etr > x.h || pos >= lim;
            const unsigned fm = (__ballot_sync(gmask, out) >> gshift) & ((SUB == 32) ? kFull : ((1u << SUB) - 1u));
            const bool valid = !out && (fm == 0 || j < (uint32_t)(__ffs(fm) - 1)) && etr > x.tr_prev;
            if (valid) {
                if (STATS) { c.st[ST_ENTRIES]++; c.st[ST_BYTES] += G.kind == ANCHOR_GLOBAL ? 12 : 8; }
                const uint32_t ch = bfs::find_child(s.nodes, G, bfs::entry_class<MAXV>(G, x.m2g, e1, e2));
                if (ch != kNone) {
                    const lane::LNode dn = s.nodes[ch];
                    if (dn.flags & NODE_COMPLETION) {
                        bfs::count_add(c, dn.slot, 1);
                        if (STATS) c.st[ST_MATCHES]++;
                    }
                    if (dn.flags & NODE_INNER)
                        spawn<MAXV, STATS>(w, bp, s.nodes, s.groups, G, dn, ch, x, pos, etr, e1, e2, c);
                }
            }
            if (fm) break;
        }
    }
    bfs::flush<STATS>(bp, s, c);
}

}  // namespace wave
