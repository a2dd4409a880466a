// wdfs.cuh -- warp-synchronous depth-first co-mining over a shared-memory stack of window
// pieces (the default depth-first phase of the hybrid form), included by comine.cu after
// flat.cuh.
//
// Algorithm 3 "Co-Mining" walks, from every root edge, the MG-Tree
// depth-first: at a node it scans the candidate window of each anchor group (Algo 1
// l.210-217: entries after the previous edge, up to t_root + delta), tests each candidate
// (Algo 1 l.219 + full injectivity, reading R4), counts completions (Algo 3 l.661) and
// descends into inner children (Algo 3 l.665-669).
//
// Mapping to a warp.  The depth-first lane kernel (lane.cuh) gives each lane its
// own search and spends ~10.7 warp instructions per window entry on a divergent per-lane state
// machine (profiles/r2a_C4.md).  Here the WARP owns one depth-first search frontier, kept as a
// LIFO stack of window pieces in shared memory; one piece = one anchor-group window of one
// partial match, with everything needed to test its entries:
//     { group g, first list position, candidate count n, tr_prev, hi(root), root edge, m2g }
// Every round the warp takes the top pieces until it has 32 candidate entries (the last piece
// possibly split) and gives ONE ENTRY TO EACH LANE: an OR-reduction of the pieces' start
// offsets lets every lane find its piece with one popc/clz; then load, time test, class of the
// neighbour against the piece's m2g, SIMD child lookup, completion count -- straight-line code
// on full warps.  A lane whose entry matched an inner child builds the child partial match
// (its successor pointers were loaded with the entry) and locates the child's windows: start
// from P / R / search (exact), length bounded by six independent probes at offsets
// 0, 1, 3, 7, 15, 31 (windows of >= 32 entries: galloping + bisection to a 32-entry bracket);
// entries past the window fail the time test.  The new pieces are pushed on top (warp-
// aggregated), so the search stays depth-first and the stack small.  When the stack holds
// fewer than 32 candidates the warp takes the next 32 items (partial matches written by the
// breadth-first level, light roots, or root edges) from a global cursor.
// Stack overflow never loses work: the lane mines that subtree serially (bfs::dfs).
// Counts are identical to every other kernel form (tests/test_gpu_forms.py).

namespace wdfs {

#ifndef WDFS_SLOTS
#define WDFS_SLOTS 2  // candidate entries per lane per round
#endif
constexpr int kSlots = WDFS_SLOTS;
#ifndef WDFS_CNT16
#define WDFS_CNT16 1  // u16 lane counters (flushed at 65535): half the shared memory of u32, more L1 (C4 68.6 -> 66.0 ms)
#endif
#if WDFS_CNT16
typedef uint16_t cnt_t;
#else
typedef uint32_t cnt_t;
#endif
#ifndef WDFS_MINB
#define WDFS_MINB 5  // resident blocks per SM the register allocation targets (96 registers)
#endif

constexpr int kWB = 128;                 // threads per block
constexpr int kWarps = kWB / 32;
#ifndef WDFS_CAP
#define WDFS_CAP 96  // r2 sweep on C4: 64 / 80 / 96 / 128 -> 78.1 / 77.3 / 75.4 / 77.8 ms
#endif
constexpr int kCap = WDFS_CAP;           // pieces per warp stack in shared memory
#ifndef WDFS_PROBE8
#define WDFS_PROBE8 1  // window lengths from 8 consecutive loads (0: 4 probes + bisection; C4 -3 %, C3 -5 %)
#endif
#ifndef WDFS_PRE
#define WDFS_PRE 1  // anchor groups of a new partial match whose windows are located together (with PROBE8: 1 beats 2 by 0.7 %, 3 spills; w47)
#endif
constexpr int kPre = WDFS_PRE;
constexpr int kCapSmall = 64;            // test instance (MAYURA_WDFS_SMALL=1): spills early and often
constexpr uint8_t NODE_NEEDP = 16;       // LNode flag: a group of the node needs its edge's successor
                                         // pointers (a START_P* group that is not a same-list continuation)

// WDFS_CHECK builds (A/B variant, tools/gpu_dbg.sh): device-side bounds checks that print and trap
#ifdef WDFS_CHECK
#define WCHECK(cond, fmt, ...)                                                                      \
    do {                                                                                            \
        if (!(cond)) {                                                                              \
            printf("WDFS_CHECK %s:%d block %d lane %d: " fmt "\n", __FILE__, __LINE__, blockIdx.x,   \
                   threadIdx.x, __VA_ARGS__);                                                       \
            __trap();                                                                               \
        }                                                                                           \
    } while (0)
#else
#define WCHECK(cond, fmt, ...) \
    do {                       \
    } while (0)
#endif

template <int MAXV>
struct Piece {
    // words per piece: 0 group, 1 pos, 2 n, 3 tr_prev, 4 h, 5 root, 6.. m2g[MAXV]
    // (shared memory: SoA, field f of piece i at f * CAP + i; spill area: AoS, F words per piece)
    static constexpr int F = 6 + MAXV;
};

struct WParams {
    bfs::BParams b;          // graph arrays, table, counts, fallback counter; b.in = the breadth-first
                             // level's partial-match records (hybrid), b.light = its light roots
    const uint32_t *gwant;   // per group: wants of its first 4 children (bytes, 0xFD pad)
    uint32_t *lb;            // [0]: item cursor (zeroed per query by the launcher)
    uint32_t *spill;         // per warp spill_cap pieces (AoS): the bottom of a full stack
    uint32_t spill_cap;
    uint32_t direct;         // 1: the items are the root edges [r0, r0 + n_roots) themselves
    uint32_t o_cnt, o_stk;   // dynamic shared memory offsets: lane counters, stacks
    uint32_t lanecnt;        // 1: per-lane u32 counters; 0: block u64 atomics (many slots)
    uint32_t chunk_max;      // items a warp takes from the cursor at once (multiple of 32)
    uint32_t ent_len;        // adjacency entries (E + V, sentinels included) -- WDFS_CHECK only
};

// dynamic shared memory: nodes | groups | slot totals (u64) | node info | group info | group wants |
// lane counters | per-warp stacks + staging
__host__ __device__ inline size_t off_info(uint32_t nn, uint32_t ng, uint32_t ns) {
    return lane::align16((size_t)nn * sizeof(lane::LNode)) + lane::align16((size_t)ng * sizeof(DGroup)) +
           lane::align16((size_t)ns * 8);
}
__host__ __device__ inline size_t off_cnt(uint32_t nn, uint32_t ng, uint32_t ns) {
    return off_info(nn, ng, ns) + lane::align16((size_t)nn * 4) + 3 * lane::align16((size_t)ng * 4);
}
__host__ __device__ inline size_t off_stk(uint32_t nn, uint32_t ng, uint32_t ns, bool lanecnt) {
    return lane::align16(off_cnt(nn, ng, ns) + (lanecnt ? (size_t)ns * kWB * sizeof(cnt_t) : 0));
}
__host__ __device__ inline size_t smem_bytes(uint32_t nn, uint32_t ng, uint32_t ns, bool lanecnt, int maxv, int cap) {
    return off_stk(nn, ng, ns, lanecnt) + (size_t)kWarps * ((6 + maxv) * cap + (kSlots - 1) * (10 + maxv) * 32) * 4;
}

// Length of a window: entries [lo, lo + n) are the entries of list `ent` from lo with time
// rank <= h, stopping at the list's sentinel (index `sent`).  Four independent probes at offsets
// 0, 1, 3, 7 (two 32-byte sectors; lists are padded past their last sentinel, so lo + 7 is in
// bounds; an index at or past the sentinel is out whatever it holds) bracket n; a bisection inside
// the bracket makes it exact (<= 2 dependent loads on the sectors the probes just brought in).
// Windows of >= 8 entries gallop on (15, 31, 63, ...: dependent loads, the rarer case).  Wider
// unconditional probes cost more L2 sectors than they save round trips (profiles/README.md r2).
__device__ __forceinline__ bool in_window(const uint2 *ent, uint32_t lo, uint32_t o, uint32_t sent, uint32_t h) {
    return lo + o < sent && __ldg(&ent[lo + o].x) <= h;
}
__device__ __forceinline__ uint32_t window_len(const uint2 *ent, uint32_t lo, uint32_t sent, uint32_t h) {
#if WDFS_PROBE8
    // every entry of the first 8 (two sectors): exact for windows of <= 7 entries, no dependent load
    uint32_t v[8];
#pragma unroll
    for (int k = 0; k < 8; k++) v[k] = __ldg(&ent[lo + k].x);
    uint32_t b = kNone;
#pragma unroll
    for (int k = 7; k >= 0; k--)
        if (lo + k >= sent || v[k] > h) b = k;
    if (b != kNone) return b;
    uint32_t a = 7;
    b = 15;
    {
#else
    const uint32_t o[4] = {0, 1, 3, 7};
    uint32_t v[4];
#pragma unroll
    for (int k = 0; k < 4; k++) v[k] = __ldg(&ent[lo + o[k]].x);
    uint32_t b = kNone, a = 0;  // out at offset b; in at every probe below it
#pragma unroll
    for (int k = 3; k >= 0; k--)
        if (lo + o[k] >= sent || v[k] > h) b = o[k];
    if (b == 0) return 0;
    if (b != kNone) {
        a = b == 1 ? 0 : (b - 1) / 2;  // the previous probe offset (in)
    } else {  // >= 8 entries: gallop
#endif
        a = 7;
        b = 15;
        for (;;) {
            if (lo + b >= sent) {
                b = sent - lo;
                break;
            }
            if (__ldg(&ent[lo + b].x) > h) break;
            a = b;
            b = 2 * b + 1;
        }
    }
    while (b - a > 1) {  // in(a), out(b): n in (a, b]
        const uint32_t m = a + ((b - a) >> 1);
        if (in_window(ent, lo, m, sent, h)) a = m;
        else b = m;
    }
    return b;
}

// Window of group G for partial match x: first position and length (exact up to entries tied
// with tr_prev, which the time test skips).
template <int MAXV, bool GEN>
__device__ __forceinline__ uint32_t window(const bfs::BParams &p, const DGroup &G, const bfs::PM<MAXV> &x,
                                           uint32_t &n) {
    if (GEN && G.kind == ANCHOR_GLOBAL) {  // edge ids after tr_prev's tie group, up to hi(root) (R6)
        uint32_t lo = x.tr_prev, hi2 = x.h + 1;
        while (lo < hi2) {
            const uint32_t mid = lo + ((hi2 - lo) >> 1);
            if (__ldg(p.tr + mid) > x.tr_prev) hi2 = mid;
            else lo = mid + 1;
        }
        n = x.h + 1 > lo ? x.h + 1 - lo : 0;
        return lo;
    }
    const bool out = G.kind == ANCHOR_OUT;
    const uint2 *ent = out ? p.out_ent : p.in_ent;
    const uint32_t *off = out ? p.out_off : p.in_off;
    const uint32_t v = lane::m2g_get<MAXV>(x.m2g, G.anchor);
    const uint32_t sent = __ldg(off + v + 1) - 1;
    uint32_t lo;
    if (G.start < START_R0) {
        lo = lane::pick4(x.P, G.start);  // exact: successor pointer of the node's own edge
    } else if (!GEN || G.start < START_SEARCH) {
        const uint4 R = __ldg(p.eptr + x.root);  // lower bound from the root edge: skip to > tr_prev
        lo = flat::first_gt(ent, lane::pick4(R, G.start - START_R0), sent, x.tr_prev);
    } else {  // search the anchor's list for the first entry after tr_prev
        uint32_t a = __ldg(off + v), b = sent;
        while (a < b) {
            const uint32_t mid = a + ((b - a) >> 1);
            if (__ldg(&ent[mid].x) > x.tr_prev) b = mid;
            else a = mid + 1;
        }
        lo = a;
    }
    n = window_len(ent, lo, sent, x.h);
    WCHECK(lo <= sent && lo + n <= sent, "window lo %u n %u sent %u start %u anchor %u v %u", lo, n, sent,
           (unsigned)G.start, (unsigned)G.anchor, v);
    return lo;
}

// Warp-collective: move the bottom m pieces of the shared-memory stack to the warp's spill area
// (coalesced AoS writes) and shift the rest down, 32 pieces at a time in ascending order, each
// chunk read before it is written (no chunk's destination overlaps a later chunk's source).
template <int MAXV, int CAP>
__device__ __noinline__ void spill_bottom(uint32_t *stk, uint32_t ps, uint32_t m, uint32_t *sp, uint32_t sp_top) {
    constexpr int F = Piece<MAXV>::F;
    const uint32_t lane_id = threadIdx.x & 31;
    for (uint32_t wi = lane_id; wi < m * F; wi += 32) {
        const uint32_t i = wi / F, f = wi - i * F;
        sp[(size_t)(sp_top + i) * F + f] = stk[f * CAP + i];
    }
    __syncwarp();
    for (uint32_t c = 0; c < ps - m; c += 32) {
        const uint32_t i = c + lane_id;
        uint32_t t[F];
#pragma unroll
        for (int f = 0; f < F; f++) t[f] = i < ps - m ? stk[f * CAP + m + i] : 0u;
        __syncwarp();
        if (i < ps - m)
#pragma unroll
            for (int f = 0; f < F; f++) stk[f * CAP + i] = t[f];
        __syncwarp();
    }
}

// Warp-collective: move the top m pieces of the spill area onto the (empty) stack.
template <int MAXV, int CAP>
__device__ __noinline__ void reload(uint32_t *stk, uint32_t m, const uint32_t *sp, uint32_t sp_top) {
    constexpr int F = Piece<MAXV>::F;
    const uint32_t lane_id = threadIdx.x & 31;
    for (uint32_t wi = lane_id; wi < m * F; wi += 32) {
        const uint32_t i = wi / F, f = wi - i * F;
        stk[f * CAP + i] = sp[(size_t)(sp_top - m + i) * F + f];
    }
    __syncwarp();
}

// Packed table words (wdfs_kernel prologue): per group, kind | SIMD child lookup possible | a
// child locates a window from the entry's successor pointers | first child << 16; per node,
// completion slot | completion | inner | n_new << 18 | nv << 24.
constexpr uint32_t GI_KIND = 3u, GI_SIMD = 4u, GI_NEEDP = 8u;
constexpr uint32_t NI_COMPLETION = 1u << 16, NI_INNER = 1u << 17;
__device__ __forceinline__ uint32_t group_info(const DGroup &G, const lane::LNode *nodes) {
    bool np = false;
    for (uint32_t ch = G.child_begin; ch < G.child_end; ch++) {
        const lane::LNode dn = nodes[ch];
        np = np || ((dn.flags & NODE_INNER) && (dn.flags & NODE_NEEDP));
    }
    const bool simd = G.child_end - G.child_begin <= 4;
    return (uint32_t)G.kind | (simd ? GI_SIMD : 0u) | (np ? GI_NEEDP : 0u) | ((uint32_t)G.child_begin << 16);
}
__device__ __forceinline__ uint32_t node_info(const lane::LNode &n) {
    return (uint32_t)(n.slot & 0xFFFFu) | ((n.flags & NODE_COMPLETION) ? NI_COMPLETION : 0u) |
           ((n.flags & NODE_INNER) ? NI_INNER : 0u) | ((uint32_t)(n.n_new & 3u) << 18) | ((uint32_t)n.nv << 24);
}

// Per group, the shape of the star chains' last level: exactly one child, a leaf (a completion
// with no children) that wants a NEW vertex from an OUT/IN list.  GL_FLAG | mapped vertices of the
// parent << 16 | the child's completion slot; 0 otherwise.  A round whose candidates all belong to
// such a group runs the specialised leaf_round<NV> (NV compile-time: the m2g compares unrolled to
// exactly the mapped vertices, the slot an operand, no child lookup).
constexpr uint32_t GL_FLAG = 1u << 31;
__device__ __forceinline__ uint32_t group_leaf(const DGroup &G, const lane::LNode *nodes) {
    if (G.kind == ANCHOR_GLOBAL || G.child_end - G.child_begin != 1) return 0u;
    const lane::LNode c = nodes[G.child_begin];
    if ((c.flags & NODE_INNER) || !(c.flags & NODE_COMPLETION) || c.want != CLS_NEW || c.n_new != 1) return 0u;
    return GL_FLAG | ((uint32_t)(c.nv - 1) << 16) | (uint32_t)(c.slot & 0xFFFFu);
}

// Per-warp staging area (shared memory, SoA, 32 slots = one per lane) of the children found by a
// round's second slots, expanded after the first slots' ones.  Words: 0 node | c_out << 31,
// 1 tr_prev, 2 h, 3 root, 4..7 P, 8 c_lo, 9 c_end, 10.. m2g[MAXV]
template <int MAXV>
struct Stage {
    static constexpr int F = 10 + MAXV;
};
template <int MAXV>
__device__ __forceinline__ void stage_put(uint32_t *sg, uint32_t lane, const bfs::PM<MAXV> &x, uint32_t c_lo,
                                          uint32_t c_end, bool c_out) {
    sg[0 * 32 + lane] = x.node | (c_out ? 0x80000000u : 0u);
    sg[1 * 32 + lane] = x.tr_prev;
    sg[2 * 32 + lane] = x.h;
    sg[3 * 32 + lane] = x.root;
    sg[4 * 32 + lane] = x.P.x;
    sg[5 * 32 + lane] = x.P.y;
    sg[6 * 32 + lane] = x.P.z;
    sg[7 * 32 + lane] = x.P.w;
    sg[8 * 32 + lane] = c_lo;
    sg[9 * 32 + lane] = c_end;
#pragma unroll
    for (int k = 0; k < MAXV; k++) sg[(10 + k) * 32 + lane] = x.m2g[k];
}
template <int MAXV>
__device__ __forceinline__ void stage_get(const uint32_t *sg, uint32_t lane, bfs::PM<MAXV> &x, uint32_t &c_lo,
                                          uint32_t &c_end, bool &c_out, const lane::LNode *s_nodes) {
    const uint32_t w0 = sg[0 * 32 + lane];
    x.node = w0 & 0xFFFFu;
    c_out = (w0 >> 31) != 0;
    x.nv = s_nodes[x.node].nv;
    x.tr_prev = sg[1 * 32 + lane];
    x.h = sg[2 * 32 + lane];
    x.root = sg[3 * 32 + lane];
    x.P = make_uint4(sg[4 * 32 + lane], sg[5 * 32 + lane], sg[6 * 32 + lane], sg[7 * 32 + lane]);
    c_lo = sg[8 * 32 + lane];
    c_end = sg[9 * 32 + lane];
#pragma unroll
    for (int k = 0; k < MAXV; k++) x.m2g[k] = sg[(10 + k) * 32 + lane];
}

// Warp-collective: every lane with `has` locates the windows of x's anchor groups and pushes the
// non-empty ones on the warp's stack (warp-aggregated).  A full stack spills its bottom half to
// global memory; a full spill area makes the lane mine x from that group on depth-first itself
// (exact; counted in p.fallback).
// A child matched at list position c_lo - 1 of its parent's window [.., c_end) continues on the
// same list in every group flagged in its node's `same` mask: that window is [c_lo, c_end), no
// memory access needed (items from a global cursor pass c_end = 0: no continuation).
template <int MAXV, bool GEN, int CAP, bool STATS>
__device__ __forceinline__ void open_push(const WParams &w, const lane::LNode *s_nodes, const DGroup *s_groups,
                                          uint32_t *stk, uint32_t &ps, uint32_t *sp, uint32_t &sp_top, bool has,
                                          const bfs::PM<MAXV> &x, uint32_t c_lo, uint32_t c_end, bool c_out,
                                          cnt_t *my_cnt, unsigned long long *s_tot, unsigned long long *st) {
    const bfs::BParams &p = w.b;
    const uint32_t lane_id = threadIdx.x & 31;
    uint32_t gb = 0, ng = 0, same = 0;
    if (has) {
        const lane::LNode xn = s_nodes[x.node];
        gb = xn.group_begin;
        ng = xn.group_end - xn.group_begin;
        same = c_end ? xn.same : 0u;
    }
    const uint32_t mg = __reduce_max_sync(kFull, ng);
    // the windows of the first kPre groups are located together (independent loads in flight at
    // once), before any is pushed
    uint32_t plo[kPre], pn[kPre];
#pragma unroll
    for (int q = 0; q < kPre; q++) {
        plo[q] = 0;
        pn[q] = 0;
        if ((uint32_t)q < ng) {
            if ((same >> q) & 1u) {
                plo[q] = c_lo;
                pn[q] = c_end > c_lo ? c_end - c_lo : 0u;
                WCHECK(c_lo <= c_end + 1, "continuation c_lo %u c_end %u node %u", c_lo, c_end, x.node);
            } else {
                plo[q] = window<MAXV, GEN>(p, s_groups[gb + q], x, pn[q]);
            }
        }
    }
    bool fell = false;
    for (uint32_t q = 0; q < mg; q++) {
        uint32_t lo = 0, n = 0;
        const bool mine = q < ng && !fell;
        if (q < (uint32_t)kPre) {
#pragma unroll
            for (int k = 0; k < kPre; k++)
                if ((uint32_t)k == q) {
                    lo = plo[k];
                    n = pn[k];
                }
        } else if (mine) {
            if ((same >> q) & 1u) {
                lo = c_lo;
                n = c_end > c_lo ? c_end - c_lo : 0u;
            } else {
                lo = window<MAXV, GEN>(p, s_groups[gb + q], x, n);
            }
        }
        const bool v = mine && n > 0;
        const unsigned bm = __ballot_sync(kFull, v);
        const uint32_t cnt = __popc(bm);
        if (ps + cnt > CAP && ps >= 2 && sp_top + ps / 2 <= w.spill_cap) {
            spill_bottom<MAXV, CAP>(stk, ps, ps / 2, sp, sp_top);
            sp_top += ps / 2;
            ps -= ps / 2;
            if (STATS && lane_id == 0) st[ST_OFFLOADS]++;
        }
        const uint32_t slot = ps + __popc(bm & ((1u << lane_id) - 1u));
        if (v) {
            if (slot < CAP) {
                stk[0 * CAP + slot] = gb + q;
                stk[1 * CAP + slot] = lo;
                stk[2 * CAP + slot] = n;
                stk[3 * CAP + slot] = x.tr_prev;
                stk[4 * CAP + slot] = x.h;
                stk[5 * CAP + slot] = x.root;
#pragma unroll
                for (int k = 0; k < MAXV; k++) stk[(6 + k) * CAP + slot] = x.m2g[k];
            } else {
                if (p.fallback) atomicAdd(p.fallback, 1u);
                bfs::PM<MAXV> y = x;
                if (c_end)  // a child: its successor pointers may not have been loaded with the entry
                    y.P = __ldg((c_out ? p.out_ptr : p.in_ptr) + (c_lo - 1));
                bfs::Ctx c;  // built here only: a Ctx whose address escapes lives in local memory
                c.cnt = sizeof(cnt_t) == 4 ? reinterpret_cast<uint32_t *>(my_cnt) : nullptr;  // u16: block atomics
                c.stride = kWB;
                c.tot = s_tot;
                c.em_next = c.em_end = 0;
                bfs::dfs<MAXV, false>(p, s_nodes, s_groups, y, c, gb + q);
                fell = true;
            }
        }
        ps = min(ps + cnt, (uint32_t)CAP);
        if (STATS && lane_id == 0) st[ST_WINDOWS] += cnt;
    }
    __syncwarp();
}

template <int MAXV, bool GEN, int CAP, bool STATS>
__global__ void __launch_bounds__(kWB, WDFS_MINB) wdfs_kernel(const __grid_constant__ WParams w) {
    pdl_begin();
    const bfs::BParams &p = w.b;
    extern __shared__ __align__(16) unsigned char smem[];
    lane::LNode *s_nodes = reinterpret_cast<lane::LNode *>(smem);
    DGroup *s_groups = reinterpret_cast<DGroup *>(smem + lane::align16((size_t)p.n_nodes * sizeof(lane::LNode)));
    unsigned long long *s_tot = reinterpret_cast<unsigned long long *>(
        smem + lane::align16((size_t)p.n_nodes * sizeof(lane::LNode)) + lane::align16((size_t)p.n_groups * sizeof(DGroup)));
    cnt_t *s_cnt = w.lanecnt ? reinterpret_cast<cnt_t *>(smem + w.o_cnt) : nullptr;
    const uint32_t tid = threadIdx.x, lane_id = tid & 31;
    constexpr int F = Piece<MAXV>::F;
    constexpr int SF = Stage<MAXV>::F;
    uint32_t *stk = reinterpret_cast<uint32_t *>(smem + w.o_stk) + (size_t)(tid >> 5) * (F * CAP + (kSlots - 1) * SF * 32);
    uint32_t *sg = stk + F * CAP;
    uint32_t *sp = w.spill + (size_t)(blockIdx.x * kWarps + (tid >> 5)) * w.spill_cap * F;
    __shared__ uint32_t s_pref[bfs::kStripes + 1];
    // Packed per-node / per-group words (one 32-bit shared load per candidate instead of the 12- and
    // 8-byte table rows and their byte extraction) and the groups' packed child wants
    uint32_t *s_ninfo = reinterpret_cast<uint32_t *>(smem + off_info(p.n_nodes, p.n_groups, p.n_slots));
    uint32_t *s_ginfo = s_ninfo + lane::align16((size_t)p.n_nodes * 4) / 4;
    uint32_t *s_gw = s_ginfo + lane::align16((size_t)p.n_groups * 4) / 4;
    uint32_t *s_gleaf = s_gw + lane::align16((size_t)p.n_groups * 4) / 4;
    for (uint32_t i = tid; i < p.n_nodes; i += kWB) s_nodes[i] = p.nodes[i];
    for (uint32_t i = tid; i < p.n_groups; i += kWB) s_groups[i] = p.groups[i];
    for (uint32_t i = tid; i < p.n_groups; i += kWB) s_gw[i] = w.gwant[i];
    for (uint32_t g = tid; g < p.n_groups; g += kWB) s_ginfo[g] = group_info(p.groups[g], p.nodes);
    for (uint32_t n = tid; n < p.n_nodes; n += kWB) s_ninfo[n] = node_info(p.nodes[n]);
    for (uint32_t g = tid; g < p.n_groups; g += kWB) s_gleaf[g] = group_leaf(p.groups[g], p.nodes);
    for (uint32_t i = tid; i < p.n_slots; i += kWB) s_tot[i] = 0;
    if (s_cnt)
        for (uint32_t i = 0; i < p.n_slots; i++) s_cnt[i * kWB + tid] = 0;
    if (tid == 0) {
        uint32_t acc = 0;
        for (int i = 0; i < bfs::kStripes; i++) {
            s_pref[i] = acc;
            acc += (!w.direct && p.in.data) ? min(p.in.cnt[i], p.in.seg_cap) : 0u;
        }
        s_pref[bfs::kStripes] = acc;
    }
    __syncthreads();

    // completion counters: this lane's u32 per slot (flushed to the block's u64 before 2^31), or
    // block u64 atomics when the group has too many slots (kept in registers, not in a bfs::Ctx:
    // the fallback passes one by address, which would put it in local memory)
    cnt_t *const my_cnt = s_cnt ? s_cnt + tid : nullptr;
    auto cnt_add = [&](uint32_t slot, uint32_t inc = 1u) {
        if (my_cnt) {
            cnt_t *q = my_cnt + slot * kWB;
            uint32_t v = *q + inc;
            if (v >= (sizeof(cnt_t) == 4 ? 0x80000000u : 0xFFF0u)) {
                atomicAdd(&s_tot[slot], (unsigned long long)v);
                v = 0;
            }
            *q = (cnt_t)v;
        } else {
            atomicAdd(&s_tot[slot], (unsigned long long)inc);
        }
    };
    unsigned long long st[ST_N];
#pragma unroll
    for (int i = 0; i < ST_N; i++) st[i] = 0;

    const lane::LNode root = s_nodes[0];
    const uint32_t n_pm = s_pref[bfs::kStripes];
    const uint32_t n_items = w.direct ? p.n_roots : n_pm + (p.light ? *(volatile const uint32_t *)p.light_cnt : 0u);

    uint32_t ps = 0;           // warp-uniform stack height (shared memory)
    uint32_t sp_top = 0;       // warp-uniform spilled pieces (global memory)
    uint32_t cb = 0, cl = 0;   // warp-uniform item chunk
    bool items_left = true;

    // The specialised round of a leaf group (all candidates in one group whose only child is a leaf
    // wanting a NEW vertex, with NV mapped vertices before it): per slot, the entry, the time test
    // and NV compares against the piece's mapped vertices; the completion slot is an operand.
    auto leaf_round = [&](auto nv_tag, const uint32_t (&spi)[kSlots], const uint32_t (&sat)[kSlots], uint32_t T,
                          uint32_t gl) {
        constexpr int NV = decltype(nv_tag)::value;
        const uint32_t slot = gl & 0xFFFFu;
        const bool out = (s_ginfo[stk[0 * CAP + spi[0]]] & GI_KIND) == ANCHOR_OUT;
        const uint2 *ent = out ? p.out_ent : p.in_ent;
        uint32_t nf = 0;  // completions of this lane's slots: one counter update per lane and round
#pragma unroll
        for (int sl = 0; sl < kSlots; sl++) {
            if (lane_id + 32u * sl < T) {
                const uint32_t pi = spi[sl];
                const uint2 e = __ldg(ent + stk[1 * CAP + pi] + sat[sl]);
                const uint32_t tp = stk[3 * CAP + pi], h = stk[4 * CAP + pi];
                bool fresh = e.x > tp && e.x <= h;
#pragma unroll
                for (int k = 0; k < NV; k++) fresh = fresh && stk[(6 + k) * CAP + pi] != e.y;
                nf += fresh ? 1u : 0u;
            }
        }
        if (nf) cnt_add(slot, nf);
    };

    // Test the candidate entry of one slot: window entry `at` of piece `pi`.  Completions are
    // counted; an inner hit fills y (the child partial match) and its continuation window.
    auto test_slot = [&](uint32_t pi, uint32_t at, bfs::PM<MAXV> &y, uint32_t &y_lo, uint32_t &y_end,
                         bool &y_out) -> bool {
        const uint32_t g = stk[0 * CAP + pi];
        const uint32_t p0 = stk[1 * CAP + pi];
        const uint32_t pos = p0 + at;
        WCHECK(pi < ps && at < stk[2 * CAP + pi] && g < p.n_groups, "slot pi %u ps %u at %u n %u g %u", pi, ps, at,
               stk[2 * CAP + pi], g);
        WCHECK((s_groups[g].kind == ANCHOR_GLOBAL && pos < p.E) || (s_groups[g].kind != ANCHOR_GLOBAL && pos < w.ent_len),
               "entry pos %u (p0 %u at %u) kind %u", pos, p0, at, (unsigned)s_groups[g].kind);
        const uint32_t tp = stk[3 * CAP + pi];
        const uint32_t h = stk[4 * CAP + pi];
        const uint32_t gi = s_ginfo[g];
        const bool glob = GEN && (gi & GI_KIND) == ANCHOR_GLOBAL;
        // successor pointers of the entry's edge, loaded with the entry (no extra round trip)
        // when a child of this group locates a window from them
        const bool needp = (gi & GI_NEEDP) != 0;
        uint32_t etr, e1, e2 = 0;
        uint4 P = make_uint4(0, 0, 0, 0);
        const bool out = (gi & GI_KIND) == ANCHOR_OUT;
        if (glob) {
            etr = __ldg(p.tr + pos);
            e1 = __ldg(p.src + pos);
            e2 = __ldg(p.dst + pos);
            if (needp) P = __ldg(p.eptr + pos);
        } else {
            const uint2 e = __ldg((out ? p.out_ent : p.in_ent) + pos);
            etr = e.x;
            e1 = e.y;
            if (needp) P = __ldg((out ? p.out_ptr : p.in_ptr) + pos);
        }
        uint32_t m2g[MAXV];
#pragma unroll
        for (int k = 0; k < MAXV; k++) m2g[k] = stk[(6 + k) * CAP + pi];
        const bool valid = etr > tp && etr <= h;
        if (STATS) st[ST_ENTRIES] += valid ? 1 : 0;
        uint32_t cls;
        if (glob)
            cls = (e1 != e2 && lane::classify<MAXV>(m2g, e1) == CLS_NEW &&
                   lane::classify<MAXV>(m2g, e2) == CLS_NEW) ? CLS_NEW : 0xFEu;
        else
            cls = lane::classify<MAXV>(m2g, e1);
        uint32_t hit = kNone;
        if (gi & GI_SIMD) {
            const uint32_t eq = __vcmpeq4(s_gw[g], cls * 0x01010101u);
            hit = eq ? (gi >> 16) + ((__ffs(eq) - 1) >> 3) : kNone;
        } else {
            hit = bfs::find_child(s_nodes, s_groups[g], cls);
        }
        if (!valid || hit == kNone) return false;
        const uint32_t ni = s_ninfo[hit];
        if (ni & NI_COMPLETION) cnt_add(ni & 0xFFFFu);
        if (STATS) st[ST_MATCHES] += (ni & NI_COMPLETION) ? 1 : 0;
        if (!(ni & NI_INNER)) return false;
        // the child partial match (Algo 3 l.665-669)
        const uint32_t n_new = (ni >> 18) & 3u, nv = ni >> 24;
#pragma unroll
        for (int k = 0; k < MAXV; k++) y.m2g[k] = m2g[k];
        if (n_new == 2) {
            lane::m2g_set<MAXV>(y.m2g, nv - 2u, e1);
            lane::m2g_set<MAXV>(y.m2g, nv - 1u, e2);
        } else if (n_new == 1) {
            lane::m2g_set<MAXV>(y.m2g, nv - 1u, e1);
        }
        y.node = hit;
        y.nv = nv;
        y.tr_prev = etr;
        y.h = h;
        y.root = stk[5 * CAP + pi];
        y.P = P;
        y_lo = glob ? 0u : pos + 1;
        y_end = glob ? 0u : p0 + stk[2 * CAP + pi];
        y_out = out;
        if (STATS) st[ST_NODES]++;
        return true;
    };

    for (;;) {
        // ---- the top 32 * kSlots pieces: candidate counts and their running sum (top first); lane l
        // holds pieces kSlots * l + i (one prefix sum of the per-lane sums)
        const uint32_t top = ps;
        uint32_t pn[kSlots], incl[kSlots], pg[kSlots];
        uint32_t lsum = 0;
#pragma unroll
        for (int i = 0; i < kSlots; i++) {
            const uint32_t idx = kSlots * lane_id + i;
            pn[i] = idx < top ? stk[2 * CAP + top - 1 - idx] : 0u;
            pg[i] = idx < top ? stk[0 * CAP + top - 1 - idx] : 0u;  // its group (the leaf-round test)
            lsum += pn[i];
        }
        uint32_t linc = lsum;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const uint32_t v = __shfl_up_sync(kFull, linc, o);
            if (lane_id >= (uint32_t)o) linc += v;
        }
        {
            uint32_t acc = linc - lsum;
#pragma unroll
            for (int i = 0; i < kSlots; i++) {
                acc += pn[i];
                incl[i] = acc;  // inclusive sum up to piece kSlots * l + i
            }
        }
        const uint32_t tot = __shfl_sync(kFull, linc, 31);
        bfs::PM<MAXV> x;   // this lane's new partial match: an item, or the first slot's child
        bool has = false;
        uint32_t hmask = 0;  // bit s: slot s (>= 1) staged a child
        uint32_t c_lo = 0, c_end = 0;  // a child's continuation window on its parent's list
        bool c_out = false;
        if (top == 0 && sp_top > 0) {
            // ---- the stack ran empty: bring back the most recently spilled pieces (depth first)
            const uint32_t m = min(sp_top, (uint32_t)CAP / 2);
            reload<MAXV, CAP>(stk, m, sp, sp_top);
            sp_top -= m;
            ps = m;
            if (STATS && lane_id == 0) st[ST_CONTEXTS]++;
            continue;
        }
        if (tot < 32 && items_left && sp_top == 0) {
            // ---- fewer than 32 candidates stacked: take the next items (one per lane)
            if (cl == 0) {
                uint32_t b = 0, sz = 0;
                if (lane_id == 0) {
                    const uint32_t cur = *(volatile uint32_t *)w.lb;
                    const uint32_t rem = cur < n_items ? n_items - cur : 0u;
                    sz = max(32u, min(w.chunk_max, (rem / (4u * gridDim.x * kWarps)) & ~31u));
                    b = atomicAdd(w.lb, sz);
                }
                b = __shfl_sync(kFull, b, 0);
                sz = __shfl_sync(kFull, sz, 0);
                if (b >= n_items) {
                    items_left = false;
                    continue;
                }
                cb = b;
                cl = min(sz, n_items - b);
            }
            const uint32_t take = min(32u, cl);
            const uint32_t item = cb + lane_id;
            cb += take;
            cl -= take;
            if (lane_id < take) {
                if (w.direct) {  // a root edge: count the root node's completion, expand it if inner
                    const uint32_t r = p.r0 + item;
                    if (bfs::load_root<MAXV>(p, r, x)) {
                        if (root.flags & NODE_COMPLETION) cnt_add(root.slot);
                        has = (root.flags & NODE_INNER) != 0;
                    }
                } else if (item < n_pm) {  // a partial match of the breadth-first level (counted there)
                    bfs::load_rec<MAXV>(p, s_pref, item, x);
                    has = x.node != bfs::kHole;
                } else {  // a light root (its completion was counted by the breadth-first level)
                    has = bfs::load_root<MAXV>(p, __ldg(p.light + (item - n_pm)), x);
                }
            }
            if (STATS && lane_id == 0) st[ST_ROOTS] += take;
        } else {
            if (top == 0) break;  // no items left, nothing stacked or spilled
            // ---- this round: T <= 32 * kSlots entries, kSlots slots per lane (lane + 32 s), from the
            // top pieces (the last one possibly split)
            const uint32_t T = min(tot, 32u * kSlots);
            uint32_t xs[kSlots], m[kSlots], kf = 0;
            bool same = true;  // every candidate of the round is in the top piece's group
            const uint32_t g0 = __shfl_sync(kFull, pg[0], 0);
            {
                uint32_t c[kSlots];
#pragma unroll
                for (int wv = 0; wv < kSlots; wv++) c[wv] = 0;
#pragma unroll
                for (int i = 0; i < kSlots; i++) {
                    xs[i] = incl[i] - pn[i];  // first slot of piece kSlots * l + i (pn = 0 past the top)
                    const bool pc = kSlots * lane_id + i < top && xs[i] < T;
                    const uint32_t bit = pc ? 1u << (xs[i] & 31) : 0u;
#pragma unroll
                    for (int wv = 0; wv < kSlots; wv++) c[wv] |= (xs[i] >> 5) == (uint32_t)wv ? bit : 0u;
                    same = same && (!pc || pg[i] == g0);
                }
#pragma unroll
                for (int wv = 0; wv < kSlots; wv++) m[wv] = __reduce_or_sync(kFull, c[wv]);
            }
#pragma unroll
            for (int i = 0; i < kSlots; i++)
                kf += __popc(__ballot_sync(kFull, kSlots * lane_id + i < top && incl[i] <= T));  // taken whole
            // the contributing pieces are a prefix (0, 1, ...) of the top pieces, one start bit each:
            // slot j belongs to piece (start bits <= j) - 1, which starts at the highest one
            const unsigned le = (2u << lane_id) - 1u;
            uint32_t before = 0, last = 0;  // start bits in the words below; highest start slot below
            if (STATS && lane_id == 0) {
                st[ST_BATCHES]++;
                st[ST_PROBES] += T;
            }
            uint32_t spi[kSlots], sat[kSlots];
#pragma unroll
            for (int sl = 0; sl < kSlots; sl++) {
                const uint32_t up = m[sl] & le;
                const uint32_t r = before + __popc(up) - 1u;                   // piece of slot lane + 32 sl
                const uint32_t s0 = up ? 32u * sl + 31 - __clz(up) : last;     // its first slot
                spi[sl] = top - 1 - r;
                sat[sl] = lane_id + 32u * sl - s0;
                before += __popc(m[sl]);
                if (m[sl]) last = 32u * sl + 31 - __clz(m[sl]);
            }
            const uint32_t gl = s_gleaf[g0];
            if (!STATS && gl && __all_sync(kFull, same)) {
                // a leaf round: the group's single child is a leaf wanting a NEW vertex
                const uint32_t nvp = (gl >> 16) & 0xFFu;
                if (nvp <= 2) leaf_round(std::integral_constant<int, 2>{}, spi, sat, T, gl);
                else if (nvp == 3 || MAXV <= 3) leaf_round(std::integral_constant<int, (MAXV < 3 ? MAXV : 3)>{}, spi, sat, T, gl);
                else if (nvp == 4 || MAXV <= 4) leaf_round(std::integral_constant<int, (MAXV < 4 ? MAXV : 4)>{}, spi, sat, T, gl);
                else if (nvp == 5 || MAXV <= 5) leaf_round(std::integral_constant<int, (MAXV < 5 ? MAXV : 5)>{}, spi, sat, T, gl);
                else if (nvp == 6 || MAXV <= 6) leaf_round(std::integral_constant<int, (MAXV < 6 ? MAXV : 6)>{}, spi, sat, T, gl);
                else leaf_round(std::integral_constant<int, MAXV>{}, spi, sat, T, gl);
            } else {
#pragma unroll
                for (int sl = 0; sl < kSlots; sl++) {
                    if (lane_id + 32u * sl < T) {
                        if (sl == 0) {
                            has = test_slot(spi[sl], sat[sl], x, c_lo, c_end, c_out);
                        } else {
                            bfs::PM<MAXV> yb;
                            uint32_t b_lo = 0, b_end = 0;
                            bool b_out = false;
                            const bool hb = test_slot(spi[sl], sat[sl], yb, b_lo, b_end, b_out);
                            if (hb) stage_put<MAXV>(sg + (sl - 1) * Stage<MAXV>::F * 32, lane_id, yb, b_lo, b_end, b_out);
                            hmask |= hb ? 1u << sl : 0u;
                        }
                    }
                }
            }
            __syncwarp();
            // ---- pop the pieces taken whole; advance the split one (piece kf)
            if (kf < top && kf < 32u * kSlots && kf / kSlots == lane_id) {
                uint32_t xk = xs[0];
#pragma unroll
                for (int i = 1; i < kSlots; i++)
                    if (kf % kSlots == (uint32_t)i) xk = xs[i];
                if (xk < T) {
                    stk[1 * CAP + top - 1 - kf] += T - xk;
                    stk[2 * CAP + top - 1 - kf] -= T - xk;
                }
            }
            ps = top - kf;
            __syncwarp();
        }
        // ---- the new partial matches' windows go on top of the stack (depth first): the first
        // slot's children (or the items) from registers, then the second slot's from staging
        for (int sl = 0; sl < kSlots; sl++) {
            if (sl >= 1) {
                has = (hmask >> sl) & 1u;
            }
            if (!__any_sync(kFull, has)) continue;
            if (sl >= 1 && has)
                stage_get<MAXV>(sg + (sl - 1) * Stage<MAXV>::F * 32, lane_id, x, c_lo, c_end, c_out, s_nodes);
            open_push<MAXV, GEN, CAP, STATS>(w, s_nodes, s_groups, stk, ps, sp, sp_top, has, x, c_lo, c_end, c_out,
                                             my_cnt, s_tot, st);
        }
    }

    // ---- counters: lanes -> block -> global, once per block
    __syncthreads();
    if (s_cnt) {
        for (uint32_t sl = tid >> 5; sl < p.n_slots; sl += kWarps) {
            unsigned long long v = 0;
            for (uint32_t i = lane_id; i < kWB; i += 32) v += s_cnt[sl * kWB + i];
#pragma unroll
            for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(kFull, v, o);
            if (lane_id == 0) s_tot[sl] += v;
        }
        __syncthreads();
    }
    for (uint32_t i = tid; i < p.n_motifs; i += kWB) {
        const unsigned long long v = s_tot[s_nodes[p.motif_node[i]].slot];
        if (v) atomicAdd(p.counts + i, v);
    }
    if (STATS) {
#pragma unroll
        for (int i = 0; i < ST_N; i++) {
            unsigned long long v = st[i];
#pragma unroll
            for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(kFull, v, o);
            if (lane_id == 0 && v) atomicAdd(p.stats + i, v);
        }
    }
}

}  // namespace wdfs
