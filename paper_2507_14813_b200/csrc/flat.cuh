// flat.cuh -- level-synchronous, entry-parallel co-mining (MAYURA_KERNEL=flat), included by
// comine.cu after bfs.cuh (it reuses bfs:: records, counters, window starts and the dfs fallback).
//
// Algorithm 3 "Co-Mining" advanced one MG-Tree level at a time over ALL
// partial matches of the level, in two kernels per level k:
//   flat_win_kernel    thread per partial match x of F_k (F_0 = the root edges): the exact
//                      window [lo, lo + n) of every anchor group of node(x) (Algo 1 l.210-214:
//                      entries with tr_prev < tr <= hi(root)), located by successor pointers /
//                      search and a galloping search for its end; windows are appended as
//                      pieces of <= kPiece entries {x, group, start, n} (warp-aggregated).
//   flat_entry_kernel  warp per 32 pieces, LANE PER WINDOW ENTRY: a warp-wide prefix sum of the
//                      pieces' lengths assigns entries to lanes 32 at a time, so every lane
//                      tests one candidate (class against the owner's m2g, at most one child
//                      per class -- Algo 1 l.219 + R4); completion children are counted
//                      (Algo 3 l.661), inner children appended to F_{k+1} (warp-aggregated).
// The depth-first lane kernel spends most of its issue slots on a divergent per-lane state
// machine (profiles/README.md r03: 22 warp instructions per window entry, 13.6 active lanes);
// here the per-entry work is straight-line code on full warps.  A full window or frontier
// buffer never loses work: the thread mines the rest of that subtree depth-first (bfs::dfs).
// Counts are identical to every other kernel form.

namespace flat {

constexpr int kTB = 256;
constexpr uint32_t kPiece = 64;  // entries per window piece (bounds one warp-round batch)

struct FParams {
    bfs::BParams b;        // graph, table, frontier in (F_k) / out (F_{k+1}), counts
    uint4 *win;            // window pieces (Piece<MAXV>); kStripes segments of win_seg_cap pieces (a
                           // warp appends to stripe warp mod kStripes: one hot counter would
                           // serialise every append)
    uint32_t *win_cnt;     // kStripes counters: pieces appended (may exceed win_seg_cap)
    uint32_t win_seg_cap;
    const uint32_t *gwant; // per group: wants of its first 4 children (bytes, 0xFD pad)
};

// A window piece carries everything the entry pass needs about its partial match, so the
// entry pass loads nothing but the piece and the window entries:
//   words [root, group | nv << 16, start, n, node, h, m2g[0..MAXV-1]], padded to uint4s
template <int MAXV>
struct Piece {
    static constexpr int W = (6 + MAXV + 3) & ~3;
};

// first position q in [lo, sent] with ent[q].x > key; ent[sent] is the list's sentinel (> any
// key).  Galloping from lo: windows are short, so this costs one or two dependent loads.
__device__ __forceinline__ uint32_t first_gt(const uint2 *ent, uint32_t lo, uint32_t sent, uint32_t key) {
    uint32_t a = lo, b = sent, step = 1;
    while (a < b) {
        const uint32_t probe = min(b, a + step - 1);
        if (__ldg(&ent[probe].x) > key) {
            b = probe;
            break;
        }
        a = probe + 1;
        step <<= 1;
    }
    while (a < b) {
        const uint32_t mid = a + ((b - a) >> 1);
        if (__ldg(&ent[mid].x) > key) b = mid;
        else a = mid + 1;
    }
    return a;
}

// The exact window of group G for partial match x: start and entry count.
template <int MAXV>
__device__ __forceinline__ uint32_t window(const bfs::BParams &p, const DGroup &G, const bfs::PM<MAXV> &x,
                                           uint32_t &n, bfs::Ctx &c) {
    uint32_t lim;
    uint32_t lo = bfs::window_start<MAXV, false>(p, G, x, lim, c);
    if (G.kind == ANCHOR_GLOBAL) {  // edge ids (tr_prev-tie-group end, hi(root)] (reading R6)
        n = x.h + 1 > lo ? x.h + 1 - lo : 0;
        return lo;
    }
    const uint2 *ent = (G.kind == ANCHOR_OUT) ? p.out_ent : p.in_ent;
    const uint32_t *off = (G.kind == ANCHOR_OUT) ? p.out_off : p.in_off;
    const uint32_t sent = __ldg(off + lane::m2g_get<MAXV>(x.m2g, G.anchor) + 1) - 1;
    if (G.start >= START_R0 && G.start < START_SEARCH) lo = first_gt(ent, lo, sent, x.tr_prev);  // lower bound
    n = first_gt(ent, lo, sent, x.h) - lo;
    return lo;
}

template <int MAXV, bool L0>
__global__ void __launch_bounds__(kTB) flat_win_kernel(const __grid_constant__ FParams f) {
    pdl_begin();
    extern __shared__ __align__(16) unsigned char smem[];
    const bfs::BParams &p = f.b;
    const bfs::Smem s = bfs::smem_setup(p, smem, L0);
    bfs::Ctx c;
    c.cnt = s.cnt ? s.cnt + threadIdx.x : nullptr;
    c.stride = blockDim.x;
    c.tot = s.tot;
#pragma unroll
    for (int i = 0; i < ST_N; i++) c.st[i] = 0;
    c.em_next = c.em_end = 0;
    const uint32_t n_items = L0 ? p.n_roots : s.pref[bfs::kStripes];
    const lane::LNode root = s.nodes[0];
    const uint32_t lane_id = threadIdx.x & 31;
    for (uint32_t base = blockIdx.x * blockDim.x + (threadIdx.x & ~31u); base < n_items;
         base += gridDim.x * blockDim.x) {  // warp-uniform trip count (aggregated appends below)
        const uint32_t item = base + lane_id;
        bfs::PM<MAXV> x;
        bool go = item < n_items;
        uint32_t xid = item;
        if (L0) {
            xid = p.r0 + item;
            if (go && !bfs::load_root<MAXV>(p, xid, x)) go = false;
            if (go && p.T) {  // hi(root) computed here (no window_end_kernel) and kept for later passes
                x.h = window_end_of(p.T, p.E, p.delta, xid);
                p.hi_w[xid] = x.h;
            }
            if (go && (root.flags & NODE_COMPLETION)) bfs::count_add(c, root.slot, 1);
            if (!(root.flags & NODE_INNER)) go = false;
            if (p.light) {  // mixed form: light roots go to the depth-first kernel whole (listed here)
                const bool light = go && !lane::heavy_root<MAXV>(s.nodes, s.groups, root, x.P, x.h, x.m2g[0],
                                                                x.m2g[1], p.out_off, p.out_ent, p.in_off,
                                                                p.in_ent, p.heavy_min);
                const unsigned lm = __ballot_sync(kFull, light);
                if (lm) {
                    uint32_t b = 0;
                    if (lane_id == 0) b = atomicAdd(p.light_cnt, (uint32_t)__popc(lm));
                    b = __shfl_sync(kFull, b, 0);
                    if (light) p.light[b + __popc(lm & ((1u << lane_id) - 1u))] = xid;
                }
                go = go && !light;
            }
        } else if (go) {
            bfs::load_rec<MAXV>(p, s.pref, item, x);
            go = x.node != bfs::kHole;
        }
        const lane::LNode xn = s.nodes[go ? x.node : 0];
        const uint32_t ng = go ? (uint32_t)(xn.group_end - xn.group_begin) : 0u;
        const uint32_t maxg = __reduce_max_sync(kFull, ng);
        bool fell = false;  // the window buffer was full: x's remaining groups were mined depth-first
        for (uint32_t gi = 0; gi < maxg; gi++) {
            const bool mine = gi < ng && !fell;
            const uint32_t g = xn.group_begin + gi;
            uint32_t lo = 0, n = 0;
            if (mine) lo = window<MAXV>(p, s.groups[g], x, n, c);
            const uint32_t np = (n + kPiece - 1) / kPiece;
            uint32_t incl = np;
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const uint32_t v = __shfl_up_sync(kFull, incl, o);
                if (lane_id >= (uint32_t)o) incl += v;
            }
            const uint32_t total = __shfl_sync(kFull, incl, 31);
            uint32_t wb = 0;
            const uint32_t seg = bfs::out_seg();
            if (lane_id == 0 && total) wb = atomicAdd(f.win_cnt + seg, total);
            wb = __shfl_sync(kFull, wb, 0);
            const uint32_t at = wb + incl - np;
            constexpr int PW = Piece<MAXV>::W / 4;  // uint4s per piece
            uint4 *wseg = f.win + (size_t)seg * f.win_seg_cap * PW;
            if (np) {
                if (at + np <= f.win_seg_cap) {
                    for (uint32_t q = 0; q < np; q++) {
                        uint4 *pc = wseg + (size_t)(at + q) * PW;
                        pc[0] = make_uint4(x.root, g | (x.nv << 16), lo + q * kPiece, min(kPiece, n - q * kPiece));
                        uint32_t w[PW * 4 - 4];
                        w[0] = x.node;
                        w[1] = x.h;
#pragma unroll
                        for (int k = 0; k < MAXV; k++) w[2 + k] = x.m2g[k];
#pragma unroll
                        for (int k = 2 + MAXV; k < PW * 4 - 4; k++) w[k] = 0;
#pragma unroll
                        for (int k = 1; k < PW; k++) pc[k] = make_uint4(w[4 * k - 4], w[4 * k - 3], w[4 * k - 2], w[4 * k - 1]);
                    }
                } else {  // no room: empty the reserved slots that exist, mine the rest in place
                    for (uint32_t q = at; q < at + np && q < f.win_seg_cap; q++) wseg[(size_t)q * PW] = make_uint4(0, 0, 0, 0);
                    if (p.fallback) atomicAdd(p.fallback, 1u);
                    bfs::dfs<MAXV, false>(p, s.nodes, s.groups, x, c, g);
                    fell = true;
                }
            }
        }
    }
    bfs::flush<false>(p, s, c);
}

template <int MAXV, bool L0>
__global__ void __launch_bounds__(kTB) flat_entry_kernel(const __grid_constant__ FParams f) {
    pdl_begin();
    extern __shared__ __align__(16) unsigned char smem[];
    const bfs::BParams &p = f.b;
    const bfs::Smem s = bfs::smem_setup(p, smem, L0);
    bfs::Ctx c;
    c.cnt = s.cnt ? s.cnt + threadIdx.x : nullptr;
    c.stride = blockDim.x;
    c.tot = s.tot;
#pragma unroll
    for (int i = 0; i < ST_N; i++) c.st[i] = 0;
    c.em_next = c.em_end = 0;
    const uint32_t lane_id = threadIdx.x & 31;
    __shared__ uint32_t s_wpre[bfs::kStripes + 1];  // prefix of the pieces per stripe
    if (threadIdx.x == 0) {
        uint32_t acc = 0;
        for (int i = 0; i < bfs::kStripes; i++) {
            s_wpre[i] = acc;
            acc += min(f.win_cnt[i], f.win_seg_cap);
        }
        s_wpre[bfs::kStripes] = acc;
    }
    __syncthreads();
    const uint32_t n_win = s_wpre[bfs::kStripes];
    const uint32_t gw = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, n_warps = (gridDim.x * blockDim.x) >> 5;
    // pieces are <= kPiece entries, so a static interleaved batch assignment balances well and
    // needs no shared cursor
    constexpr int PW = Piece<MAXV>::W / 4;
    __shared__ uint32_t s_gw[lane::kGwMax];
    for (uint32_t i = threadIdx.x; i < p.n_groups && i < lane::kGwMax; i += blockDim.x) s_gw[i] = f.gwant[i];
    __syncthreads();
    // piece wi of the level (global index over the stripes) -> registers (zeros past the end)
    auto load_piece = [&](uint32_t wi, uint32_t (&pw)[PW * 4]) {
#pragma unroll
        for (int k = 0; k < PW * 4; k++) pw[k] = 0;
        if (wi < n_win) {
            int lo = 0, hi = bfs::kStripes - 1;  // stripe s with s_wpre[s] <= wi < s_wpre[s + 1]
            while (lo < hi) {
                const int mid = (lo + hi + 1) >> 1;
                if (s_wpre[mid] <= wi) lo = mid;
                else hi = mid - 1;
            }
            const uint4 *pc = f.win + ((size_t)lo * f.win_seg_cap + (wi - s_wpre[lo])) * PW;
#pragma unroll
            for (int k = 0; k < PW; k++) {
                const uint4 v = __ldcs(pc + k);  // streamed: read once
                pw[4 * k] = v.x; pw[4 * k + 1] = v.y; pw[4 * k + 2] = v.z; pw[4 * k + 3] = v.w;
            }
        }
    };
    for (uint32_t wb = gw * 32u; wb < n_win; wb += n_warps * 32u) {
        uint32_t pw[PW * 4];
        load_piece(wb + lane_id, pw);
        const uint4 w = make_uint4(pw[0], pw[1], pw[2], pw[3]);
        const uint32_t n = w.w;
        bfs::PM<MAXV> x;
        x.root = pw[0];
        x.nv = pw[1] >> 16;
        x.node = pw[4];
        x.h = pw[5];
#pragma unroll
        for (int k = 0; k < MAXV; k++) x.m2g[k] = pw[6 + k];
        uint32_t incl = n;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const uint32_t v = __shfl_up_sync(kFull, incl, o);
            if (lane_id >= (uint32_t)o) incl += v;
        }
        const uint32_t excl = incl - n, T = __shfl_sync(kFull, incl, 31);
        for (uint32_t rb = 0; rb < T; rb += 32) {
            const uint32_t j = rb + lane_id;
            const bool act = j < T;
            uint32_t o = 0;  // owner: the first lane whose inclusive sum exceeds j
#pragma unroll
            for (uint32_t st = 16; st; st >>= 1)
                if (__shfl_sync(kFull, incl, o + st - 1) <= j) o += st;
            o = min(o, 31u);
            bfs::PM<MAXV> xo;
#pragma unroll
            for (int k = 0; k < MAXV; k++) xo.m2g[k] = __shfl_sync(kFull, x.m2g[k], o);
            xo.node = __shfl_sync(kFull, x.node, o);
            xo.nv = __shfl_sync(kFull, x.nv, o);
            xo.root = __shfl_sync(kFull, x.root, o);
            xo.h = __shfl_sync(kFull, x.h, o);
            const uint32_t g = __shfl_sync(kFull, w.y, o) & 0xffffu;
            const uint32_t pos = __shfl_sync(kFull, w.z, o) + (j - __shfl_sync(kFull, excl, o));
            uint32_t ch = kNone, etr = 0, e1 = 0, e2 = 0;
            DGroup G = s.groups[act ? g : 0];
            if (act) {
                bfs::load_entry(p, G, pos, kNone, etr, e1, e2);
                const uint32_t cls = bfs::entry_class<MAXV>(G, xo.m2g, e1, e2);
                if (G.child_end - G.child_begin <= 4 && g < lane::kGwMax) {  // one SIMD byte compare
                    const uint32_t eq = __vcmpeq4(s_gw[g], cls * 0x01010101u);
                    ch = eq ? G.child_begin + ((__ffs(eq) - 1) >> 3) : kNone;
                } else {
                    ch = bfs::find_child(s.nodes, G, cls);
                }
            }
            bool inner = false;
            if (ch != kNone) {
                const lane::LNode dn = s.nodes[ch];
                if (dn.flags & NODE_COMPLETION) bfs::count_add(c, dn.slot, 1);
                inner = (dn.flags & NODE_INNER) != 0;
            }
            if (inner) {
                bfs::PM<MAXV> y;
                bfs::make_child<MAXV>(p, G, s.nodes[ch], ch, xo, pos, etr, e1, e2, y);
                bfs::emit<MAXV, false, false>(p, s.nodes, s.groups, y, c);  // warp-aggregated append
            }
        }
    }
    bfs::flush<false>(p, s, c);
}

}  // namespace flat
