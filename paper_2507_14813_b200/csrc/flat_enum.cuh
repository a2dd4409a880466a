// flat_enum.cuh -- enumeration in the flat (level-synchronous, entry-parallel) form, included
// by comine.cu after flat.cuh.  Same passes as the counting flat form (flat.cuh), with the
// input ranks of the partial match's edges (its "prefix", root first) carried in every record
// and window piece; a completion writes prefix + the matched edge as one tuple (PAPER.md:130,
// Algo 1 l.201) at a position reserved with one atomic per (warp, motif slot) and round.
// Tuples of a motif land in arbitrary order (reading R19); a full frontier or piece buffer
// sets `overflow` and the host re-runs the query in the depth-first enumeration form.

namespace flat {

constexpr int kPre = MAYURA_MAX_EDGES;  // prefix words carried (edges of a partial match < 8)

// record: [node|nv<<16, root, tr_prev, h, P(4), m2g(MAXV), plen, pre(kPre)]
template <int MAXV>
struct ERec {
    static constexpr int W = (8 + MAXV + 1 + kPre + 3) & ~3;
};
// piece: [root, group|nv<<16, start, n, node, h, plen, 0, m2g(MAXV), pre(kPre)]
template <int MAXV>
struct EPiece {
    static constexpr int W = (8 + MAXV + kPre + 3) & ~3;
};

struct EParams {
    bfs::BParams b;                        // graph, table, frontier in/out (ERec layout)
    uint4 *win;                            // pieces (EPiece layout), kStripes segments
    uint32_t *win_cnt;
    uint32_t win_seg_cap;
    const uint32_t *perm, *out_rank, *in_rank;
    uint32_t *out;                         // tuples
    const unsigned long long *slot_word;   // first word of each completion slot's region
    unsigned long long *cursor;            // tuples written per slot
    uint32_t *overflow;                    // set when a buffer was full (host re-runs depth-first)
};

template <int MAXV>
struct EPM {
    bfs::PM<MAXV> x;
    uint32_t plen;
    uint32_t pre[kPre];
};

// All 32 lanes call together: lanes with `want` each write the tuple pre[0..plen) + last of
// completion slot `slot`; one atomic per distinct slot in the warp.
__device__ __forceinline__ void warp_put(const EParams &f, bool want, uint32_t slot, const uint32_t (&pre)[kPre],
                                         uint32_t plen, uint32_t last) {
    if (!__any_sync(kFull, want)) return;
    const uint32_t lane_id = threadIdx.x & 31;
    const unsigned grp = __match_any_sync(kFull, want ? slot : 0xFFFFFFFFu);
    const int leader = __ffs(grp) - 1;
    unsigned long long base = 0;
    if (want && (int)lane_id == leader) base = atomicAdd(f.cursor + slot, (unsigned long long)__popc(grp));
    base = __shfl_sync(kFull, base, leader);
    if (want) {
        const unsigned long long idx = base + __popc(grp & ((1u << lane_id) - 1u));
        uint32_t *o = f.out + f.slot_word[slot] + idx * (plen + 1);
#pragma unroll
        for (int i = 0; i < kPre; i++)
            if ((uint32_t)i < plen) o[i] = pre[i];
        o[plen] = last;
    }
}

template <int MAXV>
__device__ __forceinline__ void load_erec(const bfs::BParams &p, const uint32_t *s_pref, uint32_t item, EPM<MAXV> &y) {
    constexpr int W = ERec<MAXV>::W;
    int lo = 0, hi = bfs::kStripes - 1;
    while (lo < hi) {
        const int mid = (lo + hi + 1) >> 1;
        if (s_pref[mid] <= item) lo = mid;
        else hi = mid - 1;
    }
    const uint32_t *r = p.in.data + ((size_t)lo * p.in.seg_cap + (item - s_pref[lo])) * W;
    uint32_t w[W];
#pragma unroll
    for (int q = 0; q < W / 4; q++) {
        const uint4 v = __ldcs(reinterpret_cast<const uint4 *>(r) + q);
        w[4 * q] = v.x; w[4 * q + 1] = v.y; w[4 * q + 2] = v.z; w[4 * q + 3] = v.w;
    }
    y.x.node = w[0] & 0xffffu;
    y.x.nv = w[0] >> 16;
    y.x.root = w[1];
    y.x.tr_prev = w[2];
    y.x.h = w[3];
    y.x.P = make_uint4(w[4], w[5], w[6], w[7]);
#pragma unroll
    for (int k = 0; k < MAXV; k++) y.x.m2g[k] = w[8 + k];
    y.plen = w[8 + MAXV];
#pragma unroll
    for (int k = 0; k < kPre; k++) y.pre[k] = w[9 + MAXV + k];
}

template <int MAXV, bool L0>
__global__ void __launch_bounds__(kTB) flat_enum_win_kernel(const __grid_constant__ EParams f) {
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
    constexpr int PW = EPiece<MAXV>::W / 4;
    for (uint32_t base = blockIdx.x * blockDim.x + (threadIdx.x & ~31u); base < n_items;
         base += gridDim.x * blockDim.x) {
        const uint32_t item = base + lane_id;
        EPM<MAXV> y;
        bool go = item < n_items;
        if (L0) {
            const uint32_t r = p.r0 + item;
            if (go && !bfs::load_root<MAXV>(p, r, y.x)) go = false;
            y.plen = 1;
            y.pre[0] = go ? __ldg(f.perm + r) : 0u;
#pragma unroll
            for (int k = 1; k < kPre; k++) y.pre[k] = 0;
            uint32_t none[kPre];
#pragma unroll
            for (int k = 0; k < kPre; k++) none[k] = 0;
            warp_put(f, go && (root.flags & NODE_COMPLETION), root.slot, none, 0, y.pre[0]);  // 1-edge motifs
            if (!(root.flags & NODE_INNER)) go = false;
        } else if (go) {
            load_erec<MAXV>(p, s.pref, item, y);
            go = y.x.node != bfs::kHole;
        }
        const lane::LNode xn = s.nodes[go ? y.x.node : 0];
        const uint32_t ng = go ? (uint32_t)(xn.group_end - xn.group_begin) : 0u;
        const uint32_t maxg = __reduce_max_sync(kFull, ng);
        for (uint32_t gi = 0; gi < maxg; gi++) {
            const uint32_t g = xn.group_begin + gi;
            uint32_t lo = 0, n = 0;
            if (gi < ng) lo = window<MAXV>(p, s.groups[g], y.x, n, c);
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
            uint4 *wseg = f.win + (size_t)seg * f.win_seg_cap * PW;
            if (np) {
                if (at + np <= f.win_seg_cap) {
                    for (uint32_t q = 0; q < np; q++) {
                        uint32_t w[PW * 4];
                        w[0] = y.x.root;
                        w[1] = g | (y.x.nv << 16);
                        w[2] = lo + q * kPiece;
                        w[3] = min(kPiece, n - q * kPiece);
                        w[4] = y.x.node;
                        w[5] = y.x.h;
                        w[6] = y.plen;
                        w[7] = 0;
#pragma unroll
                        for (int k = 0; k < MAXV; k++) w[8 + k] = y.x.m2g[k];
#pragma unroll
                        for (int k = 0; k < kPre; k++) w[8 + MAXV + k] = y.pre[k];
#pragma unroll
                        for (int k = 8 + MAXV + kPre; k < PW * 4; k++) w[k] = 0;
                        uint4 *pc = wseg + (size_t)(at + q) * PW;
#pragma unroll
                        for (int k = 0; k < PW; k++) pc[k] = make_uint4(w[4 * k], w[4 * k + 1], w[4 * k + 2], w[4 * k + 3]);
                    }
                } else {  // no room: empty the reserved slots that exist; the host re-runs depth-first
                    for (uint32_t q = at; q < at + np && q < f.win_seg_cap; q++) wseg[(size_t)q * PW] = make_uint4(0, 0, 0, 0);
                    atomicOr(f.overflow, 1u);
                }
            }
        }
    }
}

template <int MAXV>
__global__ void __launch_bounds__(kTB) flat_enum_entry_kernel(const __grid_constant__ EParams f) {
    pdl_begin();
    extern __shared__ __align__(16) unsigned char smem[];
    const bfs::BParams &p = f.b;
    const bfs::Smem s = bfs::smem_setup(p, smem, true);
    const uint32_t lane_id = threadIdx.x & 31;
    __shared__ uint32_t s_wpre[bfs::kStripes + 1];
    __shared__ uint32_t s_gw[lane::kGwMax];
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
    constexpr int PW = EPiece<MAXV>::W / 4;
    constexpr int RW = ERec<MAXV>::W;
    (void)s_gw;
    for (uint32_t wb = gw * 32u; wb < n_win; wb += n_warps * 32u) {
        const uint32_t wi = wb + lane_id;
        uint32_t pw[PW * 4];
#pragma unroll
        for (int k = 0; k < PW * 4; k++) pw[k] = 0;
        if (wi < n_win) {
            int lo = 0, hi = bfs::kStripes - 1;
            while (lo < hi) {
                const int mid = (lo + hi + 1) >> 1;
                if (s_wpre[mid] <= wi) lo = mid;
                else hi = mid - 1;
            }
            const uint4 *pc = f.win + ((size_t)lo * f.win_seg_cap + (wi - s_wpre[lo])) * PW;
#pragma unroll
            for (int k = 0; k < PW; k++) {
                const uint4 v = __ldcs(pc + k);
                pw[4 * k] = v.x; pw[4 * k + 1] = v.y; pw[4 * k + 2] = v.z; pw[4 * k + 3] = v.w;
            }
        }
        const uint32_t n = pw[3];
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
            uint32_t o = 0;
#pragma unroll
            for (uint32_t st = 16; st; st >>= 1)
                if (__shfl_sync(kFull, incl, o + st - 1) <= j) o += st;
            o = min(o, 31u);
            bfs::PM<MAXV> xo;
#pragma unroll
            for (int k = 0; k < MAXV; k++) xo.m2g[k] = __shfl_sync(kFull, pw[8 + k], o);
            uint32_t pre[kPre];
#pragma unroll
            for (int k = 0; k < kPre; k++) pre[k] = __shfl_sync(kFull, pw[8 + MAXV + k], o);
            const uint32_t plen = __shfl_sync(kFull, pw[6], o);
            xo.root = __shfl_sync(kFull, pw[0], o);
            const uint32_t gnv = __shfl_sync(kFull, pw[1], o);
            xo.nv = gnv >> 16;
            const uint32_t g = gnv & 0xffffu;
            xo.node = __shfl_sync(kFull, pw[4], o);
            xo.h = __shfl_sync(kFull, pw[5], o);
            const uint32_t pos = __shfl_sync(kFull, pw[2], o) + (j - __shfl_sync(kFull, excl, o));
            uint32_t ch = kNone, etr = 0, e1 = 0, e2 = 0;
            const DGroup G = s.groups[act ? g : 0];
            if (act) {
                bfs::load_entry(p, G, pos, kNone, etr, e1, e2);
                ch = bfs::find_child(s.nodes, G, bfs::entry_class<MAXV>(G, xo.m2g, e1, e2));
            }
            uint32_t rk = 0, flags = 0, slot = 0;
            if (ch != kNone) {
                const lane::LNode dn = s.nodes[ch];
                flags = dn.flags;
                slot = dn.slot;
                rk = __ldg(G.kind == ANCHOR_GLOBAL ? f.perm + pos : (G.kind == ANCHOR_OUT ? f.out_rank : f.in_rank) + pos);
            }
            warp_put(f, (flags & NODE_COMPLETION) != 0, slot, pre, plen, rk);
            const bool inner = (flags & NODE_INNER) != 0;
            const unsigned im = __ballot_sync(kFull, inner);
            if (im) {  // inner children -> next level's records (warp-aggregated append)
                const uint32_t seg = bfs::out_seg();
                uint32_t b = 0;
                if (lane_id == 0) b = atomicAdd(p.out.cnt + seg, (uint32_t)__popc(im));
                b = __shfl_sync(kFull, b, 0);
                if (inner) {
                    const uint32_t idx = b + __popc(im & ((1u << lane_id) - 1u));
                    if (idx < p.out.seg_cap) {
                        bfs::PM<MAXV> y;
                        bfs::make_child<MAXV>(p, G, s.nodes[ch], ch, xo, pos, etr, e1, e2, y);
                        uint32_t w[RW];
                        w[0] = y.node | (y.nv << 16);
                        w[1] = y.root;
                        w[2] = y.tr_prev;
                        w[3] = y.h;
                        w[4] = y.P.x; w[5] = y.P.y; w[6] = y.P.z; w[7] = y.P.w;
#pragma unroll
                        for (int k = 0; k < MAXV; k++) w[8 + k] = y.m2g[k];
                        w[8 + MAXV] = plen + 1;
#pragma unroll
                        for (int k = 0; k < kPre; k++) w[9 + MAXV + k] = (uint32_t)k < plen ? pre[k] : ((uint32_t)k == plen ? rk : 0u);
#pragma unroll
                        for (int k = 9 + MAXV + kPre; k < RW; k++) w[k] = 0;
                        uint4 *r = reinterpret_cast<uint4 *>(p.out.data + ((size_t)seg * p.out.seg_cap + idx) * RW);
#pragma unroll
                        for (int k = 0; k < RW / 4; k++) r[k] = make_uint4(w[4 * k], w[4 * k + 1], w[4 * k + 2], w[4 * k + 3]);
                    } else {
                        atomicOr(f.overflow, 1u);
                    }
                }
            }
        }
    }
}

}  // namespace flat
