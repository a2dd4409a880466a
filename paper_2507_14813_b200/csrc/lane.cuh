// lane.cuh -- lane-per-search co-mining kernel (kernel v3), included by comine.cu.
//
// Algorithm 3 "Co-Mining" with one search per ROOT EDGE per LANE:
// every lane of a warp walks the MG-Tree table depth-first for its own root (the
// paper's thread-per-first-edge mapping), so a warp makes progress
// on 32 independent searches at once.  Profiles of the warp-per-root kernel (v2,
// profiles/r01_*.md) showed windows average ~2 entries: a whole warp per window spent
// ~2,200 issue slots per root on warp-uniform overhead.  Here every loop iteration
// processes ONE window entry (or one control transition) per lane, with a body of a
// few dozen instructions that all lanes execute in lockstep:
//   - window start (Algo 1 l.210-214): successor pointers P(e) of the edge matched at
//     the node (exact), the root's R (lower bound; pre-window entries are skipped by
//     the time test), a per-lane binary search (other anchors), or a binary search of
//     the edge array (GLOBAL anchor, reading R6);
//   - candidate test (Algo 1 l.219 + full injectivity R4): classify the neighbour
//     against the lane's m2g registers -> which mapped motif vertex it is, or NEW;
//     in an anchor group at most one child wants a given class;
//   - completion child: count[Q_N]++ (Algo 3 l.661) in a lane-private shared-memory
//     counter; inner child: push a frame (lane-private shared memory) and descend
//     (Algo 3 l.665-669); window end ("time rank > hi(root)", sentinel-terminated
//     lists) -> next anchor group -> pop.
// Roots are handed out by a warp-aggregated atomic cursor (guided chunk sizes):
// a lane that finishes its search takes the next root at the next iteration.
// Long windows (>= kHelpMin entries) are not scanned lane-serially: the lane parks the
// window and the whole warp scans it 32 entries per step (coalesced loads, ballot per
// child), queueing descents back to the owning lane -- see `warp_help`.

namespace lane {

constexpr int kLB = 128;                 // threads per block
constexpr int kFrameWords = 8;           // node|g<<16, pos, tr_prev, lim, P.x, P.y, P.z, P.w
constexpr uint32_t kHelpMin = 12;       // leaf windows of >= this many entries are scanned by the warp
constexpr uint32_t kAgeMin = 64;        // steps on one search before its descents are handed out
constexpr uint32_t kStackCap = 32;      // per-warp task stack (tasks)
constexpr int kPmStripes = 64;          // segments of a partial-match source (bfs::kStripes)
constexpr uint32_t kGwMax = 64;         // groups whose packed child wants are kept in shared memory
constexpr int kPreMax = MAYURA_MAX_EDGES;  // ENUM: edges of a search's base prefix (root / task start)
// ENUM frames carry one more word: the input rank of the edge matched when the frame was pushed
__host__ __device__ constexpr int frame_words(bool en) { return en ? kFrameWords + 1 : kFrameWords; }
// task-stack words per task: node|nv, tr_prev, h, P(4), R(4), m2g(MAXV) [+ ENUM: prefix length, prefix]
__host__ __device__ constexpr int task_words(int maxv, bool en) { return 11 + maxv + (en ? 1 + kPreMax : 0); }

struct __align__(4) LNode {  // 12 bytes
    uint8_t want, n_new, nv, flags;
    uint16_t group_begin, group_end;
    uint16_t slot;                      // completion counter slot (0xFFFF: none)
    uint16_t same;                      // bit q: group q of this node scans the same list as the
                                        // group this node was matched in (wdfs.cuh continuation)
};

struct LParams {
    const uint32_t *src, *dst, *tr, *hi;
    const uint4 *eptr;
    const uint32_t *out_off, *in_off;
    const uint2 *out_ent, *in_ent;
    const uint4 *out_ptr, *in_ptr;
    const LNode *nodes;
    const DGroup *groups;
    const uint32_t *motif_node;
    const uint32_t *gwant;              // per group: wants of its first 4 children (bytes, 0xFD pad)
    uint32_t n_nodes, n_groups, n_motifs, n_slots, n_frames;
    uint32_t r0, n_roots;
    uint32_t *lb;                       // load-balancer words (LB_*), zeroed per launch
    unsigned long long *dbg;            // STATS + debug: per-warp timeline records (or null)
    // hybrid mode: the searches start from partial matches a BFS pass wrote (striped
    // records: node|nv<<16, root, tr_prev, h, P, m2g) instead of from root edges
    const uint32_t *pm;                 // null: root edges [r0, r0 + n_roots)
    const uint32_t *pm_cnt;             // kPmStripes counters
    uint32_t pm_seg_cap, pm_words;
    uint32_t heavy_min;                 // hybrid: also mine the LIGHT roots of [r0, r0 + n_roots)
                                        // (heavy ones were split by the breadth-first level, which
                                        // also counted every root's completion); 0: no roots
    const uint32_t *light;              // heavy_min > 0: the light roots the breadth-first level listed
    const uint32_t *light_cnt;          //   ([0] = entries)
    unsigned long long *counts;
    unsigned long long *stats;
    // dynamic shared-memory byte offsets (set by the launcher; kernel-constant operands instead
    // of address arithmetic the compiler rematerialises under the 64-register cap)
    uint32_t o_groups, o_tot, o_cnt, o_fr, o_stk, o_pre, o_enum;
    // enumeration (ENUM kernels, mayura_enumerate): roots are mapped to warps
    // statically (32-root chunk c -> warp c mod n_warps), so pass 1 (count per warp) and pass 2
    // (write) see the same per-warp match sets and pass 2 writes at exact, prefix-summed positions
    uint32_t enum_pass;                  // 1: per-warp counts into wcnt, 2: tuples into out
    unsigned long long *wcnt;            // [slot * n_warps + warp]
    const unsigned long long *wpre;      // exclusive prefix sum of wcnt
    const unsigned long long *slot_word; // first word of a slot's tuple region in out
    const uint32_t *slot_len;            // edges per tuple of a slot
    uint32_t *out;                       // tuples: input ranks of the matched edges, in motif edge order
    const uint32_t *perm, *out_rank, *in_rank;  // input rank of an edge id / of a list position's edge
};

__host__ __device__ inline size_t align16(size_t x) { return (x + 15) & ~(size_t)15; }

// dynamic shared memory layout: nodes | groups | slot totals (u64) | lane counters (u32,
// LANECNT only) | frames
__host__ __device__ inline size_t off_groups(uint32_t nn) { return align16((size_t)nn * sizeof(LNode)); }
__host__ __device__ inline size_t off_tot(uint32_t nn, uint32_t ng) { return off_groups(nn) + align16((size_t)ng * sizeof(DGroup)); }
__host__ __device__ inline size_t off_cnt(uint32_t nn, uint32_t ng, uint32_t ns) {
    return off_tot(nn, ng) + align16((size_t)ns * 8);
}
__host__ __device__ inline size_t off_frames(uint32_t nn, uint32_t ng, uint32_t ns, bool lanecnt) {
    return off_cnt(nn, ng, ns) + (lanecnt ? (size_t)ns * kLB * 4 : 0);
}
__host__ __device__ inline size_t off_stk(uint32_t nn, uint32_t ng, uint32_t ns, uint32_t nf, bool lanecnt, bool en) {
    return off_frames(nn, ng, ns, lanecnt) + (size_t)(nf ? nf : 1) * frame_words(en) * kLB * 4;
}
__host__ __device__ inline size_t off_pre(uint32_t nn, uint32_t ng, uint32_t ns, uint32_t nf, bool lanecnt, int maxv,
                                          bool en) {
    return off_stk(nn, ng, ns, nf, lanecnt, en) + (size_t)(kLB / 32) * task_words(maxv, en) * kStackCap * 4;
}
// ENUM: per lane kPreMax prefix words; per (warp, slot) a u32 cursor and a u64 base; per slot
// its u64 region start and u32 tuple length
__host__ __device__ inline size_t off_enum(uint32_t nn, uint32_t ng, uint32_t ns, uint32_t nf, bool lanecnt, int maxv,
                                           bool en) {
    return align16(off_pre(nn, ng, ns, nf, lanecnt, maxv, en) + (en ? (size_t)kPreMax * kLB * 4 : 0));
}
__host__ __device__ inline size_t smem_total(uint32_t nn, uint32_t ng, uint32_t ns, uint32_t nf, bool lanecnt,
                                             int maxv, bool en = false) {
    return off_enum(nn, ng, ns, nf, lanecnt, maxv, en) +
           (en ? (size_t)(kLB / 32) * ns * 12 + (size_t)ns * 12 + 16 : 0);
}

// m2g[k] == kNone for every motif vertex k that is not mapped (k >= nv), so the class
// of a graph vertex is one compare per slot (vertex ids are < 2^31).
// Entries [start, start + k) of vertex x's list all lie inside the window (time rank <= h)?
// The probe must stop at x's sentinel: the next vertex's list follows it, and its entries'
// time ranks say nothing about this window.
__device__ __forceinline__ bool window_has(const uint2 *ent, const uint32_t *off, uint32_t x, uint32_t start,
                                           uint32_t k, uint32_t h) {
    const uint32_t last = __ldg(off + x + 1) - 1;  // the sentinel's position
    return start + k - 1 < last && __ldg(&ent[start + k - 1].x) <= h;
}

// Hybrid split rule, applied identically by the breadth-first level (bfs.cuh) and this
// kernel: a root is heavy if one of its root-node windows that starts from the root's own
// successor pointers (START_P*/START_R*) has >= hmin entries (one probe load per window).
template <int MAXV>
__device__ __forceinline__ bool heavy_root(const LNode *nodes, const DGroup *groups, const LNode &root, const uint4 &P,
                                           uint32_t h, uint32_t rs, uint32_t rd, const uint32_t *out_off,
                                           const uint2 *out_ent, const uint32_t *in_off, const uint2 *in_ent,
                                           uint32_t hmin) {
    bool heavy = false;
    for (uint32_t g = root.group_begin; g < root.group_end && !heavy; ++g) {
        const DGroup G = groups[g];
        if (G.start >= START_SEARCH) continue;
        const uint32_t k = G.start < START_R0 ? G.start : G.start - START_R0;
        const uint32_t start = k == 0 ? P.x : k == 1 ? P.y : k == 2 ? P.z : P.w;
        const uint32_t x = (k == 0 || k == 3) ? rs : rd;  // P/R order: out(src), in(dst), out(dst), in(src)
        heavy = G.kind == ANCHOR_OUT ? window_has(out_ent, out_off, x, start, hmin, h)
                                     : window_has(in_ent, in_off, x, start, hmin, h);
    }
    (void)nodes;
    return heavy;
}

template <int MAXV>
__device__ __forceinline__ uint32_t classify(const uint32_t (&m)[MAXV], uint32_t x) {
    uint32_t c = CLS_NEW;
#pragma unroll
    for (int k = 0; k < MAXV; k++) c = (m[k] == x) ? (uint32_t)k : c;
    return c;
}
// Opaque select: keeps m2g in registers (the compiler otherwise re-rolls the unrolled
// select chains into an indexed local-memory array).
__device__ __forceinline__ uint32_t selp(uint32_t a, uint32_t b, bool c) {
    uint32_t r;
    asm("{ .reg .pred q; setp.ne.u32 q, %3, 0; selp.b32 %0, %1, %2, q; }" : "=r"(r) : "r"(a), "r"(b), "r"((uint32_t)c));
    return r;
}
template <int MAXV>
__device__ __forceinline__ void m2g_set(uint32_t (&m)[MAXV], uint32_t i, uint32_t x) {
#pragma unroll
    for (int k = 0; k < MAXV; k++) m[k] = selp(x, m[k], k == (int)i);
}
template <int MAXV>
__device__ __forceinline__ uint32_t m2g_get(const uint32_t (&m)[MAXV], uint32_t i) {
    uint32_t r = 0;
#pragma unroll
    for (int k = 0; k < MAXV; k++) r = selp(m[k], r, k == (int)i);
    return r;
}
__device__ __forceinline__ uint32_t pick4(const uint4 &v, uint32_t k) {
    return k == 0 ? v.x : k == 1 ? v.y : k == 2 ? v.z : v.w;
}

// GEN: the tree has anchor groups that need a search (START_SEARCH) or scan the edge array
// (GLOBAL); trees without them compile those paths out.
template <int MAXV, bool LANECNT, bool STATS, bool GEN, bool ENUM = false>
__global__ void __launch_bounds__(kLB, 8) comine_lane_kernel(const __grid_constant__ LParams p) {
    constexpr int FW = frame_words(ENUM);
    pdl_begin();
    constexpr int TW = task_words(MAXV, ENUM);
    extern __shared__ __align__(16) unsigned char smem[];
    LNode *s_nodes = reinterpret_cast<LNode *>(smem);
    DGroup *s_groups = reinterpret_cast<DGroup *>(smem + p.o_groups);
    unsigned long long *s_tot = reinterpret_cast<unsigned long long *>(smem + p.o_tot);
    uint32_t *s_cnt = reinterpret_cast<uint32_t *>(smem + p.o_cnt);
    uint32_t *s_fr = reinterpret_cast<uint32_t *>(smem + p.o_fr);
    uint32_t *s_stk = reinterpret_cast<uint32_t *>(smem + p.o_stk);
    __shared__ uint32_t s_pref[kPmStripes + 1];
    __shared__ uint32_t s_gw[kGwMax];  // packed child wants (trees of <= kGwMax groups)
    for (uint32_t i = threadIdx.x; i < p.n_groups && i < kGwMax; i += kLB) s_gw[i] = p.gwant[i];
    if (p.pm && threadIdx.x == 0) {
        uint32_t acc = 0;
        for (int i = 0; i < kPmStripes; i++) {
            s_pref[i] = acc;
            acc += min(p.pm_cnt[i], p.pm_seg_cap);
        }
        s_pref[kPmStripes] = acc;
    }

    const int tid = threadIdx.x, lane = tid & 31;
    for (uint32_t i = tid; i < p.n_nodes; i += kLB) s_nodes[i] = p.nodes[i];
    for (uint32_t i = tid; i < p.n_groups; i += kLB) s_groups[i] = p.groups[i];
    for (uint32_t i = tid; i < p.n_slots; i += kLB) s_tot[i] = 0;
    if (LANECNT)
        for (uint32_t i = 0; i < p.n_slots; i++) s_cnt[i * kLB + tid] = 0;
    // ENUM: s_pre = per-lane base prefix; s_ecur/s_ebase = per (warp, slot) cursor / base (pass 1:
    // u64 overflow of the lane counters); s_eword/s_elen = per-slot region start / tuple length
    uint32_t *s_pre = reinterpret_cast<uint32_t *>(smem + p.o_pre);
    unsigned long long *s_ebase = reinterpret_cast<unsigned long long *>(smem + p.o_enum);
    unsigned long long *s_eword = s_ebase + (kLB / 32) * p.n_slots;
    uint32_t *s_ecur = reinterpret_cast<uint32_t *>(s_eword + p.n_slots);
    uint32_t *s_elen = s_ecur + (kLB / 32) * p.n_slots;
    const uint32_t gwarp = blockIdx.x * (kLB / 32) + (threadIdx.x >> 5), n_warps = gridDim.x * (kLB / 32);
    if (ENUM) {
        for (uint32_t i = tid; i < (kLB / 32) * p.n_slots; i += kLB) {
            const uint32_t w = i / p.n_slots, sl = i % p.n_slots;
            const uint32_t gw = blockIdx.x * (kLB / 32) + w;
            s_ecur[i] = 0;
            s_ebase[i] = p.enum_pass == 2 ? p.wpre[(size_t)sl * n_warps + gw] - p.wpre[(size_t)sl * n_warps] : 0ull;
        }
        if (p.enum_pass == 2)
            for (uint32_t i = tid; i < p.n_slots; i += kLB) {
                s_eword[i] = p.slot_word[i];
                s_elen[i] = p.slot_len[i];
            }
    }
    __syncthreads();

    uint32_t *myfr = s_fr + tid;    // frame d, word f at myfr[(d * FW + f) * kLB]
    uint32_t *wstk = s_stk + (size_t)(tid >> 5) * TW * kStackCap;  // word q of slot i: [q * kStackCap + i]
    const uint32_t wbase = (uint32_t)tid & ~31u;
    // add n matches to lane `ln`'s counter of `slot` (ln = this lane, or a parked lane of
    // this warp whose window the warp scans for it)
    auto count_n = [&](uint32_t slot, uint32_t ln, uint32_t n) {
        if (LANECNT) {
            uint32_t *c = s_cnt + slot * kLB + ln;
            uint32_t v = *c + n;
            if (v >= 0x80000000u) {
                atomicAdd(&s_tot[slot], (unsigned long long)v);
                if (ENUM) atomicAdd(&s_ebase[(ln >> 5) * p.n_slots + slot], (unsigned long long)v);
                v = 0;
            }
            *c = v;
        } else {
            atomicAdd(&s_tot[slot], (unsigned long long)n);
        }
    };
    // ENUM pass 2: write one tuple of `slot` for lane ln's search: its base prefix (bo words),
    // the ranks in its frames 0..dd-1, then `last` (the matched edge; kNone: none)
    auto emit = [&](uint32_t slot, uint32_t ln, uint32_t bo, uint32_t dd, uint32_t last) {
        const uint32_t wi = (ln >> 5) * p.n_slots + slot;
        const uint32_t idx = atomicAdd(&s_ecur[wi], 1u);
        uint32_t *o = p.out + s_eword[slot] + (s_ebase[wi] + idx) * s_elen[slot];
        for (uint32_t i = 0; i < bo; i++) *o++ = s_pre[i * kLB + ln];
        for (uint32_t i = 0; i < dd; i++) *o++ = s_fr[(i * FW + kFrameWords) * kLB + ln];
        if (last != kNone) *o = last;
    };
    const bool wr = ENUM && p.enum_pass == 2;
    uint32_t bpre = 0;                 // ENUM: words of this lane's base prefix in s_pre
    uint32_t wk = 0;                   // ENUM: chunks this warp has taken (static mapping)
    unsigned long long st[ST_N];
#pragma unroll
    for (int i = 0; i < ST_N; i++) st[i] = 0;

    const LNode root = s_nodes[0];
    const bool root_inner = (root.flags & NODE_INNER) != 0;
    const uint32_t n_pm = p.pm ? s_pref[kPmStripes] : 0u;
    const uint32_t n_items = n_pm + (p.light ? *(volatile const uint32_t *)p.light_cnt : !p.pm ? p.n_roots : 0u);

    // ------------------------------------------------------------ lane state
    bool active = false, scan = false, help = false, fresh = false;
    uint32_t chk = kNone;              // fresh leaf window: its anchor vertex, for the long-window probe
    uint32_t age = 0;                  // steps since this lane took its root / task
    uint32_t stop = 0;                 // warp-uniform: tasks on this warp's stack
    uint32_t m2g[MAXV];
#pragma unroll
    for (int k = 0; k < MAXV; k++) m2g[k] = kNone;
    uint32_t h = 0, tr_prev = 0, node = 0, nv = 2, g = 0, g_end = 0, pos = 0, lim = kNone, d = 0;
    uint4 P = make_uint4(0, 0, 0, 0), R = make_uint4(0, 0, 0, 0);

    // warp-uniform root chunk
    uint32_t cb = 0, cl = 0;
    bool roots_left = true;
    const unsigned lt_mask = (1u << lane) - 1u;

    unsigned long long t_start = 0, n_iter = 0, n_help = 0, n_roots_w = 0, t_roots_done = 0;
    if (STATS && p.dbg) asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_start));
    for (;;) {
        if (STATS && p.dbg) {
            n_iter++;
            if (!roots_left && t_roots_done == 0) asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_roots_done));
        }
        // ---------------------------------------------------- (0) this warp's task stack first
        // Partial matches handed out by heavy lanes (section 2) wait in a per-warp LIFO in
        // shared memory; idle lanes pop them before taking new roots.  The warp runs this
        // loop in lockstep, so the stack needs no atomics (ballot ranks + a uniform top).
        {
            const unsigned needq = __ballot_sync(kFull, !active);
            const uint32_t k = min((uint32_t)__popc(needq), stop);
            if (k) {
                __syncwarp();
                const uint32_t rank = __popc(needq & lt_mask);
                if (((needq >> lane) & 1u) && rank < k) {
                    const uint32_t slot = stop - 1 - rank;
                    const uint32_t w0 = wstk[0 * kStackCap + slot];
                    node = w0 & 0xffffu;
                    nv = w0 >> 16;
                    tr_prev = wstk[1 * kStackCap + slot];
                    h = wstk[2 * kStackCap + slot];
                    P = make_uint4(wstk[3 * kStackCap + slot], wstk[4 * kStackCap + slot], wstk[5 * kStackCap + slot],
                                   wstk[6 * kStackCap + slot]);
                    R = make_uint4(wstk[7 * kStackCap + slot], wstk[8 * kStackCap + slot], wstk[9 * kStackCap + slot],
                                   wstk[10 * kStackCap + slot]);
#pragma unroll
                    for (int q = 0; q < MAXV; q++) m2g[q] = wstk[(11 + q) * kStackCap + slot];
                    if (wr) {
                        bpre = wstk[(11 + MAXV) * kStackCap + slot];
                        for (uint32_t i = 0; i < bpre; i++) s_pre[i * kLB + tid] = wstk[(12 + MAXV + i) * kStackCap + slot];
                    }
                    const LNode dn = s_nodes[node];
                    g = dn.group_begin;
                    g_end = dn.group_end;
                    lim = kNone; d = 0; scan = false; active = true; age = 0;
                    if (STATS) st[ST_CONTEXTS]++;
                }
                stop -= k;
                __syncwarp();
            }
        }

        // ---------------------------------------------------- (1) roots for the rest
        unsigned need = __ballot_sync(kFull, !active);
        while (need && roots_left) {
            if (cl == 0) {
                uint32_t b = 0, sz = 0;
                if (ENUM) {  // static: chunk gwarp + wk * n_warps (identical in both passes)
                    b = (gwarp + wk * n_warps) * 32u;
                    if ((b >> 5) != gwarp + wk * n_warps) b = n_items;  // overflow: no more chunks
                    sz = 32;
                    wk++;
                } else {
                    if (lane == 0) {
                        const uint32_t cur = *(volatile uint32_t *)(p.lb + LB_ROOT);
                        const uint32_t rem = cur < n_items ? n_items - cur : 0u;
                        sz = max(32u, min(256u, rem / (4u * gridDim.x * (kLB / 32))));
                        b = atomicAdd(p.lb + LB_ROOT, sz);
                    }
                    b = __shfl_sync(kFull, b, 0);
                    sz = __shfl_sync(kFull, sz, 0);
                }
                if (b >= n_items) {
                    roots_left = false;
                    break;
                }
                cb = b;
                cl = min(sz, n_items - b);
            }
            const uint32_t take = min((uint32_t)__popc(need), cl);
            const uint32_t rank = __popc(need & lt_mask);
            const bool mine = ((need >> lane) & 1u) && rank < take;
            const uint32_t item = cb + rank;
            if (mine && item < n_pm) {  // a partial match: its node's completion was counted when it was made
                int lo = 0, hi2 = kPmStripes - 1;
                while (lo < hi2) {
                    const int mid = (lo + hi2 + 1) >> 1;
                    if (s_pref[mid] <= item) lo = mid;
                    else hi2 = mid - 1;
                }
                const uint4 *rec = reinterpret_cast<const uint4 *>(
                    p.pm + ((size_t)lo * p.pm_seg_cap + (item - s_pref[lo])) * p.pm_words);
                const uint4 a = __ldcs(rec), b4 = __ldcs(rec + 1);
                node = a.x & 0xffffu;
                nv = a.x >> 16;
                const uint32_t rt = a.y;
                const bool hole = node == 0xFFFFu;  // unused slot of a reserved run (bfs::kHole)
                if (hole) node = 0;
                tr_prev = a.z;
                h = a.w;
                P = b4;
#pragma unroll
                for (int q = 0; q < (MAXV + 3) / 4; q++) {
                    const uint4 m4 = __ldcs(rec + 2 + q);
                    if (4 * q + 0 < MAXV) m2g[(4 * q + 0) % MAXV] = m4.x;
                    if (4 * q + 1 < MAXV) m2g[(4 * q + 1) % MAXV] = m4.y;
                    if (4 * q + 2 < MAXV) m2g[(4 * q + 2) % MAXV] = m4.z;
                    if (4 * q + 3 < MAXV) m2g[(4 * q + 3) % MAXV] = m4.w;
                }
                if (!hole) {
                    R = __ldg(p.eptr + rt);
                    const LNode dn = s_nodes[node];
                    g = dn.group_begin; g_end = dn.group_end;
                    lim = kNone; d = 0; scan = false; age = 0;
                    active = true;
                }
            } else if (mine && p.light) {  // hybrid / mixed: a light root, mined whole (listed by the
                                           // breadth-first level, which also counted its completion)
                const uint32_t r = __ldg(p.light + (item - n_pm));
#pragma unroll
                for (int k = 2; k < MAXV; k++) m2g[k] = kNone;
                m2g[0] = __ldg(p.src + r);
                m2g[1] = __ldg(p.dst + r);
                h = __ldg(p.hi + r);
                tr_prev = __ldg(p.tr + r);
                R = __ldg(p.eptr + r);
                P = R;
                node = 0; nv = 2; g = root.group_begin; g_end = root.group_end;
                lim = kNone; d = 0; scan = false; age = 0;
                active = true;
            } else if (mine) {
                const uint32_t r = p.r0 + (item - n_pm);
                const uint32_t rs = __ldg(p.src + r), rd = __ldg(p.dst + r);
                if (rs != rd) {  // a self-loop never matches canonical 0->1 (reading R7)
                    uint32_t rk = 0;
                    if (wr) {
                        rk = __ldg(p.perm + r);
                        s_pre[tid] = rk;
                        bpre = 1;
                    }
                    if (root.flags & NODE_COMPLETION) {
                        if (wr) emit(root.slot, tid, 0, 0, rk);
                        else count_n(root.slot, tid, 1);
                    }
                    if (STATS) {
                        st[ST_ROOTS]++;
                        st[ST_BYTES] += 16 + (root_inner ? 16 : 0);
                        st[ST_MATCHES] += (root.flags & NODE_COMPLETION) ? 1 : 0;
                    }
                    if (root_inner) {
#pragma unroll
                        for (int k = 2; k < MAXV; k++) m2g[k] = kNone;
                        m2g[0] = rs;
                        m2g[1] = rd;
                        h = __ldg(p.hi + r);
                        tr_prev = __ldg(p.tr + r);
                        R = __ldg(p.eptr + r);
                        P = R;
                        node = 0; nv = 2; g = root.group_begin; g_end = root.group_end;
                        lim = kNone; d = 0; scan = false; age = 0;
                        active = true;
                        if (STATS) st[ST_NODES]++;
                    }
                } else if (STATS) {
                    st[ST_BYTES] += 16;
                }
            }
            const unsigned served = __ballot_sync(kFull, mine);
            if (STATS) n_roots_w += __popc(served);
            need &= ~served;
            cb += take;
            cl -= take;
        }

        // ---------------------------------------------------- one step of this lane's search
        fresh = false;
        do {
            if (!active) break;
            ++age;
            if (!scan) {
                if (g == g_end) {  // all anchor groups of `node` done: pop
                    if (d == 0) {
                        active = false;
                        break;
                    }
                    --d;
                    const uint32_t w0 = myfr[(d * FW + 0) * kLB];
                    pos = myfr[(d * FW + 1) * kLB];
                    tr_prev = myfr[(d * FW + 2) * kLB];
                    lim = myfr[(d * FW + 3) * kLB];
                    P.x = myfr[(d * FW + 4) * kLB];
                    P.y = myfr[(d * FW + 5) * kLB];
                    P.z = myfr[(d * FW + 6) * kLB];
                    P.w = myfr[(d * FW + 7) * kLB];
                    node = w0 & 0xffffu;
                    g = w0 >> 16;
                    const LNode dn = s_nodes[node];
                    nv = dn.nv;
                    g_end = dn.group_end;
#pragma unroll
                    for (int k = 2; k < MAXV; k++) m2g[k] = selp(m2g[k], kNone, (uint32_t)k < nv);
                } else {
                    const DGroup G = s_groups[g];
                    if (G.start < START_R0) {
                        pos = pick4(P, G.start);
                        lim = kNone;
                    } else if (G.start < START_SEARCH) {
                        pos = pick4(R, G.start - START_R0);
                        lim = kNone;
                    } else if (GEN && G.start == START_SEARCH) {
                        const uint32_t x = m2g_get<MAXV>(m2g, G.anchor);
                        const uint32_t *off = (G.kind == ANCHOR_OUT) ? p.out_off : p.in_off;
                        const uint2 *ent = (G.kind == ANCHOR_OUT) ? p.out_ent : p.in_ent;
                        uint32_t lo = __ldg(off + x), hi2 = __ldg(off + x + 1) - 1;
                        while (lo < hi2) {  // first entry with time rank > tr_prev
                            const uint32_t mid = lo + ((hi2 - lo) >> 1);
                            if (__ldg(&ent[mid].x) > tr_prev) hi2 = mid;
                            else lo = mid + 1;
                            if (STATS) st[ST_PROBES]++;
                        }
                        pos = lo;
                        lim = kNone;
                        if (STATS) st[ST_BYTES] += 8;
                    } else if (GEN) {  // GLOBAL: edge ids after the tie group of the previous edge, up to hi(root)
                        uint32_t lo = tr_prev, hi2 = h + 1;
                        while (lo < hi2) {
                            const uint32_t mid = lo + ((hi2 - lo) >> 1);
                            if (__ldg(p.tr + mid) > tr_prev) hi2 = mid;
                            else lo = mid + 1;
                            if (STATS) st[ST_PROBES]++;
                        }
                        pos = lo;
                        lim = h + 1;
                    }
                    if (STATS) {
                        st[ST_WINDOWS]++;
                        st[ST_BYTES] += G.kind == ANCHOR_GLOBAL ? 12 : 8;  // the terminating entry
                    }
                    // a long window of leaf children is scanned by the whole warp (below); the
                    // probe is issued with the window's first entry (no extra round trip)
                    if (G.n_inner == 0 && G.kind != ANCHOR_GLOBAL) chk = m2g_get<MAXV>(m2g, G.anchor);
                }
                scan = true;
            }

            // scan one entry of the current window
            const uint32_t gc = g;  // this entry's group (g may advance below when the window closes)
            const DGroup G = s_groups[gc];
            uint32_t etr, e1, e2 = 0;
            const bool glob = GEN && G.kind == ANCHOR_GLOBAL;
            if (glob) {
                etr = pos < lim ? __ldg(p.tr + pos) : kNone;
                if (etr != kNone) {
                    e1 = __ldg(p.src + pos);
                    e2 = __ldg(p.dst + pos);
                } else {
                    e1 = 0;
                }
            }
            // lists: the next entry is loaded with this one (independent load), so the window's
            // terminator does not cost an iteration of its own
            bool last = false;
            if (!glob) {
                const uint2 *lp = (G.kind == ANCHOR_OUT ? p.out_ent : p.in_ent) + pos;
                const uint2 e = __ldg(lp);
                const uint32_t nxt = __ldg(&lp[1].x);
                if (chk != kNone) {  // fresh leaf window: >= kHelpMin entries (within the anchor's list)?
                    const uint32_t sent = __ldg((G.kind == ANCHOR_OUT ? p.out_off : p.in_off) + chk + 1) - 1;
                    const uint32_t far = __ldg(&lp[kHelpMin - 1].x);
                    chk = kNone;
                    if (pos + kHelpMin - 1 < sent && far <= h) {
                        help = true;
                        break;
                    }
                }
                etr = e.x;
                e1 = e.y;
                last = nxt > h;
            }
            if (STATS) st[ST_BATCHES]++;
            if (etr > h || pos >= lim) {  // window end
                ++g;
                scan = false;
                break;
            }
            ++pos;
            if (last) {  // this entry closes the window: the next step starts the next group
                ++g;
                scan = false;
            }
            if (etr <= tr_prev) break;  // before the window (lower-bound start)
            if (STATS) {
                st[ST_ENTRIES]++;
                st[ST_BYTES] += glob ? 12 : 8;
            }
            uint32_t cls;
            if (glob)
                cls = (e1 != e2 && classify<MAXV>(m2g, e1) == CLS_NEW && classify<MAXV>(m2g, e2) == CLS_NEW)
                          ? CLS_NEW : 0xFEu;
            else
                cls = classify<MAXV>(m2g, e1);
            uint32_t hit = kNone;
            if (G.child_end - G.child_begin <= 4 && gc < kGwMax) {  // one SIMD byte compare
                const uint32_t eq = __vcmpeq4(s_gw[gc], cls * 0x01010101u);
                hit = eq ? G.child_begin + ((__ffs(eq) - 1) >> 3) : kNone;
            } else {
                for (uint32_t c = G.child_begin; c < G.child_end; ++c)
                    if (s_nodes[c].want == cls) {
                        hit = c;
                        break;
                    }
            }
            if (hit == kNone) break;
            const LNode dn = s_nodes[hit];
            uint32_t erk = 0;  // ENUM pass 2: input rank of the matched edge
            if (wr) erk = glob ? __ldg(p.perm + (pos - 1))
                               : __ldg((G.kind == ANCHOR_OUT ? p.out_rank : p.in_rank) + (pos - 1));
            if (dn.flags & NODE_COMPLETION) {
                if (wr) emit(dn.slot, tid, bpre, d, erk);
                else count_n(dn.slot, tid, 1);
                if (STATS) st[ST_MATCHES]++;
            }
            if (dn.flags & NODE_INNER) {
                if (wr) myfr[(d * FW + kFrameWords) * kLB] = erk;
                // the parent resumes at pos in its group (undo the early window close)
                myfr[(d * FW + 0) * kLB] = node | (gc << 16);
                myfr[(d * FW + 1) * kLB] = pos;
                myfr[(d * FW + 2) * kLB] = tr_prev;
                myfr[(d * FW + 3) * kLB] = lim;
                myfr[(d * FW + 4) * kLB] = P.x;
                myfr[(d * FW + 5) * kLB] = P.y;
                myfr[(d * FW + 6) * kLB] = P.z;
                myfr[(d * FW + 7) * kLB] = P.w;
                ++d;
                if (dn.n_new >= 1) m2g_set<MAXV>(m2g, nv, e1);
                if (dn.n_new == 2) m2g_set<MAXV>(m2g, nv + 1, e2);
                nv = dn.nv;
                tr_prev = etr;
                P = glob ? __ldg(p.eptr + (pos - 1))
                         : __ldg((G.kind == ANCHOR_OUT ? p.out_ptr : p.in_ptr) + (pos - 1));
                node = hit;
                g = dn.group_begin;
                g_end = dn.group_end;
                lim = kNone;
                scan = false;
                fresh = true;
                if (STATS) {
                    st[ST_NODES]++;
                    st[ST_BYTES] += 16;
                }
            }
        } while (0);

        // ---------------------------------------------------- warp cooperation
        // (1) long leaf windows: the whole warp scans each parked window, 32 entries per
        //     step, one ballot per leaf child, and credits the owning lane's counters.
        unsigned hm = __ballot_sync(kFull, help);
        while (hm) {
            const int j = __ffs(hm) - 1;
            hm &= hm - 1;
            const uint32_t gj = __shfl_sync(kFull, g, j);
            const uint32_t hj = __shfl_sync(kFull, h, j);
            const uint32_t tpj = __shfl_sync(kFull, tr_prev, j);
            const uint32_t nvj = __shfl_sync(kFull, nv, j);
            const uint32_t bj = __shfl_sync(kFull, bpre, j), dj = __shfl_sync(kFull, d, j);
            uint32_t mj[MAXV];
#pragma unroll
            for (int k = 0; k < MAXV; k++) mj[k] = __shfl_sync(kFull, m2g[k], j);
            const DGroup G = s_groups[gj];
            const uint2 *ent = (G.kind == ANCHOR_OUT) ? p.out_ent : p.in_ent;
            uint32_t b = __shfl_sync(kFull, pos, j);
            for (;;) {
                const uint2 e = __ldg(ent + b + lane);
                const unsigned fm = __ballot_sync(kFull, e.x > hj);
                const unsigned inmask = fm ? ((1u << (__ffs(fm) - 1)) - 1u) : kFull;
                const bool w = ((inmask >> lane) & 1u) && e.x > tpj;
                const uint32_t cls = classify<MAXV>(mj, e.y);
                for (uint32_t c = G.child_begin; c < G.child_end; ++c) {
                    const LNode dn = s_nodes[c];
                    const unsigned mc = __ballot_sync(kFull, w && cls == dn.want);
                    if (wr) {
                        if (w && cls == dn.want && (dn.flags & NODE_COMPLETION))
                            emit(dn.slot, wbase + j, bj, dj,
                                 __ldg((G.kind == ANCHOR_OUT ? p.out_rank : p.in_rank) + b + lane));
                    } else if (lane == 0 && mc && (dn.flags & NODE_COMPLETION)) count_n(dn.slot, wbase + j, __popc(mc));
                    if (STATS && lane == 0) st[ST_MATCHES] += __popc(mc);
                }
                if (STATS) {
                    const uint32_t we = __popc(__ballot_sync(kFull, w));
                    if (lane == 0) {
                        st[ST_ENTRIES] += we;
                        st[ST_BYTES] += 8ull * we;
                        st[ST_BATCHES]++;
                    }
                    n_help++;
                }
                if (fm) break;
                b += 32;
            }
            if (lane == j) {
                help = false;
                scan = false;
                ++g;
            }
        }
        // (2) split heavy searches: a lane that has run for more than kAgeMin steps on one
        //     root/task hands each partial match it descends into to this warp's task stack
        //     (the paper's intra-warp balancing); any idle lane of the warp
        //     mines that subtree only (its frame stack starts there) and the donor returns to
        //     its parent's window.  Sibling exclusivity holds by
        //     construction: a task is one partial match, handed over before any child of it
        //     was examined.
        {
            const unsigned don = __ballot_sync(kFull, fresh && active && (age > kAgeMin || !roots_left));
            const uint32_t n = min((uint32_t)__popc(don), kStackCap - stop);
            if (n) {
                const uint32_t rank = __popc(don & lt_mask);
                if (((don >> lane) & 1u) && rank < n) {
                    const uint32_t slot = stop + rank;
                    wstk[0 * kStackCap + slot] = node | (nv << 16);
                    wstk[1 * kStackCap + slot] = tr_prev;
                    wstk[2 * kStackCap + slot] = h;
                    wstk[3 * kStackCap + slot] = P.x;
                    wstk[4 * kStackCap + slot] = P.y;
                    wstk[5 * kStackCap + slot] = P.z;
                    wstk[6 * kStackCap + slot] = P.w;
                    wstk[7 * kStackCap + slot] = R.x;
                    wstk[8 * kStackCap + slot] = R.y;
                    wstk[9 * kStackCap + slot] = R.z;
                    wstk[10 * kStackCap + slot] = R.w;
#pragma unroll
                    for (int q = 0; q < MAXV; q++) wstk[(11 + q) * kStackCap + slot] = m2g[q];
                    if (wr) {  // the task's base prefix: this search's prefix + its frames' edges
                        wstk[(11 + MAXV) * kStackCap + slot] = bpre + d;
                        for (uint32_t i = 0; i < bpre; i++) wstk[(12 + MAXV + i) * kStackCap + slot] = s_pre[i * kLB + tid];
                        for (uint32_t i = 0; i < d; i++)
                            wstk[(12 + MAXV + bpre + i) * kStackCap + slot] = myfr[(i * FW + kFrameWords) * kLB];
                    }
                    g = g_end;  // handed out: pop back to the parent at the next step
                    fresh = false;
                    if (STATS) st[ST_OFFLOADS]++;
                }
                stop += n;
            }
        }

        // ---------------------------------------------------- (3) termination
        if (!roots_left && stop == 0 && !__any_sync(kFull, active)) break;
    }

    if (STATS && p.dbg && lane == 0) {
        unsigned long long t_end, smid;
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_end));
        uint32_t sm32;
        asm("mov.u32 %0, %%smid;" : "=r"(sm32));
        smid = sm32;
        unsigned long long *r = p.dbg + (size_t)(blockIdx.x * (kLB / 32) + (tid >> 5)) * 8;
        r[0] = t_start; r[1] = t_end; r[2] = n_iter; r[3] = n_help; r[4] = n_roots_w; r[5] = t_roots_done;
        r[6] = smid; r[7] = 0;
    }
    // ---- counters: lanes -> block -> global, once per block
    __syncthreads();
    if (ENUM && p.enum_pass == 1) {  // per-warp match counts (lane counters + their u64 overflow)
        for (uint32_t sl = 0; sl < p.n_slots; sl++) {
            unsigned long long v = s_cnt[sl * kLB + tid];
#pragma unroll
            for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(kFull, v, o);
            if (lane == 0) p.wcnt[(size_t)sl * n_warps + gwarp] = v + s_ebase[(tid >> 5) * p.n_slots + sl];
        }
    }
    if (LANECNT) {
        for (uint32_t s = (uint32_t)tid >> 5; s < p.n_slots; s += kLB / 32) {
            unsigned long long v = 0;
            for (int i = lane; i < kLB; i += 32) v += s_cnt[s * kLB + i];
#pragma unroll
            for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(kFull, v, o);
            if (lane == 0) s_tot[s] += v;
        }
        __syncthreads();
    }
    for (uint32_t i = tid; i < p.n_motifs; i += kLB) {
        const unsigned long long v = s_tot[s_nodes[p.motif_node[i]].slot];
        if (v) atomicAdd(p.counts + i, v);
    }
    if (STATS) {
#pragma unroll
        for (int i = 0; i < ST_N; i++) {
            unsigned long long v = st[i];
#pragma unroll
            for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(kFull, v, o);
            if (lane == 0 && v) atomicAdd(p.stats + i, v);
        }
    }
}

}  // namespace lane
