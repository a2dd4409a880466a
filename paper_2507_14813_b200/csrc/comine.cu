// comine.cu -- sm_100a kernels of the co-mining hot path + the device side of the C ABI.
//
// Steps:
//   a2  window_end_kernel: hi[r] = last edge id with t <= t_r + delta
//   a3-a7 comine_kernel:   persistent grid; each warp claims 32 root edges at a
//       time from a global atomic queue ("distributes these
//       candidate edges across warps"), then runs one depth-first co-mining
//       search per root along the MG-Tree table (Algorithm 3):
//         - window location (Algo 1 l.210-214): the edge matched at the current
//           node carries successor pointers P(e) -- the first position after t_e
//           in out(src), in(dst), out(dst), in(src) -- so a window anchored at one
//           of its endpoints starts with no search; lists are sentinel-terminated so
//           the window ends on "time rank > hi(root)" alone.  Other anchors use the
//           root edge's pointers as a lower bound, or a lane-cooperative 32-ary search;
//         - candidate filter: lane i takes window entry i (coalesced 8-byte loads);
//           the entry's neighbour is classified against the warp-uniform register
//           map m2g (which mapped motif vertex it is, or NEW); each child of the anchor
//           group tests its structural constraint with one compare + __ballot_sync
//           (Algo 1 l.219 + full injectivity, reading R4) -- the paper's predicated /
//           LUT-simplified checks;
//         - completion children add __popc(mask) to a lane-resident counter
//           (count[Q_N]++, Algo 3 l.661) without descending; inner children push a
//           frame on the per-warp shared-memory DFS stack and descend with the
//           candidate as the new partial match (Algo 3 l.665-669);
//         - dynamic load balance (PAPER.md:758-774 inter-warp balancing, 893-904
//           multi-offload): once warps go idle, a busy warp that reaches the next batch
//           of a long window fans the rest of the window out as chunk contexts in a
//           global queue (and the node's remaining anchor groups as one more context).
//       Counters are reduced per block in shared memory, then flushed once per
//       block with 64-bit atomics ("context ... maintained locally").
// All arithmetic is integer (u32 ids and time ranks, i64 timestamps, u64 counts).
#include <cuda_runtime.h>

#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <mutex>

#include "internal.h"

namespace mayura {

namespace {

constexpr int kWarps = 8;
constexpr int kBlock = kWarps * 32;
constexpr int kMaxDepth = MAYURA_MAX_EDGES;  // frames 0..max_edges-2
constexpr int kMaxGroupChildren = MAYURA_MAX_V + 1;
constexpr unsigned kFull = 0xffffffffu;
constexpr uint32_t kNone = 0xffffffffu;
constexpr int kCtxWords = 32;               // one context = 128 bytes
constexpr uint32_t kCtxCap = 1u << 20;      // contexts per launch (128 MiB)
constexpr uint32_t kSmallRows = 64;         // trees up to this many rows/groups: table in parameter space
constexpr uint32_t kSweepMax = 32;          // leaf sweep: longest per-lane window
enum { S_GROUP = 0, S_BATCH = 1, S_ITER = 2 };
enum { ST_ROOTS, ST_NODES, ST_WINDOWS, ST_ENTRIES, ST_PROBES, ST_BATCHES, ST_BYTES, ST_MATCHES,
       ST_OFFLOADS, ST_CONTEXTS, ST_N };
// load-balancer words (zeroed by window_end_kernel)
enum { LB_ROOT = 0, LB_TAIL = 1, LB_HEAD = 2, LB_IDLE = 3, LB_WORK = 4, LB_ERR = 5, LB_N = 8 };

struct KParams {
    const uint32_t *src, *dst, *tr, *hi;
    const uint4 *eptr;                 // P(e) per edge id
    const uint32_t *out_off, *in_off;  // list x = [off[x], off[x+1]-1), sentinel at off[x+1]-1
    const uint2 *out_ent, *in_ent;     // (tr, nbr)
    const uint4 *out_ptr, *in_ptr;     // P(e) of each entry's edge
    const DNode *nodes;
    const DGroup *groups;
    const uint32_t *motif_node;
    uint32_t n_nodes, n_groups, n_motifs;
    uint32_t r0, n_roots;
    uint32_t *lb;
    uint32_t *ctx;
    uint32_t ctx_cap, epoch;
    unsigned long long *counts;
    unsigned long long *stats;
    DNode tn[kSmallRows];   // small trees: the table itself (parameter space)
    DGroup tg[kSmallRows];
};

struct __align__(16) Frame {  // one per warp per DFS depth (shared memory), 3 x 16 bytes
    uint32_t node_g, ci, tr_prev, pos;
    uint32_t batch, mask, lim, g_end;
    uint4 P;
};

__device__ __forceinline__ uint32_t ld_acquire(const uint32_t *p) {
    uint32_t v;
    asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ uint32_t ld_relaxed(const uint32_t *p) {
    uint32_t v;
    asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ void st_release(uint32_t *p, uint32_t v) {
    asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

template <int MAXV>
__device__ __forceinline__ uint32_t m2g_get(const uint32_t (&m)[MAXV], uint32_t i) {
    uint32_t r = 0;
#pragma unroll
    for (int k = 0; k < MAXV; k++) r = (k == (int)i) ? m[k] : r;
    return r;
}
template <int MAXV>
__device__ __forceinline__ void m2g_set(uint32_t (&m)[MAXV], uint32_t i, uint32_t x) {
#pragma unroll
    for (int k = 0; k < MAXV; k++) m[k] = (k == (int)i) ? x : m[k];
}
// Which mapped motif vertex (index < nv) the graph vertex x already is, or CLS_NEW.
template <int MAXV>
__device__ __forceinline__ uint32_t classify(const uint32_t (&m)[MAXV], uint32_t nv, uint32_t x) {
    uint32_t c = CLS_NEW;
#pragma unroll
    for (int k = 0; k < MAXV; k++) c = ((uint32_t)k < nv && m[k] == x) ? (uint32_t)k : c;
    return c;
}
__device__ __forceinline__ uint32_t pick(const uint4 &v, uint32_t k) {
    return k == 0 ? v.x : k == 1 ? v.y : k == 2 ? v.z : v.w;
}
__device__ __forceinline__ uint4 shfl4(const uint4 &v, int src) {
    return make_uint4(__shfl_sync(kFull, v.x, src), __shfl_sync(kFull, v.y, src), __shfl_sync(kFull, v.z, src),
                      __shfl_sync(kFull, v.w, src));
}

// Write one search context (lane l writes word l; word 31 = publication flag, written later):
// [0] node | group << 16 (kNone = no-op), [1] window position (kNone = start the group fresh),
// [2] position limit, [3] tr_prev, [4] hi(root), [5..8] P, [9..12] R, [13..] m2g.
template <int MAXV>
__device__ __forceinline__ void put_ctx(uint32_t *slot, int lane, uint32_t w0, uint32_t w1, uint32_t w2,
                                        uint32_t w3, uint32_t w4, const uint4 &P, const uint4 &R,
                                        const uint32_t (&m2g)[MAXV]) {
    uint32_t v;
    switch (lane) {
        case 0: v = w0; break;
        case 1: v = w1; break;
        case 2: v = w2; break;
        case 3: v = w3; break;
        case 4: v = w4; break;
        case 5: v = P.x; break;
        case 6: v = P.y; break;
        case 7: v = P.z; break;
        case 8: v = P.w; break;
        case 9: v = R.x; break;
        case 10: v = R.y; break;
        case 11: v = R.z; break;
        case 12: v = R.w; break;
        default: v = (lane - 13 < MAXV) ? m2g_get<MAXV>(m2g, lane - 13) : 0u; break;
    }
    if (lane < 31) slot[lane] = v;
}
// Make contexts [base, base+n) visible: every lane fences its own stores; lane 0 adds the
// published contexts to the work counter (so "work == 0" implies an empty queue), then sets
// the flags.
__device__ __forceinline__ void publish_ctx(uint32_t *ctx, uint32_t cap, uint32_t base, uint32_t n, uint32_t epoch,
                                            uint32_t *work, int lane) {
    __syncwarp();
    __threadfence();
    __syncwarp();
    if (lane == 0) {
        const uint32_t npub = base >= cap ? 0u : min(n, cap - base);
        if (npub) atomicAdd(work, npub);
        for (uint32_t j = 0; j < npub; j++) st_release(ctx + (size_t)(base + j) * 32 + 31, epoch);
    }
}

// Lane-cooperative 32-ary search: returns lo' <= (first index in [lo, end) whose key exceeds
// x) with that index - lo' < 32, so the 32-entry batch at lo' reaches it.  key(i) = time rank
// of list entry i (kind OUT/IN) or of edge i (GLOBAL).  One sample load per lane per step.
template <bool STATS>
__device__ __forceinline__ uint32_t locate(bool global, const uint2 *__restrict__ ent,
                                           const uint32_t *__restrict__ trg, uint32_t lo, uint32_t end,
                                           uint32_t x, int lane, unsigned long long &probes) {
    uint32_t hi = end;
    while (hi - lo > 32) {
        const uint32_t n = hi - lo;
        const uint32_t step = (n + 31) >> 5;
        const uint32_t i = (uint32_t)lane * step;
        uint32_t key = kNone;
        if (i < n) key = global ? __ldg(trg + lo + i) : __ldg(&ent[lo + i].x);
        if (STATS) probes++;
        const unsigned b = __ballot_sync(kFull, key > x);
        if (b == 0) {
            lo += 31 * step + 1;
        } else {
            const uint32_t j = (uint32_t)(__ffs(b) - 1);
            if (j == 0) break;
            const uint32_t nlo = lo + (j - 1) * step + 1;
            hi = min(lo + j * step + 1, hi);
            lo = nlo;
        }
    }
    return lo;
}

// CNT > 0 ("small" trees, <= 64 rows and groups): the table lives in the kernel's parameter
// space (constant bank; warp-uniform indexed loads) and the counters in lane registers.
// CNT == 0: table and counters in dynamic shared memory.
template <int MAXV, int CNT, bool STATS>
__global__ void __launch_bounds__(kBlock, 4) comine_kernel(const __grid_constant__ KParams p) {
    extern __shared__ __align__(16) unsigned char smem[];
    __shared__ Frame s_frames[kWarps * kMaxDepth];
    __shared__ uint32_t s_masks[kWarps * kMaxDepth * kMaxGroupChildren];
    __shared__ unsigned long long s_cnt_small[CNT > 0 ? kSmallRows : 1];
    unsigned long long *s_cnt = CNT > 0 ? s_cnt_small : reinterpret_cast<unsigned long long *>(smem);
    DNode *s_nodes = reinterpret_cast<DNode *>(reinterpret_cast<unsigned long long *>(smem) + p.n_nodes);
    DGroup *s_groups = reinterpret_cast<DGroup *>(s_nodes + p.n_nodes);
#define NODE(i) (CNT > 0 ? p.tn[(i)] : s_nodes[(i)])
#define GROUP(i) (CNT > 0 ? p.tg[(i)] : s_groups[(i)])

    for (uint32_t i = threadIdx.x; i < p.n_nodes; i += blockDim.x) {
        if (CNT == 0) s_nodes[i] = p.nodes[i];
        s_cnt[i] = 0;
    }
    if (CNT == 0)
        for (uint32_t i = threadIdx.x; i < p.n_groups; i += blockDim.x) s_groups[i] = p.groups[i];
    __syncthreads();

    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    Frame *F = s_frames + warp * kMaxDepth;
    uint32_t *MS = s_masks + warp * kMaxDepth * kMaxGroupChildren;
    unsigned long long cnt[CNT > 0 ? CNT : 1];
#pragma unroll
    for (int s = 0; s < (CNT > 0 ? CNT : 1); s++) cnt[s] = 0;
    unsigned long long st[ST_N];
#pragma unroll
    for (int i = 0; i < ST_N; i++) st[i] = 0;

    // counter of trie node c (warp-uniform c, m): lane c%32 owns it (CNT > 0) or shared memory
    // add n (warp-uniform) matches to trie node c's counter
    auto count = [&](uint32_t c, uint32_t n) {
        if (CNT == 0) {
            if (lane == 0 && n) atomicAdd(&s_cnt[c], (unsigned long long)n);
        } else {
#pragma unroll
            for (int s = 0; s < (CNT > 0 ? CNT : 1); s++)
                if (c == (uint32_t)(lane + 32 * s)) cnt[s] += n;
        }
        if (STATS && lane == 0) st[ST_MATCHES] += n;
    };

    const DNode root = NODE(0);
    bool roots_done = false, idle = false;
    uint32_t ticket = kNone;  // lane 0: claimed queue slot not yet published

    // ---------------------------------------------------------------- DFS state
    uint32_t m2g[MAXV];
    uint4 R, P;                    // successor pointers of the root edge / the node's edge
    uint32_t h = 0, tr_prev = 0, node = 0, nv = 2, g = 0, g_end = 0, kind = 0, pos = 0, lim = kNone;
    uint32_t batch = 0, ci = 0, c_end = 0, mask = 0, nbatch = 0;
    int depth = 0, state = S_GROUP;
    uint32_t etr = 0, e1 = 0, e2 = 0;  // this lane's batch entry: time rank, neighbour / (src, dst)
    uint4 ep = make_uint4(0, 0, 0, 0); // P of this lane's entry edge

    for (;;) {
        // ------------------------------------------------------- acquire work
        uint32_t chunk_base = kNone, chunk_len = 0, ctx_slot = kNone;
        bool quit = false;
        if (!roots_done) {
            // guided self-scheduling: chunks shrink from 32 roots to 1 as the queue drains,
            // so the root queue lasts until the end of the launch
            uint32_t b = 0, sz = 0;
            if (lane == 0) {
                const uint32_t cur = ld_relaxed(p.lb + LB_ROOT);
                const uint32_t rem = cur < p.n_roots ? p.n_roots - cur : 0u;
                sz = max(1u, min(32u, rem / (2u * gridDim.x * kWarps)));
                b = atomicAdd(p.lb + LB_ROOT, sz);
                if (b < p.n_roots) atomicAdd(p.lb + LB_WORK, 1u);
            }
            b = __shfl_sync(kFull, b, 0);
            sz = __shfl_sync(kFull, sz, 0);
            if (b < p.n_roots) {
                chunk_base = b;
                chunk_len = min(sz, p.n_roots - b);
            } else {
                roots_done = true;
            }
        }
        if (chunk_base == kNone) {
            // context phase: take a ticket (queue slot) and wait for it to be published, or exit
            // once LB_WORK -- warps holding work + published contexts not yet finished -- is 0
            uint32_t got = kNone, ex = 0;
            if (lane == 0) {
                if (!idle) {
                    atomicAdd(p.lb + LB_IDLE, 1u);
                    idle = true;
                }
                if (ticket == kNone) ticket = atomicAdd(p.lb + LB_HEAD, 1u);
                // polls are relaxed loads: a gpu-scope acquire would invalidate this SM's L1
                // (CCTL.IVALL) on every poll; one fence follows a successful poll instead
                for (int spin = 0;; spin++) {
                    if (ticket < p.ctx_cap &&
                        ld_relaxed(p.ctx + (size_t)ticket * kCtxWords + (kCtxWords - 1)) == p.epoch) {
                        got = ticket;
                        ticket = kNone;
                        __threadfence();
                        break;
                    }
                    if (ld_relaxed(p.lb + LB_WORK) == 0) {
                        ex = 1;
                        break;
                    }
                    // exponential backoff: waiting warps must not steal issue slots from working ones
                    __nanosleep(64u << (spin < 5 ? spin : 5));
                }
                if (got != kNone) {
                    atomicSub(p.lb + LB_IDLE, 1u);
                    idle = false;
                }
            }
            got = __shfl_sync(kFull, got, 0);
            ex = __shfl_sync(kFull, ex, 0);
            idle = __shfl_sync(kFull, (int)idle, 0) != 0;
            if (ex) quit = true;
            else ctx_slot = got;
        }
        if (quit) break;

        // ---------------------------------------------- root chunk: 32 roots
        uint32_t rs = 0, rd = 0, rt = 0, rh = 0;
        uint4 rp = make_uint4(0, 0, 0, 0);
        unsigned pending = 0;
        if (chunk_base != kNone) {
            const bool valid = (uint32_t)lane < chunk_len;
            const uint32_t r = p.r0 + chunk_base + lane;
            if (valid) {
                rs = __ldg(p.src + r);
                rd = __ldg(p.dst + r);
                rt = __ldg(p.tr + r);
                rh = __ldg(p.hi + r);
                if (root.flags & NODE_INNER) rp = __ldg(p.eptr + r);
            }
            pending = __ballot_sync(kFull, valid && rs != rd);  // a self-loop never matches 0->1
            if (STATS) {
                const unsigned vm = __ballot_sync(kFull, valid);
                if (lane == 0) {
                    st[ST_ROOTS] += __popc(pending);
                    st[ST_BYTES] += 16ull * __popc(vm) + ((root.flags & NODE_INNER) ? 16ull * __popc(pending) : 0);
                }
            }
            if (root.flags & NODE_COMPLETION) count(0, __popc(pending));
            if (!(root.flags & NODE_INNER)) pending = 0;
        }

        // one search per pending root (or one context)
        for (;;) {
            if (chunk_base != kNone) {
                if (!pending) break;
                const int j = __ffs(pending) - 1;
                pending &= pending - 1;
                if (pending) {
                    // idle warps exist: hand this chunk's other pending roots to the queue
                    uint32_t n_idle = 0;
                    if (lane == 0) n_idle = ld_relaxed(p.lb + LB_IDLE);
                    n_idle = __shfl_sync(kFull, n_idle, 0);
                    if (n_idle > 0) {
                        const uint32_t total = __popc(pending);
                        uint32_t base = 0;
                        if (lane == 0) base = atomicAdd(p.lb + LB_TAIL, total);
                        base = __shfl_sync(kFull, base, 0);
                        const bool fits = base + total <= p.ctx_cap;
                        unsigned rest = pending;
                        for (uint32_t q = 0; q < total && base + q < p.ctx_cap; q++) {
                            const int b = __ffs(rest) - 1;
                            rest &= rest - 1;
                            uint32_t rm[MAXV];
#pragma unroll
                            for (int k = 0; k < MAXV; k++) rm[k] = 0;
                            rm[0] = __shfl_sync(kFull, rs, b);
                            rm[1] = __shfl_sync(kFull, rd, b);
                            const uint4 rr = shfl4(rp, b);
                            put_ctx<MAXV>(p.ctx + (size_t)(base + q) * kCtxWords, lane,
                                          fits ? (uint32_t)root.group_begin << 16 : kNone, kNone, kNone,
                                          __shfl_sync(kFull, rt, b), __shfl_sync(kFull, rh, b), rr, rr, rm);
                        }
                        publish_ctx(p.ctx, p.ctx_cap, base, total, p.epoch, p.lb + LB_WORK, lane);
                        if (fits) {
                            pending = 0;
                            if (STATS && lane == 0) st[ST_OFFLOADS]++;
                        }
                    }
                }
#pragma unroll
                for (int k = 0; k < MAXV; k++) m2g[k] = 0;
                m2g[0] = __shfl_sync(kFull, rs, j);
                m2g[1] = __shfl_sync(kFull, rd, j);
                h = __shfl_sync(kFull, rh, j);
                tr_prev = __shfl_sync(kFull, rt, j);
                R = shfl4(rp, j);
                P = R;
                node = 0; nv = 2; g = root.group_begin; g_end = root.group_end;
                lim = kNone; depth = 0; state = S_GROUP;
                if (STATS && lane == 0) st[ST_NODES]++;
            } else {
                if (ctx_slot == kNone) break;
                uint32_t w = 0;
                if (ctx_slot < p.ctx_cap) {
                    __syncwarp();  // lane 0 observed the flag and fenced
                    w = __ldcg(p.ctx + (size_t)ctx_slot * kCtxWords + lane);
                } else {
                    w = kNone;
                }
                ctx_slot = kNone;
                const uint32_t w0 = __shfl_sync(kFull, w, 0);
                if (w0 == kNone) continue;  // no-op context (overflowed reservation)
                node = w0 & 0xffffu;
                g = w0 >> 16;
                pos = __shfl_sync(kFull, w, 1);
                lim = __shfl_sync(kFull, w, 2);
                tr_prev = __shfl_sync(kFull, w, 3);
                h = __shfl_sync(kFull, w, 4);
                P = make_uint4(__shfl_sync(kFull, w, 5), __shfl_sync(kFull, w, 6), __shfl_sync(kFull, w, 7),
                               __shfl_sync(kFull, w, 8));
                R = make_uint4(__shfl_sync(kFull, w, 9), __shfl_sync(kFull, w, 10), __shfl_sync(kFull, w, 11),
                               __shfl_sync(kFull, w, 12));
#pragma unroll
                for (int k = 0; k < MAXV; k++) m2g[k] = __shfl_sync(kFull, w, 13 + k);
                const DNode dn = NODE(node);
                nv = dn.nv;
                g_end = (lim != kNone) ? g + 1 : dn.group_end;
                depth = 0;
                if (pos == kNone) {
                    state = S_GROUP;
                } else {
                    kind = GROUP(g).kind;
                    nbatch = 1;  // a continuation: may split again
                    state = S_BATCH;
                }
                if (STATS && lane == 0) st[ST_CONTEXTS]++;
            }

            // ---------------------------------------------------- the search
            for (;;) {
                if (state == S_GROUP) {
                    if (g == g_end) {  // all anchor groups of `node` done: pop
                        if (depth == 0) break;
                        --depth;
                        __syncwarp();
                        const Frame f = F[depth];
                        node = f.node_g & 0xffffu; g = f.node_g >> 16; ci = f.ci; tr_prev = f.tr_prev;
                        pos = f.pos; batch = f.batch; mask = f.mask; lim = f.lim; g_end = f.g_end; P = f.P;
                        const DGroup G = GROUP(g);
                        nv = NODE(node).nv;
                        kind = G.kind; c_end = G.child_end;
                        const uint32_t idx = batch + lane;
                        if (kind == ANCHOR_GLOBAL) {
                            etr = __ldg(p.tr + idx); e1 = __ldg(p.src + idx); e2 = __ldg(p.dst + idx);
                            ep = __ldg(p.eptr + idx);
                        } else {
                            const uint2 e = __ldg((kind == ANCHOR_OUT ? p.out_ent : p.in_ent) + idx);
                            etr = e.x; e1 = e.y;
                            ep = __ldg((kind == ANCHOR_OUT ? p.out_ptr : p.in_ptr) + idx);
                        }
                        state = S_ITER;
                    } else {
                        const DGroup G = GROUP(g);
                        kind = G.kind;
                        nbatch = 0;
                        if (G.start < START_R0) {
                            pos = pick(P, G.start);
                        } else if (G.start < START_SEARCH) {
                            pos = pick(R, G.start - START_R0);
                        } else if (G.start == START_SEARCH) {
                            const uint32_t x = m2g_get<MAXV>(m2g, G.anchor);
                            const uint32_t *off = (kind == ANCHOR_OUT) ? p.out_off : p.in_off;
                            const uint32_t lo = __ldg(off + x), end = __ldg(off + x + 1) - 1;
                            pos = locate<STATS>(false, kind == ANCHOR_OUT ? p.out_ent : p.in_ent, p.tr, lo, end,
                                                tr_prev, lane, st[ST_PROBES]);
                            if (STATS && lane == 0) st[ST_BYTES] += 8;
                        } else {  // GLOBAL: edge ids (tie group of the previous edge, hi(root)]
                            pos = locate<STATS>(true, nullptr, p.tr, tr_prev, h + 1, tr_prev, lane, st[ST_PROBES]);
                        }
                        // a fresh window is bounded by hi(root) alone (edge ids for GLOBAL);
                        // chunk contexts enter S_BATCH directly with their own limit
                        lim = (kind == ANCHOR_GLOBAL) ? h + 1 : kNone;
                        if (STATS && lane == 0) st[ST_WINDOWS]++;
                        state = S_BATCH;
                    }
                }
                if (state == S_BATCH) {
                    const DGroup G = GROUP(g);
                    if (pos >= lim) {
                        ++g;
                        state = S_GROUP;
                        continue;
                    }
                    // ---- dynamic load balance: split the rest of a long window when warps idle
                    if (nbatch > 0) {
                        uint32_t n_idle = 0;
                        if (lane == 0) n_idle = ld_relaxed(p.lb + LB_IDLE);
                        n_idle = __shfl_sync(kFull, n_idle, 0);
                        if (n_idle > 0) {
                            // window end: first position in [pos, list end) with time rank > h
                            uint32_t wend;
                            if (kind == ANCHOR_GLOBAL) {
                                wend = lim;
                            } else {
                                const uint32_t x = m2g_get<MAXV>(m2g, G.anchor);
                                const uint32_t *off = (kind == ANCHOR_OUT) ? p.out_off : p.in_off;
                                const uint2 *ent = (kind == ANCHOR_OUT) ? p.out_ent : p.in_ent;
                                const uint32_t end = __ldg(off + x + 1);  // one past the sentinel
                                uint32_t lo = locate<STATS>(false, ent, p.tr, pos, end, h, lane, st[ST_PROBES]);
                                const uint32_t idx = lo + lane;
                                const uint32_t k2 = idx < end ? __ldg(&ent[idx].x) : kNone;
                                const unsigned b = __ballot_sync(kFull, k2 > h);
                                wend = b ? lo + (uint32_t)(__ffs(b) - 1) : end;
                                wend = min(wend, lim);
                            }
                            const uint32_t nb = wend > pos ? (wend - pos + 31) / 32 : 0;
                            uint32_t per = G.n_inner ? 1u : 4u;
                            uint32_t nctx = (nb + per - 1) / per;
                            if (nctx > 32) {
                                per = (nb + 31) / 32;
                                nctx = (nb + per - 1) / per;
                            }
                            const uint32_t extra = (g + 1 < g_end) ? 1u : 0u;
                            const uint32_t total = nctx + extra;
                            if (nb >= 2) {
                                uint32_t base = 0;
                                if (lane == 0) base = atomicAdd(p.lb + LB_TAIL, total);
                                base = __shfl_sync(kFull, base, 0);
                                const bool fits = base + total <= p.ctx_cap;
                                for (uint32_t j = 0; j < total && base + j < p.ctx_cap; j++) {
                                    const bool chunk = j < nctx;
                                    put_ctx<MAXV>(p.ctx + (size_t)(base + j) * kCtxWords, lane,
                                                  fits ? (node | ((chunk ? g : g + 1) << 16)) : kNone,
                                                  chunk ? pos + j * per * 32 : kNone,
                                                  chunk ? min(wend, pos + (j + 1) * per * 32) : kNone, tr_prev, h,
                                                  P, R, m2g);
                                }
                                publish_ctx(p.ctx, p.ctx_cap, base, total, p.epoch, p.lb + LB_WORK, lane);
                                if (fits) {
                                    if (STATS && lane == 0) st[ST_OFFLOADS]++;
                                    g = g_end;  // this node's remaining work now lives in the queue
                                    state = S_GROUP;
                                    continue;
                                }
                            }
                        }
                    }
                    // ---- load one batch of 32 window entries
                    const uint32_t idx = pos + lane;
                    bool fail;
                    const bool inner = G.n_inner != 0;
                    if (kind == ANCHOR_GLOBAL) {
                        fail = idx >= lim;
                        etr = kNone;
                        if (!fail) {
                            etr = __ldg(p.tr + idx); e1 = __ldg(p.src + idx); e2 = __ldg(p.dst + idx);
                            if (inner) ep = __ldg(p.eptr + idx);
                        }
                    } else {
                        const uint2 e = __ldg((kind == ANCHOR_OUT ? p.out_ent : p.in_ent) + idx);
                        etr = e.x; e1 = e.y;
                        if (inner) ep = __ldg((kind == ANCHOR_OUT ? p.out_ptr : p.in_ptr) + idx);
                        fail = etr > h || idx >= lim;
                    }
                    const unsigned fm = __ballot_sync(kFull, fail);
                    const unsigned inmask = fm ? ((1u << (__ffs(fm) - 1)) - 1u) : kFull;  // lanes before the window end
                    const bool w = ((inmask >> lane) & 1u) && etr > tr_prev;
                    const unsigned wm = __ballot_sync(kFull, w);
                    batch = pos;
                    pos = fm ? kNone : pos + 32;
                    ++nbatch;
                    if (STATS && lane == 0) {
                        st[ST_BATCHES]++;
                        st[ST_ENTRIES] += __popc(wm);
                        st[ST_BYTES] += (kind == ANCHOR_GLOBAL ? 12ull : 8ull) * (__popc(wm) + (fm ? 1 : 0)) +
                                        (inner ? 16ull * __popc(wm) : 0ull);
                    }
                    if (wm == 0) {
                        // forward skip from a lower-bound start: the whole batch precedes the window
                        const uint32_t last = __shfl_sync(kFull, etr, 31);
                        if (!fm && G.start >= START_R0 && G.start < START_SEARCH && nbatch >= 2 && last <= tr_prev) {
                            const uint32_t x = m2g_get<MAXV>(m2g, G.anchor);
                            const uint32_t *off = (kind == ANCHOR_OUT) ? p.out_off : p.in_off;
                            const uint32_t end = __ldg(off + x + 1) - 1;
                            pos = locate<STATS>(false, kind == ANCHOR_OUT ? p.out_ent : p.in_ent, p.tr, pos, end,
                                                tr_prev, lane, st[ST_PROBES]);
                            nbatch = 0;
                        }
                        continue;
                    }
                    uint32_t cls;
                    if (kind == ANCHOR_GLOBAL)
                        cls = (e1 != e2 && classify<MAXV>(m2g, nv, e1) == CLS_NEW &&
                               classify<MAXV>(m2g, nv, e2) == CLS_NEW) ? CLS_NEW : 0xFEu;
                    else
                        cls = classify<MAXV>(m2g, nv, e1);
                    bool any_inner = false;
                    for (uint32_t c = G.child_begin; c < G.child_end; ++c) {
                        const DNode dn = NODE(c);
                        unsigned mc = __ballot_sync(kFull, w && cls == dn.want);
                        if (dn.flags & NODE_COMPLETION) count(c, __popc(mc));
                        if ((dn.flags & NODE_SWEEP) && mc) {
                            // ---- leaf sweep: child c's subtree is one level of completions; each
                            // lane takes one candidate and scans its (short) windows itself
                            bool act = (mc >> lane) & 1u;
                            // windows of >= kSweepMax entries go to the warp path (descent)
                            for (uint32_t g2 = dn.group_begin; g2 < dn.group_end; ++g2) {
                                const DGroup G2 = GROUP(g2);
                                const uint32_t s0 = G2.start < START_R0 ? pick(ep, G2.start)
                                                                        : pick(R, G2.start - START_R0);
                                const uint2 *ent2 = G2.kind == ANCHOR_OUT ? p.out_ent : p.in_ent;
                                if (act && __ldg(&ent2[s0 + kSweepMax].x) <= h) act = false;
                            }
                            const unsigned fb = __ballot_sync(kFull, ((mc >> lane) & 1u) && !act);
                            if (fb != mc) {
                                const uint32_t xa = e1, xb = e2, tl = etr;  // the candidate edge
                                for (uint32_t g2 = dn.group_begin; g2 < dn.group_end; ++g2) {
                                    const DGroup G2 = GROUP(g2);
                                    uint32_t s0 = G2.start < START_R0 ? pick(ep, G2.start)
                                                                      : pick(R, G2.start - START_R0);
                                    const uint2 *ent2 = G2.kind == ANCHOR_OUT ? p.out_ent : p.in_ent;
                                    const uint32_t nch = G2.child_end - G2.child_begin;
                                    const uint32_t w0 = NODE(G2.child_begin).want;
                                    const uint32_t w1 = nch > 1 ? NODE(G2.child_begin + 1).want : 0xFDu;
                                    const uint32_t w2 = nch > 2 ? NODE(G2.child_begin + 2).want : 0xFDu;
                                    const uint32_t w3 = nch > 3 ? NODE(G2.child_begin + 3).want : 0xFDu;
                                    uint32_t n0 = 0, n1 = 0, n2 = 0, n3 = 0, ne = 0;
                                    bool go = act;
                                    while (__any_sync(kFull, go)) {
                                        if (go) {
                                            const uint2 e = __ldg(ent2 + s0);
                                            if (e.x > h) {
                                                go = false;
                                            } else {
                                                if (e.x > tl) {
                                                    const uint32_t cl =
                                                        (dn.n_new >= 1 && e.y == xa) ? nv
                                                        : (dn.n_new == 2 && e.y == xb) ? nv + 1
                                                        : classify<MAXV>(m2g, nv, e.y);
                                                    n0 += cl == w0;
                                                    n1 += cl == w1;
                                                    n2 += cl == w2;
                                                    n3 += cl == w3;
                                                    ++ne;
                                                }
                                                ++s0;
                                            }
                                        }
                                    }
                                    count(G2.child_begin, __reduce_add_sync(kFull, n0));
                                    if (nch > 1) count(G2.child_begin + 1, __reduce_add_sync(kFull, n1));
                                    if (nch > 2) count(G2.child_begin + 2, __reduce_add_sync(kFull, n2));
                                    if (nch > 3) count(G2.child_begin + 3, __reduce_add_sync(kFull, n3));
                                    if (STATS) {
                                        const uint32_t te = __reduce_add_sync(kFull, ne);
                                        const uint32_t tw = __popc(__ballot_sync(kFull, act));
                                        if (lane == 0) {
                                            st[ST_WINDOWS] += tw;
                                            st[ST_ENTRIES] += te;
                                            st[ST_BYTES] += 8ull * (te + tw);
                                        }
                                    }
                                }
                                if (STATS && lane == 0) st[ST_NODES] += __popc(mc & ~fb);
                            }
                            mc = fb;
                        }
                        if (dn.flags & NODE_INNER) {
                            if (lane == 0) MS[depth * kMaxGroupChildren + (c - G.child_begin)] = mc;
                            any_inner |= (mc != 0);
                        }
                    }
                    if (!any_inner) continue;  // next batch
                    __syncwarp();
                    ci = G.child_begin;
                    c_end = G.child_end;
                    mask = (NODE(ci).flags & NODE_INNER) ? MS[depth * kMaxGroupChildren] : 0u;
                    state = S_ITER;
                }
                // ---- S_ITER: next (inner child, candidate) pair of the current batch
                while (mask == 0) {
                    if (++ci >= c_end) break;
                    const uint32_t cb = GROUP(g).child_begin;
                    mask = (NODE(ci).flags & NODE_INNER) ? MS[depth * kMaxGroupChildren + (ci - cb)] : 0u;
                }
                if (mask == 0) {
                    state = S_BATCH;
                    continue;
                }
                const int b = __ffs(mask) - 1;
                mask &= mask - 1;
                const uint32_t ctr = __shfl_sync(kFull, etr, b);
                const uint32_t c1 = __shfl_sync(kFull, e1, b);
                const uint32_t c2 = __shfl_sync(kFull, e2, b);
                const uint4 cp = shfl4(ep, b);
                if (lane == 0) {
                    Frame f;
                    f.node_g = node | (g << 16); f.ci = ci; f.tr_prev = tr_prev; f.pos = pos;
                    f.batch = batch; f.mask = mask; f.lim = lim; f.g_end = g_end; f.P = P;
                    F[depth] = f;
                }
                const DNode dc = NODE(ci);
                if (dc.n_new >= 1) m2g_set<MAXV>(m2g, nv, c1);
                if (dc.n_new == 2) m2g_set<MAXV>(m2g, nv + 1, c2);
                nv = dc.nv;
                tr_prev = ctr;
                P = cp;
                node = ci;
                g = dc.group_begin;
                g_end = dc.group_end;
                lim = kNone;
                ++depth;
                state = S_GROUP;
                if (STATS && lane == 0) st[ST_NODES]++;
            }
        }
        if (lane == 0) atomicSub(p.lb + LB_WORK, 1u);
    }

    // ---- counters: lanes -> block (shared) -> global, once per block
    if (CNT > 0) {
#pragma unroll
        for (int s = 0; s < (CNT > 0 ? CNT : 1); s++) {
            const uint32_t c = lane + 32 * s;
            if (c < p.n_nodes && cnt[s]) atomicAdd(&s_cnt[c], cnt[s]);
        }
    }
    __syncthreads();
    for (uint32_t i = threadIdx.x; i < p.n_motifs; i += blockDim.x) {
        const unsigned long long v = s_cnt[p.motif_node[i]];
        if (v) atomicAdd(p.counts + i, v);
    }
    if (STATS && lane == 0) {
#pragma unroll
        for (int i = 0; i < ST_N; i++)
            if (st[i]) atomicAdd(p.stats + i, st[i]);
    }
}

#include "lane.cuh"
#include "bfs.cuh"
#include "wave.cuh"
#include "tile.cuh"

// a2: hi[r] = (last edge id e with t[e] <= t[r] + delta), by galloping from r (windows
// are short) then binary search.  Also zeroes the load-balancer words and the output
// counts of this call, so a co-mining query is exactly two launches.
__global__ void window_end_kernel(const int64_t *__restrict__ T, uint32_t E, int64_t delta, uint32_t r0,
                                  uint32_t n_roots, uint32_t *__restrict__ hi, uint32_t *lb, uint32_t n_lb,
                                  unsigned long long *counts, uint32_t n_counts) {
    const uint32_t tid = blockIdx.x * blockDim.x + threadIdx.x;
    if (tid < n_lb) lb[tid] = 0;
    if (tid < n_counts) counts[tid] = 0;
    for (uint32_t k = tid; k < n_roots; k += gridDim.x * blockDim.x) {
        const uint32_t r = r0 + k;
        const int64_t x = __ldg(T + r);
        const int64_t lim = (delta > INT64_MAX - x) ? INT64_MAX : x + delta;
        uint32_t a = r + 1, step = 1;  // invariant: T[a-1] <= lim
        uint32_t b = E;
        while (a < E) {
            const uint32_t probe = min(E - 1, a + step - 1);
            if (__ldg(T + probe) > lim) {
                b = probe;
                break;
            }
            a = probe + 1;
            step <<= 1;
        }
        while (a < b) {  // first index in [a, b) with T > lim
            const uint32_t m = a + ((b - a) >> 1);
            if (__ldg(T + m) > lim) b = m;
            else a = m + 1;
        }
        hi[r] = a - 1;
    }
}

struct DeviceTable {
    DNode *nodes;
    DGroup *groups;
    uint32_t *motif_node;
    lane::LNode *lnodes;
    uint32_t *gwant;
    uint32_t n_nodes, n_groups, n_motifs, max_vertices, max_edges, n_slots;
};

// per group: wants of its first 4 children packed in bytes (0xFD: no child), for the
// SIMD-compare child lookup of the tile kernels
std::vector<uint32_t> group_wants(const Table &t) {
    std::vector<uint32_t> out(t.groups.size());
    for (size_t gi = 0; gi < t.groups.size(); gi++) {
        uint32_t v = 0xFDFDFDFDu;
        const DGroup &G = t.groups[gi];
        for (uint32_t c = G.child_begin, k = 0; c < G.child_end && k < 4; c++, k++)
            v = (v & ~(0xFFu << (8 * k))) | ((uint32_t)t.nodes[c].want << (8 * k));
        out[gi] = v;
    }
    return out;
}

// Lane-kernel node rows: the DNode fields plus a completion-counter slot per node.
std::vector<lane::LNode> lane_nodes(const Table &t, uint32_t &n_slots) {
    std::vector<lane::LNode> out(t.nodes.size());
    n_slots = 0;
    for (size_t i = 0; i < t.nodes.size(); i++) {
        const DNode &a = t.nodes[i];
        lane::LNode &b = out[i];
        b.want = a.want; b.n_new = a.n_new; b.nv = a.nv; b.flags = a.flags;
        b.group_begin = a.group_begin; b.group_end = a.group_end;
        b.slot = (a.flags & NODE_COMPLETION) ? (uint16_t)n_slots++ : (uint16_t)0xFFFF;
        b.pad = 0;
        if (a.flags & NODE_INNER) {  // pre-leaf: every child is a leaf
            bool pre = true;
            for (uint32_t gi = a.group_begin; gi < a.group_end; gi++)
                for (uint32_t c = t.groups[gi].child_begin; c < t.groups[gi].child_end; c++)
                    pre = pre && !(t.nodes[c].flags & NODE_INNER);
            if (pre) b.flags |= bfs::NODE_PRELEAF;
        }
    }
    return out;
}

bool small_table(uint32_t n_nodes, uint32_t n_groups) { return n_nodes <= kSmallRows && n_groups <= kSmallRows; }

// dynamic shared memory: only large trees keep their counters, rows and groups there
size_t smem_bytes(uint32_t n_nodes, uint32_t n_groups) {
    if (small_table(n_nodes, n_groups)) return 0;
    return (size_t)n_nodes * sizeof(unsigned long long) + (size_t)n_nodes * sizeof(DNode) +
           (size_t)n_groups * sizeof(DGroup);
}

mayura_status cuda_fail(cudaError_t e, const char *what) {
    return fail(MAYURA_E_CUDA, std::string(what) + ": " + cudaGetErrorString(e));
}

#define CK(call, what)                                     \
    do {                                                   \
        cudaError_t e_ = (call);                           \
        if (e_ != cudaSuccess) return cuda_fail(e_, what); \
    } while (0)

template <int MAXV, int CNT, bool STATS>
cudaError_t launch_comine_t(const KParams &p, size_t smem, cudaStream_t s, int sms) {
    auto kern = comine_kernel<MAXV, CNT, STATS>;
    // occupancy is queried once per (kernel instance, shared-memory size, device)
    static std::mutex mu;
    static size_t cached_smem = 0;
    static int cached_dev = -1, cached_per_sm = 0;
    int dev = 0;
    cudaGetDevice(&dev);
    int per_sm = 0;
    {
        std::lock_guard<std::mutex> lk(mu);
        if (cached_smem == smem && cached_dev == dev) per_sm = cached_per_sm;
    }
    if (per_sm == 0) {
        cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        if (e != cudaSuccess) return e;
        e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, kBlock, smem);
        if (e != cudaSuccess) return e;
        if (per_sm < 1) per_sm = 1;
        std::lock_guard<std::mutex> lk(mu);
        cached_smem = smem;
        cached_dev = dev;
        cached_per_sm = per_sm;
    }
    uint32_t grid = (uint32_t)(sms * per_sm);
    const uint32_t need = (p.n_roots + 32 * kWarps - 1) / (32 * kWarps);
    if (need < grid) grid = need ? need : 1;
    kern<<<grid, kBlock, smem, s>>>(p);
    return cudaGetLastError();
}

template <int MAXV>
cudaError_t launch_comine_v(const KParams &p, bool stats, cudaStream_t s, int sms) {
    const size_t smem = smem_bytes(p.n_nodes, p.n_groups);
    const bool small = small_table(p.n_nodes, p.n_groups);
    if (small && p.n_nodes <= 32)
        return stats ? launch_comine_t<MAXV, 1, true>(p, smem, s, sms) : launch_comine_t<MAXV, 1, false>(p, smem, s, sms);
    if (small)
        return stats ? launch_comine_t<MAXV, 2, true>(p, smem, s, sms) : launch_comine_t<MAXV, 2, false>(p, smem, s, sms);
    return stats ? launch_comine_t<MAXV, 0, true>(p, smem, s, sms) : launch_comine_t<MAXV, 0, false>(p, smem, s, sms);
}

cudaError_t launch_comine(const KParams &p, uint32_t max_vertices, bool stats, cudaStream_t s, int sms) {
    if (max_vertices <= 4) return launch_comine_v<4>(p, stats, s, sms);
    if (max_vertices <= 6) return launch_comine_v<6>(p, stats, s, sms);
    if (max_vertices <= 8) return launch_comine_v<8>(p, stats, s, sms);
    return launch_comine_v<16>(p, stats, s, sms);
}

// ---- lane kernel (v3) launch: MAXV and counter mode by tree; grid = SMs x resident blocks
template <int MAXV, bool LANECNT, bool STATS>
cudaError_t launch_lane_t(const lane::LParams &p, size_t smem, cudaStream_t s, int sms) {
    auto kern = lane::comine_lane_kernel<MAXV, LANECNT, STATS>;
    static std::mutex mu;
    static size_t cached_smem = 0;
    static int cached_dev = -1, cached_per_sm = 0;
    int dev = 0;
    cudaGetDevice(&dev);
    int per_sm = 0;
    {
        std::lock_guard<std::mutex> lk(mu);
        if (cached_smem == smem && cached_dev == dev) per_sm = cached_per_sm;
    }
    if (per_sm == 0) {
        cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        if (e != cudaSuccess) return e;
        e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, lane::kLB, smem);
        if (e != cudaSuccess) return e;
        if (per_sm < 1) per_sm = 1;
        std::lock_guard<std::mutex> lk(mu);
        cached_smem = smem;
        cached_dev = dev;
        cached_per_sm = per_sm;
    }
    uint32_t grid = (uint32_t)(sms * per_sm);
    const uint32_t need = (p.n_roots + lane::kLB - 1) / lane::kLB;
    if (need < grid) grid = need ? need : 1;
    kern<<<grid, lane::kLB, smem, s>>>(p);
    return cudaGetLastError();
}

constexpr size_t kLaneCntSmem = 48 * 1024;  // lane-private counters while they fit this budget

template <int MAXV>
cudaError_t launch_lane_v(const lane::LParams &p, bool stats, cudaStream_t s, int sms) {
    const bool lanecnt = (size_t)p.n_slots * lane::kLB * 4 <= kLaneCntSmem;
    const size_t smem = lane::smem_total(p.n_nodes, p.n_groups, p.n_slots, p.n_frames, lanecnt, MAXV);
    if (lanecnt)
        return stats ? launch_lane_t<MAXV, true, true>(p, smem, s, sms) : launch_lane_t<MAXV, true, false>(p, smem, s, sms);
    return stats ? launch_lane_t<MAXV, false, true>(p, smem, s, sms) : launch_lane_t<MAXV, false, false>(p, smem, s, sms);
}

cudaError_t launch_lane(const lane::LParams &p, uint32_t max_vertices, bool stats, cudaStream_t s, int sms) {
    if (max_vertices <= 4) return launch_lane_v<4>(p, stats, s, sms);
    if (max_vertices <= 6) return launch_lane_v<6>(p, stats, s, sms);
    if (max_vertices <= 8) return launch_lane_v<8>(p, stats, s, sms);
    return launch_lane_v<16>(p, stats, s, sms);
}

// Kernel choice (MAYURA_KERNEL): "bfs" level-synchronous passes (v4, default), "lane" one
// search per lane (v3), "warp" one search per warp (v2).  All three return identical counts.
enum KernelKind { K_BFS = 0, K_LANE = 1, K_WARP = 2, K_WAVE = 3, K_TILE = 4, K_HYBRID = 5 };
KernelKind kernel_kind() {
    static int v = -1;
    if (v < 0) {
        const char *e = getenv("MAYURA_KERNEL");
        v = !e ? K_HYBRID : std::strcmp(e, "warp") == 0 ? K_WARP : std::strcmp(e, "lane") == 0 ? K_LANE
          : std::strcmp(e, "bfs") == 0 ? K_BFS : std::strcmp(e, "wave") == 0 ? K_WAVE
          : std::strcmp(e, "tile") == 0 ? K_TILE : K_HYBRID;
    }
    return (KernelKind)v;
}
// hybrid: BFS levels before the depth-first lane kernel (MAYURA_HYBRID_LEVELS, default 1)
uint32_t hybrid_levels() {
    static int v = -1;
    if (v < 0) {
        const char *e = getenv("MAYURA_HYBRID_LEVELS");
        v = e ? std::max(0, atoi(e)) : 1;
    }
    return (uint32_t)v;
}
bool use_warp_kernel() { return kernel_kind() == K_WARP; }

// ---- BFS passes (v4): per level an expand pass and a long-window pass
constexpr uint32_t kCtlWords = bfs::kStripes + 2;  // per level: stripe counters, long counter, pad

template <int MAXV, bool L0, bool STATS>
cudaError_t launch_bfs_pass(const bfs::BParams &p, bool long_pass, cudaStream_t s, int sms) {
    auto kern = long_pass ? bfs::long_kernel<MAXV, L0, STATS> : bfs::expand_kernel<MAXV, L0, STATS>;
    const size_t smem = bfs::smem_bytes(p.n_nodes, p.n_groups, p.n_slots, bfs::kTB);
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    int per_sm = 0;
    e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, bfs::kTB, smem);
    if (e != cudaSuccess) return e;
    uint32_t grid = (uint32_t)(sms * (per_sm > 0 ? per_sm : 1));
    if (L0 && !long_pass) {
        const uint32_t need = (p.n_roots + bfs::kTB - 1) / bfs::kTB;
        grid = std::max(1u, std::min(grid, need));
    }
    kern<<<grid, bfs::kTB, smem, s>>>(p);
    return cudaGetLastError();
}

template <int MAXV>
cudaError_t launch_bfs_v(bfs::BParams &p, uint32_t levels, uint32_t *bufs[2], uint32_t *ctl, uint32_t seg_cap,
                         bool stats, cudaStream_t s, int sms) {
    for (uint32_t L = 0; L < levels; L++) {
        p.in.data = L ? bufs[(L - 1) & 1] : nullptr;
        p.in.cnt = L ? ctl + (L - 1) * kCtlWords : nullptr;
        p.in.seg_cap = seg_cap;
        p.out.data = bufs[L & 1];
        p.out.cnt = ctl + L * kCtlWords;
        p.out.seg_cap = seg_cap;
        p.long_cnt = ctl + L * kCtlWords + bfs::kStripes;
        for (int lp = 0; lp < 2; lp++) {
            cudaError_t e;
            if (L == 0) e = stats ? launch_bfs_pass<MAXV, true, true>(p, lp, s, sms) : launch_bfs_pass<MAXV, true, false>(p, lp, s, sms);
            else e = stats ? launch_bfs_pass<MAXV, false, true>(p, lp, s, sms) : launch_bfs_pass<MAXV, false, false>(p, lp, s, sms);
            if (e != cudaSuccess) return e;
        }
    }
    return cudaSuccess;
}

cudaError_t launch_bfs(bfs::BParams &p, uint32_t max_vertices, uint32_t levels, uint32_t *bufs[2], uint32_t *ctl,
                       uint32_t seg_cap, bool stats, cudaStream_t s, int sms) {
    if (max_vertices <= 4) return launch_bfs_v<4>(p, levels, bufs, ctl, seg_cap, stats, s, sms);
    if (max_vertices <= 6) return launch_bfs_v<6>(p, levels, bufs, ctl, seg_cap, stats, s, sms);
    if (max_vertices <= 8) return launch_bfs_v<8>(p, levels, bufs, ctl, seg_cap, stats, s, sms);
    return launch_bfs_v<16>(p, levels, bufs, ctl, seg_cap, stats, s, sms);
}

// ---- waves of window tasks (v5)
constexpr uint32_t kWaveCtl = 3 * wave::kStripes;  // per wave: record, normal-task, long-task counters

template <typename K>
cudaError_t launch_wave_kernel(K kern, const wave::WParams &w, uint32_t items, cudaStream_t s, int sms) {
    const size_t smem = wave::smem_bytes(w.n_nodes, w.n_groups, w.n_slots);
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    int per_sm = 0;
    e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, wave::kTB, smem);
    if (e != cudaSuccess) return e;
    uint32_t grid = (uint32_t)(sms * (per_sm > 0 ? per_sm : 1));
    if (items) grid = std::max(1u, std::min(grid, (items + wave::kTB - 1) / wave::kTB));
    kern<<<grid, wave::kTB, smem, s>>>(w);
    return cudaGetLastError();
}

struct WaveBufs {
    uint32_t *pm[2], *norm[2], *lng[2], *ctl;
    uint32_t pm_seg_cap, norm_seg_cap, long_seg_cap;
};

template <int MAXV>
cudaError_t launch_wave_v(wave::WParams &w, uint32_t waves, const WaveBufs &b, bool stats, cudaStream_t s, int sms) {
    auto lists = [&](uint32_t k, wave::List &nl, wave::List &ll) {  // task lists written by wave k
        nl.data = b.norm[k & 1]; nl.cnt = b.ctl + k * kWaveCtl + wave::kStripes; nl.seg_cap = b.norm_seg_cap;
        ll.data = b.lng[k & 1]; ll.cnt = b.ctl + k * kWaveCtl + 2 * wave::kStripes; ll.seg_cap = b.long_seg_cap;
    };
    // wave 0: root windows
    w.in_pm = nullptr;
    w.in_tasks = wave::List{nullptr, nullptr, 0};
    w.out_pm = b.pm[0]; w.out_pm_cnt = b.ctl; w.pm_seg_cap = b.pm_seg_cap;
    lists(0, w.out_norm, w.out_long);
    cudaError_t e = stats ? launch_wave_kernel(wave::root_kernel<MAXV, true>, w, w.n_roots, s, sms)
                          : launch_wave_kernel(wave::root_kernel<MAXV, false>, w, w.n_roots, s, sms);
    if (e != cudaSuccess) return e;
    for (uint32_t k = 1; k <= waves; k++) {
        wave::List in_n, in_l;
        lists(k - 1, in_n, in_l);
        w.in_pm = k >= 2 ? b.pm[(k - 2) & 1] : nullptr;     // records written by wave k-1
        w.out_pm = b.pm[(k - 1) & 1];
        w.out_pm_cnt = b.ctl + k * kWaveCtl;
        lists(k, w.out_norm, w.out_long);
        for (int lp = 0; lp < 2; lp++) {
            w.in_tasks = lp ? in_l : in_n;
            if (k == 1) {
                if (lp) e = stats ? launch_wave_kernel(wave::scan_kernel<MAXV, 32, true, true>, w, 0, s, sms)
                                  : launch_wave_kernel(wave::scan_kernel<MAXV, 32, true, false>, w, 0, s, sms);
                else e = stats ? launch_wave_kernel(wave::scan_kernel<MAXV, wave::kSub, true, true>, w, 0, s, sms)
                               : launch_wave_kernel(wave::scan_kernel<MAXV, wave::kSub, true, false>, w, 0, s, sms);
            } else {
                if (lp) e = stats ? launch_wave_kernel(wave::scan_kernel<MAXV, 32, false, true>, w, 0, s, sms)
                                  : launch_wave_kernel(wave::scan_kernel<MAXV, 32, false, false>, w, 0, s, sms);
                else e = stats ? launch_wave_kernel(wave::scan_kernel<MAXV, wave::kSub, false, true>, w, 0, s, sms)
                               : launch_wave_kernel(wave::scan_kernel<MAXV, wave::kSub, false, false>, w, 0, s, sms);
            }
            if (e != cudaSuccess) return e;
        }
    }
    return cudaSuccess;
}

cudaError_t launch_wave(wave::WParams &w, uint32_t max_vertices, uint32_t waves, const WaveBufs &b, bool stats,
                        cudaStream_t s, int sms) {
    if (max_vertices <= 4) return launch_wave_v<4>(w, waves, b, stats, s, sms);
    if (max_vertices <= 6) return launch_wave_v<6>(w, waves, b, stats, s, sms);
    if (max_vertices <= 8) return launch_wave_v<8>(w, waves, b, stats, s, sms);
    return launch_wave_v<16>(w, waves, b, stats, s, sms);
}

// Record / task / control buffers of the waves, allocated once per graph, grown on demand.
// Capacities: records 8 per edge, normal tasks 12 per edge, long tasks 2 per edge
// (each >= 2^20 and <= 2^26 items per buffer); overflow is handled in place (exact).
mayura_status ensure_wave_buffers(mayura_graph_s *g, uint32_t words) {
    auto segs = [&](uint64_t per_edge) {
        return (uint32_t)((std::min<uint64_t>(std::max<uint64_t>(per_edge * g->E, 1u << 20), 1u << 26) +
                           wave::kStripes - 1) / wave::kStripes);
    };
    uint32_t pm_seg = segs(8), n_seg = segs(12), l_seg = segs(2);
    if (const char *e = getenv("MAYURA_BFS_SEG_CAP")) pm_seg = n_seg = l_seg = (uint32_t)std::max(1L, atol(e));
    const size_t pm_bytes = (size_t)pm_seg * wave::kStripes * words * 4;
    const size_t n_bytes = (size_t)n_seg * wave::kStripes * wave::kTaskWords * 4;
    const size_t l_bytes = (size_t)l_seg * wave::kStripes * wave::kTaskWords * 4;
    const size_t total = 2 * (pm_bytes + n_bytes + l_bytes) + sizeof(uint32_t) * (kWaveCtl * (bfs::kMaxLevels + 1) + 16);
    if (g->wave_bytes < total) {
        if (g->d_wave) cudaFree(g->d_wave);
        g->d_wave = nullptr;
        g->device_bytes -= g->wave_bytes;
        g->wave_bytes = 0;
        CK(cudaMalloc(&g->d_wave, total), "cudaMalloc(wave buffers)");
        g->wave_bytes = total;
        g->device_bytes += total;
    }
    g->wave_pm_seg = pm_seg; g->wave_n_seg = n_seg; g->wave_l_seg = l_seg;
    g->wave_pm_bytes = pm_bytes; g->wave_n_bytes = n_bytes; g->wave_l_bytes = l_bytes;
    return MAYURA_OK;
}

// ---- waves of window tiles (v6)
template <typename K>
cudaError_t launch_tile_kernel(K kern, const tile::TParams &w, uint32_t items, cudaStream_t s, int sms) {
    const size_t smem = tile::smem_bytes(w.n_nodes, w.n_groups, w.n_slots);
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    int per_sm = 0;
    e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, tile::kTB, smem);
    if (e != cudaSuccess) return e;
    uint32_t grid = (uint32_t)(sms * (per_sm > 0 ? per_sm : 1));
    if (items) grid = std::max(1u, std::min(grid, (items + tile::kTB - 1) / tile::kTB));
    kern<<<grid, tile::kTB, smem, s>>>(w);
    return cudaGetLastError();
}

struct TileBufs {
    uint32_t *norm[2], *lng, *ctl;   // ctl: per wave k, [normal-task counters | long-task counters]
    uint32_t norm_seg_cap, long_seg_cap;
};

template <int MAXV>
cudaError_t launch_tile_v(tile::TParams &w, uint32_t waves, const TileBufs &b, bool stats, cudaStream_t s, int sms) {
    auto nlist = [&](uint32_t k) {  // tasks of wave k
        return wave::List{b.norm[k & 1], b.ctl + k * 2 * wave::kStripes, b.norm_seg_cap};
    };
    auto llist = [&](uint32_t k) {
        return wave::List{b.lng, b.ctl + k * 2 * wave::kStripes + wave::kStripes, b.long_seg_cap};
    };
    cudaError_t e;
    for (uint32_t k = 0; k < waves; k++) {
        w.out_norm = nlist(k + 1);
        w.out_long = llist(k);
        if (k == 0) {
            w.in_tasks = wave::List{nullptr, nullptr, 0};
            e = stats ? launch_tile_kernel(tile::root_kernel<MAXV, true>, w, w.n_roots, s, sms)
                      : launch_tile_kernel(tile::root_kernel<MAXV, false>, w, w.n_roots, s, sms);
        } else {
            w.in_tasks = nlist(k);
            e = stats ? launch_tile_kernel(tile::tile_kernel<MAXV, true>, w, 0, s, sms)
                      : launch_tile_kernel(tile::tile_kernel<MAXV, false>, w, 0, s, sms);
        }
        if (e != cudaSuccess) return e;
        w.in_tasks = llist(k);
        e = stats ? launch_tile_kernel(tile::long_kernel<MAXV, true>, w, 0, s, sms)
                  : launch_tile_kernel(tile::long_kernel<MAXV, false>, w, 0, s, sms);
        if (e != cudaSuccess) return e;
    }
    return cudaSuccess;
}

cudaError_t launch_tile(tile::TParams &w, uint32_t max_vertices, uint32_t waves, const TileBufs &b, bool stats,
                        cudaStream_t s, int sms) {
    if (max_vertices <= 4) return launch_tile_v<4>(w, waves, b, stats, s, sms);
    if (max_vertices <= 6) return launch_tile_v<6>(w, waves, b, stats, s, sms);
    if (max_vertices <= 8) return launch_tile_v<8>(w, waves, b, stats, s, sms);
    return launch_tile_v<16>(w, waves, b, stats, s, sms);
}

uint32_t task_words(uint32_t max_vertices) {
    const uint32_t mv = max_vertices <= 4 ? 4 : max_vertices <= 6 ? 6 : max_vertices <= 8 ? 8 : 16;
    return (5 + mv + 3) & ~3u;
}

// Task lists of the tile waves, allocated once per graph and grown on demand: normal tasks
// 8 per edge (x2, ping-pong), long tasks 2 per edge (each >= 2^20, <= 2^26 tasks);
// overflow is mined in place (exact).
mayura_status ensure_tile_buffers(mayura_graph_s *g, uint32_t words) {
    auto segs = [&](uint64_t per_edge) {
        return (uint32_t)((std::min<uint64_t>(std::max<uint64_t>(per_edge * g->E, 1u << 20), 1u << 26) +
                           wave::kStripes - 1) / wave::kStripes);
    };
    uint32_t n_seg = segs(8), l_seg = segs(2);
    if (const char *e = getenv("MAYURA_BFS_SEG_CAP")) n_seg = l_seg = (uint32_t)std::max(1L, atol(e));
    const size_t n_bytes = (size_t)n_seg * wave::kStripes * words * 4;
    const size_t l_bytes = (size_t)l_seg * wave::kStripes * words * 4;
    const size_t ctl = sizeof(uint32_t) * (2 * wave::kStripes * (bfs::kMaxLevels + 1) + 16);
    const size_t total = 2 * n_bytes + l_bytes + ctl;
    if (g->tile_bytes < total) {
        if (g->d_tile) cudaFree(g->d_tile);
        g->d_tile = nullptr;
        g->device_bytes -= g->tile_bytes;
        g->tile_bytes = 0;
        CK(cudaMalloc(&g->d_tile, total), "cudaMalloc(tile buffers)");
        g->tile_bytes = total;
        g->device_bytes += total;
    }
    g->tile_n_seg = n_seg; g->tile_l_seg = l_seg; g->tile_n_bytes = n_bytes; g->tile_l_bytes = l_bytes;
    return MAYURA_OK;
}

uint32_t rec_words(uint32_t max_vertices) {
    const uint32_t mv = max_vertices <= 4 ? 4 : max_vertices <= 6 ? 6 : max_vertices <= 8 ? 8 : 16;
    return (8 + mv + 3) & ~3u;
}

// Frontier / long-item / control buffers of the BFS passes, allocated once per graph and
// grown on demand.  Capacity: 4 records per edge (>= 2^20, <= 2^26) per buffer.
mayura_status ensure_bfs_buffers(mayura_graph_s *g, uint32_t words) {
    const uint64_t recs = std::min<uint64_t>(std::max<uint64_t>(8 * g->E, 1u << 20), 1u << 26);
    uint32_t seg_cap = (uint32_t)((recs + bfs::kStripes - 1) / bfs::kStripes);
    // test hook: tiny capacities force the depth-first fallback / in-place long windows
    if (const char *e = getenv("MAYURA_BFS_SEG_CAP")) seg_cap = (uint32_t)std::max(1L, atol(e));
    const size_t bytes = (size_t)seg_cap * bfs::kStripes * words * 4;
    if (g->bfs_bytes < bytes) {
        for (int i = 0; i < 2; i++)
            if (g->d_bfs[i]) cudaFree(g->d_bfs[i]), g->d_bfs[i] = nullptr;
        g->device_bytes -= 2 * g->bfs_bytes;
        g->bfs_bytes = 0;
        for (int i = 0; i < 2; i++) CK(cudaMalloc(&g->d_bfs[i], bytes), "cudaMalloc(frontier)");
        g->bfs_bytes = bytes;
        g->device_bytes += 2 * bytes;
    }
    g->bfs_seg_cap = std::min(seg_cap, (uint32_t)(g->bfs_bytes / ((size_t)bfs::kStripes * words * 4)));
    if (!g->d_bfs_ctl) {
        CK(cudaMalloc(&g->d_bfs_ctl, sizeof(uint32_t) * (kCtlWords * bfs::kMaxLevels + 16)), "cudaMalloc(bfs ctl)");
        g->bfs_long_cap = (uint32_t)std::min<uint64_t>(std::max<uint64_t>(g->E / 2, 1u << 20), 1u << 26);
        if (const char *e = getenv("MAYURA_BFS_LONG_CAP")) g->bfs_long_cap = (uint32_t)std::max(1L, atol(e));
        CK(cudaMalloc(&g->d_bfs_long, sizeof(uint32_t) * 3 * (size_t)g->bfs_long_cap), "cudaMalloc(long items)");
        g->device_bytes += sizeof(uint32_t) * 3 * (size_t)g->bfs_long_cap;
    }
    return MAYURA_OK;
}

void table_view(const Table &t, uint32_t n_motifs, char *buf, DeviceTable &d) {
    const size_t bn = t.nodes.size() * sizeof(DNode), bg = t.groups.size() * sizeof(DGroup),
                 bm = lane::align16(t.motif_node.size() * sizeof(uint32_t));
    d.nodes = reinterpret_cast<DNode *>(buf);
    d.groups = reinterpret_cast<DGroup *>(buf + bn);
    d.motif_node = reinterpret_cast<uint32_t *>(buf + bn + bg);
    d.lnodes = reinterpret_cast<lane::LNode *>(buf + bn + bg + bm);
    d.gwant = reinterpret_cast<uint32_t *>(buf + bn + bg + bm + lane::align16(t.nodes.size() * sizeof(lane::LNode)));
    d.n_nodes = (uint32_t)t.nodes.size();
    d.n_groups = (uint32_t)t.groups.size();
    d.n_motifs = n_motifs;
    d.max_vertices = t.max_vertices;
    d.max_edges = t.max_edges;
    d.n_slots = 0;
    for (const DNode &x : t.nodes) d.n_slots += (x.flags & NODE_COMPLETION) ? 1 : 0;
}

mayura_status upload_table(const Table &t, uint32_t n_motifs, DeviceTable &d, void *&owner) {
    const size_t bn = t.nodes.size() * sizeof(DNode), bg = t.groups.size() * sizeof(DGroup),
                 bm = t.motif_node.size() * sizeof(uint32_t), bm16 = lane::align16(bm);
    uint32_t n_slots = 0;
    const std::vector<lane::LNode> ln = lane_nodes(t, n_slots);
    const size_t bl = lane::align16(ln.size() * sizeof(lane::LNode));
    const std::vector<uint32_t> gw = group_wants(t);
    char *buf = nullptr;
    CK(cudaMalloc(&buf, bn + bg + bm16 + bl + gw.size() * 4 + 16), "cudaMalloc(mgtree table)");
    owner = buf;
    CK(cudaMemcpy(buf, t.nodes.data(), bn, cudaMemcpyHostToDevice), "cudaMemcpy(table)");
    if (bg) CK(cudaMemcpy(buf + bn, t.groups.data(), bg, cudaMemcpyHostToDevice), "cudaMemcpy(table)");
    CK(cudaMemcpy(buf + bn + bg, t.motif_node.data(), bm, cudaMemcpyHostToDevice), "cudaMemcpy(table)");
    CK(cudaMemcpy(buf + bn + bg + bm16, ln.data(), ln.size() * sizeof(lane::LNode), cudaMemcpyHostToDevice),
       "cudaMemcpy(table)");
    if (!gw.empty())
        CK(cudaMemcpy(buf + bn + bg + bm16 + bl, gw.data(), gw.size() * 4, cudaMemcpyHostToDevice), "cudaMemcpy(table)");
    table_view(t, n_motifs, buf, d);
    return MAYURA_OK;
}

void free_tables(mayura_mgtree_s *m) {
    if (m->dev >= 0) {
        int prev = 0;
        cudaGetDevice(&prev);
        cudaSetDevice(m->dev);
        for (void *p : m->d_tables)
            if (p) cudaFree(p);
        cudaSetDevice(prev);
    }
    m->d_tables.clear();
    m->dev = -1;
}

// Device copies of the group table ([0]) and the single-motif tables ([1..k]), uploaded once
// per (tree, device) and cached in the tree handle.
mayura_status ensure_tables(mayura_mgtree_s *m, int dev, std::vector<DeviceTable> &out) {
    if (m->dev != dev) free_tables(m);
    out.resize(1 + m->single.size());
    if (m->dev == dev && m->d_tables.size() == out.size()) {
        for (size_t i = 0; i < out.size(); i++)
            table_view(i == 0 ? m->group : m->single[i - 1], i == 0 ? m->n_motifs : 1, (char *)m->d_tables[i], out[i]);
        return MAYURA_OK;
    }
    std::vector<void *> owners(out.size(), nullptr);
    for (size_t i = 0; i < out.size(); i++) {
        const Table &t = i == 0 ? m->group : m->single[i - 1];
        mayura_status s = upload_table(t, i == 0 ? m->n_motifs : 1, out[i], owners[i]);
        if (s != MAYURA_OK) {
            for (void *p : owners)
                if (p) cudaFree(p);
            return s;
        }
    }
    m->d_tables = owners;
    m->dev = dev;
    return MAYURA_OK;
}

struct DeviceGuard {
    int prev = -1;
    explicit DeviceGuard(int dev) {
        cudaGetDevice(&prev);
        if (prev != dev) cudaSetDevice(dev);
    }
    ~DeviceGuard() {
        int cur = -1;
        cudaGetDevice(&cur);
        if (prev >= 0 && cur != prev) cudaSetDevice(prev);
    }
};

int sm_count(int dev) {
    int n = 0;
    cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
    return n > 0 ? n : 1;
}

// mode 0: co-mine, 1: independent (one launch per motif); stats: instrumented kernel.
mayura_status run(mayura_graph_s *g, mayura_mgtree_s *m, uint64_t rb, uint64_t re, void *stream,
                  uint64_t *counts_out, int on_device, int mode, unsigned long long *stats_host,
                  void *mid_event = nullptr) {
    if (!g || !m) return fail(MAYURA_E_INVALID, "mayura_comine: NULL handle");
    if (g->device < 0) return fail(MAYURA_E_STATE, "mayura_comine: graph is host-only (device = -1)");
    if (rb > re || re > g->E) return fail(MAYURA_E_INVALID, "mayura_comine: bad root range");
    if (!counts_out && !stats_host) return fail(MAYURA_E_INVALID, "mayura_comine: counts_out is NULL");
    DeviceGuard guard(g->device);
    cudaStream_t s = (cudaStream_t)stream;
    std::vector<DeviceTable> tabs;
    mayura_status st = ensure_tables(m, g->device, tabs);
    if (st != MAYURA_OK) return st;
    const uint32_t k = m->n_motifs;
    unsigned long long *d_counts = reinterpret_cast<unsigned long long *>(counts_out);
    if (!on_device || stats_host) {
        if (g->d_counts_cap < k) {
            if (g->d_counts) cudaFree(g->d_counts);
            g->d_counts = nullptr;
            g->d_counts_cap = 0;
            CK(cudaMalloc(&g->d_counts, sizeof(unsigned long long) * k), "cudaMalloc(counts)");
            g->d_counts_cap = k;
        }
        d_counts = g->d_counts;
    }
    if (!g->d_ctx) {
        CK(cudaMalloc(&g->d_ctx, sizeof(uint32_t) * kCtxWords * (size_t)kCtxCap), "cudaMalloc(contexts)");
        CK(cudaMemset(g->d_ctx, 0, sizeof(uint32_t) * kCtxWords * (size_t)kCtxCap), "cudaMemset(contexts)");
        g->ctx_cap = kCtxCap;
        g->device_bytes += sizeof(uint32_t) * kCtxWords * (size_t)kCtxCap;
    }
    if (stats_host && !g->d_stats) CK(cudaMalloc(&g->d_stats, sizeof(unsigned long long) * ST_N), "cudaMalloc(stats)");
    // MAYURA_DEBUG_WARPS=<file>: the instrumented lane kernel writes one timeline record per warp
    // (start ns, end ns, iterations, warp-help batches, roots taken, root-queue-empty ns, SM id)
    const char *dbg_path = stats_host ? getenv("MAYURA_DEBUG_WARPS") : nullptr;
    const size_t kDbgWarps = 1u << 16;
    if (dbg_path && !g->d_dbg) CK(cudaMalloc(&g->d_dbg, sizeof(unsigned long long) * 8 * kDbgWarps), "cudaMalloc(dbg)");
    if (dbg_path) CK(cudaMemsetAsync(g->d_dbg, 0, sizeof(unsigned long long) * 8 * kDbgWarps, s), "cudaMemsetAsync(dbg)");
    if (!dbg_path && stats_host && g->d_dbg) {
        cudaFree(g->d_dbg);
        g->d_dbg = nullptr;
    }
    if (stats_host) CK(cudaMemsetAsync(g->d_stats, 0, sizeof(unsigned long long) * ST_N, s), "cudaMemsetAsync(stats)");
    const uint32_t n_roots = (uint32_t)(re - rb);
    const size_t n_launch = mode == 1 ? k : 1;
    const uint32_t n_lb = (uint32_t)(LB_N * n_launch);
    {
        const int threads = 256;
        uint32_t blocks = (n_roots + threads - 1) / threads;
        const uint32_t minb = (std::max(n_lb, k) + threads - 1) / threads;
        blocks = std::max(blocks, minb);
        blocks = std::min<uint32_t>(blocks, 148u * 32u);
        if (blocks == 0) blocks = 1;
        window_end_kernel<<<blocks, threads, 0, s>>>(g->d_t, (uint32_t)g->E, m->delta, (uint32_t)rb, n_roots,
                                                     g->d_hi, g->d_queue, n_lb, d_counts, k);
        CK(cudaGetLastError(), "window_end_kernel launch");
    }
    if (mid_event) CK(cudaEventRecord((cudaEvent_t)mid_event, s), "cudaEventRecord(mid_event)");
    const int sms = sm_count(g->device);
    if (n_roots > 0) {
        for (size_t i = 0; i < n_launch; i++) {
            const DeviceTable &dt = mode == 1 ? tabs[1 + i] : tabs[0];
            KParams p;
            p.src = g->d_src; p.dst = g->d_dst; p.tr = g->d_tr; p.hi = g->d_hi;
            p.eptr = reinterpret_cast<const uint4 *>(g->d_eptr);
            p.out_off = g->d_out_off; p.in_off = g->d_in_off;
            p.out_ent = reinterpret_cast<const uint2 *>(g->d_out_ent);
            p.in_ent = reinterpret_cast<const uint2 *>(g->d_in_ent);
            p.out_ptr = reinterpret_cast<const uint4 *>(g->d_out_ptr);
            p.in_ptr = reinterpret_cast<const uint4 *>(g->d_in_ptr);
            p.nodes = dt.nodes; p.groups = dt.groups; p.motif_node = dt.motif_node;
            p.n_nodes = dt.n_nodes; p.n_groups = dt.n_groups; p.n_motifs = dt.n_motifs;
            std::memset(p.tn, 0, sizeof(p.tn));
            std::memset(p.tg, 0, sizeof(p.tg));
            if (small_table(dt.n_nodes, dt.n_groups)) {
                const Table &ht = mode == 1 ? m->single[i] : m->group;
                std::memcpy(p.tn, ht.nodes.data(), sizeof(DNode) * ht.nodes.size());
                std::memcpy(p.tg, ht.groups.data(), sizeof(DGroup) * ht.groups.size());
            }
            p.r0 = (uint32_t)rb; p.n_roots = n_roots;
            p.lb = g->d_queue + LB_N * i;
            p.ctx = g->d_ctx;
            p.ctx_cap = g->ctx_cap;
            p.epoch = ++g->epoch;
            if (p.epoch == 0) p.epoch = ++g->epoch;  // 0 marks a never-written slot
            p.counts = d_counts + (mode == 1 ? i : 0);
            p.stats = g->d_stats;
            if (kernel_kind() == K_TILE) {
                const uint32_t words = task_words(dt.max_vertices);
                mayura_status ts = ensure_tile_buffers(g, words);
                if (ts != MAYURA_OK) return ts;
                char *base = reinterpret_cast<char *>(g->d_tile);
                TileBufs tb;
                tb.norm[0] = reinterpret_cast<uint32_t *>(base);
                tb.norm[1] = reinterpret_cast<uint32_t *>(base + g->tile_n_bytes);
                tb.lng = reinterpret_cast<uint32_t *>(base + 2 * g->tile_n_bytes);
                tb.ctl = reinterpret_cast<uint32_t *>(base + 2 * g->tile_n_bytes + g->tile_l_bytes);
                tb.norm_seg_cap = g->tile_n_seg; tb.long_seg_cap = g->tile_l_seg;
                const size_t ctl_bytes = sizeof(uint32_t) * (2 * wave::kStripes * (bfs::kMaxLevels + 1) + 16);
                CK(cudaMemsetAsync(tb.ctl, 0, ctl_bytes, s), "cudaMemsetAsync(tile ctl)");
                tile::TParams w;
                w.src = p.src; w.dst = p.dst; w.tr = p.tr; w.hi = p.hi; w.eptr = p.eptr;
                w.out_off = p.out_off; w.in_off = p.in_off; w.out_ent = p.out_ent; w.in_ent = p.in_ent;
                w.out_ptr = p.out_ptr; w.in_ptr = p.in_ptr;
                w.nodes = dt.lnodes; w.groups = dt.groups; w.gwant = dt.gwant; w.motif_node = dt.motif_node;
                w.n_nodes = dt.n_nodes; w.n_groups = dt.n_groups; w.n_motifs = dt.n_motifs; w.n_slots = dt.n_slots;
                w.r0 = p.r0; w.n_roots = p.n_roots;
                w.fallback = tb.ctl + 2 * wave::kStripes * (bfs::kMaxLevels + 1);
                w.counts = p.counts; w.stats = p.stats;
                const uint32_t waves = dt.max_edges > 1 ? dt.max_edges - 1 : 0;
                if (waves == 0) {  // one-edge motifs only: the root kernel still counts roots
                    w.in_tasks = wave::List{nullptr, nullptr, 0};
                    w.out_norm = wave::List{tb.norm[1], tb.ctl, tb.norm_seg_cap};
                    w.out_long = wave::List{tb.lng, tb.ctl + wave::kStripes, tb.long_seg_cap};
                    if (dt.max_vertices <= 4)
                        CK(stats_host ? launch_tile_kernel(tile::root_kernel<4, true>, w, w.n_roots, s, sms)
                                      : launch_tile_kernel(tile::root_kernel<4, false>, w, w.n_roots, s, sms),
                           "tile root launch");
                } else {
                    CK(launch_tile(w, dt.max_vertices, waves, tb, stats_host != nullptr, s, sms), "tile launch");
                }
            } else if (kernel_kind() == K_WAVE) {
                const uint32_t words = rec_words(dt.max_vertices);
                mayura_status ws = ensure_wave_buffers(g, words);
                if (ws != MAYURA_OK) return ws;
                char *base = reinterpret_cast<char *>(g->d_wave);
                WaveBufs wb;
                wb.pm[0] = reinterpret_cast<uint32_t *>(base);
                wb.pm[1] = reinterpret_cast<uint32_t *>(base + g->wave_pm_bytes);
                base += 2 * g->wave_pm_bytes;
                wb.norm[0] = reinterpret_cast<uint32_t *>(base);
                wb.norm[1] = reinterpret_cast<uint32_t *>(base + g->wave_n_bytes);
                base += 2 * g->wave_n_bytes;
                wb.lng[0] = reinterpret_cast<uint32_t *>(base);
                wb.lng[1] = reinterpret_cast<uint32_t *>(base + g->wave_l_bytes);
                base += 2 * g->wave_l_bytes;
                wb.ctl = reinterpret_cast<uint32_t *>(base);
                wb.pm_seg_cap = g->wave_pm_seg; wb.norm_seg_cap = g->wave_n_seg; wb.long_seg_cap = g->wave_l_seg;
                const size_t ctl_bytes = sizeof(uint32_t) * (kWaveCtl * (bfs::kMaxLevels + 1) + 16);
                CK(cudaMemsetAsync(wb.ctl, 0, ctl_bytes, s), "cudaMemsetAsync(wave ctl)");
                wave::WParams w;
                w.src = p.src; w.dst = p.dst; w.tr = p.tr; w.hi = p.hi; w.eptr = p.eptr;
                w.out_off = p.out_off; w.in_off = p.in_off; w.out_ent = p.out_ent; w.in_ent = p.in_ent;
                w.out_ptr = p.out_ptr; w.in_ptr = p.in_ptr;
                w.nodes = dt.lnodes; w.groups = dt.groups; w.motif_node = dt.motif_node;
                w.n_nodes = dt.n_nodes; w.n_groups = dt.n_groups; w.n_motifs = dt.n_motifs; w.n_slots = dt.n_slots;
                w.r0 = p.r0; w.n_roots = p.n_roots;
                w.fallback = wb.ctl + kWaveCtl * (bfs::kMaxLevels + 1);
                w.counts = p.counts; w.stats = p.stats;
                const uint32_t waves = dt.max_edges > 1 ? dt.max_edges - 1 : 0;
                CK(launch_wave(w, dt.max_vertices, waves, wb, stats_host != nullptr, s, sms), "wave launch");
            } else if (kernel_kind() == K_HYBRID) {
                // BFS over the first levels (splits heavy roots into many partial matches),
                // then one depth-first search per partial match in the lane kernel
                const uint32_t words = rec_words(dt.max_vertices);
                uint32_t levels = std::min(hybrid_levels(), dt.max_edges > 2 ? dt.max_edges - 2 : 0u);
                lane::LParams q;
                q.src = p.src; q.dst = p.dst; q.tr = p.tr; q.hi = p.hi; q.eptr = p.eptr;
                q.out_off = p.out_off; q.in_off = p.in_off; q.out_ent = p.out_ent; q.in_ent = p.in_ent;
                q.out_ptr = p.out_ptr; q.in_ptr = p.in_ptr;
                q.nodes = dt.lnodes; q.groups = dt.groups; q.motif_node = dt.motif_node;
                q.n_nodes = dt.n_nodes; q.n_groups = dt.n_groups; q.n_motifs = dt.n_motifs; q.n_slots = dt.n_slots;
                q.n_frames = dt.max_edges > 2 ? dt.max_edges - 2 : 0;
                q.r0 = p.r0; q.n_roots = p.n_roots; q.lb = p.lb; q.counts = p.counts; q.stats = p.stats;
                q.dbg = stats_host ? g->d_dbg : nullptr;
                q.pm = nullptr; q.pm_cnt = nullptr; q.pm_seg_cap = 0; q.pm_words = words;
                if (levels > 0) {
                    mayura_status bs = ensure_bfs_buffers(g, words);
                    if (bs != MAYURA_OK) return bs;
                    uint32_t *ctl = g->d_bfs_ctl;
                    CK(cudaMemsetAsync(ctl, 0, sizeof(uint32_t) * (kCtlWords * bfs::kMaxLevels + 16), s),
                       "cudaMemsetAsync(ctl)");
                    bfs::BParams b;
                    b.src = p.src; b.dst = p.dst; b.tr = p.tr; b.hi = p.hi; b.eptr = p.eptr;
                    b.out_off = p.out_off; b.in_off = p.in_off; b.out_ent = p.out_ent; b.in_ent = p.in_ent;
                    b.out_ptr = p.out_ptr; b.in_ptr = p.in_ptr;
                    b.nodes = dt.lnodes; b.groups = dt.groups; b.motif_node = dt.motif_node;
                    b.n_nodes = dt.n_nodes; b.n_groups = dt.n_groups; b.n_motifs = dt.n_motifs;
                    b.n_slots = dt.n_slots;
                    b.r0 = p.r0; b.n_roots = p.n_roots;
                    b.long_items = g->d_bfs_long; b.long_cap = g->bfs_long_cap;
                    b.fallback = ctl + kCtlWords * bfs::kMaxLevels;
                    b.inline_preleaf = 0;
                    b.counts = p.counts; b.stats = p.stats;
                    uint32_t *bufs[2] = {g->d_bfs[0], g->d_bfs[1]};
                    CK(launch_bfs(b, dt.max_vertices, levels, bufs, ctl, g->bfs_seg_cap, stats_host != nullptr, s,
                                  sms), "bfs pass launch");
                    q.pm = bufs[(levels - 1) & 1];
                    q.pm_cnt = ctl + (levels - 1) * kCtlWords;
                    q.pm_seg_cap = g->bfs_seg_cap;
                }
                CK(launch_lane(q, dt.max_vertices, stats_host != nullptr, s, sms), "comine_lane_kernel launch");
            } else if (kernel_kind() == K_BFS) {
                const uint32_t words = rec_words(dt.max_vertices);
                mayura_status bs = ensure_bfs_buffers(g, words);
                if (bs != MAYURA_OK) return bs;
                uint32_t *ctl = g->d_bfs_ctl;
                CK(cudaMemsetAsync(ctl, 0, sizeof(uint32_t) * (kCtlWords * bfs::kMaxLevels + 16), s), "cudaMemsetAsync(ctl)");
                bfs::BParams b;
                b.src = p.src; b.dst = p.dst; b.tr = p.tr; b.hi = p.hi; b.eptr = p.eptr;
                b.out_off = p.out_off; b.in_off = p.in_off; b.out_ent = p.out_ent; b.in_ent = p.in_ent;
                b.out_ptr = p.out_ptr; b.in_ptr = p.in_ptr;
                b.nodes = dt.lnodes; b.groups = dt.groups; b.motif_node = dt.motif_node;
                b.n_nodes = dt.n_nodes; b.n_groups = dt.n_groups; b.n_motifs = dt.n_motifs; b.n_slots = dt.n_slots;
                b.r0 = p.r0; b.n_roots = p.n_roots;
                b.long_items = g->d_bfs_long; b.long_cap = g->bfs_long_cap;
                b.fallback = ctl + kCtlWords * bfs::kMaxLevels;
                b.inline_preleaf = 1;
                b.counts = p.counts; b.stats = p.stats;
                uint32_t *bufs[2] = {g->d_bfs[0], g->d_bfs[1]};
                const uint32_t levels = dt.max_edges > 1 ? dt.max_edges - 1 : 1;
                CK(launch_bfs(b, dt.max_vertices, levels, bufs, ctl, g->bfs_seg_cap, stats_host != nullptr, s, sms),
                   "bfs pass launch");
            } else if (use_warp_kernel()) {
                CK(launch_comine(p, dt.max_vertices, stats_host != nullptr, s, sms), "comine_kernel launch");
            } else {
                lane::LParams q;
                q.src = p.src; q.dst = p.dst; q.tr = p.tr; q.hi = p.hi; q.eptr = p.eptr;
                q.out_off = p.out_off; q.in_off = p.in_off; q.out_ent = p.out_ent; q.in_ent = p.in_ent;
                q.out_ptr = p.out_ptr; q.in_ptr = p.in_ptr;
                q.nodes = dt.lnodes; q.groups = dt.groups; q.motif_node = dt.motif_node;
                q.n_nodes = dt.n_nodes; q.n_groups = dt.n_groups; q.n_motifs = dt.n_motifs; q.n_slots = dt.n_slots;
                q.n_frames = dt.max_edges > 2 ? dt.max_edges - 2 : 0;
                q.r0 = p.r0; q.n_roots = p.n_roots; q.lb = p.lb; q.counts = p.counts; q.stats = p.stats;
                q.dbg = stats_host ? g->d_dbg : nullptr;
                q.pm = nullptr; q.pm_cnt = nullptr; q.pm_seg_cap = 0; q.pm_words = 0;
                CK(launch_lane(q, dt.max_vertices, stats_host != nullptr, s, sms), "comine_lane_kernel launch");
            }
        }
    }
    if (stats_host) {
        CK(cudaMemcpyAsync(stats_host, g->d_stats, sizeof(unsigned long long) * ST_N, cudaMemcpyDeviceToHost, s),
           "cudaMemcpyAsync(stats)");
    }
    if (!on_device && counts_out) {
        CK(cudaMemcpyAsync(counts_out, d_counts, sizeof(unsigned long long) * k, cudaMemcpyDeviceToHost, s),
           "cudaMemcpyAsync(counts)");
    }
    if (!on_device || stats_host) {
        CK(cudaStreamSynchronize(s), "cudaStreamSynchronize");
        if (dbg_path && g->d_dbg) {
            std::vector<unsigned long long> rec(8 * kDbgWarps);
            CK(cudaMemcpy(rec.data(), g->d_dbg, rec.size() * 8, cudaMemcpyDeviceToHost), "cudaMemcpy(dbg)");
            if (FILE *f = fopen(dbg_path, "wb")) {
                fwrite(rec.data(), 8, rec.size(), f);
                fclose(f);
            }
        }
        // the lane kernel's load-balancer watchdog (never expected to fire) marks LB_ERR
        std::vector<uint32_t> lbw(n_lb);
        CK(cudaMemcpy(lbw.data(), g->d_queue, sizeof(uint32_t) * n_lb, cudaMemcpyDeviceToHost), "cudaMemcpy(lb)");
        for (size_t i = 0; i < n_launch; i++)
            if (lbw[LB_N * i + LB_ERR])
                return fail(MAYURA_E_CUDA, "mayura_comine: load-balancer watchdog fired (counts invalid)");
    }
    return MAYURA_OK;
}

void free_device(mayura_graph_s *g) {
    if (g->device < 0) return;
    DeviceGuard guard(g->device);
    void *ptrs[] = {g->d_src, g->d_dst, g->d_tr, g->d_hi, g->d_t, g->d_out_off, g->d_in_off, g->d_out_ent,
                    g->d_in_ent, g->d_eptr, g->d_out_ptr, g->d_in_ptr, g->d_ctx, g->d_queue, g->d_counts,
                    g->d_stats, g->d_dbg, g->d_bfs[0], g->d_bfs[1], g->d_bfs_ctl, g->d_bfs_long,
                    g->d_wave, g->d_tile};
    for (void *p : ptrs)
        if (p) cudaFree(p);
}

// Upload h plus `pad` trailing elements filled with byte `fill` (so 32-wide batches never
// read past the allocation).
template <typename T>
mayura_status up(T *&d, const std::vector<T> &h, size_t min_elems, size_t pad, int fill, uint64_t &bytes) {
    const size_t n = std::max(h.size(), min_elems) + pad;
    CK(cudaMalloc(&d, sizeof(T) * (n ? n : 1)), "cudaMalloc(graph)");
    if (n > h.size()) CK(cudaMemset(d, fill, sizeof(T) * n), "cudaMemset(graph)");
    if (!h.empty()) CK(cudaMemcpy(d, h.data(), sizeof(T) * h.size(), cudaMemcpyHostToDevice), "cudaMemcpy(graph)");
    bytes += sizeof(T) * n;
    return MAYURA_OK;
}

}  // namespace

void free_mgtree_device(mayura_mgtree_s *m) { free_tables(m); }

}  // namespace mayura

using namespace mayura;

extern "C" mayura_status mayura_load_graph(const uint32_t *src, const uint32_t *dst, const int64_t *t,
                                           uint64_t n_edges, uint32_t n_vertices, int device, mayura_graph *out) {
    clear_error();
    if (!out) return fail(MAYURA_E_INVALID, "mayura_load_graph: out is NULL");
    if (n_edges > 0 && (!src || !dst || !t)) return fail(MAYURA_E_INVALID, "mayura_load_graph: NULL edge array");
    if (n_edges > MAYURA_MAX_E) return fail(MAYURA_E_LIMIT, "mayura_load_graph: more than MAYURA_MAX_E edges");
    if (n_vertices > MAYURA_MAX_VERTICES) return fail(MAYURA_E_LIMIT, "mayura_load_graph: too many vertices");
    if (device < -1) return fail(MAYURA_E_INVALID, "mayura_load_graph: bad device");
    mayura_graph_s *g = new (std::nothrow) mayura_graph_s();
    if (!g) return fail(MAYURA_E_OOM, "mayura_load_graph: out of host memory");
    mayura_status s;
    try {
        s = build_graph_host(src, dst, t, n_edges, n_vertices, g);
    } catch (const std::bad_alloc &) {
        s = fail(MAYURA_E_OOM, "mayura_load_graph: out of host memory");
    }
    if (s != MAYURA_OK) {
        delete g;
        return s;
    }
    if (device >= 0) {
        int ndev = 0;
        cudaError_t e = cudaGetDeviceCount(&ndev);
        if (e != cudaSuccess || device >= ndev) {
            delete g;
            return fail(MAYURA_E_CUDA, std::string("mayura_load_graph: no CUDA device ") + std::to_string(device) +
                                           (e != cudaSuccess ? std::string(": ") + cudaGetErrorString(e) : ""));
        }
        g->device = device;
        DeviceGuard guard(device);
        uint64_t bytes = 0;
        std::vector<uint32_t> none;
        const size_t E = (size_t)n_edges;
        const size_t PADE = 32;  // 32 trailing elements per array
        mayura_status u = MAYURA_OK;
        if (u == MAYURA_OK) u = up(g->d_src, g->src, 0, PADE, 0, bytes);
        if (u == MAYURA_OK) u = up(g->d_dst, g->dst, 0, PADE, 0, bytes);
        if (u == MAYURA_OK) u = up(g->d_tr, g->tr, 0, PADE, 0xFF, bytes);
        if (u == MAYURA_OK) u = up(g->d_t, g->t, 0, 0, 0, bytes);
        if (u == MAYURA_OK) u = up(g->d_hi, none, E, PADE, 0, bytes);
        if (u == MAYURA_OK) u = up(g->d_eptr, g->eptr, 0, 4 * PADE, 0, bytes);
        if (u == MAYURA_OK) u = up(g->d_out_off, g->out_off, 0, 0, 0, bytes);
        if (u == MAYURA_OK) u = up(g->d_in_off, g->in_off, 0, 0, 0, bytes);
        // sentinel padding: a batch (32) or a leaf-sweep length probe (kSweepMax) never reads past it
        if (u == MAYURA_OK) u = up(g->d_out_ent, g->out_ent, 0, 2 * (PADE + kSweepMax), 0xFF, bytes);
        if (u == MAYURA_OK) u = up(g->d_in_ent, g->in_ent, 0, 2 * (PADE + kSweepMax), 0xFF, bytes);
        if (u == MAYURA_OK) u = up(g->d_out_ptr, g->out_ptr, 0, 4 * PADE, 0, bytes);
        if (u == MAYURA_OK) u = up(g->d_in_ptr, g->in_ptr, 0, 4 * PADE, 0, bytes);
        if (u == MAYURA_OK) u = up(g->d_queue, none, (size_t)LB_N * (MAYURA_MAX_MOTIFS + 1), 0, 0, bytes);
        if (u != MAYURA_OK) {
            free_device(g);
            delete g;
            return u;
        }
        g->device_bytes = bytes;
    }
    *out = g;
    return MAYURA_OK;
}

extern "C" void mayura_free_graph(mayura_graph g) {
    if (!g) return;
    free_device(g);
    delete g;
}

extern "C" mayura_status mayura_comine(mayura_graph g, mayura_mgtree m, uint64_t root_begin, uint64_t root_end,
                                       void *cuda_stream, uint64_t *counts_out, int counts_on_device) {
    clear_error();
    return run(g, m, root_begin, root_end, cuda_stream, counts_out, counts_on_device, 0, nullptr);
}

extern "C" mayura_status mayura_mine_independent(mayura_graph g, mayura_mgtree m, uint64_t root_begin,
                                                 uint64_t root_end, void *cuda_stream, uint64_t *counts_out,
                                                 int counts_on_device) {
    clear_error();
    return run(g, m, root_begin, root_end, cuda_stream, counts_out, counts_on_device, 1, nullptr);
}

extern "C" mayura_status mayura_comine_ex(mayura_graph g, mayura_mgtree m, uint64_t root_begin, uint64_t root_end,
                                          void *cuda_stream, uint64_t *counts_out, int counts_on_device,
                                          int independent, void *mid_event) {
    clear_error();
    return run(g, m, root_begin, root_end, cuda_stream, counts_out, counts_on_device, independent ? 1 : 0,
               nullptr, mid_event);
}

extern "C" mayura_status mayura_comine_stats(mayura_graph g, mayura_mgtree m, uint64_t root_begin,
                                             uint64_t root_end, int independent, uint64_t *stats_out) {
    clear_error();
    if (!stats_out) return fail(MAYURA_E_INVALID, "mayura_comine_stats: stats_out is NULL");
    return run(g, m, root_begin, root_end, nullptr, nullptr, 0, independent ? 1 : 0,
               reinterpret_cast<unsigned long long *>(stats_out));
}
