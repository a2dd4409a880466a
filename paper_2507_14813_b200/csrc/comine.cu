// comine.cu -- sm_100a kernels of the co-mining hot path + the device side of the C ABI.
//
// Steps:
//   a2  window_end_kernel: hi[r] = last edge id with t <= t_r + delta
//   a3-a7 comine_kernel:   persistent grid; each warp claims 32 root edges at a
//       time from a global atomic queue ("distributes these
//       candidate edges across warps"), then runs one depth-first co-mining
//       search per root along the MG-Tree table (Algorithm 3):
//         - window location: lane-cooperative 32-ary search for the first entry
//           with time rank > tr_prev in the anchor list (Algo 1 l.210-214);
//         - candidate filter: lane i takes window entry i (coalesced 8-byte
//           loads); the entry's neighbour is classified against the warp-uniform
//           register map m2g (which mapped motif vertex it equals, or NEW); every
//           child of the anchor group tests its structural constraint with one
//           compare and a __ballot_sync (Algo 1 l.219 + full injectivity R4) --
//           the paper's predicated / LUT-simplified checks;
//         - completion children add __popc(mask) to a per-block counter
//           (count[Q_N]++, Algo 3 l.661) without descending; inner children
//           push a frame on the per-warp shared-memory DFS stack and descend
//           with the candidate as the new partial match (Algo 3 l.665-669).
//       Per-block shared counters are flushed once per block.
// All arithmetic is integer (u32 ids and time ranks, i64 timestamps, u64 counts).
#include <cuda_runtime.h>

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
enum { S_GROUP = 0, S_BATCH = 1, S_ITER = 2 };
enum { ST_ROOTS, ST_NODES, ST_WINDOWS, ST_ENTRIES, ST_PROBES, ST_BATCHES, ST_BYTES, ST_MATCHES, ST_N };

struct KParams {
    const uint32_t *src, *dst, *tr, *hi;
    const uint32_t *out_off, *in_off;
    const uint2 *out_ent, *in_ent;
    const DNode *nodes;
    const DGroup *groups;
    const uint32_t *motif_node;
    uint32_t n_nodes, n_groups, n_motifs;
    uint32_t r0, n_roots;
    uint32_t *queue;
    unsigned long long *counts;
    unsigned long long *stats;
};

struct Frame {  // one per warp per DFS depth (shared memory)
    uint32_t node, g, g_end, tr_prev, nv, kind, pos, end, batch, ci, mask, c_end;
};

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

// Coarse lane-cooperative 32-ary search: returns lo' <= first index in [lo, end) whose
// time rank exceeds tr_prev, with (first - lo') < 32, so the first 32-entry batch
// from lo' (or its successor) reaches the window.  One sample load per lane per step.
template <bool STATS>
__device__ __forceinline__ uint32_t locate(uint32_t kind, const uint2 *__restrict__ ent,
                                           const uint32_t *__restrict__ trg, uint32_t lo, uint32_t end,
                                           uint32_t tr_prev, int lane, unsigned long long &probes) {
    uint32_t hi = end;
    while (hi - lo > 32) {
        const uint32_t n = hi - lo;
        const uint32_t step = (n + 31) >> 5;
        const uint32_t i = (uint32_t)lane * step;
        uint32_t key = 0xffffffffu;
        if (i < n) key = (kind == ANCHOR_GLOBAL) ? __ldg(trg + lo + i) : __ldg(&ent[lo + i].x);
        if (STATS) probes++;
        const unsigned b = __ballot_sync(kFull, key > tr_prev);
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

template <int MAXV, bool STATS>
__global__ void __launch_bounds__(kBlock) comine_kernel(KParams p) {
    extern __shared__ __align__(16) unsigned char smem[];
    DNode *s_nodes = reinterpret_cast<DNode *>(smem);
    DGroup *s_groups = reinterpret_cast<DGroup *>(s_nodes + p.n_nodes);
    unsigned long long *s_cnt = reinterpret_cast<unsigned long long *>(s_groups + p.n_groups);
    Frame *s_frames = reinterpret_cast<Frame *>(s_cnt + p.n_nodes);
    uint32_t *s_masks = reinterpret_cast<uint32_t *>(s_frames + kWarps * kMaxDepth);

    for (uint32_t i = threadIdx.x; i < p.n_nodes; i += blockDim.x) {
        s_nodes[i] = p.nodes[i];
        s_cnt[i] = 0;
    }
    for (uint32_t i = threadIdx.x; i < p.n_groups; i += blockDim.x) s_groups[i] = p.groups[i];
    __syncthreads();

    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    Frame *F = s_frames + warp * kMaxDepth;
    uint32_t *MS = s_masks + warp * kMaxDepth * kMaxGroupChildren;
    const DNode root = s_nodes[0];
    unsigned long long st[ST_N];
#pragma unroll
    for (int i = 0; i < ST_N; i++) st[i] = 0;

    for (;;) {
        uint32_t base = 0;
        if (lane == 0) base = atomicAdd(p.queue, 32u);
        base = __shfl_sync(kFull, base, 0);
        if (base >= p.n_roots) break;
        const bool valid = base + lane < p.n_roots;
        const uint32_t r = p.r0 + base + lane;
        uint32_t rs = 0, rd = 0, rt = 0, rh = 0;
        if (valid) {
            rs = __ldg(p.src + r);
            rd = __ldg(p.dst + r);
            rt = __ldg(p.tr + r);
            rh = __ldg(p.hi + r);
        }
        unsigned ok = __ballot_sync(kFull, valid && rs != rd);  // a self-loop never matches 0->1
        if (STATS) {
            const unsigned vm = __ballot_sync(kFull, valid);
            if (lane == 0) {
                st[ST_ROOTS] += __popc(ok);
                st[ST_BYTES] += 16ull * __popc(vm);
            }
        }
        if ((root.flags & NODE_COMPLETION) && lane == 0 && ok) {
            atomicAdd(&s_cnt[0], (unsigned long long)__popc(ok));
            if (STATS) st[ST_MATCHES] += __popc(ok);
        }
        if (!(root.flags & NODE_INNER)) continue;

        while (ok) {
            const int j = __ffs(ok) - 1;
            ok &= ok - 1;
            uint32_t m2g[MAXV];
#pragma unroll
            for (int k = 0; k < MAXV; k++) m2g[k] = 0;
            m2g[0] = __shfl_sync(kFull, rs, j);
            m2g[1] = __shfl_sync(kFull, rd, j);
            const uint32_t h = __shfl_sync(kFull, rh, j);
            uint32_t tr_prev = __shfl_sync(kFull, rt, j);

            int depth = 0;
            uint32_t node = 0, nv = 2, g = root.group_begin, g_end = root.group_end;
            uint32_t kind = 0, pos = 0, end = 0, batch = 0, ci = 0, mask = 0, c_end = 0;
            uint32_t etr = 0, e1 = 0, e2 = 0;  // this lane's batch entry: time rank, neighbour / (src, dst)
            int state = S_GROUP;
            if (STATS && lane == 0) st[ST_NODES]++;

            for (;;) {
                if (state == S_GROUP) {
                    if (g == g_end) {  // all children groups of `node` done: pop
                        if (depth == 0) break;
                        --depth;
                        __syncwarp();
                        const Frame f = F[depth];
                        node = f.node; g = f.g; g_end = f.g_end; tr_prev = f.tr_prev; nv = f.nv;
                        kind = f.kind; pos = f.pos; end = f.end; batch = f.batch; ci = f.ci;
                        mask = f.mask; c_end = f.c_end;
                        const uint32_t idx = batch + lane;
                        if (idx < end) {
                            if (kind == ANCHOR_GLOBAL) {
                                etr = __ldg(p.tr + idx); e1 = __ldg(p.src + idx); e2 = __ldg(p.dst + idx);
                            } else {
                                const uint2 e = __ldg((kind == ANCHOR_OUT ? p.out_ent : p.in_ent) + idx);
                                etr = e.x; e1 = e.y;
                            }
                        }
                        state = S_ITER;
                        continue;
                    }
                    const DGroup G = s_groups[g];
                    kind = G.kind;
                    if (kind == ANCHOR_GLOBAL) {
                        pos = tr_prev;  // first edge of the previous edge's tie group
                        end = h + 1;
                    } else {
                        const uint32_t x = m2g_get<MAXV>(m2g, G.anchor);
                        const uint32_t *off = (kind == ANCHOR_OUT) ? p.out_off : p.in_off;
                        pos = __ldg(off + x);
                        end = __ldg(off + x + 1);
                        if (STATS && lane == 0) st[ST_BYTES] += 8;
                    }
                    pos = locate<STATS>(kind, kind == ANCHOR_OUT ? p.out_ent : p.in_ent, p.tr, pos, end,
                                        tr_prev, lane, st[ST_PROBES]);
                    if (STATS && lane == 0) st[ST_WINDOWS]++;
                    state = S_BATCH;
                }
                if (state == S_BATCH) {
                    if (pos >= end) {
                        ++g;
                        state = S_GROUP;
                        continue;
                    }
                    batch = pos;
                    const uint32_t idx = pos + lane;
                    bool in = idx < end;
                    etr = 0xffffffffu;
                    if (in) {
                        if (kind == ANCHOR_GLOBAL) {
                            etr = __ldg(p.tr + idx); e1 = __ldg(p.src + idx); e2 = __ldg(p.dst + idx);
                        } else {
                            const uint2 e = __ldg((kind == ANCHOR_OUT ? p.out_ent : p.in_ent) + idx);
                            etr = e.x; e1 = e.y;
                        }
                    }
                    in = in && etr <= h;
                    const bool w = in && etr > tr_prev;
                    const bool more = __shfl_sync(kFull, (int)in, 31) != 0;
                    pos = more ? pos + 32 : end;
                    uint32_t cls;
                    if (kind == ANCHOR_GLOBAL)
                        cls = (classify<MAXV>(m2g, nv, e1) == CLS_NEW && classify<MAXV>(m2g, nv, e2) == CLS_NEW &&
                               e1 != e2) ? CLS_NEW : 0xFEu;
                    else
                        cls = classify<MAXV>(m2g, nv, e1);
                    const DGroup G = s_groups[g];
                    if (STATS) {
                        const unsigned wm = __ballot_sync(kFull, w);
                        if (lane == 0) {
                            st[ST_BATCHES]++;
                            st[ST_ENTRIES] += __popc(wm);
                            st[ST_BYTES] += (kind == ANCHOR_GLOBAL ? 12ull : 8ull) *
                                            (__popc(wm) + (more ? 0 : 1));
                        }
                    }
                    bool any_inner = false;
                    for (uint32_t c = G.child_begin; c < G.child_end; ++c) {
                        const DNode dn = s_nodes[c];
                        const unsigned mc = __ballot_sync(kFull, w && cls == dn.want);
                        if ((dn.flags & NODE_COMPLETION) && mc && lane == 0) {
                            atomicAdd(&s_cnt[c], (unsigned long long)__popc(mc));
                            if (STATS) st[ST_MATCHES] += __popc(mc);
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
                    mask = (s_nodes[ci].flags & NODE_INNER) ? MS[depth * kMaxGroupChildren] : 0u;
                    state = S_ITER;
                }
                // S_ITER: next (inner child, candidate) pair of the current batch
                while (mask == 0) {
                    if (++ci >= c_end) break;
                    const uint32_t cb = s_groups[g].child_begin;
                    mask = (s_nodes[ci].flags & NODE_INNER) ? MS[depth * kMaxGroupChildren + (ci - cb)] : 0u;
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
                if (lane == 0) {
                    Frame f;
                    f.node = node; f.g = g; f.g_end = g_end; f.tr_prev = tr_prev; f.nv = nv; f.kind = kind;
                    f.pos = pos; f.end = end; f.batch = batch; f.ci = ci; f.mask = mask; f.c_end = c_end;
                    F[depth] = f;
                }
                const DNode dc = s_nodes[ci];
                if (dc.n_new >= 1) m2g_set<MAXV>(m2g, nv, c1);
                if (dc.n_new == 2) m2g_set<MAXV>(m2g, nv + 1, c2);
                nv = dc.nv;
                tr_prev = ctr;
                node = ci;
                g = dc.group_begin;
                g_end = dc.group_end;
                ++depth;
                state = S_GROUP;
                if (STATS && lane == 0) st[ST_NODES]++;
            }
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

// a2: hi[r] = (last edge id e with t[e] <= t[r] + delta), by galloping from r (windows
// are short) then binary search.  Also zeroes the work-queue cursors and the output
// counts of this call, so a co-mining query is exactly two launches.
__global__ void window_end_kernel(const int64_t *__restrict__ T, uint32_t E, int64_t delta, uint32_t r0,
                                  uint32_t n_roots, uint32_t *__restrict__ hi, uint32_t *queue, uint32_t n_queue,
                                  unsigned long long *counts, uint32_t n_counts) {
    const uint32_t tid = blockIdx.x * blockDim.x + threadIdx.x;
    if (tid < n_queue) queue[tid] = 0;
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
    uint32_t n_nodes, n_groups, n_motifs, max_vertices;
};

size_t smem_bytes(uint32_t n_nodes, uint32_t n_groups) {
    return (size_t)n_nodes * sizeof(DNode) + (size_t)n_groups * sizeof(DGroup) +
           (size_t)n_nodes * sizeof(unsigned long long) + sizeof(Frame) * kWarps * kMaxDepth +
           sizeof(uint32_t) * kWarps * kMaxDepth * kMaxGroupChildren;
}

mayura_status cuda_fail(cudaError_t e, const char *what) {
    return fail(MAYURA_E_CUDA, std::string(what) + ": " + cudaGetErrorString(e));
}

#define CK(call, what)                                  \
    do {                                                \
        cudaError_t e_ = (call);                        \
        if (e_ != cudaSuccess) return cuda_fail(e_, what); \
    } while (0)

template <int MAXV, bool STATS>
cudaError_t launch_comine_t(const KParams &p, size_t smem, cudaStream_t s, int sms) {
    auto kern = comine_kernel<MAXV, STATS>;
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

cudaError_t launch_comine(const KParams &p, uint32_t max_vertices, bool stats, cudaStream_t s, int sms) {
    const size_t smem = smem_bytes(p.n_nodes, p.n_groups);
    if (stats) {
        if (max_vertices <= 4) return launch_comine_t<4, true>(p, smem, s, sms);
        if (max_vertices <= 8) return launch_comine_t<8, true>(p, smem, s, sms);
        return launch_comine_t<16, true>(p, smem, s, sms);
    }
    if (max_vertices <= 4) return launch_comine_t<4, false>(p, smem, s, sms);
    if (max_vertices <= 8) return launch_comine_t<8, false>(p, smem, s, sms);
    return launch_comine_t<16, false>(p, smem, s, sms);
}

mayura_status upload_table(const Table &t, uint32_t n_motifs, DeviceTable &d, void *&owner) {
    const size_t bn = t.nodes.size() * sizeof(DNode), bg = t.groups.size() * sizeof(DGroup),
                 bm = t.motif_node.size() * sizeof(uint32_t);
    char *buf = nullptr;
    CK(cudaMalloc(&buf, bn + bg + bm + 16), "cudaMalloc(mgtree table)");
    CK(cudaMemcpy(buf, t.nodes.data(), bn, cudaMemcpyHostToDevice), "cudaMemcpy(table)");
    CK(cudaMemcpy(buf + bn, t.groups.data(), bg, cudaMemcpyHostToDevice), "cudaMemcpy(table)");
    CK(cudaMemcpy(buf + bn + bg, t.motif_node.data(), bm, cudaMemcpyHostToDevice), "cudaMemcpy(table)");
    owner = buf;
    d.nodes = reinterpret_cast<DNode *>(buf);
    d.groups = reinterpret_cast<DGroup *>(buf + bn);
    d.motif_node = reinterpret_cast<uint32_t *>(buf + bn + bg);
    d.n_nodes = (uint32_t)t.nodes.size();
    d.n_groups = (uint32_t)t.groups.size();
    d.n_motifs = n_motifs;
    d.max_vertices = t.max_vertices;
    return MAYURA_OK;
}

void free_tables(mayura_mgtree_s *m) {
    if (m->dev >= 0) {
        int prev = 0;
        cudaGetDevice(&prev);
        cudaSetDevice(m->dev);
        for (void *p : m->d_tables) cudaFree(p);
        cudaSetDevice(prev);
    }
    m->d_tables.clear();
    m->dev = -1;
}

mayura_status ensure_tables(mayura_mgtree_s *m, int dev, std::vector<DeviceTable> &out) {
    if (m->dev != dev) free_tables(m);
    out.resize(1 + m->single.size());
    std::vector<void *> owners(out.size(), nullptr);
    // (re)upload each call is cheap but we cache per device
    if (m->dev == dev && m->d_tables.size() == out.size()) {
        for (size_t i = 0; i < out.size(); i++) {
            const Table &t = i == 0 ? m->group : m->single[i - 1];
            char *buf = (char *)m->d_tables[i];
            const size_t bn = t.nodes.size() * sizeof(DNode), bg = t.groups.size() * sizeof(DGroup);
            out[i].nodes = reinterpret_cast<DNode *>(buf);
            out[i].groups = reinterpret_cast<DGroup *>(buf + bn);
            out[i].motif_node = reinterpret_cast<uint32_t *>(buf + bn + bg);
            out[i].n_nodes = (uint32_t)t.nodes.size();
            out[i].n_groups = (uint32_t)t.groups.size();
            out[i].n_motifs = i == 0 ? m->n_motifs : 1;
            out[i].max_vertices = t.max_vertices;
        }
        return MAYURA_OK;
    }
    for (size_t i = 0; i < out.size(); i++) {
        const Table &t = i == 0 ? m->group : m->single[i - 1];
        mayura_status s = upload_table(t, i == 0 ? m->n_motifs : 1, out[i], owners[i]);
        if (s != MAYURA_OK) {
            for (void *p : owners) if (p) cudaFree(p);
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

// mode 0: co-mine, 1: independent (one launch per motif), stats: instrumented kernel.
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
    if (stats_host && !g->d_stats) CK(cudaMalloc(&g->d_stats, sizeof(unsigned long long) * ST_N), "cudaMalloc(stats)");
    if (stats_host) CK(cudaMemsetAsync(g->d_stats, 0, sizeof(unsigned long long) * ST_N, s), "cudaMemsetAsync(stats)");
    const uint32_t n_roots = (uint32_t)(re - rb);
    const uint32_t n_queue = mode == 1 ? k : 1;
    {
        const int threads = 256;
        uint32_t blocks = (n_roots + threads - 1) / threads;
        const uint32_t minb = (std::max(n_queue, k) + threads - 1) / threads;
        blocks = std::max(blocks, minb);
        blocks = std::min<uint32_t>(blocks, 148u * 32u);
        if (blocks == 0) blocks = 1;
        window_end_kernel<<<blocks, threads, 0, s>>>(g->d_t, (uint32_t)g->E, m->delta, (uint32_t)rb, n_roots,
                                                     g->d_hi, g->d_queue, n_queue, d_counts, k);
        CK(cudaGetLastError(), "window_end_kernel launch");
    }
    if (mid_event) CK(cudaEventRecord((cudaEvent_t)mid_event, s), "cudaEventRecord(mid_event)");
    const int sms = sm_count(g->device);
    if (n_roots > 0) {
        const size_t n_launch = mode == 1 ? k : 1;
        for (size_t i = 0; i < n_launch; i++) {
            const DeviceTable &dt = mode == 1 ? tabs[1 + i] : tabs[0];
            KParams p;
            p.src = g->d_src; p.dst = g->d_dst; p.tr = g->d_tr; p.hi = g->d_hi;
            p.out_off = g->d_out_off; p.in_off = g->d_in_off;
            p.out_ent = reinterpret_cast<const uint2 *>(g->d_out_ent);
            p.in_ent = reinterpret_cast<const uint2 *>(g->d_in_ent);
            p.nodes = dt.nodes; p.groups = dt.groups; p.motif_node = dt.motif_node;
            p.n_nodes = dt.n_nodes; p.n_groups = dt.n_groups; p.n_motifs = dt.n_motifs;
            p.r0 = (uint32_t)rb; p.n_roots = n_roots;
            p.queue = g->d_queue + i;
            p.counts = d_counts + (mode == 1 ? i : 0);
            p.stats = g->d_stats;
            CK(launch_comine(p, dt.max_vertices, stats_host != nullptr, s, sms), "comine_kernel launch");
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
    if (!on_device || stats_host) CK(cudaStreamSynchronize(s), "cudaStreamSynchronize");
    return MAYURA_OK;
}

void free_device(mayura_graph_s *g) {
    if (g->device < 0) return;
    DeviceGuard guard(g->device);
    void *ptrs[] = {g->d_src, g->d_dst, g->d_tr, g->d_hi, g->d_t, g->d_out_off, g->d_in_off,
                    g->d_out_ent, g->d_in_ent, g->d_queue, g->d_counts, g->d_stats};
    for (void *p : ptrs)
        if (p) cudaFree(p);
}

template <typename T>
mayura_status up(T *&d, const std::vector<T> &h, size_t min_elems, uint64_t &bytes) {
    const size_t n = std::max(h.size(), min_elems);
    CK(cudaMalloc(&d, sizeof(T) * (n ? n : 1)), "cudaMalloc(graph)");
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
        mayura_status u = MAYURA_OK;
        if (u == MAYURA_OK) u = up(g->d_src, g->src, 0, bytes);
        if (u == MAYURA_OK) u = up(g->d_dst, g->dst, 0, bytes);
        if (u == MAYURA_OK) u = up(g->d_tr, g->tr, 0, bytes);
        if (u == MAYURA_OK) u = up(g->d_t, g->t, 0, bytes);
        if (u == MAYURA_OK) u = up(g->d_hi, none, E, bytes);
        if (u == MAYURA_OK) u = up(g->d_out_off, g->out_off, 0, bytes);
        if (u == MAYURA_OK) u = up(g->d_in_off, g->in_off, 0, bytes);
        if (u == MAYURA_OK) u = up(g->d_out_ent, g->out_ent, 0, bytes);
        if (u == MAYURA_OK) u = up(g->d_in_ent, g->in_ent, 0, bytes);
        if (u == MAYURA_OK) u = up(g->d_queue, none, MAYURA_MAX_MOTIFS + 1, bytes);
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
