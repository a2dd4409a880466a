// comine.cu -- device side of the C ABI: the co-mining launch sequence (SURVEY.md §8(a)
// steps a2-a7) and graph/tree residency on the GPU.
//
//   a2  window_end_kernel   hi[r] = last edge id with t <= t_r + delta
//   a3-a7, default "hybrid" (MAYURA_KERNEL unset):
//       bfs::expand_kernel + bfs::long_kernel (bfs.cuh) expand every root edge by
//           MAYURA_HYBRID_LEVELS (default 1) MG-Tree levels: thread per partial match,
//           warp per long window; counts completions, writes the next partial matches;
//       lane::comine_lane_kernel (lane.cuh) then mines every partial match depth-first,
//           one search per lane (Algorithm 3), with per-warp task
//           stacks and warp-cooperative long leaf windows for balance.
//     Splitting the heavy hub roots into many partial matches first is what balances the
//     depth-first phase (profiles/README.md).  MAYURA_KERNEL=lane (depth-first from the
//     roots) and MAYURA_KERNEL=bfs (all levels breadth-first) select the two pure forms;
//     all return identical counts.
// All arithmetic is integer (u32 ids and time ranks, i64 timestamps, u64 counts).
#include <cuda_runtime.h>

#include <cub/device/device_scan.cuh>
#include <nvtx3/nvToolsExt.h>  // header-only NVTX ranges (visible under nsys / ncu --nvtx)

#include <algorithm>
#include <type_traits>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <mutex>

#include "internal.h"

namespace mayura {

namespace {

// NVTX range for the scope of one C-ABI call (a no-op unless a profiler is attached)
struct NvtxRange {
    explicit NvtxRange(const char *name) { nvtxRangePushA(name); }
    ~NvtxRange() { nvtxRangePop(); }
};

constexpr unsigned kFull = 0xffffffffu;
constexpr uint32_t kNone = 0xffffffffu;
enum { ST_ROOTS, ST_NODES, ST_WINDOWS, ST_ENTRIES, ST_PROBES, ST_BATCHES, ST_BYTES, ST_MATCHES,
       ST_OFFLOADS, ST_CONTEXTS, ST_N };
// per-launch scheduler words (zeroed by window_end_kernel): [LB_ROOT] = root / item cursor
enum { LB_ROOT = 0, LB_N = 8 };

// Programmatic dependent launch (sm_90+): every kernel of a query lets the next one be
// scheduled at once (its blocks take SM slots as this grid's blocks retire, hiding launch
// latency and the tail), then waits for the previous grid to complete and flush before it
// touches anything -- so the dependency chain is unchanged.
__device__ __forceinline__ void pdl_begin() {
    asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
    asm volatile("griddepcontrol.wait;" ::: "memory");
}

// hi(r) = last edge id with T <= T[r] + delta: galloping from r (windows are
// short) then binary search
__device__ __forceinline__ uint32_t window_end_of(const int64_t *__restrict__ T, uint32_t E, int64_t delta, uint32_t r) {
    const int64_t x = __ldg(T + r);
    int64_t lim = (x > INT64_MAX - delta) ? INT64_MAX : x + delta;  // delta >= 0: no overflow
    uint32_t a = r + 1, step = 1;  // invariant: T[a-1] <= lim
    uint32_t b = E;
#ifdef MAYURA_PLANT_BUG
    // PLANTED BUG (test build only, tests/test_planted_bug.py): the window closes BEFORE t_r + delta
    // (t_m - t_1 < delta instead of <= delta) -- the parity suite must turn red
    if (lim != INT64_MIN) lim -= 1;
#endif
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
    return a - 1;
}

#include "lane.cuh"
#include "bfs.cuh"
#include "flat.cuh"
#include "flat_enum.cuh"
#include "wdfs.cuh"

// a2: hi[r] = (last edge id e with t[e] <= t[r] + delta), by galloping from r (windows
// are short) then binary search.  Also zeroes the load-balancer words and the output
// counts of this call, so a co-mining query is exactly two launches.
__global__ void window_end_kernel(const int64_t *__restrict__ T, uint32_t E, int64_t delta, uint32_t r0,
                                  uint32_t n_roots, uint32_t *__restrict__ hi, uint32_t *lb, uint32_t n_lb,
                                  unsigned long long *counts, uint32_t n_counts) {
    pdl_begin();
    const uint32_t tid = blockIdx.x * blockDim.x + threadIdx.x;
    if (tid < n_lb) lb[tid] = 0;
    if (tid < n_counts) counts[tid] = 0;
    for (uint32_t k = tid; k < n_roots; k += gridDim.x * blockDim.x) {
        const uint32_t r = r0 + k;
        hi[r] = window_end_of(T, E, delta, r);
    }
}

bool pdl_enabled() {  // MAYURA_PDL=0 launches without the attribute (A/B)
    static int v = -1;
    if (v < 0) {
        const char *e = getenv("MAYURA_PDL");
        v = (e && atoi(e) == 0) ? 0 : 1;
    }
    return v == 1;
}

template <typename... KArgs, typename... Args>
cudaError_t launch_pdl(void (*kern)(KArgs...), uint32_t grid, uint32_t block, size_t smem, cudaStream_t s,
                       Args &&...args) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(grid);
    cfg.blockDim = dim3(block);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = s;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[0].val.programmaticStreamSerializationAllowed = pdl_enabled() ? 1 : 0;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    return cudaLaunchKernelEx(&cfg, kern, std::forward<Args>(args)...);
}

struct DeviceTable {
    DNode *nodes;
    DGroup *groups;
    uint32_t *motif_node;
    lane::LNode *lnodes;
    uint32_t *gwant;
    uint32_t n_nodes, n_groups, n_motifs, max_vertices, max_edges, n_slots;
    uint32_t max_groups;  // anchor groups of the widest node
    bool generic;  // some anchor group searches its list or scans the edge array
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
        // Same-list groups (wdfs.cuh): node i was matched as an entry of its parent's group G; a
        // group of i with G's kind and anchor scans the same adjacency list, and its window starts
        // right after that entry (START_P0 = out(src), START_P1 = in(dst) of i's own edge) and ends
        // where G's window ends (same hi(root)) -- a suffix of the parent's window.
        b.same = 0;
        for (uint32_t pg = 0; pg < t.groups.size(); pg++) {
            const DGroup &G = t.groups[pg];
            if (i < G.child_begin || i >= G.child_end || G.kind == ANCHOR_GLOBAL) continue;
            for (uint32_t q = 0; q < (uint32_t)(a.group_end - a.group_begin) && q < 16; q++) {
                const DGroup &G2 = t.groups[a.group_begin + q];
                const uint8_t want_start = G.kind == ANCHOR_OUT ? START_P0 : START_P1;
                if (G2.kind == G.kind && G2.anchor == G.anchor && G2.start == want_start) b.same |= (uint16_t)(1u << q);
            }
        }
        // NODE_NEEDP: some group of this node starts from the successor pointers of its own edge
        // and is not a same-list continuation (the warp kernel loads P with the entry only then)
        for (uint32_t q = 0; q < (uint32_t)(a.group_end - a.group_begin); q++) {
            const DGroup &G2 = t.groups[a.group_begin + q];
            if (G2.start < START_R0 && !(q < 16 && ((b.same >> q) & 1u))) b.flags |= wdfs::NODE_NEEDP;
        }
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

mayura_status cuda_fail(cudaError_t e, const char *what) {
    return fail(MAYURA_E_CUDA, std::string(what) + ": " + cudaGetErrorString(e));
}

#define CK(call, what)                                     \
    do {                                                   \
        cudaError_t e_ = (call);                           \
        if (e_ != cudaSuccess) return cuda_fail(e_, what); \
    } while (0)

// Resident blocks per SM of kernel `kern` at `block` threads and `smem` dynamic bytes, with the
// opt-in shared-memory attribute set -- both driver calls made once per (kernel, device, smem)
// and cached: a C2 query issues 6 launches, and the per-launch attribute + occupancy queries
// were ~12 driver calls of host overhead on the end-to-end path.
struct OccKey {
    const void *kern;
    int dev;
    size_t smem;
};
cudaError_t blocks_per_sm(const void *kern, int block, size_t smem, int *per_sm) {
    static std::mutex mu;
    static std::vector<std::pair<OccKey, int>> cache;
    int dev = 0;
    cudaGetDevice(&dev);
    {
        std::lock_guard<std::mutex> lk(mu);
        for (const auto &e : cache)
            if (e.first.kern == kern && e.first.dev == dev && e.first.smem == smem) {
                *per_sm = e.second;
                return cudaSuccess;
            }
    }
    // the attribute is a per-(kernel, device) maximum: never lower it below a size another
    // cached entry launches with
    size_t mx = smem;
    {
        std::lock_guard<std::mutex> lk(mu);
        for (const auto &e : cache)
            if (e.first.kern == kern && e.first.dev == dev) mx = std::max(mx, e.first.smem);
    }
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)mx);
    if (e != cudaSuccess) return e;
    int n = 0;
    e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&n, kern, block, smem);
    if (e != cudaSuccess) return e;
    if (n < 1) n = 1;
    std::lock_guard<std::mutex> lk(mu);
    cache.push_back({OccKey{kern, dev, smem}, n});
    *per_sm = n;
    return cudaSuccess;
}

template <int MAXV, bool LANECNT, bool STATS, bool GEN, bool ENUM = false>
cudaError_t launch_lane_t(const lane::LParams &p, size_t smem, cudaStream_t s, int sms, uint32_t *grid_out = nullptr) {
    auto kern = lane::comine_lane_kernel<MAXV, LANECNT, STATS, GEN, ENUM>;
    int per_sm = 0;
    {
        cudaError_t e = blocks_per_sm((const void *)kern, lane::kLB, smem, &per_sm);
        if (e != cudaSuccess) return e;
    }
    uint32_t grid = (uint32_t)(sms * per_sm);
    const uint32_t need = (p.n_roots + lane::kLB - 1) / lane::kLB;
    if (need < grid) grid = need ? need : 1;
    if (grid_out) {  // ENUM: the caller sizes the per-warp arrays from the grid first
        if (*grid_out == 0) {
            *grid_out = grid;
            return cudaSuccess;
        }
        grid = *grid_out;
    }
    cudaError_t le = launch_pdl(kern, grid, lane::kLB, smem, s, p);
    count_launch();
    return le != cudaSuccess ? le : cudaGetLastError();
}

constexpr size_t kLaneCntSmem = 48 * 1024;  // lane-private counters while they fit this budget

template <int MAXV>
cudaError_t launch_lane_v(lane::LParams p, bool stats, bool generic, cudaStream_t s, int sms) {
    const bool lanecnt = (size_t)p.n_slots * lane::kLB * 4 <= kLaneCntSmem;
    const size_t smem = lane::smem_total(p.n_nodes, p.n_groups, p.n_slots, p.n_frames, lanecnt, MAXV);
    p.o_groups = (uint32_t)lane::off_groups(p.n_nodes);
    p.o_tot = (uint32_t)lane::off_tot(p.n_nodes, p.n_groups);
    p.o_cnt = (uint32_t)lane::off_cnt(p.n_nodes, p.n_groups, p.n_slots);
    p.o_fr = (uint32_t)lane::off_frames(p.n_nodes, p.n_groups, p.n_slots, lanecnt);
    p.o_stk = (uint32_t)lane::off_stk(p.n_nodes, p.n_groups, p.n_slots, p.n_frames, lanecnt, false);
    p.o_pre = (uint32_t)lane::off_pre(p.n_nodes, p.n_groups, p.n_slots, p.n_frames, lanecnt, MAXV, false);
    p.o_enum = (uint32_t)lane::off_enum(p.n_nodes, p.n_groups, p.n_slots, p.n_frames, lanecnt, MAXV, false);
    if (stats)  // the instrumented kernel is always the generic one
        return lanecnt ? launch_lane_t<MAXV, true, true, true>(p, smem, s, sms)
                       : launch_lane_t<MAXV, false, true, true>(p, smem, s, sms);
    if (lanecnt)
        return generic ? launch_lane_t<MAXV, true, false, true>(p, smem, s, sms)
                       : launch_lane_t<MAXV, true, false, false>(p, smem, s, sms);
    return generic ? launch_lane_t<MAXV, false, false, true>(p, smem, s, sms)
                   : launch_lane_t<MAXV, false, false, false>(p, smem, s, sms);
}

// ENUM kernels (mayura_enumerate): lane counters always, no stats.  *grid == 0: only compute the
// grid (returned in *grid); else launch on exactly that grid (both passes must agree).
template <int MAXV>
cudaError_t launch_enum_v(lane::LParams p, bool generic, cudaStream_t s, int sms, uint32_t *grid) {
    const size_t smem = lane::smem_total(p.n_nodes, p.n_groups, p.n_slots, p.n_frames, true, MAXV, true);
    p.o_groups = (uint32_t)lane::off_groups(p.n_nodes);
    p.o_tot = (uint32_t)lane::off_tot(p.n_nodes, p.n_groups);
    p.o_cnt = (uint32_t)lane::off_cnt(p.n_nodes, p.n_groups, p.n_slots);
    p.o_fr = (uint32_t)lane::off_frames(p.n_nodes, p.n_groups, p.n_slots, true);
    p.o_stk = (uint32_t)lane::off_stk(p.n_nodes, p.n_groups, p.n_slots, p.n_frames, true, true);
    p.o_pre = (uint32_t)lane::off_pre(p.n_nodes, p.n_groups, p.n_slots, p.n_frames, true, MAXV, true);
    p.o_enum = (uint32_t)lane::off_enum(p.n_nodes, p.n_groups, p.n_slots, p.n_frames, true, MAXV, true);
    return generic ? launch_lane_t<MAXV, true, false, true, true>(p, smem, s, sms, grid)
                   : launch_lane_t<MAXV, true, false, false, true>(p, smem, s, sms, grid);
}

cudaError_t launch_enum(const lane::LParams &p, uint32_t max_vertices, bool generic, cudaStream_t s, int sms,
                        uint32_t *grid) {
    if (max_vertices <= 4) return launch_enum_v<4>(p, generic, s, sms, grid);
    if (max_vertices <= 6) return launch_enum_v<6>(p, generic, s, sms, grid);
    if (max_vertices <= 8) return launch_enum_v<8>(p, generic, s, sms, grid);
    return launch_enum_v<16>(p, generic, s, sms, grid);
}

// ---- warp-synchronous depth-first kernel (wdfs.cuh)
// MAYURA_WDFS_SMALL=1 (test hook, read per call): the 64-piece stack instance, which spills to
// global memory early and often
bool wdfs_small() {
    const char *e = getenv("MAYURA_WDFS_SMALL");
    return e && atoi(e) != 0;
}
// MAYURA_WDFS_STATS=1: mayura_comine_stats runs the instrumented warp kernel (round / spill
// counters in the stats fields, see mayura.py) instead of the instrumented lane kernel
bool wdfs_stats() {
    const char *e = getenv("MAYURA_WDFS_STATS");
    return e && atoi(e) != 0;
}

template <int MAXV, bool GEN, int CAP, bool STATS>
cudaError_t launch_wdfs_t(const wdfs::WParams &w, size_t smem, cudaStream_t s, int sms) {
    auto kern = wdfs::wdfs_kernel<MAXV, GEN, CAP, STATS>;
    int per_sm = 0;
    cudaError_t e = blocks_per_sm((const void *)kern, wdfs::kWB, smem, &per_sm);
    if (e != cudaSuccess) return e;
    cudaError_t le = launch_pdl(kern, (uint32_t)(sms * per_sm), wdfs::kWB, smem, s, w);
    count_launch();
    return le != cudaSuccess ? le : cudaGetLastError();
}

template <int MAXV, int CAP>
cudaError_t launch_wdfs_c(wdfs::WParams w, bool generic, bool stats, cudaStream_t s, int sms) {
    const bfs::BParams &b = w.b;
    w.lanecnt = (size_t)b.n_slots * wdfs::kWB * sizeof(wdfs::cnt_t) <= kLaneCntSmem ? 1u : 0u;
    w.o_cnt = (uint32_t)wdfs::off_cnt(b.n_nodes, b.n_groups, b.n_slots);
    w.o_stk = (uint32_t)wdfs::off_stk(b.n_nodes, b.n_groups, b.n_slots, w.lanecnt != 0);
    const size_t smem = wdfs::smem_bytes(b.n_nodes, b.n_groups, b.n_slots, w.lanecnt != 0, MAXV, CAP);
    if (stats) return launch_wdfs_t<MAXV, true, CAP, true>(w, smem, s, sms);
    return generic ? launch_wdfs_t<MAXV, true, CAP, false>(w, smem, s, sms)
                   : launch_wdfs_t<MAXV, false, CAP, false>(w, smem, s, sms);
}

template <int MAXV>
cudaError_t launch_wdfs_v(wdfs::WParams w, bool generic, bool stats, cudaStream_t s, int sms) {
    return wdfs_small() ? launch_wdfs_c<MAXV, wdfs::kCapSmall>(w, generic, stats, s, sms)
                        : launch_wdfs_c<MAXV, wdfs::kCap>(w, generic, stats, s, sms);
}

uint32_t mv_class(uint32_t max_vertices) {
    return max_vertices <= 4 ? 4 : max_vertices <= 6 ? 6 : max_vertices <= 8 ? 8 : 16;
}

// Spill area of the warp kernel: per resident warp, room for the bottom halves of its stack
// (1,024 pieces; 64 MiB - 1 GiB in total, at most 5 % of the free memory), allocated per graph.
mayura_status ensure_wspill(mayura_graph_s *g, uint32_t mv, int sms, uint32_t *spill_cap) {
    const size_t piece = 4 * (6 + (size_t)mv_class(mv));
    const size_t warps = (size_t)sms * 16 * wdfs::kWarps;  // >= resident warps of any instance
    if (!g->d_wspill) {
        size_t free_b = 0, total_b = 0;
        cudaMemGetInfo(&free_b, &total_b);
        const size_t want = std::max<size_t>(64ull << 20, std::min<size_t>({1ull << 30, (size_t)(free_b * 0.05),
                                                                          warps * 1024 * 4 * 22}));
        CK((cudaError_t)dmalloc((void **)&g->d_wspill, want), "cudaMalloc(warp stack spill)");
        g->wspill_bytes = want;
        g->device_bytes += want;
        g->fresh_alloc = true;
    }
    *spill_cap = (uint32_t)std::min<size_t>(g->wspill_bytes / (warps * piece), 0xFFFFFFFFu);
    // test hook: a tiny spill area forces the depth-first fallback of full stacks
    if (const char *e = getenv("MAYURA_WDFS_SPILL_CAP")) *spill_cap = std::min<uint32_t>(*spill_cap, (uint32_t)atoi(e));
    return MAYURA_OK;
}

mayura_status launch_wdfs(mayura_graph_s *g, wdfs::WParams w, uint32_t max_vertices, bool generic, bool stats,
                          cudaStream_t s, int sms) {
    mayura_status ms = ensure_wspill(g, max_vertices, sms, &w.spill_cap);
    if (ms != MAYURA_OK) return ms;
    if (g->fresh_alloc) {
        CK(cudaStreamSynchronize(0), "cudaStreamSynchronize");
        g->fresh_alloc = false;
    }
    w.spill = g->d_wspill;
    w.ent_len = (uint32_t)(g->E + g->V);
    {  // MAYURA_WDFS_CHUNK: items per cursor grab (tuning; default 256)
        const char *ev = getenv("MAYURA_WDFS_CHUNK");
        w.chunk_max = ev ? std::max<uint32_t>(32u, (uint32_t)atoi(ev) & ~31u) : 32u;  // r2 sweep: 32 best
    }
    cudaError_t e;
    if (max_vertices <= 4) e = launch_wdfs_v<4>(w, generic, stats, s, sms);
    else if (max_vertices <= 6) e = launch_wdfs_v<6>(w, generic, stats, s, sms);
    else if (max_vertices <= 8) e = launch_wdfs_v<8>(w, generic, stats, s, sms);
    else e = launch_wdfs_v<16>(w, generic, stats, s, sms);
    CK(e, "wdfs_kernel launch");
    return MAYURA_OK;
}

// the warp kernel's stacks fit the block's shared memory (else the lane kernel is used)
bool wdfs_fits(const DeviceTable &dt) {
    const bool lc = (size_t)dt.n_slots * wdfs::kWB * sizeof(wdfs::cnt_t) <= kLaneCntSmem;
    return wdfs::smem_bytes(dt.n_nodes, dt.n_groups, dt.n_slots, lc, (int)mv_class(dt.max_vertices), wdfs::kCap) <=
           200 * 1024;
}

// depth-first phase: MAYURA_DFS=lane selects the lane kernel (A/B), default the warp kernel
bool use_wdfs() {
    const char *e = getenv("MAYURA_DFS");
    return !(e && std::strcmp(e, "lane") == 0);
}

cudaError_t launch_lane(const lane::LParams &p, uint32_t max_vertices, bool stats, bool generic, cudaStream_t s,
                        int sms) {
    if (max_vertices <= 4) return launch_lane_v<4>(p, stats, generic, s, sms);
    if (max_vertices <= 6) return launch_lane_v<6>(p, stats, generic, s, sms);
    if (max_vertices <= 8) return launch_lane_v<8>(p, stats, generic, s, sms);
    return launch_lane_v<16>(p, stats, generic, s, sms);
}

// Kernel form (MAYURA_KERNEL overrides): "mixed" (heavy roots in the flat form, light roots
// depth-first), "flat" (level-synchronous, entry-parallel; flat.cuh), "warp" (the warp-
// synchronous depth-first kernel straight from the roots; wdfs.cuh), "hybrid" (one breadth-first
// level + the warp kernel, MAYURA_DFS=lane: + the lane kernel), "lane", "bfs".  Default: flat when
// the graph arrays fit in L2, else warp (r2: C4 92.7 ms hybrid-lane -> 75.4 ms warp).  Measured (profiles/README.md r04): flat
// C1 0.172 -> 0.076 ms, C2 0.527 -> 0.321 ms; on DRAM-resident graphs its per-level frontier
// and window-piece traffic loses (C3 4.9 ms hybrid vs 7.8 ms flat).
enum KernelKind { K_HYBRID = 0, K_LANE = 1, K_BFS = 2, K_FLAT = 3, K_MIXED = 4, K_WARP = 5 };
bool l2_resident(const mayura_graph_s *g) {
    int l2 = 0;
    cudaDeviceGetAttribute(&l2, cudaDevAttrL2CacheSize, g->device);
    return g->graph_bytes <= (uint64_t)l2;
}
KernelKind kernel_kind(const mayura_graph_s *g) {  // read per call (tests switch forms within one process)
    const char *e = getenv("MAYURA_KERNEL");
    if (e && std::strcmp(e, "lane") == 0) return K_LANE;
    if (e && std::strcmp(e, "bfs") == 0) return K_BFS;
    if (e && std::strcmp(e, "flat") == 0) return K_FLAT;
    if (e && std::strcmp(e, "hybrid") == 0) return K_HYBRID;
    if (e && std::strcmp(e, "mixed") == 0) return K_MIXED;
    if (e && std::strcmp(e, "warp") == 0) return K_WARP;
    return l2_resident(g) ? K_FLAT : K_WARP;
}
// hybrid: a root is split breadth-first only if one of its root-node windows has >= this
// many entries; the breadth-first level lists the light ones for the depth-first kernel.
// Measured sweep (profiles/README.md r04, H in {0,4,8,16,32}): graphs that fit in L2 are
// best at 8 (C2 0.575 ms at 0 -> 0.524 at 8), DRAM-resident graphs at 16 (C3 8.3 ms at 0 ->
// 4.79 at 16).  MAYURA_HEAVY_MIN overrides (0 = split every root).
uint32_t heavy_min(const mayura_graph_s *g) {
    static int v = -2;
    if (v == -2) {
        const char *e = getenv("MAYURA_HEAVY_MIN");
        v = e ? std::max(0, atoi(e)) : -1;
    }
    if (v >= 0) return (uint32_t)v;
    return l2_resident(g) ? 8u : 16u;
}
// hybrid: breadth-first levels before the depth-first lane kernel (MAYURA_HYBRID_LEVELS)
uint32_t hybrid_levels() {
    static int v = -1;
    if (v < 0) {
        const char *e = getenv("MAYURA_HYBRID_LEVELS");
        v = e ? std::max(0, atoi(e)) : 1;
    }
    return (uint32_t)v;
}

// ---- BFS passes (v4): per level an expand pass and a long-window pass
constexpr uint32_t kCtlWords = bfs::kStripes + 2;  // per level: stripe counters, long counter, pad
// control words: per level kCtlWords | 16 misc (fallback count, light-root count) | flat form:
// per level kStripes window-piece stripe counters
constexpr uint32_t kCtlFlat = kCtlWords * bfs::kMaxLevels + 16;
constexpr uint32_t kCtlTotal = kCtlFlat + bfs::kStripes * bfs::kMaxLevels;

template <int MAXV, bool L0, bool STATS>
cudaError_t launch_bfs_pass(const bfs::BParams &p, bool long_pass, cudaStream_t s, int sms) {
    auto kern = long_pass ? bfs::long_kernel<MAXV, L0, STATS> : bfs::expand_kernel<MAXV, L0, STATS>;
    const size_t smem = bfs::smem_bytes(p.n_nodes, p.n_groups, p.n_slots, bfs::kTB);
    int per_sm = 0;
    cudaError_t e = blocks_per_sm((const void *)kern, bfs::kTB, smem, &per_sm);
    if (e != cudaSuccess) return e;
    uint32_t grid = (uint32_t)(sms * (per_sm > 0 ? per_sm : 1));
    if (L0 && !long_pass) {
        const uint32_t need = (p.n_roots + bfs::kTB - 1) / bfs::kTB;
        grid = std::max(1u, std::min(grid, need));
    }
    cudaError_t le = launch_pdl(kern, grid, bfs::kTB, smem, s, p);
    count_launch();
    return le != cudaSuccess ? le : cudaGetLastError();
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

// ---- flat (level-synchronous, entry-parallel): per level a window pass and an entry pass
template <int MAXV, bool L0>
cudaError_t launch_flat_level(const flat::FParams &f, cudaStream_t s, int sms) {
    const size_t smem = bfs::smem_bytes(f.b.n_nodes, f.b.n_groups, f.b.n_slots, flat::kTB);
    for (int pass = 0; pass < 2; pass++) {
        auto kern = pass == 0 ? flat::flat_win_kernel<MAXV, L0> : flat::flat_entry_kernel<MAXV, L0>;
        int per_sm = 0;
        cudaError_t e = blocks_per_sm((const void *)kern, flat::kTB, smem, &per_sm);
        if (e != cudaSuccess) return e;
        uint32_t grid = (uint32_t)(sms * (per_sm > 0 ? per_sm : 1));
        if (L0 && pass == 0) grid = std::max(1u, std::min(grid, (f.b.n_roots + flat::kTB - 1) / flat::kTB));
        e = launch_pdl(kern, grid, flat::kTB, smem, s, f);
        count_launch();
        if (e == cudaSuccess) e = cudaGetLastError();
        if (e != cudaSuccess) return e;
    }
    return cudaSuccess;
}

template <int MAXV>
cudaError_t launch_flat_v(bfs::BParams p, uint32_t levels, uint32_t *bufs[2], uint32_t *ctl, uint32_t seg_cap,
                          uint4 *win, uint32_t win_cap, const uint32_t *gwant, cudaStream_t s, int sms);

uint32_t rec_words(uint32_t max_vertices) {
    const uint32_t mv = max_vertices <= 4 ? 4 : max_vertices <= 6 ? 6 : max_vertices <= 8 ? 8 : 16;
    return (8 + mv + 3) & ~3u;
}

// Frontier / long-item / control buffers of the BFS passes, allocated once per graph and
// grown on demand.  Capacity: 4 records per edge (>= 2^20, <= 2^26) per buffer.
// Frontier buffers of the breadth-first levels (nbufs = 1 for the hybrid's single level, 2 to
// ping-pong), allocated per graph from the retained pool and grown on demand.  Capacity: 16
// records per edge, at most 2^32 - 1 records and at most 40 % of the free device memory (a
// full segment is still exact: that subtree is mined depth-first in place).  Long-window items:
// 1 per edge (>= 2^20).
mayura_status ensure_bfs_buffers(mayura_graph_s *g, uint32_t words, int nbufs) {
    const size_t rb = (size_t)words * 4;
    if (g->bfs_bytes && g->bfs_nbufs >= nbufs && g->bfs_words >= words && !getenv("MAYURA_BFS_SEG_CAP")) {
        // sized once per graph (the query path must not pay cudaMemGetInfo)
        g->bfs_seg_cap = (uint32_t)std::min<size_t>(g->bfs_bytes / ((size_t)bfs::kStripes * rb), 0xFFFFFFFFu);
        return MAYURA_OK;
    }
    size_t free_b = 0, total_b = 0;
    cudaMemGetInfo(&free_b, &total_b);
    const size_t rec_bytes = (size_t)words * 4;
    // the buffers held now are freed before the new ones are allocated: count them as free
    const uint64_t by_mem = (uint64_t)((free_b + (size_t)g->bfs_nbufs * g->bfs_bytes) * 0.4) / (rec_bytes * nbufs);
    const uint64_t recs = std::max<uint64_t>(1u << 20, std::min<uint64_t>({16 * g->E, by_mem, 0xFFFFFFFFull}));
    uint32_t seg_cap = (uint32_t)((recs + bfs::kStripes - 1) / bfs::kStripes);
    // test hook: tiny capacities force the depth-first fallback / in-place long windows
    if (const char *e = getenv("MAYURA_BFS_SEG_CAP")) seg_cap = (uint32_t)std::max(1L, atol(e));
    const size_t bytes = (size_t)seg_cap * bfs::kStripes * rec_bytes;
    if (g->bfs_bytes < bytes || (nbufs == 2 && !g->d_bfs[1])) {
        // keep the old size only when the buffer count is unchanged (two buffers of a size
        // budgeted for one would take 80 % of the device)
        const size_t want = g->bfs_nbufs >= nbufs ? std::max(bytes, g->bfs_bytes) : bytes;
        // queries already enqueued on any stream (e.g. enqueue-only calls with counts_on_device
        // = 1 on a non-blocking stream) may still read the old buffers: dfree orders on the
        // legacy stream only, so drain the device before the memory returns to the pool
        if (g->d_bfs[0] || g->d_bfs[1]) cudaDeviceSynchronize();
        for (int i = 0; i < 2; i++)
            if (g->d_bfs[i]) dfree(g->d_bfs[i]), g->d_bfs[i] = nullptr;
        g->device_bytes -= g->bfs_nbufs * g->bfs_bytes;
        g->bfs_bytes = 0;
        g->bfs_nbufs = 0;
        for (int i = 0; i < nbufs; i++)
            CK((cudaError_t)dmalloc((void **)&g->d_bfs[i], want), "cudaMalloc(frontier)");
        g->fresh_alloc = true;
        g->bfs_bytes = want;
        g->bfs_nbufs = nbufs;
        g->bfs_words = std::max(g->bfs_words, words);
        g->device_bytes += nbufs * want;
    }
    g->bfs_seg_cap = std::min(seg_cap, (uint32_t)(g->bfs_bytes / ((size_t)bfs::kStripes * rec_bytes)));
    if (!g->d_bfs_ctl) {
        CK((cudaError_t)dmalloc((void **)&g->d_bfs_ctl, sizeof(uint32_t) * kCtlTotal),
           "cudaMalloc(bfs ctl)");
        g->fresh_alloc = true;
        g->bfs_long_cap = (uint32_t)std::min<uint64_t>(std::max<uint64_t>(g->E, 1u << 20), 1u << 28);
        if (const char *e = getenv("MAYURA_BFS_LONG_CAP")) g->bfs_long_cap = (uint32_t)std::max(1L, atol(e));
        CK((cudaError_t)dmalloc((void **)&g->d_bfs_long, sizeof(uint32_t) * 3 * (size_t)g->bfs_long_cap),
           "cudaMalloc(long items)");
        g->device_bytes += sizeof(uint32_t) * 3 * (size_t)g->bfs_long_cap;
        CK((cudaError_t)dmalloc((void **)&g->d_light, sizeof(uint32_t) * ((size_t)g->E + 32)), "cudaMalloc(light roots)");
        g->device_bytes += sizeof(uint32_t) * ((size_t)g->E + 32);
    }
    return MAYURA_OK;
}

template <int MAXV>
cudaError_t launch_flat_v(bfs::BParams p, uint32_t levels, uint32_t *bufs[2], uint32_t *ctl, uint32_t seg_cap,
                          uint4 *win, uint32_t win_cap, const uint32_t *gwant, cudaStream_t s, int sms) {
    for (uint32_t L = 0; L < levels; L++) {
        p.in.data = L ? bufs[(L - 1) & 1] : nullptr;
        p.in.cnt = L ? ctl + (L - 1) * kCtlWords : nullptr;
        p.in.seg_cap = seg_cap;
        p.out.data = bufs[L & 1];
        p.out.cnt = ctl + L * kCtlWords;
        p.out.seg_cap = seg_cap;
        flat::FParams f;
        f.b = p;
        f.win = win;
        f.win_cnt = ctl + kCtlFlat + L * bfs::kStripes;
        f.win_seg_cap = win_cap / bfs::kStripes;
        f.gwant = gwant;
        cudaError_t e = L == 0 ? launch_flat_level<MAXV, true>(f, s, sms) : launch_flat_level<MAXV, false>(f, s, sms);
        if (e != cudaSuccess) return e;
    }
    return cudaSuccess;
}

cudaError_t launch_flat(const bfs::BParams &p, uint32_t max_vertices, uint32_t levels, uint32_t *bufs[2], uint32_t *ctl,
                        uint32_t seg_cap, uint4 *win, uint32_t win_cap, const uint32_t *gwant, cudaStream_t s, int sms) {
    if (max_vertices <= 4) return launch_flat_v<4>(p, levels, bufs, ctl, seg_cap, win, win_cap, gwant, s, sms);
    if (max_vertices <= 6) return launch_flat_v<6>(p, levels, bufs, ctl, seg_cap, win, win_cap, gwant, s, sms);
    if (max_vertices <= 8) return launch_flat_v<8>(p, levels, bufs, ctl, seg_cap, win, win_cap, gwant, s, sms);
    return launch_flat_v<16>(p, levels, bufs, ctl, seg_cap, win, win_cap, gwant, s, sms);
}

// Window-piece buffer of the flat form: bytes for 8 pieces of 48 B per edge, >= 48 MiB, <= 15 %
// of the free memory; its capacity in pieces depends on the tree's piece size.
uint32_t piece_bytes(uint32_t max_vertices) {
    const uint32_t mv = max_vertices <= 4 ? 4 : max_vertices <= 6 ? 6 : max_vertices <= 8 ? 8 : 16;
    return 4 * ((6 + mv + 3) & ~3u);
}
mayura_status ensure_flat_win(mayura_graph_s *g) {
    if (g->d_flat_win) return MAYURA_OK;
    size_t free_b = 0, total_b = 0;
    cudaMemGetInfo(&free_b, &total_b);
    const uint64_t bytes = std::max<uint64_t>(48ull << 20, std::min<uint64_t>(8 * 48 * g->E, (uint64_t)(free_b * 0.15)));
    CK((cudaError_t)dmalloc((void **)&g->d_flat_win, bytes), "cudaMalloc(window pieces)");
    g->flat_win_bytes = bytes;
    g->device_bytes += bytes;
    g->fresh_alloc = true;
    return MAYURA_OK;
}
uint32_t flat_win_cap(const mayura_graph_s *g, uint32_t max_vertices) {
    uint64_t cap = std::min<uint64_t>(g->flat_win_bytes / piece_bytes(max_vertices), 0xFFFFFFFFull);
    if (const char *e = getenv("MAYURA_FLAT_WIN_CAP")) cap = std::min<uint64_t>(cap, (uint64_t)std::max(1L, atol(e)));
    return (uint32_t)cap;  // (MAYURA_FLAT_WIN_CAP: test hook forcing the depth-first fallback)
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
    d.max_groups = 1;
    for (const DNode &x : t.nodes) {
        d.n_slots += (x.flags & NODE_COMPLETION) ? 1 : 0;
        d.max_groups = std::max<uint32_t>(d.max_groups, (uint32_t)(x.group_end - x.group_begin));
    }
    d.generic = false;
    for (const DGroup &x : t.groups) d.generic = d.generic || x.kind == ANCHOR_GLOBAL || x.start == START_SEARCH;
}

mayura_status upload_table(const Table &t, uint32_t n_motifs, DeviceTable &d, void *&owner) {
    const size_t bn = t.nodes.size() * sizeof(DNode), bg = t.groups.size() * sizeof(DGroup),
                 bm = t.motif_node.size() * sizeof(uint32_t), bm16 = lane::align16(bm);
    uint32_t n_slots = 0;
    const std::vector<lane::LNode> ln = lane_nodes(t, n_slots);
    const size_t bl = lane::align16(ln.size() * sizeof(lane::LNode));
    const std::vector<uint32_t> gw = group_wants(t);
    char *buf = nullptr;
    CK((cudaError_t)dmalloc((void **)&buf, bn + bg + bm16 + bl + gw.size() * 4 + 16), "cudaMalloc(mgtree table)");
    CK(cudaStreamSynchronize(0), "cudaStreamSynchronize");
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
        cudaDeviceSynchronize();
        for (void *p : m->d_tables) dfree(p);
        cudaStreamSynchronize(0);
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
            for (void *p : owners) dfree(p);
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

lane::LParams lane_params(const mayura_graph_s *g, const DeviceTable &dt, uint32_t r0, uint32_t n_roots,
                          uint32_t *lb, unsigned long long *counts, unsigned long long *stats, bool dbg) {
    lane::LParams q;
    q.src = g->d_src; q.dst = g->d_dst; q.tr = g->d_tr; q.hi = g->d_hi;
    q.eptr = reinterpret_cast<const uint4 *>(g->d_eptr);
    q.out_off = g->d_out_off; q.in_off = g->d_in_off;
    q.out_ent = reinterpret_cast<const uint2 *>(g->d_out_ent);
    q.in_ent = reinterpret_cast<const uint2 *>(g->d_in_ent);
    q.out_ptr = reinterpret_cast<const uint4 *>(g->d_out_ptr);
    q.in_ptr = reinterpret_cast<const uint4 *>(g->d_in_ptr);
    q.nodes = dt.lnodes; q.groups = dt.groups; q.motif_node = dt.motif_node; q.gwant = dt.gwant;
    q.n_nodes = dt.n_nodes; q.n_groups = dt.n_groups; q.n_motifs = dt.n_motifs; q.n_slots = dt.n_slots;
    q.n_frames = dt.max_edges > 2 ? dt.max_edges - 2 : 0;
    q.r0 = r0; q.n_roots = n_roots; q.lb = lb; q.counts = counts; q.stats = stats;
    q.dbg = dbg ? g->d_dbg : nullptr;
    q.pm = nullptr; q.pm_cnt = nullptr; q.pm_seg_cap = 0; q.pm_words = 0; q.heavy_min = 0;
    q.light = nullptr; q.light_cnt = nullptr;
    q.enum_pass = 0; q.wcnt = nullptr; q.wpre = nullptr; q.slot_word = nullptr; q.slot_len = nullptr; q.out = nullptr;
    q.perm = g->d_perm; q.out_rank = g->d_out_rank; q.in_rank = g->d_in_rank;
    return q;
}

bfs::BParams bfs_params(const mayura_graph_s *g, const DeviceTable &dt, uint32_t r0, uint32_t n_roots,
                        unsigned long long *counts, unsigned long long *stats, uint32_t inline_preleaf) {
    bfs::BParams b;
    b.src = g->d_src; b.dst = g->d_dst; b.tr = g->d_tr; b.hi = g->d_hi;
    b.eptr = reinterpret_cast<const uint4 *>(g->d_eptr);
    b.out_off = g->d_out_off; b.in_off = g->d_in_off;
    b.out_ent = reinterpret_cast<const uint2 *>(g->d_out_ent);
    b.in_ent = reinterpret_cast<const uint2 *>(g->d_in_ent);
    b.out_ptr = reinterpret_cast<const uint4 *>(g->d_out_ptr);
    b.in_ptr = reinterpret_cast<const uint4 *>(g->d_in_ptr);
    b.nodes = dt.lnodes; b.groups = dt.groups; b.motif_node = dt.motif_node;
    b.n_nodes = dt.n_nodes; b.n_groups = dt.n_groups; b.n_motifs = dt.n_motifs; b.n_slots = dt.n_slots;
    b.r0 = r0; b.n_roots = n_roots;
    b.long_items = g->d_bfs_long; b.long_cap = g->bfs_long_cap;
    // diagnostic counters in the control words; null when this graph has none allocated (the warp
    // form allocates no breadth-first scratch): the kernels skip the count then
    b.fallback = g->d_bfs_ctl ? g->d_bfs_ctl + kCtlWords * bfs::kMaxLevels : nullptr;
    b.inline_preleaf = inline_preleaf;
    b.heavy_min = 0;  // set by mine() for the hybrid's single breadth-first level
    b.T = nullptr;    // set by the flat path: its level-0 pass computes (and stores) hi itself
    b.delta = 0;
    b.E = (uint32_t)g->E;
    b.hi_w = g->d_hi;
    b.light = nullptr;
    b.light_cnt = g->d_bfs_ctl ? g->d_bfs_ctl + kCtlWords * bfs::kMaxLevels + 1 : nullptr;
    b.counts = counts; b.stats = stats;
    return b;
}

// One co-mining pass of table dt over roots [r0, r0 + n_roots) into counts (already zeroed).
mayura_status mine(mayura_graph_s *g, const DeviceTable &dt, uint32_t r0, uint32_t n_roots, uint32_t *lb,
                   unsigned long long *counts, unsigned long long *stats, cudaStream_t s, int sms, int64_t delta) {
    const bool st = stats != nullptr;
    const KernelKind kind = kernel_kind(g);
    const uint32_t words = rec_words(dt.max_vertices);
    uint32_t levels = 0;  // breadth-first levels before the depth-first phase
    if (kind == K_HYBRID) levels = std::min(hybrid_levels(), dt.max_edges > 2 ? dt.max_edges - 2 : 0u);
    if (kind == K_BFS) levels = dt.max_edges > 1 ? dt.max_edges - 1 : 1;
    if (kind == K_FLAT && !st) {  // (the instrumented run uses the hybrid's counters)
        const uint32_t fl = dt.max_edges > 1 ? dt.max_edges - 1 : 1;
        mayura_status bs = ensure_bfs_buffers(g, words, 2);
        if (bs != MAYURA_OK) return bs;
        bs = ensure_flat_win(g);
        if (bs != MAYURA_OK) return bs;
        uint32_t *ctl = g->d_bfs_ctl;
        CK(cudaMemsetAsync(ctl, 0, sizeof(uint32_t) * kCtlTotal, s), "cudaMemsetAsync(ctl)");
        bfs::BParams b = bfs_params(g, dt, r0, n_roots, counts, nullptr, 0u);
        b.T = g->d_t;  // no window_end_kernel before the flat form: level 0 computes hi
        b.delta = delta;
        uint32_t *bufs[2] = {g->d_bfs[0], g->d_bfs[1]};
        CK(launch_flat(b, dt.max_vertices, fl, bufs, ctl, g->bfs_seg_cap, reinterpret_cast<uint4 *>(g->d_flat_win),
                       flat_win_cap(g, dt.max_vertices), dt.gwant, s, sms),
           "flat pass launch");
        return MAYURA_OK;
    }
    if (kind == K_MIXED && !st && dt.max_edges > 2) {  // heavy roots flat, then light roots depth-first
        const uint32_t fl = dt.max_edges - 1;
        mayura_status bs = ensure_bfs_buffers(g, words, 2);
        if (bs != MAYURA_OK) return bs;
        bs = ensure_flat_win(g);
        if (bs != MAYURA_OK) return bs;
        uint32_t *ctl = g->d_bfs_ctl;
        CK(cudaMemsetAsync(ctl, 0, sizeof(uint32_t) * kCtlTotal, s), "cudaMemsetAsync(ctl)");
        bfs::BParams b = bfs_params(g, dt, r0, n_roots, counts, nullptr, 0u);
        b.heavy_min = heavy_min(g);
        b.light = g->d_light;
        uint32_t *bufs[2] = {g->d_bfs[0], g->d_bfs[1]};
        CK(launch_flat(b, dt.max_vertices, fl, bufs, ctl, g->bfs_seg_cap, reinterpret_cast<uint4 *>(g->d_flat_win),
                       flat_win_cap(g, dt.max_vertices), dt.gwant, s, sms),
           "flat pass launch");
        lane::LParams q = lane_params(g, dt, r0, n_roots, lb, counts, nullptr, false);
        q.light = g->d_light;
        q.light_cnt = b.light_cnt;
        q.heavy_min = b.heavy_min;
        CK(launch_lane(q, dt.max_vertices, false, dt.generic, s, sms), "comine_lane_kernel launch");
        return MAYURA_OK;
    }
    if (kind == K_WARP && (!st || wdfs_stats()) && wdfs_fits(dt)) {  // the warp kernel straight from the roots
        wdfs::WParams w;
        w.b = bfs_params(g, dt, r0, n_roots, counts, stats, 0u);
        w.b.in.data = nullptr;
        w.gwant = dt.gwant;
        w.lb = lb;
        w.direct = 1;
        return launch_wdfs(g, w, dt.max_vertices, dt.generic, st, s, sms);
    }
    if (kind == K_FLAT || kind == K_MIXED) levels = std::min(hybrid_levels(), dt.max_edges > 2 ? dt.max_edges - 2 : 0u);
    lane::LParams q = lane_params(g, dt, r0, n_roots, lb, counts, stats, st);
    if (levels > 0) {
        mayura_status bs = ensure_bfs_buffers(g, words, levels >= 2 ? 2 : 1);
        if (bs != MAYURA_OK) return bs;
        uint32_t *ctl = g->d_bfs_ctl;
        CK(cudaMemsetAsync(ctl, 0, sizeof(uint32_t) * kCtlTotal, s), "cudaMemsetAsync(ctl)");
        bfs::BParams b = bfs_params(g, dt, r0, n_roots, counts, stats, kind == K_BFS ? 1u : 0u);
        if (kind == K_HYBRID && levels == 1) b.heavy_min = heavy_min(g);
        if (b.heavy_min) b.light = g->d_light;  // light roots are listed for the depth-first kernel
        uint32_t *bufs[2] = {g->d_bfs[0], g->d_bfs[1]};
        CK(launch_bfs(b, dt.max_vertices, levels, bufs, ctl, g->bfs_seg_cap, st, s, sms), "bfs pass launch");
        if (kind == K_BFS) return MAYURA_OK;
        if (kind == K_HYBRID && levels == 1 && (!st || wdfs_stats()) && use_wdfs() && wdfs_fits(dt)) {
            // depth-first phase in the warp kernel: items = the level's partial matches + light roots
            wdfs::WParams w;
            w.b = b;
            w.b.in.data = bufs[0];
            w.b.in.cnt = ctl;
            w.b.in.seg_cap = g->bfs_seg_cap;
            w.gwant = dt.gwant;
            w.lb = lb;
            w.direct = 0;
            return launch_wdfs(g, w, dt.max_vertices, dt.generic, st, s, sms);
        }
        q.pm = bufs[(levels - 1) & 1];
        q.pm_cnt = ctl + (levels - 1) * kCtlWords;
        q.pm_seg_cap = g->bfs_seg_cap;
        q.pm_words = words;
        q.heavy_min = (levels == 1) ? heavy_min(g) : 0u;
        q.light = b.light;
        q.light_cnt = b.light_cnt;
    }
    CK(launch_lane(q, dt.max_vertices, st, dt.generic, s, sms), "comine_lane_kernel launch");
    return MAYURA_OK;
}

// mode 0: co-mine, 1: independent (one pass per motif); stats: instrumented kernels.
mayura_status run(mayura_graph_s *g, mayura_mgtree_s *m, uint64_t rb, uint64_t re, void *stream,
                  uint64_t *counts_out, int on_device, int mode, unsigned long long *stats_host,
                  void *mid_event = nullptr) {
    if (!g || !m) return fail(MAYURA_E_INVALID, "mayura_comine: NULL handle");
    if (g->device < 0) return fail(MAYURA_E_STATE, "mayura_comine: graph is host-only (device = -1)");
    if (rb > re || re > g->E) return fail(MAYURA_E_INVALID, "mayura_comine: bad root range");
    if (!counts_out && !stats_host) return fail(MAYURA_E_INVALID, "mayura_comine: counts_out is NULL");
    DeviceGuard guard(g->device);
    cudaStream_t s = (cudaStream_t)stream;
    trace("comine: enter");
    std::vector<DeviceTable> tabs;
    mayura_status st = ensure_tables(m, g->device, tabs);
    if (st != MAYURA_OK) return st;
    const uint32_t k = m->n_motifs;
    unsigned long long *d_counts = reinterpret_cast<unsigned long long *>(counts_out);
    if (!on_device || stats_host) {
        if (g->d_counts_cap < k) {
            if (g->d_counts) cudaDeviceSynchronize(), dfree(g->d_counts);  // may be in flight (see above)
            g->d_counts = nullptr;
            g->d_counts_cap = 0;
            CK((cudaError_t)dmalloc((void **)&g->d_counts, sizeof(unsigned long long) * k), "cudaMalloc(counts)");
            g->fresh_alloc = true;
            g->d_counts_cap = k;
        }
        d_counts = g->d_counts;
    }
    if (!g->d_queue) {
        CK((cudaError_t)dmalloc((void **)&g->d_queue, sizeof(uint32_t) * LB_N * (MAYURA_MAX_MOTIFS + 1)),
           "cudaMalloc(queue)");
        g->fresh_alloc = true;
        g->device_bytes += sizeof(uint32_t) * LB_N * (MAYURA_MAX_MOTIFS + 1);
    }
    if (stats_host && !g->d_stats) {
        CK((cudaError_t)dmalloc((void **)&g->d_stats, sizeof(unsigned long long) * ST_N), "cudaMalloc(stats)");
        g->fresh_alloc = true;
    }
    // MAYURA_DEBUG_WARPS=<file>: the instrumented lane kernel writes one timeline record per warp
    // (start ns, end ns, iterations, warp-help batches, roots taken, root-queue-empty ns, SM id)
    const char *dbg_path = stats_host ? getenv("MAYURA_DEBUG_WARPS") : nullptr;
    const size_t kDbgWarps = 1u << 16;
    if (dbg_path && !g->d_dbg) {
        CK((cudaError_t)dmalloc((void **)&g->d_dbg, sizeof(unsigned long long) * 8 * kDbgWarps), "cudaMalloc(dbg)");
        g->fresh_alloc = true;
    }
    if (dbg_path) CK(cudaMemsetAsync(g->d_dbg, 0, sizeof(unsigned long long) * 8 * kDbgWarps, s), "cudaMemsetAsync(dbg)");
    if (!dbg_path && stats_host && g->d_dbg) {
        dfree(g->d_dbg);
        g->d_dbg = nullptr;
    }
    if (stats_host) CK(cudaMemsetAsync(g->d_stats, 0, sizeof(unsigned long long) * ST_N, s), "cudaMemsetAsync(stats)");
    const uint32_t n_roots = (uint32_t)(re - rb);
    const size_t n_launch = mode == 1 ? k : 1;
    {
        // size the scratch of the passes below now, so the (stream-ordered, legacy-stream)
        // allocation completes before the caller's stream uses it
        uint32_t mv = tabs[0].max_vertices;
        for (size_t i = 1; i < tabs.size(); i++) mv = std::max(mv, tabs[i].max_vertices);
        const KernelKind kind = kernel_kind(g);
        if (kind != K_LANE && n_roots > 0) {
            // the warp form needs no frontier buffers (its stacks live in shared memory + the spill area)
            const uint32_t lv = kind == K_BFS || kind == K_FLAT || kind == K_MIXED ? 2u
                                : kind == K_HYBRID ? std::min(hybrid_levels(), 2u) : 0u;
            if (lv > 0) st = ensure_bfs_buffers(g, rec_words(mv), lv >= 2 ? 2 : 1);
            if (st != MAYURA_OK) return st;
            if (kind == K_FLAT || kind == K_MIXED) st = ensure_flat_win(g);
            if (st != MAYURA_OK) return st;
        }
        if (g->fresh_alloc) {
            CK(cudaStreamSynchronize(0), "cudaStreamSynchronize");
            g->fresh_alloc = false;
        }
    }
    trace("comine: tables + scratch");
    const uint32_t n_lb = (uint32_t)(LB_N * n_launch);
    // the flat form computes hi in its level-0 pass and uses no scheduler words: only the
    // counts need zeroing (one memset instead of the window_end_kernel launch)
    const bool flat_only = kernel_kind(g) == K_FLAT && !stats_host && tabs[0].max_edges > 1;
    if (flat_only) CK(cudaMemsetAsync(d_counts, 0, sizeof(unsigned long long) * k, s), "cudaMemsetAsync(counts)");
    if (!flat_only) {
        const int threads = 256;
        uint32_t blocks = (n_roots + threads - 1) / threads;
        const uint32_t minb = (std::max(n_lb, k) + threads - 1) / threads;
        blocks = std::max(blocks, minb);
        blocks = std::min<uint32_t>(blocks, 148u * 32u);
        if (blocks == 0) blocks = 1;
        CK(launch_pdl(window_end_kernel, blocks, threads, 0, s, (const int64_t *)g->d_t, (uint32_t)g->E, m->delta,
                      (uint32_t)rb, n_roots, g->d_hi, g->d_queue, n_lb, d_counts, k),
           "window_end_kernel launch");
        count_launch();
    }
    if (mid_event) CK(cudaEventRecord((cudaEvent_t)mid_event, s), "cudaEventRecord(mid_event)");
    const int sms = sm_count(g->device);
    if (n_roots > 0) {
        for (size_t i = 0; i < n_launch; i++) {
            const DeviceTable &dt = mode == 1 ? tabs[1 + i] : tabs[0];
            st = mine(g, dt, (uint32_t)rb, n_roots, g->d_queue + LB_N * i, d_counts + (mode == 1 ? i : 0),
                      stats_host ? g->d_stats : nullptr, s, sms, m->delta);
            if (st != MAYURA_OK) return st;
        }
    }
    trace("comine: kernels");
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
        trace("comine: D2H + sync");
        if (dbg_path && g->d_dbg) {
            std::vector<unsigned long long> rec(8 * kDbgWarps);
            CK(cudaMemcpy(rec.data(), g->d_dbg, rec.size() * 8, cudaMemcpyDeviceToHost), "cudaMemcpy(dbg)");
            if (FILE *f = fopen(dbg_path, "wb")) {
                fwrite(rec.data(), 8, rec.size(), f);
                fclose(f);
            }
        }
    }
    return MAYURA_OK;
}

// ---- enumeration in the flat form (graphs that fit in L2): window + entry pass per level
template <int MAXV>
cudaError_t launch_flat_enum_v(flat::EParams e, uint32_t levels, uint32_t *bufs[2], uint32_t *ctl, uint32_t seg_cap,
                               uint32_t win_cap, cudaStream_t s, int sms) {
    constexpr int PW = flat::EPiece<MAXV>::W / 4;
    (void)PW;
    const size_t smem = bfs::smem_bytes(e.b.n_nodes, e.b.n_groups, e.b.n_slots, flat::kTB);
    e.win_seg_cap = win_cap / bfs::kStripes;
    auto launch = [&](auto kern, bool roots) -> cudaError_t {
        int per_sm = 0;
        cudaError_t er = blocks_per_sm((const void *)kern, flat::kTB, smem, &per_sm);
        if (er != cudaSuccess) return er;
        uint32_t grid = (uint32_t)(sms * (per_sm > 0 ? per_sm : 1));
        if (roots) grid = std::max(1u, std::min(grid, (e.b.n_roots + flat::kTB - 1) / flat::kTB));
        er = launch_pdl(kern, grid, flat::kTB, smem, s, e);
        count_launch();
        return er != cudaSuccess ? er : cudaGetLastError();
    };
    if (levels == 0) {  // 1-edge motifs only: root completions
        e.win_cnt = ctl + kCtlFlat;
        return launch(flat::flat_enum_win_kernel<MAXV, true>, true);
    }
    for (uint32_t L = 0; L < levels; L++) {
        e.b.in.data = L ? bufs[(L - 1) & 1] : nullptr;
        e.b.in.cnt = L ? ctl + (L - 1) * kCtlWords : nullptr;
        e.b.in.seg_cap = seg_cap;
        e.b.out.data = bufs[L & 1];
        e.b.out.cnt = ctl + L * kCtlWords;
        e.b.out.seg_cap = seg_cap;
        e.win_cnt = ctl + kCtlFlat + L * bfs::kStripes;
        cudaError_t er = L == 0 ? launch(flat::flat_enum_win_kernel<MAXV, true>, true)
                                : launch(flat::flat_enum_win_kernel<MAXV, false>, false);
        if (er == cudaSuccess) er = launch(flat::flat_enum_entry_kernel<MAXV>, false);
        if (er != cudaSuccess) return er;
    }
    return cudaSuccess;
}

uint32_t erec_words(uint32_t mv) {
    return mv <= 4 ? flat::ERec<4>::W : mv <= 6 ? flat::ERec<6>::W : mv <= 8 ? flat::ERec<8>::W : flat::ERec<16>::W;
}
uint32_t epiece_bytes(uint32_t mv) {
    return 4 * (mv <= 4 ? flat::EPiece<4>::W : mv <= 6 ? flat::EPiece<6>::W : mv <= 8 ? flat::EPiece<8>::W
                                                                                      : flat::EPiece<16>::W);
}

// Flat-form enumeration attempt.  Returns MAYURA_OK with *done = true when the tuples are in
// `dout` (device); *done = false when a buffer overflowed (the caller re-runs depth-first).
mayura_status flat_enum(mayura_graph_s *g, const DeviceTable &dt, uint32_t r0, uint32_t n_roots,
                        const std::vector<unsigned long long> &slot_word, uint32_t *dout, cudaStream_t s, bool *done) {
    *done = false;
    const uint32_t ns = dt.n_slots, mv = dt.max_vertices;
    mayura_status st = ensure_bfs_buffers(g, erec_words(mv), 2);
    if (st == MAYURA_OK) st = ensure_flat_win(g);
    if (st != MAYURA_OK) return st;
    unsigned long long *sc = nullptr;  // cursor[ns] | slot_word[ns] | overflow
    CK((cudaError_t)dmalloc((void **)&sc, 16 * (size_t)ns + 16), "cudaMalloc(enumeration cursors)");
    CK(cudaStreamSynchronize(0), "cudaStreamSynchronize");
    uint32_t *ovf = reinterpret_cast<uint32_t *>(sc + 2 * ns);
    mayura_status rs = MAYURA_OK;
    cudaError_t e = cudaMemsetAsync(sc, 0, 16 * (size_t)ns + 16, s);
    if (e == cudaSuccess && ns) e = cudaMemcpyAsync(sc + ns, slot_word.data(), 8 * (size_t)ns, cudaMemcpyHostToDevice, s);
    if (e == cudaSuccess) e = cudaMemsetAsync(g->d_bfs_ctl, 0, sizeof(uint32_t) * kCtlTotal, s);
    if (e == cudaSuccess) {
        flat::EParams ep;
        ep.b = bfs_params(g, dt, r0, n_roots, nullptr, nullptr, 0u);
        ep.win = reinterpret_cast<uint4 *>(g->d_flat_win);
        ep.perm = g->d_perm;
        ep.out_rank = g->d_out_rank;
        ep.in_rank = g->d_in_rank;
        ep.out = dout;
        ep.slot_word = sc + ns;
        ep.cursor = sc;
        ep.overflow = ovf;
        uint32_t *bufs[2] = {g->d_bfs[0], g->d_bfs[1]};
        const uint32_t levels = dt.max_edges > 1 ? dt.max_edges - 1 : 0;
        uint64_t wc = std::min<uint64_t>(g->flat_win_bytes / epiece_bytes(mv), 0xFFFFFFFFull);
        if (const char *ev = getenv("MAYURA_FLAT_WIN_CAP")) wc = std::min<uint64_t>(wc, (uint64_t)std::max(1L, atol(ev)));
        const uint32_t wcap = (uint32_t)wc;  // (MAYURA_FLAT_WIN_CAP: test hook forcing the fallback)
        const int sms = sm_count(g->device);
        if (mv <= 4) e = launch_flat_enum_v<4>(ep, levels, bufs, g->d_bfs_ctl, g->bfs_seg_cap, wcap, s, sms);
        else if (mv <= 6) e = launch_flat_enum_v<6>(ep, levels, bufs, g->d_bfs_ctl, g->bfs_seg_cap, wcap, s, sms);
        else if (mv <= 8) e = launch_flat_enum_v<8>(ep, levels, bufs, g->d_bfs_ctl, g->bfs_seg_cap, wcap, s, sms);
        else e = launch_flat_enum_v<16>(ep, levels, bufs, g->d_bfs_ctl, g->bfs_seg_cap, wcap, s, sms);
    }
    uint32_t hov = 1;
    if (e == cudaSuccess) e = cudaMemcpyAsync(&hov, ovf, 4, cudaMemcpyDeviceToHost, s);
    if (e == cudaSuccess) e = cudaStreamSynchronize(s);
    if (e != cudaSuccess) rs = cuda_fail(e, "flat enumeration");
    dfree(sc);
    if (rs == MAYURA_OK) *done = hov == 0;
    return rs;
}

// Enumeration (NEXT-3; "a comprehensive list of all matching motifs
// (enumeration)", :412-413; Algo 1 l.201 / Algo 3 l.662 "add to the enumeration list").
// Two passes of the depth-first lane kernel over the same static root-to-warp mapping:
//   pass 1 counts per (completion slot, warp)   -> wcnt, and the per-motif counts
//   exclusive scan of wcnt (CUB)                -> wpre: each warp's first tuple per slot
//   pass 2 re-mines and writes every match      -> out, at exact positions (no holes)
// then duplicate motifs (sharing a slot) get a device-to-device copy of their region.
mayura_status run_enum(mayura_graph_s *g, mayura_mgtree_s *m, uint64_t rb, uint64_t re, void *stream,
                       uint32_t *out, uint64_t cap_words, int on_device, uint64_t *counts_out,
                       uint64_t *words_needed) {
    if (!g || !m) return fail(MAYURA_E_INVALID, "mayura_enumerate: NULL handle");
    if (g->device < 0) return fail(MAYURA_E_STATE, "mayura_enumerate: graph is host-only (device = -1)");
    if (rb > re || re > g->E) return fail(MAYURA_E_INVALID, "mayura_enumerate: bad root range");
    if (!counts_out) return fail(MAYURA_E_INVALID, "mayura_enumerate: counts_out is NULL");
    DeviceGuard guard(g->device);
    cudaStream_t s = (cudaStream_t)stream;
    std::vector<DeviceTable> tabs;
    mayura_status st = ensure_tables(m, g->device, tabs);
    if (st == MAYURA_OK) st = ensure_ranks(g);
    if (st != MAYURA_OK) return st;
    const DeviceTable &dt = tabs[0];
    const uint32_t k = m->n_motifs, ns = dt.n_slots;
    if ((size_t)ns * lane::kLB * 4 > kLaneCntSmem)
        return fail(MAYURA_E_LIMIT, "mayura_enumerate: more than 96 distinct motifs in the group");
    // slot of each motif (first-come order of the completion nodes) and the tuple length per slot
    uint32_t n_slots_h = 0;
    const std::vector<lane::LNode> ln = lane_nodes(m->group, n_slots_h);
    std::vector<uint32_t> slot_of(k), slot_len(ns, 0), first_of(ns, kNone);
    for (uint32_t q = 0; q < k; q++) {
        slot_of[q] = ln[m->group.motif_node[q]].slot;
        slot_len[slot_of[q]] = (uint32_t)m->canon[q].size();
        if (first_of[slot_of[q]] == kNone) first_of[slot_of[q]] = q;
    }
    const uint32_t n_roots = (uint32_t)(re - rb);
    // graphs that fit in L2: the flat form (counts from the flat counting pass, then one
    // enumeration pass per level); a full buffer falls back to the depth-first form below
    if (n_roots > 0 && !getenv("MAYURA_ENUM_LANE")) {
        std::vector<uint64_t> cnt(k, 0);
        st = run(g, m, rb, re, stream, cnt.data(), 0, 0, nullptr);
        if (st != MAYURA_OK) return st;
        for (uint32_t i = 0; i < k; i++) counts_out[i] = cnt[i];
        std::vector<uint64_t> word(k + 1, 0);
        for (uint32_t i = 0; i < k; i++) word[i + 1] = word[i] + cnt[i] * (uint64_t)m->canon[i].size();
        if (words_needed) *words_needed = word[k];
        if (!out) return MAYURA_OK;
        if (cap_words < word[k]) return fail(MAYURA_E_LIMIT, "mayura_enumerate: capacity_words < words needed");
        if (word[k] == 0) return MAYURA_OK;
        std::vector<unsigned long long> sw(ns, 0);
        for (uint32_t sl = 0; sl < ns; sl++) sw[sl] = first_of[sl] == kNone ? 0 : word[first_of[sl]];
        uint32_t *dout = out;
        if (!on_device) {
            CK((cudaError_t)dmalloc((void **)&dout, 4 * word[k]), "cudaMalloc(enumeration staging)");
            CK(cudaStreamSynchronize(0), "cudaStreamSynchronize");
        }
        bool done = false;
        mayura_status fs = flat_enum(g, dt, (uint32_t)rb, n_roots, sw, dout, s, &done);
        if (fs == MAYURA_OK && done) {
            g->last_enum_form = "flat";
            cudaError_t e = cudaSuccess;
            for (uint32_t i = 0; i < k && e == cudaSuccess; i++) {  // duplicate motifs: copy the first one's tuples
                const uint32_t q0 = first_of[slot_of[i]];
                if (q0 != i && cnt[i])
                    e = cudaMemcpyAsync(dout + word[i], dout + word[q0], 4 * cnt[i] * m->canon[i].size(),
                                        cudaMemcpyDeviceToDevice, s);
            }
            if (e == cudaSuccess && !on_device) e = cudaMemcpyAsync(out, dout, 4 * word[k], cudaMemcpyDeviceToHost, s);
            if (e == cudaSuccess) e = cudaStreamSynchronize(s);
            if (!on_device) {
                dfree(dout);
                cudaStreamSynchronize(0);
            }
            return e == cudaSuccess ? MAYURA_OK : cuda_fail(e, "flat enumeration output");
        }
        if (!on_device) {
            dfree(dout);
            cudaStreamSynchronize(0);
        }
        if (fs != MAYURA_OK) return fs;
        // overflow: fall through to the depth-first form
    }
    g->last_enum_form = "depth-first";
    const int sms = sm_count(g->device);
    lane::LParams q = lane_params(g, dt, (uint32_t)rb, n_roots, nullptr, nullptr, nullptr, false);
    uint32_t grid = 0;
    CK(launch_enum(q, dt.max_vertices, dt.generic, s, sms, &grid), "enumeration grid");
    const size_t nw = (size_t)grid * (lane::kLB / 32), nsw = (size_t)ns * nw;
    size_t scan_bytes = 0;
    CK(cub::DeviceScan::ExclusiveSum(nullptr, scan_bytes, (const unsigned long long *)nullptr,
                                     (unsigned long long *)nullptr, (int)std::max<size_t>(nsw, 1), s),
       "cub scan size");
    // scratch: counts k | wcnt nsw | wpre nsw | slot_word ns | slot_len ns | lb | scan temp
    const size_t b_counts = 8 * (size_t)k, b_w = 8 * std::max<size_t>(nsw, 1), b_sw = 8 * (size_t)std::max(ns, 1u),
                 b_sl = lane::align16(4 * (size_t)std::max(ns, 1u)), b_lb = 4 * LB_N * 4;
    const size_t need_b = lane::align16(b_counts) + 2 * b_w + b_sw + b_sl + b_lb + scan_bytes + 256;
    if (g->enum_bytes < need_b) {
        if (g->d_enum) cudaDeviceSynchronize(), dfree(g->d_enum);  // may be in flight
        g->d_enum = nullptr;
        g->enum_bytes = 0;
        CK((cudaError_t)dmalloc((void **)&g->d_enum, need_b), "cudaMalloc(enumeration scratch)");
        g->enum_bytes = need_b;
    }
    char *sc = reinterpret_cast<char *>(g->d_enum);
    unsigned long long *d_counts = reinterpret_cast<unsigned long long *>(sc);
    sc += lane::align16(b_counts);
    unsigned long long *wcnt = reinterpret_cast<unsigned long long *>(sc);
    sc += b_w;
    unsigned long long *wpre = reinterpret_cast<unsigned long long *>(sc);
    sc += b_w;
    unsigned long long *d_sw = reinterpret_cast<unsigned long long *>(sc);
    sc += b_sw;
    uint32_t *d_sl = reinterpret_cast<uint32_t *>(sc);
    sc += b_sl;
    uint32_t *d_lb = reinterpret_cast<uint32_t *>(sc);
    sc += b_lb;
    void *d_scan = lane::align16((size_t)(sc - (char *)g->d_enum)) + (char *)g->d_enum;
    CK(cudaStreamSynchronize(0), "cudaStreamSynchronize");
    // pass 1: window ends (zeroes the counts) + per-warp counts
    {
        const int threads = 256;
        uint32_t blocks = (n_roots + threads - 1) / threads;
        blocks = std::max(blocks, (std::max<uint32_t>(LB_N, k) + threads - 1) / threads);
        blocks = std::min<uint32_t>(std::max(blocks, 1u), 148u * 32u);
        window_end_kernel<<<blocks, threads, 0, s>>>(g->d_t, (uint32_t)g->E, m->delta, (uint32_t)rb, n_roots,
                                                     g->d_hi, d_lb, LB_N, d_counts, k);
        CK(cudaGetLastError(), "window_end_kernel launch");
        count_launch();
    }
    q.lb = d_lb;
    q.counts = d_counts;
    q.enum_pass = 1;
    q.wcnt = wcnt;
    if (n_roots > 0) CK(launch_enum(q, dt.max_vertices, dt.generic, s, sms, &grid), "enumeration pass 1");
    std::vector<unsigned long long> cnt(k, 0);
    CK(cudaMemcpyAsync(cnt.data(), d_counts, 8 * (size_t)k, cudaMemcpyDeviceToHost, s), "D2H(counts)");
    CK(cudaStreamSynchronize(s), "cudaStreamSynchronize");
    for (uint32_t i = 0; i < k; i++) counts_out[i] = cnt[i];
    // regions in input motif order
    std::vector<uint64_t> word(k + 1, 0);
    for (uint32_t i = 0; i < k; i++) word[i + 1] = word[i] + cnt[i] * (uint64_t)m->canon[i].size();
    if (words_needed) *words_needed = word[k];
    if (!out) return MAYURA_OK;  // size query
    if (cap_words < word[k]) return fail(MAYURA_E_LIMIT, "mayura_enumerate: capacity_words < words needed");
    if (word[k] == 0) return MAYURA_OK;
    std::vector<unsigned long long> sw(ns, 0);
    for (uint32_t sl = 0; sl < ns; sl++) sw[sl] = first_of[sl] == kNone ? 0 : word[first_of[sl]];
    CK(cudaMemcpyAsync(d_sw, sw.data(), 8 * (size_t)ns, cudaMemcpyHostToDevice, s), "H2D(slot words)");
    CK(cudaMemcpyAsync(d_sl, slot_len.data(), 4 * (size_t)ns, cudaMemcpyHostToDevice, s), "H2D(slot lengths)");
    CK(cub::DeviceScan::ExclusiveSum(d_scan, scan_bytes, wcnt, wpre, (int)nsw, s), "cub scan");
    uint32_t *dout = out;
    if (!on_device) {
        CK((cudaError_t)dmalloc((void **)&dout, 4 * word[k]), "cudaMalloc(enumeration staging)");
        CK(cudaStreamSynchronize(0), "cudaStreamSynchronize");
    }
    q.enum_pass = 2;
    q.wpre = wpre;
    q.slot_word = d_sw;
    q.slot_len = d_sl;
    q.out = dout;
    mayura_status rs = MAYURA_OK;
    cudaError_t e = launch_enum(q, dt.max_vertices, dt.generic, s, sms, &grid);
    if (e != cudaSuccess) rs = cuda_fail(e, "enumeration pass 2");
    for (uint32_t i = 0; i < k && rs == MAYURA_OK; i++) {  // duplicate motifs: copy the first one's tuples
        const uint32_t q0 = first_of[slot_of[i]];
        if (q0 != i && cnt[i]) {
            e = cudaMemcpyAsync(dout + word[i], dout + word[q0], 4 * cnt[i] * m->canon[i].size(),
                                cudaMemcpyDeviceToDevice, s);
            if (e != cudaSuccess) rs = cuda_fail(e, "D2D(duplicate motif)");
        }
    }
    if (!on_device && rs == MAYURA_OK) {
        e = cudaMemcpyAsync(out, dout, 4 * word[k], cudaMemcpyDeviceToHost, s);
        if (e != cudaSuccess) rs = cuda_fail(e, "D2H(tuples)");
    }
    e = cudaStreamSynchronize(s);
    if (e != cudaSuccess && rs == MAYURA_OK) rs = cuda_fail(e, "cudaStreamSynchronize");
    if (!on_device) {
        dfree(dout);
        cudaStreamSynchronize(0);
    }
    return rs;
}

// Per-device cache of one graph's query scratch (frontier, window pieces, control words,
// long-window items, light-root list, queue words), handed to the next graph loaded on the
// device: the e2e path builds and drops a graph per query, and sizing + allocating the
// scratch cost ~0.2 ms per new graph (MAYURA_TRACE, C2).  A graph owns its scratch while it
// lives, so distinct handles stay independent.
struct ScratchSet {
    bool valid = false;
    uint64_t e_cap = 0;  // scratch was sized for graphs of up to this many edges
    uint32_t *bfs[2] = {nullptr, nullptr};
    size_t bfs_bytes = 0;
    int bfs_nbufs = 0;
    uint32_t bfs_words = 0, bfs_seg_cap = 0, bfs_long_cap = 0;
    uint32_t *ctl = nullptr, *lng = nullptr, *light = nullptr, *flat_win = nullptr, *queue = nullptr, *wspill = nullptr;
    uint64_t flat_win_bytes = 0, bytes = 0, wspill_bytes = 0;
};
std::mutex g_scratch_mu;
ScratchSet g_scratch[64];

void free_scratch_set(ScratchSet &c) {
    void *ptrs[] = {c.bfs[0], c.bfs[1], c.ctl, c.lng, c.light, c.flat_win, c.queue, c.wspill};
    for (void *p : ptrs) dfree(p);
    c = ScratchSet();
}

// called with the graph's device current: keep g's scratch for the next graph, else free it
void stash_scratch(mayura_graph_s *g) {
    if (g->device < 0 || g->device >= 64) return;
    std::lock_guard<std::mutex> lk(g_scratch_mu);
    ScratchSet &c = g_scratch[g->device];
    if (!g->d_queue) return;  // nothing reusable (freed with the graph); other members may be null
    if (c.valid) free_scratch_set(c);
    c.valid = true;
    c.e_cap = g->E;
    c.bfs[0] = g->d_bfs[0]; c.bfs[1] = g->d_bfs[1];
    c.bfs_bytes = g->bfs_bytes; c.bfs_nbufs = g->bfs_nbufs; c.bfs_words = g->bfs_words;
    c.bfs_seg_cap = g->bfs_seg_cap; c.bfs_long_cap = g->bfs_long_cap;
    c.ctl = g->d_bfs_ctl; c.lng = g->d_bfs_long; c.light = g->d_light;
    c.flat_win = g->d_flat_win; c.flat_win_bytes = g->flat_win_bytes;
    c.queue = g->d_queue;
    c.wspill = g->d_wspill; c.wspill_bytes = g->wspill_bytes;
    g->d_bfs[0] = g->d_bfs[1] = nullptr;
    g->d_bfs_ctl = g->d_bfs_long = g->d_light = g->d_flat_win = g->d_queue = g->d_wspill = nullptr;
}

// before building a graph of E edges on `device`: drop a cached set too small for it (so its
// memory is available to the build)
void drop_small_scratch(int device, uint64_t E) {
    if (device < 0 || device >= 64) return;
    std::lock_guard<std::mutex> lk(g_scratch_mu);
    ScratchSet &c = g_scratch[device];
    if (c.valid && c.e_cap < E) {
        cudaDeviceSynchronize();
        free_scratch_set(c);
    }
}

// after building g: adopt the cached set if it was sized for at least g->E edges
void adopt_scratch(mayura_graph_s *g) {
    if (g->device < 0 || g->device >= 64) return;
    std::lock_guard<std::mutex> lk(g_scratch_mu);
    ScratchSet &c = g_scratch[g->device];
    if (!c.valid || c.e_cap < g->E) return;
    if (getenv("MAYURA_BFS_LONG_CAP")) return;  // test hook sizing: allocate afresh
    g->d_bfs[0] = c.bfs[0]; g->d_bfs[1] = c.bfs[1];
    g->bfs_bytes = c.bfs_bytes; g->bfs_nbufs = c.bfs_nbufs; g->bfs_words = c.bfs_words;
    g->bfs_seg_cap = c.bfs_seg_cap; g->bfs_long_cap = c.bfs_long_cap;
    g->d_bfs_ctl = c.ctl; g->d_bfs_long = c.lng; g->d_light = c.light;
    g->d_flat_win = c.flat_win; g->flat_win_bytes = c.flat_win_bytes;
    g->d_queue = c.queue;
    g->d_wspill = c.wspill; g->wspill_bytes = c.wspill_bytes;
    g->device_bytes += (uint64_t)c.bfs_nbufs * c.bfs_bytes + c.flat_win_bytes + 4ull * 3 * c.bfs_long_cap +
                       4ull * (c.e_cap + 32) + c.wspill_bytes;
    c = ScratchSet();
}

void free_device(mayura_graph_s *g) {
    if (g->device < 0) return;
    DeviceGuard guard(g->device);
    cudaDeviceSynchronize();  // no queued work may still use the memory returned to the pool
    stash_scratch(g);
    void *ptrs[] = {g->d_arena, g->d_queue, g->d_counts, g->d_stats, g->d_dbg, g->d_bfs[0], g->d_bfs[1],
                    g->d_bfs_ctl, g->d_bfs_long, g->d_light, g->d_enum, g->d_flat_win, g->d_wspill};  // arena: graph arrays
    for (void *p : ptrs) dfree(p);
    cudaStreamSynchronize(0);
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
    if (device < 0) {  // host-only graph: the multithreaded host builder
        try {
            s = build_graph_host(src, dst, t, n_edges, n_vertices, g);
        } catch (const std::bad_alloc &) {
            s = fail(MAYURA_E_OOM, "mayura_load_graph: out of host memory");
        }
        if (s != MAYURA_OK) {
            delete g;
            return s;
        }
        *out = g;
        return MAYURA_OK;
    }
    int ndev = 0;
    cudaError_t e = cudaGetDeviceCount(&ndev);
    if (e != cudaSuccess || device >= ndev) {
        delete g;
        return fail(MAYURA_E_CUDA, std::string("mayura_load_graph: no CUDA device ") + std::to_string(device) +
                                       (e != cudaSuccess ? std::string(": ") + cudaGetErrorString(e) : ""));
    }
    g->device = device;
    {
        NvtxRange nr("mayura_load_graph");
        DeviceGuard guard(device);
        drop_small_scratch(device, n_edges);
        s = build_graph_device(src, dst, t, n_edges, n_vertices, g);  // step a0 on the GPU (graph_gpu.cu)
        if (s == MAYURA_OK) adopt_scratch(g);
    }
    if (s != MAYURA_OK) {
        free_device(g);
        delete g;
        return s;
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
    NvtxRange nr("mayura_comine");
    return run(g, m, root_begin, root_end, cuda_stream, counts_out, counts_on_device, 0, nullptr);
}

extern "C" mayura_status mayura_mine_independent(mayura_graph g, mayura_mgtree m, uint64_t root_begin,
                                                 uint64_t root_end, void *cuda_stream, uint64_t *counts_out,
                                                 int counts_on_device) {
    clear_error();
    NvtxRange nr("mayura_mine_independent");
    return run(g, m, root_begin, root_end, cuda_stream, counts_out, counts_on_device, 1, nullptr);
}

extern "C" mayura_status mayura_comine_ex(mayura_graph g, mayura_mgtree m, uint64_t root_begin, uint64_t root_end,
                                          void *cuda_stream, uint64_t *counts_out, int counts_on_device,
                                          int independent, void *mid_event) {
    clear_error();
    NvtxRange nr(independent ? "mayura_comine_ex(independent)" : "mayura_comine_ex");
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

extern "C" mayura_status mayura_enumerate(mayura_graph g, mayura_mgtree m, uint64_t root_begin, uint64_t root_end,
                                          void *cuda_stream, uint32_t *tuples_out, uint64_t capacity_words,
                                          int tuples_on_device, uint64_t *counts_out, uint64_t *words_needed) {
    clear_error();
    NvtxRange nr("mayura_enumerate");
    return run_enum(g, m, root_begin, root_end, cuda_stream, tuples_out, capacity_words, tuples_on_device,
                    counts_out, words_needed);
}

extern "C" const char *mayura_enum_form(mayura_graph g) {
    return g ? g->last_enum_form : "none";
}

extern "C" const char *mayura_kernel_form(mayura_graph g) {
    if (!g || g->device < 0) return "none";
    switch (kernel_kind(g)) {
        case K_FLAT: return "flat";
        case K_LANE: return "lane";
        case K_BFS: return "bfs";
        case K_MIXED: return "mixed";
        case K_WARP: return "warp";
        default: return "hybrid";
    }
}
