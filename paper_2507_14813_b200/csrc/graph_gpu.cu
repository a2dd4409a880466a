// graph_gpu.cu -- step a0 on the device: the time-sorted edge arrays and per-vertex out/in
// adjacency ("Data-Loading", §4.2: "CSR ... with edges sorted in
// ascending order of timestamps"), built on the graph's GPU from the caller's host
// arrays.  Same layout and results as the host builder (graph_build.cpp, used for
// host-only graphs); tests/test_gpu_parity.py checks the two are identical array by array.
//
//   ids        stable radix sort of (t - t_min) with the input rank as value (CUB onesweep):
//              edge id i = i-th edge in (t, input rank) order; perm[i] = its input rank
//   tr[i]      first id with timestamp t[i] (binary search in the sorted t)
//   out/in CSR stable radix sort of the source (destination) with the edge id as value,
//              so every list is in edge-id (= time) order; list x occupies
//              [off[x], off[x+1]-1) followed by one sentinel entry (tr = nbr = 0xFFFFFFFF)
//   eptr[e]    successor pointers: first list position with time rank > tr[e] in
//              out(src), in(dst), out(dst), in(src) (binary searches)
//   *_ptr[p]   eptr of the edge behind each list entry (sentinels: 0)
// Host copies are made lazily (ensure_host) only when an inspection call needs them.
#include <cuda_runtime.h>

#include <cub/device/device_radix_sort.cuh>
#include <cub/device/device_reduce.cuh>
#include <cub/device/device_scan.cuh>

#include <atomic>
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <mutex>
#include <string>
#include <type_traits>

#include "internal.h"

namespace mayura {
namespace {

mayura_status cfail(cudaError_t e, const char *what) {
    return fail(MAYURA_E_CUDA, std::string("mayura_load_graph: ") + what + ": " + cudaGetErrorString(e));
}
#define GK(call, what)                                  \
    do {                                                \
        cudaError_t e_ = (call);                        \
        if (e_ != cudaSuccess) return cfail(e_, what);  \
    } while (0)

constexpr int kT = 256;

inline uint32_t blocks_for(uint64_t n) { return (uint32_t)std::max<uint64_t>(1, std::min<uint64_t>((n + kT - 1) / kT, 148u * 64u)); }

int bits_for(uint64_t maxval) {
    int b = 0;
    while (b < 64 && (maxval >> b) != 0) b++;
    return b;
}

// vertex ids checked against V and packed (src | dst << 32), so the gather after the time sort
// reads one 8-byte word per edge instead of two scattered 4-byte ones
__global__ void k_check_pack(const uint32_t *src, const uint32_t *dst, uint32_t E, uint32_t V, uint32_t *bad,
                             uint64_t *sd) {
    for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < E; i += gridDim.x * blockDim.x) {
        const uint32_t a = src[i], b = dst[i];
        if (a >= V || b >= V) atomicOr(bad, 1u);
        sd[i] = (uint64_t)a | ((uint64_t)b << 32);
    }
}

__global__ void k_iota_key(const int64_t *t, int64_t tmin, uint64_t *key, uint32_t *val, uint32_t E) {
    for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < E; i += gridDim.x * blockDim.x) {
        key[i] = (uint64_t)t[i] - (uint64_t)tmin;
        val[i] = i;
    }
}

// edge i of the time order: endpoints gathered from the packed input, the timestamp from the
// sorted key itself (t - tmin, coalesced)
__global__ void k_gather(const uint32_t *perm, const uint64_t *sd, const uint64_t *skey, int64_t tmin, uint32_t *src,
                         uint32_t *dst, int64_t *t, uint32_t E) {
    for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < E; i += gridDim.x * blockDim.x) {
        const uint64_t w = sd[perm[i]];
        src[i] = (uint32_t)w;
        dst[i] = (uint32_t)(w >> 32);
        t[i] = (int64_t)(skey[i] + (uint64_t)tmin);
    }
}

// tr[i] = first index with t == t[i] (t sorted): a backward step over the (rare) ties, a
// bisection when the tie run is long.  The list entries {tr, neighbour} of edge i are written
// beside it (out-lists: {tr, dst}, in-lists: {tr, src}), so the scatter into the lists gathers one
// 8-byte word per edge
__global__ void k_time_rank(const int64_t *t, const uint32_t *src, const uint32_t *dst, uint32_t *tr, uint2 *ent_out,
                            uint2 *ent_in, uint32_t E) {
    for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < E; i += gridDim.x * blockDim.x) {
        const int64_t x = t[i];
        uint32_t j = i;
        for (int s = 0; s < 8 && j > 0 && t[j - 1] == x; s++) j--;
        if (j > 0 && t[j - 1] == x) {
            uint32_t lo = 0, hi = j;
            while (lo < hi) {
                const uint32_t m = lo + ((hi - lo) >> 1);
                if (t[m] < x) lo = m + 1;
                else hi = m;
            }
            j = lo;
        }
        tr[i] = j;
        ent_out[i] = make_uint2(j, dst[i]);
        ent_in[i] = make_uint2(j, src[i]);
    }
}

__global__ void k_iota(uint32_t *v, uint32_t E) {
    for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < E; i += gridDim.x * blockDim.x) v[i] = i;
}

// off[x] = (number of edges whose key < x) + x   (one sentinel slot per earlier list)
__global__ void k_offsets(const uint32_t *skey, uint32_t E, uint32_t V, uint32_t *off) {
    for (uint32_t x = blockIdx.x * blockDim.x + threadIdx.x; x <= V; x += gridDim.x * blockDim.x) {
        uint32_t lo = 0, hi = E;
        while (lo < hi) {
            const uint32_t m = lo + ((hi - lo) >> 1);
            if (skey[m] < x) lo = m + 1;
            else hi = m;
        }
        off[x] = lo + x;
    }
}

// list entries in sorted (key, edge id) order; ids[pos] = edge id of list position pos, owner[pos]
// = the list's vertex
__global__ void k_scatter(const uint32_t *skey, const uint32_t *seid, const uint2 *ent_of, uint32_t E, uint2 *ent,
                          uint32_t *ids, uint32_t *owner) {
    for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < E; i += gridDim.x * blockDim.x) {
        const uint32_t e = seid[i];
        const uint32_t x = skey[i];
        const uint32_t pos = i + x;
        ent[pos] = ent_of[e];
        ids[pos] = e;
        owner[pos] = x;
    }
}

// input rank of the edge behind each list position, in place over the edge ids (enumeration only)
__global__ void k_ranks(uint32_t *ids, const uint32_t *perm, uint32_t N) {
    for (uint32_t p = blockIdx.x * blockDim.x + threadIdx.x; p < N; p += gridDim.x * blockDim.x) {
        const uint32_t e = ids[p];
        if (e != 0xFFFFFFFFu) ids[p] = perm[e];
    }
}

__device__ __forceinline__ uint32_t first_after(const uint32_t *off, const uint2 *ent, uint32_t x, uint32_t key) {
    uint32_t lo = off[x], hi = off[x + 1] - 1;  // excludes the sentinel
    while (lo < hi) {
        const uint32_t m = lo + ((hi - lo) >> 1);
        if (ent[m].x > key) hi = m;
        else lo = m + 1;
    }
    return lo;
}

// Successor pointers P(e), one thread per position of one direction's lists,
// both components that position owns: the list's own component (0 = out(src) over the out-list
// positions, 1 = in(dst) over the in-list ones) is the first position after pos with a later time
// rank -- a forward step over the (rare) ties, no search; the cross component (3 = in(src) over the
// out-list positions, 2 = out(dst) over the in-list ones) searches the owner's list of the other
// direction -- neighbouring threads search the same list at nearby keys (cache-friendly, unlike one
// thread per edge id).  The entry's time rank is its own list word (no gather of tr[e]); the two
// words written land in one 16-byte eptr row.  eptr as u32 words: P(e) component k at eptr[4e + k].
__global__ void k_succ(const uint32_t *ids, const uint2 *ent, const uint32_t *owner, const uint32_t *xoff,
                       const uint2 *xent, uint32_t N, uint32_t k_own, uint32_t k_cross, uint32_t *eptr) {
    for (uint32_t pos = blockIdx.x * blockDim.x + threadIdx.x; pos < N; pos += gridDim.x * blockDim.x) {
        const uint32_t e = ids[pos];
        if (e == 0xFFFFFFFFu) continue;  // a sentinel position
        const uint32_t key = ent[pos].x;
        const uint32_t x = owner[pos];
        uint32_t q = pos + 1;
        while (ent[q].x <= key) ++q;  // ties; the list's sentinel (time rank 0xFFFFFFFF) stops it
        eptr[4 * (size_t)e + k_own] = q;
        eptr[4 * (size_t)e + k_cross] = first_after(xoff, xent, x, key);
    }
}

__global__ void k_entry_ptr(const uint32_t *ids, const uint4 *eptr, uint32_t N, uint4 *ptr) {
    for (uint32_t p = blockIdx.x * blockDim.x + threadIdx.x; p < N; p += gridDim.x * blockDim.x) {
        const uint32_t e = ids[p];
        ptr[p] = e != 0xFFFFFFFFu ? eptr[e] : make_uint4(0, 0, 0, 0);
    }
}

// Partition proxy per root (capi.cpp): p(r) = 1 + min(s_r, 65535)^2 with s_r the level-1
// window sizes at the root's endpoints; H = last edge id with t <= t_r + delta.
__global__ void k_proxy(const int64_t *t, uint32_t E, int64_t delta, const uint32_t *src, const uint32_t *dst,
                        const uint4 *eptr, const uint32_t *out_off, const uint2 *out_ent, const uint32_t *in_off,
                        const uint2 *in_ent, unsigned long long *proxy) {
    for (uint32_t r = blockIdx.x * blockDim.x + threadIdx.x; r < E; r += gridDim.x * blockDim.x) {
        const int64_t x = t[r];
        const int64_t lim = (x > INT64_MAX - delta) ? INT64_MAX : x + delta;  // delta >= 0: no overflow
        uint32_t a = r + 1, step = 1, b = E;  // first index with t > lim, galloping from r
        while (a < E) {
            const uint32_t probe = min(E - 1, a + step - 1);
            if (t[probe] > lim) {
                b = probe;
                break;
            }
            a = probe + 1;
            step <<= 1;
        }
        while (a < b) {
            const uint32_t m = a + ((b - a) >> 1);
            if (t[m] > lim) b = m;
            else a = m + 1;
        }
        const uint32_t H = a - 1;
        const uint4 P = eptr[r];
        const uint32_t u = src[r], v = dst[r];
        const uint32_t st[4] = {P.x, P.y, P.z, P.w}, xs[4] = {u, v, v, u};
        unsigned long long s = 0;
#pragma unroll
        for (int k = 0; k < 4; k++) {
            const uint32_t *off = (k == 0 || k == 2) ? out_off : in_off;
            const uint2 *ent = (k == 0 || k == 2) ? out_ent : in_ent;
            uint32_t lo = st[k], hi = off[xs[k] + 1] - 1;
            // first position in [lo, hi] with time rank > H: gallop from lo (windows are short),
            // then bisect -- the same position the host's binary search finds
            for (uint32_t step = 1; lo < hi; step <<= 1) {
                const uint32_t probe = min(hi, lo + step - 1);
                if (ent[probe].x > H) {
                    hi = probe;
                    break;
                }
                lo = probe + 1;
            }
            while (lo < hi) {
                const uint32_t m = lo + ((hi - lo) >> 1);
                if (ent[m].x > H) hi = m;
                else lo = m + 1;
            }
            s += lo - st[k];
        }
        s = s < 65535ull ? s : 65535ull;
        proxy[r] = 1 + s * s;
    }
}

// cut[p] = first r with inclusive_prefix[r] >= target_p, + 1  (index into the exclusive prefix)
__global__ void k_cuts(const unsigned long long *inc, uint32_t E, uint32_t P, unsigned long long *cut) {
    const uint32_t p = threadIdx.x + 1;
    if (p >= P) return;
    const unsigned long long total = E ? inc[E - 1] : 0ull;
    const unsigned long long target = (total / P) * p + ((total % P) * p) / P;
    if (target == 0) {
        cut[p] = 0;
        return;
    }
    uint32_t lo = 0, hi = E;
    while (lo < hi) {
        const uint32_t m = lo + ((hi - lo) >> 1);
        if (inc[m] >= target) hi = m;
        else lo = m + 1;
    }
    cut[p] = (unsigned long long)lo + 1;
}

struct SideStream {  // per device: a non-blocking stream, two events, a pinned flag word
    std::mutex mu;
    bool init = false;
    cudaStream_t s2 = nullptr;
    cudaEvent_t ev0 = nullptr, ev2 = nullptr;
    uint32_t *hbad = nullptr;
};
SideStream &side_stream(int dev) {
    static SideStream ss[64];
    static std::mutex init_mu;
    SideStream &x = ss[dev & 63];
    std::lock_guard<std::mutex> lk(init_mu);
    if (!x.init) {
        cudaStreamCreateWithFlags(&x.s2, cudaStreamNonBlocking);
        cudaEventCreateWithFlags(&x.ev0, cudaEventDisableTiming);
        cudaEventCreateWithFlags(&x.ev2, cudaEventDisableTiming);
        cudaMallocHost((void **)&x.hbad, 16);
        x.init = true;
    }
    return x;
}

struct Tmp {  // scratch freed at scope exit
    std::vector<void *> p;
    template <typename T>
    cudaError_t get(T *&x, size_t n) {
        void *v = nullptr;
        cudaError_t e = (cudaError_t)dmalloc(&v, n * sizeof(T));
        if (e == cudaSuccess) p.push_back(v);
        x = reinterpret_cast<T *>(v);
        return e;
    }
    ~Tmp() {
        for (void *v : p) dfree(v);
    }
};

}  // namespace

static std::atomic<uint64_t> g_launches{0};
void count_launch(uint64_t n) { g_launches.fetch_add(n, std::memory_order_relaxed); }
uint64_t launch_count() { return g_launches.load(std::memory_order_relaxed); }

void trace(const char *what) {
    static int on = -1;
    if (on < 0) on = getenv("MAYURA_TRACE") ? 1 : 0;
    if (!on) return;
    static auto last = std::chrono::steady_clock::now();
    cudaDeviceSynchronize();
    const auto now = std::chrono::steady_clock::now();
    fprintf(stderr, "[mayura] %-28s %9.1f us\n", what, std::chrono::duration<double, std::micro>(now - last).count());
    last = std::chrono::steady_clock::now();
}

int dmalloc(void **p, size_t bytes) {
    static std::mutex mu;
    static bool pooled[64] = {};
    int dev = 0;
    cudaGetDevice(&dev);
    {
        std::lock_guard<std::mutex> lk(mu);
        if (dev >= 0 && dev < 64 && !pooled[dev]) {
            cudaMemPool_t pool;
            if (cudaDeviceGetDefaultMemPool(&pool, dev) == cudaSuccess) {
                uint64_t keep = UINT64_MAX;
                cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &keep);
            }
            pooled[dev] = true;
        }
    }
    return (int)cudaMallocAsync(p, bytes ? bytes : 1, 0);
}

void dfree(void *p) {
    if (p) cudaFreeAsync(p, 0);
}

mayura_status build_graph_device(const uint32_t *hsrc, const uint32_t *hdst, const int64_t *ht, uint64_t E64,
                                 uint32_t V, mayura_graph_s *g) {
    if (E64 + (uint64_t)V + 64 > 0xFFFFFFFFull)
        return fail(MAYURA_E_LIMIT, "mayura_load_graph: n_edges + n_vertices exceeds 32-bit list positions");
    const uint32_t E = (uint32_t)E64;
    const size_t N = (size_t)E + V;  // list positions incl. sentinels
    trace("load: enter");
    g->E = E;
    g->V = V;
    g->host_built = false;
    cudaStream_t s = nullptr;
    uint64_t bytes = 0;
    // all product arrays live in ONE allocation (the e2e path builds a graph per query; one
    // pool allocation instead of 15): a planning pass sums the 256-byte-aligned sizes, a
    // second pass carves the arena and fills
    char *arena = nullptr;
    size_t off = 0;
    bool plan = true;
    auto alloc = [&](auto *&d, size_t n, int fill) -> cudaError_t {
        using T = std::remove_reference_t<decltype(*d)>;
        const size_t b = (n ? n : 1) * sizeof(T);
        const size_t ab = (b + 255) & ~(size_t)255;
        if (plan) {
            off += ab;
            return cudaSuccess;
        }
        d = reinterpret_cast<T *>(arena + off);
        off += ab;
        bytes += b;
        return fill >= 0 ? cudaMemsetAsync(d, fill, b, s) : cudaSuccess;
    };
    auto product = [&]() -> mayura_status {
        GK(alloc(g->d_src, E + kPadE, 0), "cudaMalloc(src)");
        GK(alloc(g->d_dst, E + kPadE, 0), "cudaMalloc(dst)");
        GK(alloc(g->d_tr, E + kPadE, 0xFF), "cudaMalloc(tr)");
        GK(alloc(g->d_t, (size_t)E, -1), "cudaMalloc(t)");
        GK(alloc(g->d_hi, E + kPadE, 0), "cudaMalloc(hi)");
        GK(alloc(g->d_eptr, 4 * ((size_t)E + kPadE), 0), "cudaMalloc(eptr)");
        GK(alloc(g->d_out_off, (size_t)V + 1, -1), "cudaMalloc(out_off)");
        GK(alloc(g->d_in_off, (size_t)V + 1, -1), "cudaMalloc(in_off)");
        GK(alloc(g->d_out_ent, 2 * (N + kPadEnt), 0xFF), "cudaMalloc(out_ent)");
        GK(alloc(g->d_in_ent, 2 * (N + kPadEnt), 0xFF), "cudaMalloc(in_ent)");
        GK(alloc(g->d_out_ptr, 4 * (N + kPadE), 0), "cudaMalloc(out_ptr)");
        GK(alloc(g->d_in_ptr, 4 * (N + kPadE), 0), "cudaMalloc(in_ptr)");
        GK(alloc(g->d_perm, (size_t)E, -1), "cudaMalloc(perm)");
        g->graph_bytes = bytes;
        // enumeration only (mayura_enumerate): input rank of the edge behind every list position
        // (not read by the counting kernels, so not part of graph_bytes' residency estimate)
        GK(alloc(g->d_out_rank, N + kPadE, 0xFF), "cudaMalloc(out_rank)");
        GK(alloc(g->d_in_rank, N + kPadE, 0xFF), "cudaMalloc(in_rank)");
        return MAYURA_OK;
    };
    product();
    GK((cudaError_t)dmalloc(reinterpret_cast<void **>(&arena), off), "cudaMalloc(graph arrays)");
    g->d_arena = arena;
    plan = false;
    off = 0;
    if (mayura_status ps = product()) return ps;
    g->device_bytes += bytes;

    Tmp tmp;
    uint32_t *isrc, *idst, *bad, *val, *val2, *skey, *owner[2];
    int64_t *it;
    uint64_t *key, *key2;
    GK(tmp.get(isrc, E), "cudaMalloc(tmp)");
    GK(tmp.get(idst, E), "cudaMalloc(tmp)");
    GK(tmp.get(it, E), "cudaMalloc(tmp)");
    GK(tmp.get(bad, 4), "cudaMalloc(tmp)");
    uint64_t *sd;
    GK(tmp.get(sd, E), "cudaMalloc(tmp)");
    trace("load: allocations");
    // src/dst travel on a side stream while t is copied, reduced and sorted on the main one:
    // the sort by time needs only t, so the second half of the H2D traffic overlaps it
    // (issuing t's copy first and holding the side copies behind it measured the same e2e, w54)
    SideStream &ss = side_stream(g->device);
    std::unique_lock<std::mutex> side_lock(ss.mu);  // one build at a time uses this device's side stream
    GK(cudaEventRecord(ss.ev0, s), "event");
    GK(cudaStreamWaitEvent(ss.s2, ss.ev0, 0), "stream wait");
    GK(cudaMemsetAsync(bad, 0, 16, ss.s2), "memset");
    GK(cudaMemcpyAsync(isrc, hsrc, 4ull * E, cudaMemcpyHostToDevice, ss.s2), "H2D(src)");
    GK(cudaMemcpyAsync(idst, hdst, 4ull * E, cudaMemcpyHostToDevice, ss.s2), "H2D(dst)");
    if (E) {
        k_check_pack<<<blocks_for(E), kT, 0, ss.s2>>>(isrc, idst, E, V, bad, sd);
        count_launch();
    }
    GK(cudaMemcpyAsync(ss.hbad, bad, 4, cudaMemcpyDeviceToHost, ss.s2), "D2H(check)");
    GK(cudaEventRecord(ss.ev2, ss.s2), "event");
    GK(cudaMemcpyAsync(it, ht, 8ull * E, cudaMemcpyHostToDevice, s), "H2D(t)");
    // time range -> key bits
    int64_t *mm;
    GK(tmp.get(mm, 2), "cudaMalloc(tmp)");
    size_t tb = 0, tb2 = 0;
    int64_t tmin = 0, tmax = 0;
    if (E) {
        GK(cub::DeviceReduce::Min(nullptr, tb, it, mm, (int)E, s), "cub Min");
        GK(cub::DeviceReduce::Max(nullptr, tb2, it, mm + 1, (int)E, s), "cub Max");
        tb = std::max(tb, tb2);
        char *cr;
        GK(tmp.get(cr, tb), "cudaMalloc(tmp)");
        GK(cub::DeviceReduce::Min(cr, tb, it, mm, (int)E, s), "cub Min");
        GK(cub::DeviceReduce::Max(cr, tb, it, mm + 1, (int)E, s), "cub Max");
        int64_t hm[2];
        GK(cudaMemcpyAsync(hm, mm, 16, cudaMemcpyDeviceToHost, s), "D2H(minmax)");
        GK(cudaStreamSynchronize(s), "sync");
        tmin = hm[0];
        tmax = hm[1];
    }
    if (!E) {
        GK(cudaEventSynchronize(ss.ev2), "event sync");
        GK(cudaStreamWaitEvent(s, ss.ev2, 0), "stream wait");
    }
    trace("load: H2D + id check + minmax");
    // 1. stable sort by (t, input rank)
    GK(tmp.get(key, E), "cudaMalloc(tmp)");
    GK(tmp.get(key2, E), "cudaMalloc(tmp)");
    GK(tmp.get(val, E), "cudaMalloc(tmp)");
    if (E) {
        k_iota_key<<<blocks_for(E), kT, 0, s>>>(it, tmin, key, val, E); count_launch();
        const int tbits = std::max(1, bits_for((uint64_t)tmax - (uint64_t)tmin));
        size_t need = 0;
        GK(cub::DeviceRadixSort::SortPairs(nullptr, need, key, key2, val, g->d_perm, (int)E, 0, tbits, s), "cub sort");
        char *ct;
        GK(tmp.get(ct, need), "cudaMalloc(tmp)");
        GK(cub::DeviceRadixSort::SortPairs(ct, need, key, key2, val, g->d_perm, (int)E, 0, tbits, s), "cub sort");
        trace("load: time sort");
        // src/dst on the device and checked (host waits for the side stream only: the sort runs on)
        GK(cudaEventSynchronize(ss.ev2), "event sync");
        if (*ss.hbad) return fail(MAYURA_E_INVALID, "mayura_load_graph: vertex id >= n_vertices");
        GK(cudaStreamWaitEvent(s, ss.ev2, 0), "stream wait");
        k_gather<<<blocks_for(E), kT, 0, s>>>(g->d_perm, sd, key2, tmin, g->d_src, g->d_dst, g->d_t, E); count_launch();
        trace("load: gather");
        // 2. time ranks
        // the list-entry words per edge reuse the sort's input keys and the packed endpoints (both consumed)
        k_time_rank<<<blocks_for(E), kT, 0, s>>>(g->d_t, g->d_src, g->d_dst, g->d_tr, reinterpret_cast<uint2 *>(key),
                                                 reinterpret_cast<uint2 *>(sd), E); count_launch();
    }
    trace("load: time sort + ranks");
    // 3. out / in adjacency
    GK(tmp.get(skey, E), "cudaMalloc(tmp)");
    GK(tmp.get(val2, E), "cudaMalloc(tmp)");
    GK(tmp.get(owner[0], N + 1), "cudaMalloc(tmp)");
    GK(tmp.get(owner[1], N + 1), "cudaMalloc(tmp)");
    // the edge id behind each list position goes into the rank arrays (filled with 0xFF: sentinel
    // positions stay 0xFFFFFFFF); the first enumeration turns them into input ranks (ensure_ranks)
    uint32_t *ids[2] = {g->d_out_rank, g->d_in_rank};
    g->ranks_ready = false;
    const int vbits = std::max(1, bits_for(V ? V - 1 : 0));
    for (int dir = 0; dir < 2; dir++) {
        const uint32_t *k_in = dir == 0 ? g->d_src : g->d_dst;
        const uint2 *ent_of = reinterpret_cast<const uint2 *>(dir == 0 ? key : sd);
        uint32_t *off = dir == 0 ? g->d_out_off : g->d_in_off;
        uint2 *ent = reinterpret_cast<uint2 *>(dir == 0 ? g->d_out_ent : g->d_in_ent);
        if (E) {
            k_iota<<<blocks_for(E), kT, 0, s>>>(val, E); count_launch();
            size_t need = 0;
            GK(cub::DeviceRadixSort::SortPairs(nullptr, need, k_in, skey, val, val2, (int)E, 0, vbits, s), "cub sort");
            char *ct;
            GK(tmp.get(ct, need), "cudaMalloc(tmp)");
            GK(cub::DeviceRadixSort::SortPairs(ct, need, k_in, skey, val, val2, (int)E, 0, vbits, s), "cub sort");
            trace("load: vertex sort");
            k_scatter<<<blocks_for(E), kT, 0, s>>>(skey, val2, ent_of, E, ent, ids[dir], owner[dir]); count_launch();
        }
        k_offsets<<<blocks_for((uint64_t)V + 1), kT, 0, s>>>(skey, E, V, off); count_launch();
    }
    trace("load: out/in CSR");
    // 4. successor pointers, then each list entry's copy of them
    if (E) {
        // out-list positions: components 0 (own) and 3 (in(src)); in-list positions: 1 (own), 2 (out(dst))
        k_succ<<<blocks_for(N), kT, 0, s>>>(ids[0], reinterpret_cast<const uint2 *>(g->d_out_ent), owner[0], g->d_in_off,
                                            reinterpret_cast<const uint2 *>(g->d_in_ent), (uint32_t)N, 0u, 3u, g->d_eptr);
        count_launch();
        k_succ<<<blocks_for(N), kT, 0, s>>>(ids[1], reinterpret_cast<const uint2 *>(g->d_in_ent), owner[1], g->d_out_off,
                                            reinterpret_cast<const uint2 *>(g->d_out_ent), (uint32_t)N, 1u, 2u, g->d_eptr);
        count_launch();
        trace("load: successor pointers (by edge)");
    }
    if (N) {
        k_entry_ptr<<<blocks_for(N), kT, 0, s>>>(ids[0], reinterpret_cast<const uint4 *>(g->d_eptr), (uint32_t)N,
                                                 reinterpret_cast<uint4 *>(g->d_out_ptr));
        count_launch();
        k_entry_ptr<<<blocks_for(N), kT, 0, s>>>(ids[1], reinterpret_cast<const uint4 *>(g->d_eptr), (uint32_t)N,
                                                 reinterpret_cast<uint4 *>(g->d_in_ptr));
        count_launch();
    }
    GK(cudaGetLastError(), "graph build kernels");
    GK(cudaStreamSynchronize(s), "graph build");
    trace("load: entry copies");
    return MAYURA_OK;
}

mayura_status partition_device(mayura_graph_s *g, int64_t delta, uint32_t n_parts, uint64_t *cut) {
    if (n_parts > 1024) return fail(MAYURA_E_LIMIT, "mayura_partition_roots: more than 1024 parts");
    int prev = 0;
    cudaGetDevice(&prev);
    cudaSetDevice(g->device);
    struct Restore {
        int d;
        ~Restore() { cudaSetDevice(d); }
    } restore{prev};
    const uint32_t E = (uint32_t)g->E;
    Tmp tmp;
    unsigned long long *proxy, *inc, *dcut;
    cudaStream_t s = nullptr;
    GK(tmp.get(proxy, E), "cudaMalloc(proxy)");
    GK(tmp.get(inc, E), "cudaMalloc(prefix)");
    GK(tmp.get(dcut, n_parts + 1), "cudaMalloc(cuts)");
    GK(cudaMemsetAsync(dcut, 0, 8 * (n_parts + 1), s), "memset");
    if (E) {
        k_proxy<<<blocks_for(E), kT, 0, s>>>(g->d_t, E, delta, g->d_src, g->d_dst, reinterpret_cast<const uint4 *>(g->d_eptr),
                                             g->d_out_off, reinterpret_cast<const uint2 *>(g->d_out_ent), g->d_in_off,
                                             reinterpret_cast<const uint2 *>(g->d_in_ent), proxy); count_launch();
        size_t need = 0;
        GK(cub::DeviceScan::InclusiveSum(nullptr, need, proxy, inc, (int)E, s), "cub scan");
        char *ct;
        GK(tmp.get(ct, need), "cudaMalloc(tmp)");
        GK(cub::DeviceScan::InclusiveSum(ct, need, proxy, inc, (int)E, s), "cub scan");
        k_cuts<<<1, 1024, 0, s>>>(inc, E, n_parts, dcut); count_launch();
    }
    GK(cudaGetLastError(), "partition kernels");
    std::vector<unsigned long long> h(n_parts + 1);
    GK(cudaMemcpyAsync(h.data(), dcut, 8 * (n_parts + 1), cudaMemcpyDeviceToHost, s), "D2H(cuts)");
    GK(cudaStreamSynchronize(s), "partition");
    for (uint32_t p = 0; p <= n_parts; p++) cut[p] = h[p];
    return MAYURA_OK;
}

// Timestamps of a device-built graph (edge-id order), for mayura_partition_roots.
mayura_status copy_t_host(mayura_graph_s *g, std::vector<int64_t> &t) {
    int prev = 0;
    cudaGetDevice(&prev);
    cudaSetDevice(g->device);
    try {
        t.resize(g->E);
    } catch (const std::bad_alloc &) {
        cudaSetDevice(prev);
        return fail(MAYURA_E_OOM, "copy_t_host: out of host memory");
    }
    const cudaError_t e = g->E ? cudaMemcpy(t.data(), g->d_t, 8 * g->E, cudaMemcpyDeviceToHost) : cudaSuccess;
    cudaSetDevice(prev);
    if (e != cudaSuccess) return fail(MAYURA_E_CUDA, std::string("copy_t_host: ") + cudaGetErrorString(e));
    return MAYURA_OK;
}

// The enumeration's input ranks per list position, converted in place from the edge ids the build
// left there (once per graph; the counting path never reads them).
mayura_status ensure_ranks(mayura_graph_s *g) {
    if (g->ranks_ready || g->device < 0) return MAYURA_OK;
    const size_t N = (size_t)g->E + g->V;
    if (N) {
        k_ranks<<<blocks_for(N), kT>>>(g->d_out_rank, g->d_perm, (uint32_t)N);
        k_ranks<<<blocks_for(N), kT>>>(g->d_in_rank, g->d_perm, (uint32_t)N);
        count_launch(2);
    }
    GK(cudaGetLastError(), "rank kernels");
    GK(cudaStreamSynchronize(0), "ranks");
    g->ranks_ready = true;
    return MAYURA_OK;
}

// Host copies of a device-built graph, for the inspection / partitioning calls.
mayura_status ensure_host(mayura_graph_s *g) {
    if (g->host_built || g->device < 0) return MAYURA_OK;
    int prev = 0;
    cudaGetDevice(&prev);
    cudaSetDevice(g->device);
    const size_t E = g->E, V1 = (size_t)g->V + 1, N = (size_t)g->E + g->V;
    try {
        g->src.resize(E); g->dst.resize(E); g->tr.resize(E); g->t.resize(E); g->perm.resize(E);
        g->out_off.resize(V1); g->in_off.resize(V1);
        g->out_ent.resize(2 * N); g->in_ent.resize(2 * N);
        g->eptr.resize(4 * E); g->out_ptr.resize(4 * N); g->in_ptr.resize(4 * N);
    } catch (const std::bad_alloc &) {
        cudaSetDevice(prev);
        return fail(MAYURA_E_OOM, "ensure_host: out of host memory");
    }
    std::vector<uint32_t> perm32(E);
    cudaError_t e = cudaSuccess;
    auto cp = [&](void *h, const void *d, size_t b) {
        if (e == cudaSuccess && b) e = cudaMemcpy(h, d, b, cudaMemcpyDeviceToHost);
    };
    cp(g->src.data(), g->d_src, 4 * E);
    cp(g->dst.data(), g->d_dst, 4 * E);
    cp(g->tr.data(), g->d_tr, 4 * E);
    cp(g->t.data(), g->d_t, 8 * E);
    cp(perm32.data(), g->d_perm, 4 * E);
    cp(g->out_off.data(), g->d_out_off, 4 * V1);
    cp(g->in_off.data(), g->d_in_off, 4 * V1);
    cp(g->out_ent.data(), g->d_out_ent, 8 * N);
    cp(g->in_ent.data(), g->d_in_ent, 8 * N);
    cp(g->eptr.data(), g->d_eptr, 16 * E);
    cp(g->out_ptr.data(), g->d_out_ptr, 16 * N);
    cp(g->in_ptr.data(), g->d_in_ptr, 16 * N);
    cudaSetDevice(prev);
    if (e != cudaSuccess) return fail(MAYURA_E_CUDA, std::string("ensure_host: ") + cudaGetErrorString(e));
    for (size_t i = 0; i < E; i++) g->perm[i] = perm32[i];
    g->host_built = true;
    return MAYURA_OK;
}

}  // namespace mayura
