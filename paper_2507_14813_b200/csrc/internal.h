// internal.h -- shared host/device declarations of libmayura (not part of the ABI).
#pragma once

#include <stdint.h>

#include <string>
#include <vector>

#include "../../include/mayura.h"

namespace mayura {

// ------------------------------------------------------------------ errors --
mayura_status fail(mayura_status s, const std::string &msg);
void clear_error();

// ------------------------------------------------------------ device table --
// One row per trie node = one distinct canonical edge prefix.
// Rows are laid out in BFS order with the children of every node contiguous and
// grouped by anchor, so a group is a contiguous child range.
enum AnchorKind : uint8_t { ANCHOR_OUT = 0, ANCHOR_IN = 1, ANCHOR_GLOBAL = 2 };
static constexpr uint8_t CLS_NEW = 0xFF;  // "graph vertex not yet in the image of m2g"

struct DNode {             // 8 bytes
    uint8_t want;          // OUT child: mapped motif vertex the dst must equal, or CLS_NEW
    uint8_t n_new;         // motif vertices this node's edge maps for the first time (0,1,2)
    uint8_t nv;            // mapped motif vertices after this node's edge
    uint8_t flags;         // bit0: completion (some motif == this prefix), bit1: has children
    uint16_t group_begin;  // groups of this node's children
    uint16_t group_end;
};
// Where a group's window starts (DESIGN.md §5 "successor pointers"): P(e) of the edge
// matched at this node -- slot 0 out(src), 1 in(dst), 2 out(dst), 3 in(src) -- gives
// the exact first position after t_e; the root edge's R(r) gives a lower bound for
// lists of motif vertices 0/1 (forward skip); otherwise a lane-cooperative search.
enum StartKind : uint8_t {
    START_P0 = 0, START_P1, START_P2, START_P3,  // exact, from the node's own edge
    START_R0 = 4, START_R1, START_R2, START_R3,  // lower bound, from the root edge
    START_SEARCH = 8,                           // 32-ary search in the anchor's list
    START_GLOBAL = 9                            // all edges: search the time-rank array
};
struct DGroup {            // 8 bytes
    uint8_t kind;          // AnchorKind
    uint8_t anchor;        // motif vertex whose adjacency is scanned (OUT: u, IN: v)
    uint8_t n_inner;       // children that have children themselves
    uint8_t start;         // StartKind
    uint16_t child_begin;  // contiguous node rows
    uint16_t child_end;
};
// NODE_SWEEP: every child group of the node is an OUT/IN list group whose window start comes
// from successor pointers (START_P*/START_R*), holds <= kSweepChildren children, all leaves --
// the kernel counts such a node's subtree for 32 candidates at once, one lane per candidate.
static constexpr uint8_t NODE_COMPLETION = 1, NODE_INNER = 2, NODE_SWEEP = 4;
static constexpr uint32_t kSweepChildren = 4;

struct Table {
    std::vector<DNode> nodes;          // row 0 = root (canonical edge 0->1)
    std::vector<DGroup> groups;
    std::vector<uint32_t> motif_node;  // per input motif: its row
    uint32_t max_vertices = 2, max_edges = 1;
};

}  // namespace mayura

// ------------------------------------------------------------------ handles --
struct mayura_graph_s {
    uint64_t E = 0;
    uint32_t V = 0;
    int device = -1;
    bool host_built = true;                 // false: built on the GPU, host arrays made lazily
    bool fresh_alloc = false;               // device scratch allocated since the last stream sync
    const char *last_enum_form = "none";   // form of the last mayura_enumerate (mayura_enum_form)
    // host build results (edge id order)
    std::vector<uint32_t> src, dst, tr;
    std::vector<int64_t> t;
    std::vector<uint64_t> perm;
    std::vector<uint32_t> out_off, in_off;  // V+1; list x = [off[x], off[x+1]-1), sentinel at off[x+1]-1
    std::vector<uint32_t> out_ent, in_ent;  // 2(E+V): (tr, nbr); sentinel = (0xFFFFFFFF, 0xFFFFFFFF)
    std::vector<uint32_t> eptr;             // 4E: P(e) = first list position with time > t_e in
                                            //     out(src e), in(dst e), out(dst e), in(src e)
    std::vector<uint32_t> out_ptr, in_ptr;  // 4(E+V): P(e) of each list entry's edge (sentinel: 0)
    // device arrays
    uint32_t *d_src = nullptr, *d_dst = nullptr, *d_tr = nullptr, *d_hi = nullptr;
    int64_t *d_t = nullptr;
    uint32_t *d_out_off = nullptr, *d_in_off = nullptr;
    uint32_t *d_out_ent = nullptr, *d_in_ent = nullptr;  // uint2 {tr, nbr}
    uint32_t *d_eptr = nullptr, *d_out_ptr = nullptr, *d_in_ptr = nullptr;  // uint4
    uint32_t *d_perm = nullptr;                           // input rank of edge id (GPU-built graphs)
    char *d_arena = nullptr;                              // the one allocation holding the arrays above
    uint32_t *d_out_rank = nullptr, *d_in_rank = nullptr; // input rank of the edge behind each list position
    bool ranks_ready = false;  // d_*_rank hold edge ids until the first enumeration converts them (ensure_ranks)
    uint32_t *d_enum = nullptr;                           // enumeration scratch (per-warp counts / bases)
    size_t enum_bytes = 0;
    uint32_t *d_queue = nullptr;                         // work-queue cursors
    unsigned long long *d_counts = nullptr;              // scratch counts (host-output calls)
    uint32_t d_counts_cap = 0;
    unsigned long long *d_stats = nullptr;
    unsigned long long *d_dbg = nullptr;                 // MAYURA_DEBUG_WARPS timeline
    uint32_t *d_bfs[2] = {nullptr, nullptr};             // BFS frontier buffers (ping-pong)
    uint32_t *d_bfs_ctl = nullptr, *d_bfs_long = nullptr;
    uint32_t *d_flat_win = nullptr;                      // flat form: window pieces (uint4)
    uint64_t flat_win_bytes = 0;
    uint32_t *d_light = nullptr;                         // hybrid: light roots listed by the BFS level (E + 32)
    uint32_t *d_wspill = nullptr;                        // warp kernel: per-warp stack spill area
    uint64_t wspill_bytes = 0;
    size_t bfs_bytes = 0;
    int bfs_nbufs = 0;
    uint32_t bfs_words = 0;
    uint32_t bfs_seg_cap = 0, bfs_long_cap = 0;
    uint64_t device_bytes = 0;
    uint64_t graph_bytes = 0;                            // the graph arrays alone (no scratch)
};

struct mayura_mgtree_s {
    int64_t delta = 0;
    uint32_t n_motifs = 0;
    std::vector<std::vector<std::pair<uint32_t, uint32_t>>> canon;  // canonical motifs
    mayura::Table group;                  // co-mining table
    std::vector<mayura::Table> single;    // one single-motif table per motif
    // path-compressed MG-Tree view
    uint32_t n_mg_nodes = 0;
    double sm = 0.0;
    std::string dump;
    // lazily uploaded device copies: [0] = group, [1..k] = singles
    int dev = -1;
    std::vector<void *> d_tables;
};

namespace mayura {
// device padding: 32 trailing elements after every per-edge / per-position array and 64
// sentinel-valued entries after the adjacency, so batched and read-ahead loads never leave
// the allocation
constexpr size_t kPadE = 32, kPadEnt = 64;
mayura_status build_graph_device(const uint32_t *src, const uint32_t *dst, const int64_t *t, uint64_t E,
                                 uint32_t V, mayura_graph_s *g);
mayura_status ensure_host(mayura_graph_s *g);
mayura_status ensure_ranks(mayura_graph_s *g);
mayura_status copy_t_host(mayura_graph_s *g, std::vector<int64_t> &t);
// device path of mayura_partition_roots: cut[p] (1 <= p < n_parts) = first root index whose
// proxy prefix reaches floor(total * p / n_parts) (capi.cpp documents the proxy)
mayura_status partition_device(mayura_graph_s *g, int64_t delta, uint32_t n_parts, uint64_t *cut);
// Library device memory comes from the device's stream-ordered pool with a retained release
// threshold, so load / free / scratch-growth cycles reuse memory instead of paying
// cudaMalloc / cudaFree (the e2e path builds and drops a graph per step).  dmalloc/dfree
// order on the legacy default stream; callers synchronise before first use on another stream.
int dmalloc(void **p, size_t bytes);
// hand-written kernel launches enqueued by this library (mayura_launch_count)
void count_launch(uint64_t n = 1);  // cudaError_t as int (keeps this header CUDA-free)
void dfree(void *p);
mayura_status build_graph_host(const uint32_t *src, const uint32_t *dst, const int64_t *t,
                               uint64_t E, uint32_t V, mayura_graph_s *g);
mayura_status compile_tree(const uint32_t *motif_edges, const uint32_t *motif_len,
                           uint32_t n_motifs, int64_t delta, mayura_mgtree_s *m);
int host_threads();
// MAYURA_TRACE=1: synchronise the device and print the host time since the previous trace
// point (diagnostic of the e2e path; perturbs timing, never on by default)
void trace(const char *what);
}  // namespace mayura

namespace mayura {
void free_mgtree_device(mayura_mgtree_s *m);
}
