/*
 * mayura.h -- C ABI of the B200-native MG-Tree temporal motif co-mining library
 * (libmayura.so).  Paper: "Mayura: Exploiting Similarities in Motifs for Temporal
 * Co-Mining", arXiv 2507.14813 (PAPER.md in the reference tree).
 *
 * Problem statement (Fig. 4 "Example User Query"; §2.1
 * PAPER.md:117-133): given a temporal graph G, a group of delta-temporal motifs
 * MG = {M_1..M_k} and a window delta, return for every motif the number of edge
 * tuples (e_1..e_m) with t(e_1) < ... < t(e_m), t(e_m) - t(e_1) <= delta, that
 * match the motif under a one-to-one (injective) vertex map.  Co-mining walks
 * the MG-Tree (Algorithm 2) with Algorithm 3
 * and must return exactly the per-motif counts of independent mining
 * (Algorithm 1).  Readings of ambiguous passages: DESIGN.md §3.
 *
 * Conventions
 *   - Every function returns mayura_status (0 == MAYURA_OK, negative == error)
 *     except the free functions and mayura_last_error.  On error, a message is
 *     available from mayura_last_error() (thread-local, valid until the next
 *     call on the same thread); outputs are left untouched.
 *   - Input arrays are BORROWED for the duration of the call and copied; the
 *     library never retains caller pointers.
 *   - Handles are owned by the caller and released with mayura_free_*.  Calls
 *     on one handle are not re-entrant (the graph handle owns per-query
 *     scratch); distinct handles are independent.
 *   - Edge ids: edges are stably sorted by (t, input rank); id i is the i-th
 *     edge in that order.  Root ranges [root_begin, root_end) are in those ids;
 *     a match belongs to the range that contains its FIRST edge, so counts are
 *     additive over any partition of [0, E).
 *   - Timestamps are int64 and delta shares their unit.
 */
#ifndef MAYURA_H
#define MAYURA_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
    MAYURA_OK = 0,
    MAYURA_E_INVALID = -1, /* bad argument: vertex id >= n_vertices, motif self-loop edge,
                              delta < 0, bad root range, empty group, NULL pointer */
    MAYURA_E_LIMIT = -2,   /* a documented limit is exceeded (see MAYURA_MAX_*) */
    MAYURA_E_OOM = -3,     /* host or device allocation failed */
    MAYURA_E_CUDA = -4,    /* a CUDA runtime call or kernel failed (message has the CUDA error) */
    MAYURA_E_STATE = -5    /* handle in the wrong state (e.g. host-only graph passed to comine) */
} mayura_status;

#define MAYURA_MAX_EDGES 8        /* edges per motif (the paper uses <= 5) */
#define MAYURA_MAX_V 16           /* vertices per motif */
#define MAYURA_MAX_MOTIFS 4096    /* motifs per group */
#define MAYURA_MAX_TRIE_NODES 4096 /* distinct canonical edge prefixes per group */
#define MAYURA_MAX_E 0xFFFFFFFEull /* edges per graph (32-bit edge ids) */
#define MAYURA_MAX_VERTICES 0x7FFFFFFFu

typedef struct mayura_graph_s *mayura_graph;   /* opaque: host arrays (+ device arrays) */
typedef struct mayura_mgtree_s *mayura_mgtree; /* opaque: compiled MG-Tree table + delta */

/* ---------------------------------------------------------------- graph ---
 * mayura_load_graph -- build the time-sorted edge arrays and the per-vertex
 * out/in adjacency sorted by timestamp ("Data-Loading", §4.2:
 * "CSR ... with edges sorted in ascending order of timestamps"), then copy them
 * to GPU `device`.
 *   src, dst   : n_edges vertex ids (< n_vertices), host memory, input order.
 *   t          : n_edges int64 timestamps, host memory, any order, ties allowed.
 *   device     : CUDA device ordinal, or -1 for a HOST-ONLY graph (no CUDA call is
 *                made; usable with mayura_graph_info / mayura_graph_export /
 *                mayura_partition_roots, rejected by mayura_comine with E_STATE).
 *   out        : receives the new handle.
 * Self-loops and parallel edges are kept (they are distinct edges; a self-loop
 * never matches a motif edge).  Errors: E_INVALID (NULL pointers with
 * n_edges > 0, vertex id out of range), E_LIMIT (n_edges > MAYURA_MAX_E or
 * n_vertices > MAYURA_MAX_VERTICES), E_OOM, E_CUDA. */
mayura_status mayura_load_graph(const uint32_t *src, const uint32_t *dst, const int64_t *t,
                                uint64_t n_edges, uint32_t n_vertices, int device,
                                mayura_graph *out);

/* Sizes of a loaded graph.  device_bytes = bytes held on the GPU (0 if host-only).
 * Any output pointer may be NULL. */
mayura_status mayura_graph_info(mayura_graph g, uint64_t *n_edges, uint32_t *n_vertices,
                                uint64_t *device_bytes);

/* Copy the host-side build results into caller buffers (any may be NULL):
 *   src,dst,tr [E] u32 / t [E] i64 : edges in id order; tr[e] = id of the first
 *                                    edge with timestamp t[e] (time rank);
 *   perm [E] u64                   : input rank of edge id e;
 *   out_off,in_off [V+1] u32       : CSR offsets; the list of vertex x occupies
 *                                    [off[x], off[x+1]-1) and is followed by one sentinel
 *                                    entry (0xFFFFFFFF, 0xFFFFFFFF) at off[x+1]-1;
 *   out_ent,in_ent [2(E+V)] u32    : CSR entries (tr, neighbour) pairs, each list in
 *                                    increasing edge id (= timestamp) order. */
mayura_status mayura_graph_export(mayura_graph g, uint32_t *src, uint32_t *dst, int64_t *t,
                                  uint32_t *tr, uint64_t *perm, uint32_t *out_off,
                                  uint32_t *out_ent, uint32_t *in_off, uint32_t *in_ent);

/* Successor pointers of every edge, eptr [4E] u32: for edge e = (a, b),
 * eptr[4e+0..3] = first position (in out_ent / in_ent entry units) with time rank > tr[e]
 * in out(a), in(b), out(b), in(a) respectively (the sentinel position if none). */
mayura_status mayura_graph_export_succ(mayura_graph g, uint32_t *eptr);

void mayura_free_graph(mayura_graph g);

/* --------------------------------------------------------------- mg-tree ---
 * mayura_build_mgtree -- compile a motif group into an MG-Tree table
 * (Algorithm 2 "MG-Tree Construction"; node definition
 * PAPER.md:441-466).  Each motif is canonicalised (first-appearance labels, u
 * before v); the tree is the trie of canonical edge sequences (one node per
 * distinct prefix; the paper's MG-Tree is its path-compressed view, reported by
 * mayura_mgtree_info / mayura_mgtree_dump).  Per child the compiler records the
 * candidate source ("anchor"): out-adjacency of a mapped u, in-adjacency of a
 * mapped v, or the global edge array when neither endpoint is mapped (Algo 1
 * l.210; readings R5, R6).
 *   motif_edges : concatenated (u, v) pairs of all motifs, temporal order.
 *                 Labels are arbitrary uint32 (need not be dense or canonical).
 *   motif_len   : n_motifs entries, edges per motif (1..MAYURA_MAX_EDGES).
 *   delta       : window, >= 0, in timestamp units.
 * Duplicate motifs (equal after canonicalisation) are accepted; each gets the
 * same count.  Errors: E_INVALID (NULL, n_motifs == 0, motif self-loop edge,
 * delta < 0), E_LIMIT (motif length, vertices, motifs or trie nodes over
 * MAYURA_MAX_*), E_OOM.  No CUDA call is made (the device copy of the table is
 * made lazily by the first mayura_comine on a device). */
mayura_status mayura_build_mgtree(const uint32_t *motif_edges, const uint32_t *motif_len,
                                  uint32_t n_motifs, int64_t delta, mayura_mgtree *out);

/* Shape of a compiled tree (any output may be NULL):
 *   n_trie_nodes : distinct canonical prefixes (kernel table rows);
 *   n_mg_nodes   : nodes of the path-compressed MG-Tree (root, branching
 *                  prefixes, query motifs), PAPER.md:441-466;
 *   max_vertices, max_edges : over the group;
 *   sm           : Similarity Metric, PAPER.md:954-961 (§6). */
mayura_status mayura_mgtree_info(mayura_mgtree m, uint32_t *n_motifs, uint32_t *n_trie_nodes,
                                 uint32_t *n_mg_nodes, uint32_t *max_vertices,
                                 uint32_t *max_edges, double *sm);

/* Text outline of the path-compressed MG-Tree (Fig. 6 style), one node per line:
 * "<indent>[Q=i,j] C=(0>1,1>2,...)".  Writes at most cap bytes (NUL-terminated)
 * into buf (may be NULL when cap == 0) and stores the full length + 1 in *needed. */
mayura_status mayura_mgtree_dump(mayura_mgtree m, char *buf, size_t cap, size_t *needed);

void mayura_free_mgtree(mayura_mgtree m);

/* ---------------------------------------------------------------- mining ---
 * mayura_comine -- co-mine every motif of the group over root edges
 * [root_begin, root_end) on the graph's GPU (Algorithm 3 "Co-Mining",
 * PAPER.md:638-711; one depth-first search per root edge).
 *   cuda_stream      : cudaStream_t to launch on, or NULL for the legacy default stream.
 *   counts_out       : n_motifs uint64, input motif order.  Host memory if
 *                      counts_on_device == 0 (the call then synchronises the stream);
 *                      device memory on the graph's GPU if counts_on_device == 1
 *                      (the call only enqueues work; counts are valid once the stream
 *                      completes; suitable for an NCCL all-reduce).
 * Counts are overwritten (not accumulated).  Errors: E_INVALID (range, NULL),
 * E_STATE (host-only graph), E_CUDA. */
mayura_status mayura_comine(mayura_graph g, mayura_mgtree m, uint64_t root_begin,
                            uint64_t root_end, void *cuda_stream, uint64_t *counts_out,
                            int counts_on_device);

/* mayura_mine_independent -- the per-motif baseline: the same kernel run once per
 * motif on that motif's single-motif tree (what co-mining is compared against,
 * PAPER.md:930-934 §6 "The Baselines").  Same arguments and results as
 * mayura_comine; must return identical counts. */
mayura_status mayura_mine_independent(mayura_graph g, mayura_mgtree m, uint64_t root_begin,
                                      uint64_t root_end, void *cuda_stream,
                                      uint64_t *counts_out, int counts_on_device);

/* mayura_comine_ex -- mayura_comine (independent == 0) or mayura_mine_independent
 * (independent != 0), additionally recording the caller's cudaEvent_t `mid_event`
 * (may be NULL) on `cuda_stream` between the query's set-up and its co-mining kernels:
 * after window_end_kernel (warp / hybrid / lane / bfs forms), or after the counts memset
 * in the flat form (which has no window-end kernel: its level-0 pass computes the window
 * ends itself, so there the interval after the event includes step a2).  The caller times
 * the co-mining pass with events on the launching stream. */
mayura_status mayura_comine_ex(mayura_graph g, mayura_mgtree m, uint64_t root_begin,
                               uint64_t root_end, void *cuda_stream, uint64_t *counts_out,
                               int counts_on_device, int independent, void *mid_event);

/* mayura_comine_stats -- the same search in an instrumented kernel (not for timing; the
 * instrumented depth-first lane kernel, after the breadth-first level in the hybrid form):
 * stats_out[0..7] = roots visited (non-self-loop), search-tree nodes expanded (partial
 * matches whose children were examined), windows located, in-window entries examined,
 * binary-search probes (window starts located by search), lane iterations that loaded an
 * entry, implementation bytes, matches counted; stats_out[8..9] = load-
 * balance offloads (partial matches handed to a warp's task stack), contexts processed.
 * Roots, nodes, windows, entries and matches are properties of the search tree, identical
 * in every kernel form; bench.py computes SURVEY.md's B_alg from them.  With the
 * environment variable MAYURA_WDFS_STATS=1 (and the warp form) the instrumented warp kernel
 * runs instead and reuses the fields for its round counters (tools/wdfs_stats.py).
 * stats_out must hold 10 entries.  Host output; synchronises. */
mayura_status mayura_comine_stats(mayura_graph g, mayura_mgtree m, uint64_t root_begin,
                                  uint64_t root_end, int independent, uint64_t *stats_out);

/* ----------------------------------------------------------- enumeration ---
 * mayura_enumerate -- list every match instead of counting it (the paper's second
 * output: "a comprehensive list of all matching motifs (enumeration)", PAPER.md:130;
 * query option "counted or enumerated"; Algo 1 l.201 / Algo 3 l.662
 * add the match to an enumeration list).  Root edges [root_begin, root_end) as in
 * mayura_comine; a match belongs to the range of its first edge (reading R16).
 *   tuples_out     : uint32 words.  Motif q's matches occupy words
 *                    [W_q, W_q + count_q * len_q), W_q = sum_{j<q} count_j * len_j
 *                    (len_q = edges of motif q); each match is len_q consecutive
 *                    words = the INPUT indices (positions in the src/dst/t arrays given
 *                    to mayura_load_graph) of the matched edges in motif edge order
 *                    (strictly increasing time).  The order of matches within a motif
 *                    is unspecified.  Device memory on the graph's GPU if
 *                    tuples_on_device == 1, else host memory.  NULL: size query only.
 *   capacity_words : words available at tuples_out.
 *   counts_out     : host, n_motifs uint64 (always filled, as mayura_comine).
 *   words_needed   : host, may be NULL: sum_q count_q * len_q.
 * Synchronises the stream.  Errors: E_INVALID (range, NULL handle / counts_out),
 * E_STATE (host-only graph), E_LIMIT (capacity_words < words needed -- counts_out and
 * words_needed are still filled; or > 96 distinct motifs in the group), E_CUDA. */
mayura_status mayura_enumerate(mayura_graph g, mayura_mgtree m, uint64_t root_begin,
                               uint64_t root_end, void *cuda_stream, uint32_t *tuples_out,
                               uint64_t capacity_words, int tuples_on_device,
                               uint64_t *counts_out, uint64_t *words_needed);

/* mayura_comine_heuristic -- the paper's rule for whether co-mining the group beats
 * mining each motif on its own (§6 "Heuristic for Co-Mining"; the
 * listing itself is figure-only, reading R18): co-mine if the graph is
 * bipartite (co-mining "has always resulted in a performance improvement" there) or the
 * group's Similarity Metric is >= 0.44.
 *   use_comine : 1 = co-mine, 0 = mine independently.    (each output may be NULL)
 *   bipartite  : 1 if the underlying undirected graph is 2-colourable (a self-loop is
 *                an odd cycle), else 0.
 *   sm         : the group's Similarity Metric (as mayura_mgtree_info).
 * Host computation (union-find over the edges); a device-built graph's edge arrays are
 * downloaded once.  Errors: E_INVALID (NULL handle), E_OOM, E_CUDA. */
mayura_status mayura_comine_heuristic(mayura_graph g, mayura_mgtree m, int *use_comine,
                                      int *bipartite, double *sm);

/* ------------------------------------------------------------ multi-GPU ---
 * mayura_partition_roots -- split [0, E) into n_parts contiguous root ranges
 * (timestamp ranges) of balanced estimated work.  Proxy work of root r:
 * p(r) = 1 + min(s_r, 65535)^2, s_r = entries with t_r < t <= t_r + delta in the four
 * adjacency lists at the root's endpoints (out(src), in(dst), out(dst), in(src)); cut p
 * at the first root whose proxy prefix sum reaches floor(total * p / n_parts).
 * Deterministic: host arithmetic for host-only graphs, the same integer arithmetic on
 * the GPU for device-built graphs (identical bounds, tests/test_gpu_parity.py).
 * bounds_out: n_parts + 1 entries, bounds_out[0] = 0, bounds_out[n_parts] = E,
 * non-decreasing.  Errors: E_INVALID (NULL, n_parts == 0, delta < 0), E_CUDA. */
mayura_status mayura_partition_roots(mayura_graph g, int64_t delta, uint32_t n_parts,
                                     uint64_t *bounds_out);

/* Kernel form mayura_comine uses for this graph: "flat" (level-synchronous,
 * entry-parallel; the default when the graph arrays fit in L2), "warp" (the warp-synchronous
 * depth-first kernel over a shared-memory stack of window pieces; the default otherwise), or
 * "hybrid" / "lane" / "bfs" / "mixed" when forced with the MAYURA_KERNEL environment
 * variable; "none" for NULL or host-only graphs.  All forms return identical counts.
 * Static string. */
const char *mayura_kernel_form(mayura_graph g);

/* Form the last mayura_enumerate call on this graph took (enumeration row):
 * "flat" (the flat counting pass, then a window + entry pass per MG-Tree level writing
 * tuples), "depth-first" (per-warp count pass, CUB scan, write pass; used when
 * MAYURA_ENUM_LANE is set or a flat buffer overflowed), or "none" (NULL graph, or no
 * enumeration has written tuples yet).  Host-only, no CUDA call.  Static string. */
const char *mayura_enum_form(mayura_graph g);

/* Thread-local message for the last failing call on this thread ("" if none). */
const char *mayura_last_error(void);

/* Library version string, e.g. "mayura-b200 0.3 sm_100a". */
const char *mayura_version(void);

/* Number of the library's own (hand-written) kernel launches enqueued so far in this
 * process, all devices and handles (CUB's sort/scan launches inside the graph build are not
 * included).  Monotonic; the difference around a call sequence is its launch count. */
uint64_t mayura_launch_count(void);

#ifdef __cplusplus
}
#endif
#endif /* MAYURA_H */
