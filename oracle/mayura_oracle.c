/*
 * mayura_oracle.c -- CPU ORACLE.  TEST INFRASTRUCTURE ONLY.
 *
 * Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl
 * reference legs may load this library.  It shares NO code with the CUDA path
 * (paper_2507_14813_b200/): its own sort, its own adjacency, its own matcher.
 *
 * What it computes (the plain definition, §2.1 "A delta-Temporal
 * Motif" / "Temporal Motif Mining"): for a motif M = ((u_1,v_1),...,(u_m,v_m)),
 *
 *   count(M, G, delta) = #{ (e_1..e_m) : t(e_1) < ... < t(e_m),  t(e_m) - t(e_1) <= delta,
 *                           exists injective phi: V_M -> V_G, phi(u_j)=src(e_j), phi(v_j)=dst(e_j) }
 *
 * Two implementations (+ O2's enumeration form, oracle_enumerate):
 *   O1  oracle_bruteforce  -- the definition written out: enumerate increasing
 *       tuples of edges in time order, test the window, then build phi edge by
 *       edge and test consistency + injectivity.  Guarded (small inputs only).
 *   O2  oracle_backtrack   -- Algorithm 1 "Temporal Motif Mining" (PAPER.md:174-265,
 *       §2.2) step by step, mining every motif of the group INDEPENDENTLY, with
 *       the readings of DESIGN.md §3:
 *         R1 strict timestamp order (ties never co-occur)
 *         R2 inclusive window t_m - t_1 <= delta               PAPER.md:125, Algo1 l.214
 *         R3 order test skips t <= t_prev (not only <)          Algo1 l.214 garble
 *         R4 full injectivity (one-to-one correspondence)
 *         R9 RollBackEdge(u_G, v_G) (the paper passes (u,u))    Algo1 l.232 typo
 *       Candidate selection is the paper's literal rule (Algo1 l.210):
 *       out-neighbourhood N(u_G) if u_M is mapped, else ALL edges (restricted to the
 *       time window by binary search on the time-sorted edge array; the CUDA path
 *       instead uses in-adjacency -- the two must agree).
 *       Parallelised over first-edge candidates (roots) with pthreads, as the
 *       paper's CPU task manager does (§4.5).
 *
 * Edge ids: edges are stably sorted by (t, input rank); a root
 * range [root_begin, root_end) refers to those sorted ids.  A match belongs to
 * the range containing its first edge (reading R16).
 *
 * Error behaviour: functions return 0 on success, -1 on invalid input, -2 when a
 * guard is exceeded, -3 on allocation failure.
 */
#include <pthread.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#define OR_MAX_EDGES 8
#define OR_MAX_LABEL 64 /* motif vertex labels must be < 64 */

/* ------------------------------------------------------------------ graph -- */
typedef struct {
    uint64_t E;
    uint32_t V;
    uint32_t *src, *dst; /* sorted by (t, input rank) */
    int64_t *t;
    uint64_t *out_off;   /* V+1 */
    uint64_t *out_eid;   /* E: out-edges of each vertex in increasing edge id (= time) order */
    uint64_t *rank;      /* E: input rank (position in the caller's arrays) of each sorted edge */
} og_graph;

typedef struct { int64_t t; uint64_t rank; } og_key;

static int og_key_cmp(const void *a, const void *b) {
    const og_key *x = (const og_key *)a, *y = (const og_key *)b;
    if (x->t != y->t) return x->t < y->t ? -1 : 1;
    return x->rank < y->rank ? -1 : (x->rank > y->rank);
}

static void og_free(og_graph *g) {
    free(g->src); free(g->dst); free(g->t); free(g->out_off); free(g->out_eid); free(g->rank);
    memset(g, 0, sizeof(*g));
}

static int og_build(og_graph *g, const uint32_t *src, const uint32_t *dst, const int64_t *t,
                    uint64_t E, uint32_t V) {
    memset(g, 0, sizeof(*g));
    g->E = E; g->V = V;
    for (uint64_t i = 0; i < E; i++)
        if (src[i] >= V || dst[i] >= V) return -1;
    og_key *k = (og_key *)malloc(sizeof(og_key) * (E ? E : 1));
    g->src = (uint32_t *)malloc(4 * (E ? E : 1));
    g->dst = (uint32_t *)malloc(4 * (E ? E : 1));
    g->t = (int64_t *)malloc(8 * (E ? E : 1));
    g->out_off = (uint64_t *)calloc((size_t)V + 1, 8);
    g->out_eid = (uint64_t *)malloc(8 * (E ? E : 1));
    g->rank = (uint64_t *)malloc(8 * (E ? E : 1));
    if (!k || !g->src || !g->dst || !g->t || !g->out_off || !g->out_eid || !g->rank) { free(k); og_free(g); return -3; }
    for (uint64_t i = 0; i < E; i++) { k[i].t = t[i]; k[i].rank = i; }
    qsort(k, E, sizeof(og_key), og_key_cmp);
    for (uint64_t i = 0; i < E; i++) {
        uint64_t r = k[i].rank;
        g->src[i] = src[r]; g->dst[i] = dst[r]; g->t[i] = t[r]; g->rank[i] = r;
    }
    free(k);
    /* out adjacency: counting sort by source, edge ids visited in increasing order */
    for (uint64_t i = 0; i < E; i++) g->out_off[g->src[i] + 1]++;
    for (uint32_t v = 0; v < V; v++) g->out_off[v + 1] += g->out_off[v];
    uint64_t *fill = (uint64_t *)malloc(8 * ((size_t)V + 1));
    if (!fill) { og_free(g); return -3; }
    memcpy(fill, g->out_off, 8 * ((size_t)V + 1));
    for (uint64_t i = 0; i < E; i++) g->out_eid[fill[g->src[i]]++] = i;
    free(fill);
    return 0;
}

/* first index i in [lo, hi) with t[key(i)] > x, keys given by an id array (or identity) */
static uint64_t og_first_after(const og_graph *g, const uint64_t *ids, uint64_t lo, uint64_t hi, int64_t x) {
    while (lo < hi) {
        uint64_t mid = lo + (hi - lo) / 2;
        int64_t tm = g->t[ids ? ids[mid] : mid];
        if (tm > x) hi = mid; else lo = mid + 1;
    }
    return lo;
}

/* ------------------------------------------------------------ O1: brute force */
typedef struct {
    const og_graph *g;
    const uint32_t *mu, *mv; /* motif edges */
    uint32_t m;
    int64_t delta;
    uint64_t tup[OR_MAX_EDGES];
    uint64_t count;
} o1_ctx;

/* Does the tuple admit an injective phi with phi(u_j)=src(e_j), phi(v_j)=dst(e_j)? */
static int o1_structure_ok(const o1_ctx *c) {
    int64_t phi[OR_MAX_LABEL];
    for (int i = 0; i < OR_MAX_LABEL; i++) phi[i] = -1;
    for (uint32_t j = 0; j < c->m; j++) {
        uint32_t a = c->mu[j], b = c->mv[j];
        int64_t ga = c->g->src[c->tup[j]], gb = c->g->dst[c->tup[j]];
        if (phi[a] == -1) phi[a] = ga; else if (phi[a] != ga) return 0;
        if (phi[b] == -1) phi[b] = gb; else if (phi[b] != gb) return 0;
    }
    /* injective: distinct motif vertices map to distinct graph vertices */
    for (int a = 0; a < OR_MAX_LABEL; a++) {
        if (phi[a] == -1) continue;
        for (int b = a + 1; b < OR_MAX_LABEL; b++)
            if (phi[b] == phi[a]) return 0;
    }
    return 1;
}

static void o1_rec(o1_ctx *c, uint32_t j) {
    if (j == c->m) { c->count += (uint64_t)o1_structure_ok(c); return; }
    const og_graph *g = c->g;
    for (uint64_t e = c->tup[j - 1] + 1; e < g->E; e++) {
        /* window: t_m - t_1 <= delta; t_m >= t_1 here, so the difference is exact
         * in u64 for any int64 timestamps (a signed subtraction overflows for t_1 < 0 < t_m) */
        if ((uint64_t)g->t[e] - (uint64_t)g->t[c->tup[0]] > (uint64_t)c->delta) break;
        if (!(g->t[e] > g->t[c->tup[j - 1]])) continue;     /* strict order t_{j-1} < t_j */
        c->tup[j] = e;
        o1_rec(c, j + 1);
    }
}

int oracle_bruteforce(const uint32_t *src, const uint32_t *dst, const int64_t *t, uint64_t E,
                      uint32_t V, const uint32_t *motif_edges, uint32_t m, int64_t delta,
                      uint64_t root_begin, uint64_t root_end, uint64_t guard, uint64_t *count_out) {
    if (m == 0 || m > OR_MAX_EDGES || delta < 0 || root_begin > root_end || root_end > E) return -1;
    uint32_t mu[OR_MAX_EDGES], mv[OR_MAX_EDGES];
    for (uint32_t j = 0; j < m; j++) {
        mu[j] = motif_edges[2 * j]; mv[j] = motif_edges[2 * j + 1];
        if (mu[j] >= OR_MAX_LABEL || mv[j] >= OR_MAX_LABEL || mu[j] == mv[j]) return -1;
    }
    if (E > guard) return -2;
    og_graph g;
    int rc = og_build(&g, src, dst, t, E, V);
    if (rc) return rc;
    o1_ctx c;
    memset(&c, 0, sizeof(c));
    c.g = &g; c.mu = mu; c.mv = mv; c.m = m; c.delta = delta;
    for (uint64_t e = root_begin; e < root_end; e++) {
        c.tup[0] = e;
        o1_rec(&c, 1);
    }
    *count_out = c.count;
    og_free(&g);
    return 0;
}

/* --------------------------------------------------- O2: Algorithm 1 (Mackey) */
typedef struct {
    const og_graph *g;
    const uint32_t *mu, *mv;
    uint32_t m;
    int64_t delta;
    /* Book-Keeping Context (Algo 1 line 3) */
    uint64_t e_stack[OR_MAX_EDGES];
    uint32_t top;
    int64_t m2g[OR_MAX_LABEL];
    int32_t *g2m;      /* V entries, -1 = unmapped */
    uint32_t *incnt;   /* V entries */
    uint64_t count;
    uint32_t *out;     /* enumeration list (Algo 1 l.201 "add to enumeration list"), or NULL */
    uint64_t cap;      /* tuples that fit in out */
} o2_ctx;

/* RollOnEdge (Algo 1 lines 240-245) */
static void o2_roll_on(o2_ctx *c, uint32_t uM, uint32_t vM, uint32_t uG, uint32_t vG) {
    c->m2g[uM] = uG; c->g2m[uG] = (int32_t)uM;
    c->m2g[vM] = vG; c->g2m[vG] = (int32_t)vM;
    c->incnt[uG]++; c->incnt[vG]++;
}

/* RollBackEdge (Algo 1 lines 247-263), with the (u_G, v_G) reading R9 */
static void o2_roll_back(o2_ctx *c, uint32_t uG, uint32_t vG) {
    c->incnt[uG]--; c->incnt[vG]--;
    if (c->incnt[uG] == 0) { int32_t uM = c->g2m[uG]; c->g2m[uG] = -1; c->m2g[uM] = -1; }
    if (c->incnt[vG] == 0) { int32_t vM = c->g2m[vG]; c->g2m[vG] = -1; c->m2g[vM] = -1; }
}

/* Structural constraints (Algo 1 line 219) + full injectivity (R4). */
static int o2_struct_ok(const o2_ctx *c, uint32_t uM, uint32_t vM, uint32_t eu, uint32_t ev) {
    int64_t uG = c->m2g[uM], vG = c->m2g[vM];
    if (uG != -1 && eu != (uint32_t)uG) return 0;
    if (vG != -1 && ev != (uint32_t)vG) return 0;            /* paper's check */
    if (uG == -1 && c->g2m[eu] != -1) return 0;              /* R4: eu already image of another motif vertex */
    if (vG == -1 && c->g2m[ev] != -1) return 0;              /* R4 */
    if (uG == -1 && vG == -1 && eu == ev) return 0;          /* R4: two new motif vertices, one graph vertex */
    return 1;
}

/* MatchEdge (Algo 1 lines 198-236) for motif edge e_M >= 1; e_M = 0 is the root loop. */
static void o2_match_edge(o2_ctx *c, uint32_t eM) {
    if (eM == c->m) {                                        /* line 199-201 */
        if (c->out && c->count < c->cap)                     /* enumeration: input ranks of e_1..e_m */
            for (uint32_t j = 0; j < c->m; j++) c->out[c->count * c->m + j] = (uint32_t)c->g->rank[c->e_stack[j]];
        c->count++;
        return;
    }
    const og_graph *g = c->g;
    uint32_t uM = c->mu[eM], vM = c->mv[eM];
    int64_t uG = c->m2g[uM];                                 /* line 205 */
    int64_t t_prev = g->t[c->e_stack[c->top - 1]];
    /* window end t_1 + delta (R2, PAPER.md:125 t_m - t_1 <= delta), saturated at INT64_MAX: delta >= 0,
     * so "t_1 > INT64_MAX - delta" is the overflow test and itself cannot overflow */
    int64_t t_root = g->t[c->e_stack[0]];
    int64_t t_last = t_root > INT64_MAX - c->delta ? INT64_MAX : t_root + c->delta;
    if (uG != -1) {                                          /* cands = N(u_G) */
        const uint64_t *ids = g->out_eid;
        uint64_t lo = g->out_off[uG], hi = g->out_off[uG + 1];
        for (uint64_t i = og_first_after(g, ids, lo, hi, t_prev); i < hi; i++) {
            uint64_t e = ids[i];
            if (g->t[e] <= t_prev) continue;                 /* R3 */
            if (g->t[e] > t_last) break;                     /* time-sorted: early break */
            if (!o2_struct_ok(c, uM, vM, g->src[e], g->dst[e])) continue;
            c->e_stack[c->top++] = e;
            o2_roll_on(c, uM, vM, g->src[e], g->dst[e]);
            o2_match_edge(c, eM + 1);
            c->top--;
            o2_roll_back(c, g->src[e], g->dst[e]);
        }
    } else {                                                 /* cands = G.edges */
        for (uint64_t e = og_first_after(g, NULL, 0, g->E, t_prev); e < g->E; e++) {
            if (g->t[e] <= t_prev) continue;
            if (g->t[e] > t_last) break;
            if (!o2_struct_ok(c, uM, vM, g->src[e], g->dst[e])) continue;
            c->e_stack[c->top++] = e;
            o2_roll_on(c, uM, vM, g->src[e], g->dst[e]);
            o2_match_edge(c, eM + 1);
            c->top--;
            o2_roll_back(c, g->src[e], g->dst[e]);
        }
    }
}

typedef struct {
    const og_graph *g;
    const uint32_t *mu, *mv;
    uint32_t m;
    int64_t delta;
    uint64_t next, end, chunk;
    pthread_mutex_t lock;
} o2_shared;

typedef struct { o2_shared *sh; uint64_t count; int err; } o2_worker;

static void *o2_thread(void *arg) {
    o2_worker *w = (o2_worker *)arg;
    o2_shared *sh = w->sh;
    o2_ctx c;
    memset(&c, 0, sizeof(c));
    c.g = sh->g; c.mu = sh->mu; c.mv = sh->mv; c.m = sh->m; c.delta = sh->delta;
    c.g2m = (int32_t *)malloc(4 * ((size_t)sh->g->V + 1));
    c.incnt = (uint32_t *)calloc((size_t)sh->g->V + 1, 4);
    if (!c.g2m || !c.incnt) { free(c.g2m); free(c.incnt); w->err = -3; return NULL; }
    for (uint32_t v = 0; v < sh->g->V; v++) c.g2m[v] = -1;
    for (int i = 0; i < OR_MAX_LABEL; i++) c.m2g[i] = -1;
    for (;;) {
        pthread_mutex_lock(&sh->lock);                        /* dynamic scheduling */
        uint64_t b = sh->next;
        sh->next = b + sh->chunk < sh->end ? b + sh->chunk : sh->end;
        uint64_t e_end = sh->next;
        pthread_mutex_unlock(&sh->lock);
        if (b >= e_end) break;
        for (uint64_t e = b; e < e_end; e++) {               /* e_M = 0: every edge is a candidate */
            uint32_t eu = c.g->src[e], ev = c.g->dst[e];
            if (!o2_struct_ok(&c, c.mu[0], c.mv[0], eu, ev)) continue;
            c.e_stack[0] = e; c.top = 1;
            o2_roll_on(&c, c.mu[0], c.mv[0], eu, ev);
            o2_match_edge(&c, 1);
            c.top = 0;
            o2_roll_back(&c, eu, ev);
        }
    }
    w->count = c.count;
    free(c.g2m); free(c.incnt);
    return NULL;
}

#include <time.h>
static double o2_now(void) {
    struct timespec ts;
    clock_gettime(CLOCK_MONOTONIC, &ts);
    return (double)ts.tv_sec + 1e-9 * (double)ts.tv_nsec;
}

/* Mine each of n_motifs motifs independently over each of n_ranges root ranges
 * [ranges[2r], ranges[2r+1]) of ONE graph build (the build -- sort + adjacency -- costs tens of
 * seconds at 63 M edges, so sampled runs query many ranges of one build).
 * motif_edges: concatenated (u,v) pairs; motif_len: edges per motif.
 * counts_out[r * n_motifs + i] receives the count of motif i over range r.
 * secs_out (may be NULL): [0] graph build seconds, [1] mining seconds.  n_threads <= 0: 1.
 * budget_s > 0: no range is started once budget_s seconds of mining have elapsed (at least one
 * range runs); *n_done (may be NULL) receives the number of ranges mined (a prefix). */
int oracle_backtrack_ranges(const uint32_t *src, const uint32_t *dst, const int64_t *t, uint64_t E,
                            uint32_t V, const uint32_t *motif_edges, const uint32_t *motif_len,
                            uint32_t n_motifs, int64_t delta, const uint64_t *ranges, uint32_t n_ranges,
                            int n_threads, uint64_t *counts_out, double *secs_out, double budget_s,
                            uint32_t *n_done) {
    if (n_motifs == 0 || delta < 0) return -1;
    for (uint32_t r = 0; r < n_ranges; r++)
        if (ranges[2 * r] > ranges[2 * r + 1] || ranges[2 * r + 1] > E) return -1;
    uint64_t off = 0;
    for (uint32_t i = 0; i < n_motifs; i++) {
        if (motif_len[i] == 0 || motif_len[i] > OR_MAX_EDGES) return -1;
        for (uint32_t j = 0; j < motif_len[i]; j++) {
            uint32_t a = motif_edges[2 * (off + j)], b = motif_edges[2 * (off + j) + 1];
            if (a >= OR_MAX_LABEL || b >= OR_MAX_LABEL || a == b) return -1;
        }
        off += motif_len[i];
    }
    double t0 = o2_now();
    og_graph g;
    int rc = og_build(&g, src, dst, t, E, V);
    if (rc) return rc;
    double t1 = o2_now();
    if (n_threads < 1) n_threads = 1;
    pthread_t *th = (pthread_t *)malloc(sizeof(pthread_t) * n_threads);
    o2_worker *wk = (o2_worker *)calloc(n_threads, sizeof(o2_worker));
    if (!th || !wk) { free(th); free(wk); og_free(&g); return -3; }
    uint32_t r = 0;
    for (; r < n_ranges; r++) {
        if (budget_s > 0 && r > 0 && o2_now() - t1 >= budget_s) break;  /* time-bounded sample */
        off = 0;
        for (uint32_t i = 0; i < n_motifs; i++) {
            uint32_t mu[OR_MAX_EDGES], mv[OR_MAX_EDGES];
            for (uint32_t j = 0; j < motif_len[i]; j++) {
                mu[j] = motif_edges[2 * (off + j)]; mv[j] = motif_edges[2 * (off + j) + 1];
            }
            off += motif_len[i];
            o2_shared sh;
            sh.g = &g; sh.mu = mu; sh.mv = mv; sh.m = motif_len[i]; sh.delta = delta;
            sh.next = ranges[2 * r]; sh.end = ranges[2 * r + 1]; sh.chunk = 256;
            pthread_mutex_init(&sh.lock, NULL);
            for (int w = 0; w < n_threads; w++) {
                wk[w].sh = &sh; wk[w].count = 0; wk[w].err = 0;
                pthread_create(&th[w], NULL, o2_thread, &wk[w]);
            }
            uint64_t total = 0;
            for (int w = 0; w < n_threads; w++) {
                pthread_join(th[w], NULL);
                total += wk[w].count;
                if (wk[w].err) rc = wk[w].err;
            }
            pthread_mutex_destroy(&sh.lock);
            counts_out[(uint64_t)r * n_motifs + i] = total;
        }
    }
    if (secs_out) { secs_out[0] = t1 - t0; secs_out[1] = o2_now() - t1; }
    if (n_done) *n_done = r;
    free(th); free(wk); og_free(&g);
    return rc;
}

/* Mine each of n_motifs motifs independently over roots [root_begin, root_end) (one range of
 * oracle_backtrack_ranges).  counts_out[i] receives the count of motif i. */
int oracle_backtrack(const uint32_t *src, const uint32_t *dst, const int64_t *t, uint64_t E,
                     uint32_t V, const uint32_t *motif_edges, const uint32_t *motif_len,
                     uint32_t n_motifs, int64_t delta, uint64_t root_begin, uint64_t root_end,
                     int n_threads, uint64_t *counts_out) {
    const uint64_t rg[2] = {root_begin, root_end};
    return oracle_backtrack_ranges(src, dst, t, E, V, motif_edges, motif_len, n_motifs, delta, rg, 1,
                                   n_threads, counts_out, NULL, 0.0, NULL);
}

/* Exposes the oracle's own (t, input rank) sort, so tests can check that the
 * CUDA path's edge ids refer to the same edges (range parity). */
int oracle_sorted_order(const int64_t *t, uint64_t E, uint64_t *perm_out) {
    og_key *k = (og_key *)malloc(sizeof(og_key) * (E ? E : 1));
    if (!k) return -3;
    for (uint64_t i = 0; i < E; i++) { k[i].t = t[i]; k[i].rank = i; }
    qsort(k, E, sizeof(og_key), og_key_cmp);
    for (uint64_t i = 0; i < E; i++) perm_out[i] = k[i].rank;
    free(k);
    return 0;
}

/* Enumeration ("a comprehensive list of all matching motifs"; Algo 1
 * l.201): O2 for ONE motif, single-threaded, writing each match as m words = the input
 * ranks of its edges in motif edge order, in the order Algorithm 1 finds them.  At most
 * cap_tuples tuples are written; *count_out = the number of matches (returns -2 if it
 * exceeds cap_tuples). */
int oracle_enumerate(const uint32_t *src, const uint32_t *dst, const int64_t *t, uint64_t E, uint32_t V,
                     const uint32_t *motif_edges, uint32_t m, int64_t delta, uint64_t root_begin,
                     uint64_t root_end, uint32_t *out, uint64_t cap_tuples, uint64_t *count_out) {
    if (m == 0 || m > OR_MAX_EDGES || delta < 0 || root_begin > root_end || root_end > E) return -1;
    uint32_t mu[OR_MAX_EDGES], mv[OR_MAX_EDGES];
    for (uint32_t j = 0; j < m; j++) {
        mu[j] = motif_edges[2 * j]; mv[j] = motif_edges[2 * j + 1];
        if (mu[j] >= OR_MAX_LABEL || mv[j] >= OR_MAX_LABEL || mu[j] == mv[j]) return -1;
    }
    og_graph g;
    int rc = og_build(&g, src, dst, t, E, V);
    if (rc) return rc;
    o2_ctx c;
    memset(&c, 0, sizeof(c));
    c.g = &g; c.mu = mu; c.mv = mv; c.m = m; c.delta = delta; c.out = out; c.cap = cap_tuples;
    c.g2m = (int32_t *)malloc(4 * ((size_t)V + 1));
    c.incnt = (uint32_t *)calloc((size_t)V + 1, 4);
    if (!c.g2m || !c.incnt) { free(c.g2m); free(c.incnt); og_free(&g); return -3; }
    for (uint32_t v = 0; v < V; v++) c.g2m[v] = -1;
    for (int i = 0; i < OR_MAX_LABEL; i++) c.m2g[i] = -1;
    for (uint64_t e = root_begin; e < root_end; e++) {       /* e_M = 0: every edge is a candidate */
        uint32_t eu = g.src[e], ev = g.dst[e];
        if (!o2_struct_ok(&c, mu[0], mv[0], eu, ev)) continue;
        c.e_stack[0] = e; c.top = 1;
        o2_roll_on(&c, mu[0], mv[0], eu, ev);
        o2_match_edge(&c, 1);
        c.top = 0;
        o2_roll_back(&c, eu, ev);
    }
    *count_out = c.count;
    free(c.g2m); free(c.incnt); og_free(&g);
    return c.count > cap_tuples ? -2 : 0;
}
