/*
 * tmotif.h — C ABI of libtmotif.so, a B200-native (sm_100a) δ-temporal motif
 * miner for the hot path of arxiv 2310.02800 ("Everest").  PAPER.md is cited
 * as P:<line>.
 *
 * The problem: a temporal graph is a set of directed timestamped
 * edges (u_i, v_i, t_i); a δ-temporal motif is an ordered list of motif edges
 * (u_i, v_i) (list order = temporal order) plus a window δ and optional
 * per-gap bounds δ_i.  A match is a tuple of graph edges
 * (e_1, ..., e_L) with
 *     e_1 < e_2 < ... < e_L  in the (t, input position) order,
 *     t(e_L) - t(e_1) <= δ,         t(e_{i+1}) - t(e_i) <= δ_i,
 * and an injective map φ of motif vertices to graph vertices with
 * φ(u_i) = src(e_i), φ(v_i) = dst(e_i).  The library counts the
 * matches or enumerates them into a caller buffer ("enumerated or
 * counted").  DESIGN.md lists every reading of the paper this encodes
 * (ties Q1, inclusive bounds Q2, self-loops Q4, all-edges candidates Q9 ...).
 *
 * Conventions
 *  - Every call returns tm_status; TM_OK = 0.  No C++ exception crosses the
 *    ABI.  On failure tm_last_error() returns a thread-local message.
 *  - Edge ids: the graph orders its edges stably by (t, input position); the
 *    id of an edge is its rank in that order (reading Q1).  Enumerated rows
 *    hold these ids; tm_graph_sorted_to_input maps them back.
 *  - Timestamps and δ are int64 in the caller's unit.  TM_DELTA_INF = no
 *    bound.
 *  - Handles are immutable after creation: concurrent tm_count calls on
 *    different streams are allowed.  All device work of a call is ordered on
 *    opts->stream and the call returns after that stream reaches the end of
 *    the call's work (synchronous).
 *  - "device pointer" means memory the CUDA device of the handle can address
 *    (cudaMalloc'ed, e.g. a torch CUDA tensor's data_ptr()).
 */
#ifndef TMOTIF_H
#define TMOTIF_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
    TM_OK = 0,
    TM_EINVAL = 1,        /* invalid argument (message says which)                  */
    TM_ENOMEM = 2,        /* device or host allocation failed                       */
    TM_ECUDA = 3,         /* a CUDA runtime error (message carries cudaGetErrorString) */
    TM_EUNSUPPORTED = 4,  /* feature combination not supported (see tm_motif_create) */
    TM_TRUNCATED = 5      /* tm_enumerate: more matches than buffer rows            */
} tm_status;

#define TM_DELTA_INF INT64_MAX
#define TM_MAX_EDGES 6      /* motif edges L <= 6 (configs use <= 5)                 */
#define TM_MAX_VERTICES 7   /* distinct motif vertices                               */
#define TM_MAX_M 2147483647u  /* graph edges m <= 2^31 - 1 (u32 record positions)   */

typedef struct tm_graph tm_graph;
typedef struct tm_motif tm_motif;

/* ------------------------------------------------------------------ graph */

typedef struct {
    int device;           /* CUDA device ordinal; -1 = the calling thread's current */
    void *stream;         /* cudaStream_t for the build; NULL = legacy default      */
    int input_on_device;  /* 1: src/dst/t are device pointers; 0: host pointers     */
    int pair_index;       /* 1: also build the pair index — the edges of every vertex
                             pair (u, v), time-sorted, behind a hash table.  A closing
                             motif edge (both endpoints mapped) whose window in
                             a hub's list runs past 16 records is then counted from it
                             with two binary searches instead of a scan.  Pays off on
                             hub-heavy coarse-only queries (C5 slice: 232 -> 169 ms);
                             costs ~12 ms and 0.75 GB on a 63.5M-edge graph.  0: not built */
    int pair_id_bucket_log2; /* with pair_index, k > 0: also a membership filter of
                             (u, v, edge id >> k) — "the pair has an edge among these
                             2^k consecutive edge ids".  A closing motif edge whose
                             window (e_prev, H_δ(e_1)] covers at most 4 such buckets
                             reads no list unless one of them may hold an edge of its
                             pair.  Choose 2^k near the edge count of one δ.  8 bits
                             per edge.  0: not built */
} tm_graph_opts;

/* Load a temporal graph G = {(src[i], dst[i], t[i])}, i < m and
 * build, on the device, the chronologically sorted temporal edge list and the
 * two time-sorted CSR adjacency structures of P:230-231 (out- and
 * in-adjacency, each record a 64-bit (edge id << 32 | neighbour)).
 *   src, dst : m vertex ids, each < n_vertices (dense ids; the caller densifies)
 *   t        : m timestamps, each >= 0; any order (stable sort by (t, i))
 *   m        : 0 <= m <= TM_MAX_M; m == 0 is a valid empty graph
 *   o        : may be NULL (device -1, default stream, host input)
 * Ownership: the inputs are copied; the caller keeps them.  The library owns
 * *out and its device memory until tm_graph_destroy (besides the CSR: the
 * rank arrays, 16 B per edge, and the first-record-id cache, 32 B per edge,
 * filled by the first query that needs each of its four list variants and
 * reused by later ones — a property of the graph, independent of δ).  Self-loop edges are
 * kept (they take edge ids) but can never be matched (injectivity, Q4).
 * Errors: TM_EINVAL (null pointer with m > 0, id >= n_vertices, t < 0,
 * m > TM_MAX_M), TM_ENOMEM, TM_ECUDA. */
tm_status tm_graph_create(const uint32_t *src, const uint32_t *dst, const int64_t *t, uint64_t m,
                          uint32_t n_vertices, const tm_graph_opts *o, tm_graph **out);

tm_status tm_graph_destroy(tm_graph *g);

/* m, n_vertices and device ordinal of a graph (any pointer may be NULL). */
tm_status tm_graph_info(const tm_graph *g, uint64_t *m, uint32_t *n_vertices, int *device);

/* perm[id] = input position of edge id, for id < m.  perm: host, m entries,
 * caller-owned. */
tm_status tm_graph_sorted_to_input(const tm_graph *g, uint64_t *perm);

/* Copy the sorted edge list (host buffers of m entries each; any may be NULL). */
tm_status tm_graph_sorted_edges(const tm_graph *g, uint32_t *src, uint32_t *dst, int64_t *t);

/* ------------------------------------------------------------------ motif */

/* Define a δ-temporal motif with optional fine-grained bounds.
 *   L        : number of motif edges, 1..TM_MAX_EDGES
 *   mu, mv   : L motif edges (mu[i] -> mv[i]); list order = temporal order.
 *              Any vertex labels < 64; they are relabelled by first appearance.
 *   delta    : δ >= 0, or TM_DELTA_INF
 *   fine     : NULL, or L-1 entries: fine[i] = δ_{i+1} bounds t(e_{i+2}) -
 *              t(e_{i+1}) (0-based gaps), each >= 0 or TM_DELTA_INF
 * Ownership: inputs copied; library owns *out until tm_motif_destroy.
 * Errors: TM_EINVAL (L out of range, mu[i] == mv[i] (motif self-loop),
 * label >= 64, more than TM_MAX_VERTICES vertices, δ < 0, δ_i < 0).
 * A motif edge after the first that touches no earlier motif vertex
 * ("prefix-disconnected") takes its candidates from all later edges of the
 * time-sorted edge list (Algorithm 1's AllEdges branch; reading
 * Q9): such motifs run a thread-per-root search kernel (TM_KMODE_DFS) for
 * tm_count / tm_enumerate / tm_count_roots / tm_count_multi, and return
 * TM_EUNSUPPORTED with labels, anti-edges, tm_search_stats_run or
 * tm_motif_specialise. */
tm_status tm_motif_create(uint32_t L, const uint32_t *mu, const uint32_t *mv, int64_t delta,
                          const int64_t *fine, tm_motif **out);

tm_status tm_motif_destroy(tm_motif *mo);

/* --------------------------------------------- generalized query (N2) */
/* "Nodes and edges can be optionally endowed with discrete attributes/labels"
 * (P:167); a generalized motif may require labels and carry temporal
 * anti-edges.  Labels are int32 >= 0; unlabeled
 * vertices/edges have label 0. */
#define TM_ANY_LABEL (-1)   /* no requirement */
#define TM_MAX_ANTI 4       /* anti-edges per motif */

/* Attach labels to a graph: vlabels[n] per vertex, elabels[m] per edge in
 * the caller's INPUT order (NULL: leave that kind at 0).  Pointers are host,
 * or device when on_device.  The library copies them (edge labels into edge-id
 * order).  Not concurrent with queries on g.  Errors: TM_EINVAL, TM_ENOMEM,
 * TM_ECUDA. */
tm_status tm_graph_set_labels(tm_graph *g, const int32_t *vlabels, const int32_t *elabels, int on_device);

/* Require motif vertex `vertex` (the caller's label in mu/mv) to map to a
 * graph vertex with `label`, or motif edge `edge` (0-based, list order) to
 * match a graph edge with `label` (checked whenever the vertex /
 * edge is newly matched).  label = TM_ANY_LABEL clears the requirement.
 * Errors: TM_EINVAL (vertex not in the motif, edge >= L, label < -1). */
tm_status tm_motif_set_vertex_label(tm_motif *mo, uint32_t vertex, int32_t label);
tm_status tm_motif_set_edge_label(tm_motif *mo, uint32_t edge, int32_t label);

/* Attach a temporal anti-edge ¬(u, v, window) to real motif edge `attach`
 * (0-based): a match is rejected if the graph holds an edge
 * φ(u) -> φ(v), other than the match's own edges (reading Q22), with
 * t in [t(e_attach), t(e_attach) + window] (inclusive).  u, v: the caller's
 * motif vertex labels, distinct, both in the motif.  Matches are checked when
 * complete.  Motifs with labels or anti-edges run on the generic kernel.
 * Errors: TM_EINVAL (bad vertex, attach >= L, window < 0, more than
 * TM_MAX_ANTI anti-edges). */
tm_status tm_motif_add_anti_edge(tm_motif *mo, uint32_t u, uint32_t v, uint32_t attach, int64_t window);

/* Runtime specialisation ("code generator ... compiled into a
 * shared library"): compiles, with NVRTC, the mining
 * kernel template instantiated for this motif's structure (and, if the motif
 * has labels or anti-edges, with those checks) for counting and enumeration,
 * and uses it for every later query of mo.  A motif in the build-time catalog
 * without constraints is already specialised (no-op).  Blocking, ~1-2 s per
 * kernel on first use, cached per process.  Changing labels / anti-edges
 * afterwards drops the specialisation.  Errors: TM_EINVAL, TM_ECUDA (with the
 * NVRTC log in tm_last_error). */
tm_status tm_motif_specialise(tm_motif *mo);

/* Whether the motif runs on a compile-time specialised kernel (1) or on the
 * generic kernel with a runtime plan (0). */
tm_status tm_motif_specialised(const tm_motif *mo, int *specialised);

/* ------------------------------------------------------------------- runs */

typedef struct {
    void *stream;            /* cudaStream_t; NULL = legacy default stream           */
    uint64_t root_lo;        /* mine the search trees rooted at edge ids           */
    uint64_t root_hi;        /*   [root_lo, min(root_hi, m)); default 0, UINT64_MAX  */
    uint64_t edge_id_offset; /* added to every enumerated id (partitions, §8(e))     */
    int canonical;           /* tm_enumerate: sort rows lexicographically           */
    int buffers_on_device;   /* output buffers are device pointers                   */
    uint32_t grid_ctas;      /* 0 = auto (persistent: SMs x resident CTAs)           */
    uint32_t block_threads;  /* 0 = auto                                              */
    int32_t share;           /* heavy-subtree sharing (load balancing,    */
                             /* P:815-821): 0 = on: once the root queue is drained,  */
                             /* busy warps split off the shallowest pending subtrees */
                             /* (whole tasks or halves of a candidate window) to     */
                             /* idle warps through a global ticket queue; 1 = off;   */
                             /* 2 = eager (also leaf-level tasks; a test mode).      */
                             /* Results are identical in every mode.                 */
    int32_t fuse;            /* tm_count_multi: 0 = a motif that is the first l      */
                             /* edges of another motif of the call (same δ and       */
                             /* δ_1..δ_{l-1}, no labels / anti-edges) is counted     */
                             /* inside that motif's kernel — its matches are the     */
                             /* search-tree nodes at level l — instead of by its own */
                             /* kernel; 1 = off.  Counts are identical.               */
} tm_run_opts;

/* Fill *o with the defaults above. */
void tm_run_opts_default(tm_run_opts *o);

/* Exact number of matches whose first edge e_1 lies in the root range (a
 * match belongs to its root edge, reading Q16).  *count: host. */
tm_status tm_count(const tm_graph *g, const tm_motif *mo, const tm_run_opts *o, uint64_t *count);

/* Enumerate the matches of the root range into buf: row r occupies
 * buf[r*L .. r*L+L) (u32 edge ids + o->edge_id_offset).  buf is caller-owned,
 * cap rows (host, or device when o->buffers_on_device).  Row order is
 * unspecified unless o->canonical.  *n_total (host) always receives the exact
 * match count; *n_written (host) = min(n_total, cap).  Returns TM_TRUNCATED
 * (rows beyond cap dropped, which subset is unspecified) when n_total > cap
 * ("the user must define the number of matches to be enumerated"). */
tm_status tm_enumerate(const tm_graph *g, const tm_motif *mo, const tm_run_opts *o, uint32_t *buf,
                       uint64_t cap, uint64_t *n_total, uint64_t *n_written);

/* Per-root counts: counts[i] = number of matches with e_1 = roots[i].
 * roots (n ids < m) and counts (n entries) are host pointers, or device
 * pointers when o->buffers_on_device.  Root range fields of o are ignored. */
tm_status tm_count_roots(const tm_graph *g, const tm_motif *mo, const tm_run_opts *o,
                         const uint64_t *roots, uint64_t n, uint64_t *counts);

/* Search-tree instrumentation of one tm_count-equivalent run (debug kernel,
 * not the timed path).  nodes[l] (l = 1..L-1): partial matches with l edges
 * whose candidate window for motif edge l+1 was searched (each exactly once,
 * the P:719-723 candidate-caching invariant); window_sum: Σ window sizes;
 * list_sum: Σ lengths of the adjacency lists searched; probe_sum: Σ
 * ceil(log2(len+1)); matches; fast_window_sum: Σ window sizes of the lists
 * the production kernels actually scan (they may pick the other list of a
 * both-mapped motif edge), the basis of the algorithmic bytes. */
typedef struct {
    uint64_t nodes[8];
    uint64_t window_sum;
    uint64_t list_sum;
    uint64_t probe_sum;
    uint64_t matches;
    uint64_t fast_window_sum;
} tm_search_stats;

tm_status tm_search_stats_run(const tm_graph *g, const tm_motif *mo, const tm_run_opts *o,
                              tm_search_stats *out);

/* Several motifs over the same root range in one query: counts[i] = the
 * tm_count of mos[i].  The query-time structures — the δ-horizons of every
 * distinct δ / δ_i and the window-end ranks of every
 * distinct (list, gap bound) — are built once and shared, then one mining
 * kernel per motif runs on o->stream.  Unless o->fuse == 1, a motif that is
 * the first l edges of another (same δ, δ_i, no constraints) is counted as
 * that motif's level-l search nodes (Alg. 1 creates one per prefix match); a
 * motif that differs from another only in its last edge's target (a
 * "sibling", e.g. TRI of the 4-cycle) is written as rows (its matches) by
 * that motif's kernel, and a motif extending the sibling resumes its search
 * from those rows (a row buffer overflow re-counts it without fusion).  The
 * counts are the same with or without fusion.  mos: k host pointers;
 * counts: host, k entries.  Synchronous.  Errors: as tm_count; TM_EINVAL
 * for k == 0.  tm_last_kernel_info reports each motif's kernel. */
tm_status tm_count_multi(const tm_graph *g, const tm_motif *const *mos, uint32_t k, const tm_run_opts *o,
                         uint64_t *counts);

/* Per mining kernel of the calling thread's last tm_count / tm_count_multi /
 * tm_enumerate / tm_count_roots / tm_search_stats_run (one entry per motif):
 * its CUDA-event time and load balance (fields as in tm_run_info). */
typedef struct {
    float mine_ms;
    float tail_ms;
    float warp_busy;
    uint32_t grid_ctas;
    uint64_t shared_tasks;
    int32_t carried_by;      /* fusion: index of the motif whose kernel counted this one (as a prefix or
                                as sibling rows), else -1 */
    int32_t kernel_mode;     /* which kernel ran: TM_KMODE_* below; TM_KMODE_NONE when carried */
} tm_kernel_info;

#define TM_KMODE_NONE (-1)      /* no kernel of its own (carried_by >= 0, or no roots) */
#define TM_KMODE_COUNT 0        /* plain count (Alg. 1) */
#define TM_KMODE_ENUM 1         /* enumeration */
#define TM_KMODE_COUNT_PREFIX 4 /* count that also counts carried prefix motifs */
#define TM_KMODE_RESUME 5       /* count resumed from the sibling rows of another kernel */
#define TM_KMODE_COUNT_SIB 6    /* count that also writes a carried sibling motif's matches as rows */
#define TM_KMODE_DFS 7          /* thread-per-root search of a prefix-disconnected motif (count / enumerate / roots) */

/* Copies min(cap, n) entries to out (host); *n = number of kernels. */
tm_status tm_last_kernel_info(tm_kernel_info *out, uint32_t cap, uint32_t *n);

/* Fused census of the 36 two/three-node three-edge motifs (SURVEY.md §8(f)
 * N1, config C2): counts[a*6 + b] = the δ-temporal count of the
 * motif (0->1, E[a], E[b]), E = [0->1, 1->0, 0->2, 2->0, 1->2, 2->1], for the
 * roots of o's root range — the same 36 numbers as 36 tm_count calls, from
 * one traversal that shares the level-2 windows across all 36 motifs and the
 * level-3 windows across the six with the same second edge.
 *   delta : δ >= 0 or TM_DELTA_INF
 *   fine  : NULL, or 2 entries δ_1, δ_2 (gaps e1-e2, e2-e3), each >= 0 or
 *           TM_DELTA_INF
 *   counts: host, 36 entries (written on success)
 * Synchronous on o->stream.  Errors: TM_EINVAL (null argument, δ < 0,
 * δ_i < 0), TM_ENOMEM, TM_ECUDA.  tm_last_run_info reports its times. */
tm_status tm_census36(const tm_graph *g, int64_t delta, const int64_t *fine, const tm_run_opts *o,
                      uint64_t *counts);

/* Device times (ms, CUDA events on o->stream) of the calling thread's last
 * tm_count / tm_enumerate / tm_count_roots / tm_census36: horizon construction, the mining
 * kernel, and the whole call.  launches: kernels this library launched in it. */
typedef struct {
    float horizon_ms;
    float mine_ms;
    float total_ms;
    uint32_t launches;
    uint32_t grid_ctas;
    uint32_t block_threads;
    uint64_t shared_tasks;   /* subtrees handed from busy to idle warps (share != 1) */
    float tail_ms;           /* load balance of the mining kernel: time  */
                             /* from the first warp finding the root queue empty to  */
                             /* the last warp's exit                                 */
    float warp_busy;         /* Σ over warps of time spent searching ÷ (warps ×      */
                             /* kernel span): 1 = perfectly balanced                 */
} tm_run_info;

tm_status tm_last_run_info(tm_run_info *out);

/* ------------------------------------------------------------ partitioning */

/* Multi-GPU time-range partition plan.
 * Splits roots [0, m) of a sorted edge list into P contiguous ranges
 * [root_lo[p], root_lo[p+1]) (root_lo has P+1 entries, root_lo[0]=0,
 * root_lo[P]=m) balanced by `weights` (per-root work proxy; NULL = the
 * δ-window length H_δ(r) - r), and returns edge_hi[p] = one past the last
 * edge rank p must hold: H_δ(root_lo[p+1]-1) + 1 (its forward δ-halo).
 * Cuts fall only where the timestamp changes (root_lo[p] is the first edge
 * of its timestamp), so a slice holds every edge with t >= t(root_lo[p]):
 * anti-edge witnesses tied with the first root stay inside.  A tie
 * run longer than a share leaves some ranges empty.
 * t_sorted: host, m timestamps in edge-id order.  delta: the query's
 * reach (multi.reach: min(δ, Σδ_i) + the longest anti-edge window).
 * Errors: TM_EINVAL. */
tm_status tm_partition_plan(const int64_t *t_sorted, uint64_t m, int64_t delta, uint32_t P,
                            const uint64_t *weights, uint64_t *root_lo, uint64_t *edge_hi);

/* Thread-local message of the last non-OK status ("" if none). */
const char *tm_last_error(void);

/* Library version string. */
const char *tm_version(void);

#ifdef __cplusplus
}
#endif

#endif /* TMOTIF_H */
