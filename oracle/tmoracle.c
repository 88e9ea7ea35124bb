/*
 * oracle/tmoracle.c — TEST INFRASTRUCTURE, NOT PRODUCT CODE.
 *
 * A plain, slow, obviously-correct CPU implementation of δ-temporal motif
 * mining, written from the paper (arxiv 2310.02800, /root/reference/PAPER.md,
 * cited as P:<line>).  Only tests/, __graft_entry__.smoke() and bench.py's
 * cpu_baseline / `--impl reference` leg may load this library.  It shares no
 * code, header, table or helper with the CUDA path under
 * paper_2310_02800_b200/csrc/, and neither side includes the other.
 *
 * What it computes (definitions):
 *   S = { (e_1..e_L) : e_1 < ... < e_L  in the (t, input index) order (Q1),
 *                      t(e_L) - t(e_1) <= δ                 (Q2),
 *                      t(e_{i+1}) - t(e_i) <= δ_i           (Q3),
 *                      an injective φ: V_M -> V_G maps motif edge i onto
 *                      graph edge e_i                         (Q4) }
 *
 * How it computes it: Algorithm 1 of the paper (Mackey et al.)
 * step by step, in the paper's notation: the execution context MapMG[],
 * MapGM[], eCount[], eStack[], FindNextMatchingEdge,
 * NextLevel, Backtrack, StructConstraints,
 * UpdateDataStructures / RollbackDataStructures and
 * GetCandidateEdgeList with its binary search.  The main loop's
 * cursor mechanics are written as the equivalent recursion: the
 * call stack plays the role of eStack's "resume at eStack.pop()+1".
 * Timestamps are compared directly (t' = time(root) + δ, written as
 * t(c) - t(root) <= δ so δ = ∞ = INT64_MAX never overflows); the CUDA path's
 * index-horizon reformulation is deliberately NOT used here.
 *
 * Readings of the paper (full list in DESIGN.md §Readings):
 *   Q1 equal timestamps: total order (t, input index); edge id = rank.
 *   Q2 window boundary inclusive (t_l - t_1 <= δ), not Alg. 1's `<`.
 *   Q4 self-loop graph edges never match (injectivity); Alg. 1's
 *      StructConstraints would accept (a,a) when both endpoints are new.
 *   Q8 both endpoints mapped: Alg. 1 says "N_out(u_G)/N_in(v_G)";
 *      we scan the shorter list, ties -> N_in(v_G).  Results do not depend
 *      on the choice; the instrumentation counters do.
 *   Q9 a motif edge after the first that touches no earlier motif vertex
 *      takes Alg. 1's "Both u_G, v_G not mapped" branch: its
 *      candidates are all later edges of the time-sorted edge list.
 *
 * Generalized query:
 *   labels   vertex/edge labels are small integers (unlabeled = 0); a motif
 *            vertex / motif edge may require an exact label (TMO_ANY = none).
 *            Checked whenever a vertex or edge is newly matched.
 *   anti     an anti-edge ¬(u_j, v_j, δ_ij) attached to real motif edge i
 *            rejects a match if some graph edge φ(u_j) -> φ(v_j) has
 *            t in [t(e_i), t(e_i) + δ_ij] (inclusive).  Reading Q22:
 *            the witness must be an edge other than the match's own edges;
 *            the check runs when the last real edge is matched (a witness
 *            may lie after it), so it prunes nothing earlier.
 *
 *
 * Instrumentation (used to derive algorithmic bytes, and as a parity target
 * for the GPU's "every window is searched exactly once" invariant):
 *   nodes[l]    number of partial matches with l edges whose candidate list
 *               for motif edge l+1 was searched (l = 1..L-1),
 *   window_sum  Σ |{c in list : c after e_prev, within δ and δ_l}|,
 *   list_sum    Σ list length, probe_sum Σ ceil(log2(len+1)).
 */
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

#define TMO_MAXL 8      /* motif edges */
#define TMO_MAXV 16     /* motif vertex ids accepted: 0..15 */
#define TMO_INF INT64_MAX
#define TMO_MAXANTI 4
#define TMO_ANY (-1)    /* no label requirement */

enum { TMO_OK = 0, TMO_EINVAL = 1, TMO_ENOMEM = 2, TMO_EUNSUPPORTED = 3 };

typedef struct {
    uint64_t m;
    uint32_t n;
    uint32_t *src, *dst;      /* E_G, chronologically sorted       */
    int64_t *t;
    uint64_t *perm;           /* perm[id] = position in caller's input      */
    uint64_t *out_off, *in_off;   /* "Two CSR-like data structures ... storing */
    uint64_t *out_e, *in_e;       /*  their indices in the temporal edge list" */
    int32_t *vlab;            /* vertex labels (n) or NULL = all 0          */
    int32_t *elab;            /* edge labels by sorted id (m) or NULL = all 0 */
} tmo_graph;

/* Constraints of the generalized query. */
typedef struct {
    int32_t vlabel[TMO_MAXV];            /* required label per motif vertex, TMO_ANY = none */
    int32_t elabel[TMO_MAXL];            /* required label per motif edge                   */
    uint32_t n_anti;
    uint32_t anti_u[TMO_MAXANTI], anti_v[TMO_MAXANTI];   /* motif vertices                */
    uint32_t anti_attach[TMO_MAXANTI];                    /* real motif edge, 0-based      */
    int64_t anti_window[TMO_MAXANTI];                     /* δ_ij >= 0                     */
} tmo_constraints;

typedef struct {
    uint64_t nodes[TMO_MAXL];
    uint64_t window_sum;
    uint64_t list_sum;
    uint64_t probe_sum;
    uint64_t matches;
} tmo_stats;

/* ------------------------------------------------------------------ graph */

static const int64_t *g_sort_t; /* qsort has no context arg; single-threaded build */

static int cmp_time_then_index(const void *a, const void *b) {
    uint64_t i = *(const uint64_t *)a, j = *(const uint64_t *)b;
    if (g_sort_t[i] < g_sort_t[j]) return -1;
    if (g_sort_t[i] > g_sort_t[j]) return 1;
    return (i < j) ? -1 : (i > j);
}

void tmo_graph_free(tmo_graph *g) {
    if (!g) return;
    free(g->src); free(g->dst); free(g->t); free(g->perm);
    free(g->out_off); free(g->in_off); free(g->out_e); free(g->in_e);
    free(g->vlab); free(g->elab);
    free(g);
}

/* Builds the chronologically sorted temporal edge list and the two CSR-like
 * in/out structures.  Edge id = rank under (t, input index). */
int tmo_graph_build(const uint32_t *src, const uint32_t *dst, const int64_t *t,
                    uint64_t m, uint32_t n, tmo_graph **out) {
    *out = NULL;
    for (uint64_t i = 0; i < m; i++)
        if (src[i] >= n || dst[i] >= n || t[i] < 0) return TMO_EINVAL;
    tmo_graph *g = (tmo_graph *)calloc(1, sizeof(tmo_graph));
    if (!g) return TMO_ENOMEM;
    g->m = m; g->n = n;
    size_t mm = m ? m : 1;
    g->src = malloc(mm * 4); g->dst = malloc(mm * 4); g->t = malloc(mm * 8);
    g->perm = malloc(mm * 8);
    g->out_off = calloc((size_t)n + 1, 8); g->in_off = calloc((size_t)n + 1, 8);
    g->out_e = malloc(mm * 8); g->in_e = malloc(mm * 8);
    if (!g->src || !g->dst || !g->t || !g->perm || !g->out_off || !g->in_off ||
        !g->out_e || !g->in_e) { tmo_graph_free(g); return TMO_ENOMEM; }

    for (uint64_t i = 0; i < m; i++) g->perm[i] = i;
    g_sort_t = t;
    qsort(g->perm, m, sizeof(uint64_t), cmp_time_then_index);
    for (uint64_t e = 0; e < m; e++) {
        uint64_t i = g->perm[e];
        g->src[e] = src[i]; g->dst[e] = dst[i]; g->t[e] = t[i];
    }
    /* CSR by counting; filling in increasing e keeps every list ascending in e */
    for (uint64_t e = 0; e < m; e++) { g->out_off[g->src[e] + 1]++; g->in_off[g->dst[e] + 1]++; }
    for (uint32_t v = 0; v < n; v++) { g->out_off[v + 1] += g->out_off[v]; g->in_off[v + 1] += g->in_off[v]; }
    uint64_t *fo = malloc(((size_t)n + 1) * 8), *fi = malloc(((size_t)n + 1) * 8);
    if (!fo || !fi) { free(fo); free(fi); tmo_graph_free(g); return TMO_ENOMEM; }
    memcpy(fo, g->out_off, ((size_t)n + 1) * 8); memcpy(fi, g->in_off, ((size_t)n + 1) * 8);
    for (uint64_t e = 0; e < m; e++) { g->out_e[fo[g->src[e]]++] = e; g->in_e[fi[g->dst[e]]++] = e; }
    free(fo); free(fi);
    *out = g;
    return TMO_OK;
}

uint64_t tmo_graph_m(const tmo_graph *g) { return g->m; }

/* Optional labels ("nodes and edges can be optionally endowed with discrete
 * attributes/labels"): vlab[n] per vertex, elab[m] per edge in the
 * caller's INPUT order (stored by sorted id); NULL leaves that kind at 0. */
int tmo_graph_set_labels(tmo_graph *g, const int32_t *vlab, const int32_t *elab) {
    if (vlab) {
        free(g->vlab);
        g->vlab = malloc(((size_t)g->n + 1) * 4);
        if (!g->vlab) return TMO_ENOMEM;
        memcpy(g->vlab, vlab, (size_t)g->n * 4);
    }
    if (elab) {
        free(g->elab);
        g->elab = malloc((g->m ? g->m : 1) * 4);
        if (!g->elab) return TMO_ENOMEM;
        for (uint64_t e = 0; e < g->m; e++) g->elab[e] = elab[g->perm[e]];
    }
    return TMO_OK;
}

static int32_t vertex_label(const tmo_graph *g, uint32_t v) { return g->vlab ? g->vlab[v] : 0; }
static int32_t edge_label(const tmo_graph *g, uint64_t e) { return g->elab ? g->elab[e] : 0; }

/* sorted edge id -> input position, and the sorted arrays themselves */
void tmo_graph_export(const tmo_graph *g, uint64_t *perm, uint32_t *src, uint32_t *dst, int64_t *t) {
    for (uint64_t e = 0; e < g->m; e++) {
        if (perm) perm[e] = g->perm[e];
        if (src) src[e] = g->src[e];
        if (dst) dst[e] = g->dst[e];
        if (t) t[e] = g->t[e];
    }
}

/* ---------------------------------------------------------------- mining */

typedef struct {
    /* the motif */
    uint32_t L;
    uint32_t mu[TMO_MAXL], mv[TMO_MAXL];
    int64_t delta;               /* δ (TMO_INF = none)                          */
    int64_t fine[TMO_MAXL];      /* δ_i between motif edges i and i+1   */
    /* output */
    uint64_t *count_slot;        /* per-root counter, may be NULL              */
    uint32_t *enum_buf;          /* rows of L edge ids, may be NULL            */
    uint64_t cap;
    uint64_t *n_enum;            /* rows produced (written when < cap)         */
    const tmo_constraints *cons; /* labels / anti-edges, NULL = none           */
} tmo_query;

typedef struct {
    const tmo_graph *g;
    const tmo_query *q;
    /* Execution context of Algorithm 1 */
    int64_t MapMG[TMO_MAXV];     /* motif vertex -> graph vertex, -1 if none   */
    int32_t *MapGM;              /* graph vertex -> motif vertex, -1 if none   */
    uint32_t *eCount;            /* mapped-edge count per graph vertex         */
    uint64_t eStack[TMO_MAXL];
    uint32_t depth;              /* |eStack|                                   */
    uint64_t count;
    tmo_stats st;
} tmo_ctx;

/* StructConstraints: the candidate e = (u', v') is consistent with
 * the partial match.  uG/vG are MapMG of the motif edge's endpoints (-1 = not
 * mapped).  Reading Q4: two distinct motif vertices may not map to one graph
 * vertex, so when both endpoints are new they must differ (injectivity). */
static int StructConstraints(const tmo_ctx *c, uint64_t e, int64_t uG, int64_t vG) {
    uint32_t u2 = c->g->src[e], v2 = c->g->dst[e];
    int u_consistent = (uG == (int64_t)u2) || (uG < 0 && c->MapGM[u2] < 0);
    int v_consistent = (vG == (int64_t)v2) || (vG < 0 && c->MapGM[v2] < 0);
    if (uG < 0 && vG < 0 && u2 == v2) return 0;
    return u_consistent && v_consistent;
}

/* Label checks of a candidate e for motif edge eM ("whenever a
 * new vertex/edge is matched ... check their validity"): the edge's label,
 * and the label of each endpoint this edge maps for the first time. */
static int LabelConstraints(const tmo_ctx *c, uint64_t e, uint32_t eM, int64_t uG, int64_t vG) {
    const tmo_constraints *k = c->q->cons;
    if (!k) return 1;
    if (k->elabel[eM] != TMO_ANY && edge_label(c->g, e) != k->elabel[eM]) return 0;
    int32_t ru = k->vlabel[c->q->mu[eM]], rv = k->vlabel[c->q->mv[eM]];
    if (uG < 0 && ru != TMO_ANY && vertex_label(c->g, c->g->src[e]) != ru) return 0;
    if (vG < 0 && rv != TMO_ANY && vertex_label(c->g, c->g->dst[e]) != rv) return 0;
    return 1;
}

/* Temporal anti-edges of the complete match eStack[0..L-2]
 * + last: rejected if a graph edge φ(u_j) -> φ(v_j) other than the match's own
 * edges (reading Q22) has t in [t(e_attach), t(e_attach) + δ_ij].  The
 * out-list of φ(u_j) is sorted by (t, id): binary-search t >= t(e_attach),
 * then scan while t <= t(e_attach) + δ_ij. */
static int AntiConstraints(const tmo_ctx *c, uint64_t last) {
    const tmo_constraints *k = c->q->cons;
    if (!k || !k->n_anti) return 1;
    const tmo_graph *g = c->g;
    const tmo_query *q = c->q;
    uint64_t match[TMO_MAXL];
    int64_t phi[TMO_MAXV];
    for (uint32_t i = 0; i + 1 < q->L; i++) match[i] = c->eStack[i];
    match[q->L - 1] = last;
    for (uint32_t i = 0; i < q->L; i++) { phi[q->mu[i]] = g->src[match[i]]; phi[q->mv[i]] = g->dst[match[i]]; }
    for (uint32_t j = 0; j < k->n_anti; j++) {
        uint32_t x = (uint32_t)phi[k->anti_u[j]], y = (uint32_t)phi[k->anti_v[j]];
        int64_t ta = g->t[match[k->anti_attach[j]]], w = k->anti_window[j];
        const uint64_t *list = g->out_e + g->out_off[x];
        uint64_t len = g->out_off[x + 1] - g->out_off[x], lo = 0, hi = len;
        while (lo < hi) {
            uint64_t mid = lo + (hi - lo) / 2;
            if (g->t[list[mid]] >= ta) hi = mid; else lo = mid + 1;
        }
        for (uint64_t p = lo; p < len && g->t[list[p]] - ta <= w; p++) {
            uint64_t e = list[p];
            if (g->dst[e] != y) continue;
            int own = 0;
            for (uint32_t i = 0; i < q->L; i++) own |= (match[i] == e);
            if (!own) return 0;   /* the absence the anti-edge asks for is violated */
        }
    }
    return 1;
}

/* UpdateDataStructures */
static void UpdateDataStructures(tmo_ctx *c, uint64_t eG, uint32_t eM) {
    uint32_t uG = c->g->src[eG], vG = c->g->dst[eG];
    uint32_t uM = c->q->mu[eM], vM = c->q->mv[eM];
    c->MapMG[uM] = uG; c->MapMG[vM] = vG;
    c->MapGM[uG] = (int32_t)uM; c->MapGM[vG] = (int32_t)vM;
    c->eCount[uG] += 1; c->eCount[vG] += 1;
}

/* RollbackDataStructures */
static void RollbackDataStructures(tmo_ctx *c, uint64_t eG) {
    uint32_t uG = c->g->src[eG], vG = c->g->dst[eG];
    c->eCount[uG] -= 1; c->eCount[vG] -= 1;
    if (c->eCount[uG] == 0) { int32_t uM = c->MapGM[uG]; c->MapGM[uG] = -1; c->MapMG[uM] = -1; }
    if (c->eCount[vG] == 0) { int32_t vM = c->MapGM[vG]; c->MapGM[vG] = -1; c->MapMG[vM] = -1; }
}

/* "filter via binary search": first position in list[0..len) whose
 * edge comes after edge `prev` in the (t, index) order. */
static uint64_t first_after(const tmo_graph *g, const uint64_t *list, uint64_t len, uint64_t prev) {
    uint64_t lo = 0, hi = len;
    int64_t tp = g->t[prev];
    while (lo < hi) {
        uint64_t mid = lo + (hi - lo) / 2;
        uint64_t c = list[mid];
        int after = (g->t[c] > tp) || (g->t[c] == tp && c > prev);
        if (after) hi = mid; else lo = mid + 1;
    }
    return lo;
}

static uint32_t ceil_log2_plus1(uint64_t len) { /* ceil(log2(len+1)) */
    uint32_t k = 0;
    while (((uint64_t)1 << k) < len + 1) k++;
    return k;
}

/* Output a motif H using eStack */
static void emit(tmo_ctx *c, uint64_t last) {
    const tmo_query *q = c->q;
    if (!AntiConstraints(c, last)) return;
    c->count++;
    if (q->count_slot) (*q->count_slot)++;
    if (q->enum_buf) {
        uint64_t row = (*q->n_enum)++;
        if (row < q->cap) {
            uint32_t *r = q->enum_buf + row * q->L;
            for (uint32_t i = 0; i + 1 < q->L; i++) r[i] = (uint32_t)c->eStack[i];
            r[q->L - 1] = (uint32_t)last;
        }
    }
}

/* One level of the search tree: match motif edge e_M = depth (0-based) given
 * eStack[0..depth).  FindNextMatchingEdge + NextLevel + Backtrack of Alg. 1. */
static void search_level(tmo_ctx *c) {
    const tmo_graph *g = c->g;
    const tmo_query *q = c->q;
    uint32_t eM = c->depth;
    uint32_t uM = q->mu[eM], vM = q->mv[eM];
    int64_t uG = c->MapMG[uM], vG = c->MapMG[vM];
    uint64_t root = c->eStack[0], prev = c->eStack[c->depth - 1];

    /* GetCandidateEdgeList */
    const uint64_t *list = NULL; uint64_t len;
    if (uG < 0 && vG < 0) {
        /* AllEdges: a motif edge that touches no earlier motif
         * vertex takes its candidates from the whole time-sorted edge list,
         * whose p-th entry is sorted edge p (list == NULL below) */
        len = g->m;
    } else if (uG >= 0 && vG >= 0) {
        uint64_t lo_ = g->out_off[uG + 1] - g->out_off[uG];
        uint64_t li_ = g->in_off[vG + 1] - g->in_off[vG];
        if (lo_ < li_) { list = g->out_e + g->out_off[uG]; len = lo_; }
        else           { list = g->in_e + g->in_off[vG];   len = li_; }
    } else if (uG >= 0) {
        list = g->out_e + g->out_off[uG]; len = g->out_off[uG + 1] - g->out_off[uG];
    } else {  /* vG >= 0 */
        list = g->in_e + g->in_off[vG]; len = g->in_off[vG + 1] - g->in_off[vG];
    }
    c->st.nodes[c->depth]++;
    c->st.list_sum += len;
    c->st.probe_sum += ceil_log2_plus1(len);

    int64_t troot = g->t[root], tprev = g->t[prev];
    int64_t fine = q->fine[eM - 1];  /* δ_{eM} between motif edges eM and eM+1 (1-based) */
    for (uint64_t p = list ? first_after(g, list, len, prev) : prev + 1; p < len; p++) {
        uint64_t e = list ? list[p] : p;
        if (g->t[e] - troot > q->delta) break;   /* time(e) > t' : Backtrack */
        if (g->t[e] - tprev > fine) break;        /* fine-grained bound */
        c->st.window_sum++;
        if (!StructConstraints(c, e, uG, vG)) continue;
        if (!LabelConstraints(c, e, eM, uG, vG)) continue;
        /* NextLevel */
        if (eM == q->L - 1) { emit(c, e); continue; }
        UpdateDataStructures(c, e, eM);
        c->eStack[c->depth++] = e;
        search_level(c);
        /* Backtrack */
        c->depth--;
        RollbackDataStructures(c, e);
    }
}

/* Mine the search tree rooted at edge r (the root level maps motif edge 1 onto
 * every graph edge). */
static void mine_root(tmo_ctx *c, uint64_t r) {
    if (!StructConstraints(c, r, -1, -1)) return;   /* both endpoints unmapped */
    if (!LabelConstraints(c, r, 0, -1, -1)) return;
    if (c->q->L == 1) { c->depth = 0; emit(c, r); return; }
    UpdateDataStructures(c, r, 0);
    c->eStack[0] = r; c->depth = 1;                 /* t' <- time(r) + δ */
    search_level(c);
    c->depth = 0;
    RollbackDataStructures(c, r);                   /* eStack empty: t' <- ∞ */
}

/* Motif validation: 1 <= L <= TMO_MAXL, ids < TMO_MAXV, u != v, δ >= 0,
 * δ_i >= 0.  A motif edge that shares no vertex with the earlier ones
 * (prefix-disconnected) is searched with the AllEdges list (Q9). */
static int validate(uint32_t L, const uint32_t *mu, const uint32_t *mv, int64_t delta, const int64_t *fine) {
    if (L < 1 || L > TMO_MAXL || delta < 0) return TMO_EINVAL;
    for (uint32_t i = 0; i < L; i++) {
        if (mu[i] >= TMO_MAXV || mv[i] >= TMO_MAXV || mu[i] == mv[i]) return TMO_EINVAL;
        if (fine && i + 1 < L && fine[i] < 0) return TMO_EINVAL;
    }
    return TMO_OK;
}

/* Mine roots [root_lo, root_hi) (or the list `roots[0..n_roots)` when
 * non-NULL).  count: total matches.  per_root (nullable): count per root,
 * indexed like the roots iterated.  enum_buf (nullable): forces one thread;
 * rows of L sorted-edge ids in root order, lexicographic by construction;
 * *n_total gets the exact number of matches.  stats (nullable).
 * nthreads <= 0: OpenMP default. */
/* Anti-edges: at most TMO_MAXANTI, endpoints distinct motif vertices of the
 * motif, attached to a real edge, window >= 0. */
static int validate_constraints(uint32_t L, const uint32_t *mu, const uint32_t *mv, const tmo_constraints *k) {
    if (!k) return TMO_OK;
    if (k->n_anti > TMO_MAXANTI) return TMO_EINVAL;
    int seen[TMO_MAXV] = {0};
    for (uint32_t i = 0; i < L; i++) seen[mu[i]] = seen[mv[i]] = 1;
    for (uint32_t j = 0; j < k->n_anti; j++) {
        if (k->anti_u[j] >= TMO_MAXV || k->anti_v[j] >= TMO_MAXV || k->anti_u[j] == k->anti_v[j]) return TMO_EINVAL;
        if (!seen[k->anti_u[j]] || !seen[k->anti_v[j]]) return TMO_EINVAL;
        if (k->anti_attach[j] >= L || k->anti_window[j] < 0) return TMO_EINVAL;
    }
    return TMO_OK;
}

int tmo_mine(const tmo_graph *g, uint32_t L, const uint32_t *mu, const uint32_t *mv,
             int64_t delta, const int64_t *fine, const tmo_constraints *cons,
             uint64_t root_lo, uint64_t root_hi, const uint64_t *roots, uint64_t n_roots,
             int nthreads, uint64_t *count, uint64_t *per_root,
             uint32_t *enum_buf, uint64_t cap, uint64_t *n_total, tmo_stats *stats) {
    int rc = validate(L, mu, mv, delta, fine);
    if (rc) return rc;
    rc = validate_constraints(L, mu, mv, cons);
    if (rc) return rc;
    tmo_query q;
    memset(&q, 0, sizeof q);
    q.L = L; q.delta = delta; q.cons = cons;
    for (uint32_t i = 0; i < L; i++) { q.mu[i] = mu[i]; q.mv[i] = mv[i]; }
    for (uint32_t i = 0; i < TMO_MAXL; i++) q.fine[i] = TMO_INF;
    if (fine) for (uint32_t i = 0; i + 1 < L; i++) q.fine[i] = fine[i];
    if (root_hi > g->m) root_hi = g->m;
    uint64_t nr = roots ? n_roots : (root_hi > root_lo ? root_hi - root_lo : 0);
    if (roots) for (uint64_t i = 0; i < nr; i++) if (roots[i] >= g->m) return TMO_EINVAL;
    if (enum_buf || n_total) nthreads = 1;
#ifdef _OPENMP
    if (nthreads <= 0) nthreads = omp_get_max_threads();
#else
    nthreads = 1;
#endif
    uint64_t total = 0, n_enum = 0;
    tmo_stats agg;
    memset(&agg, 0, sizeof agg);
    int fail = 0;
    if (per_root) memset(per_root, 0, nr * 8);

#pragma omp parallel num_threads(nthreads) reduction(+:total)
    {
        tmo_ctx c;
        memset(&c, 0, sizeof c);
        c.g = g;
        for (int i = 0; i < TMO_MAXV; i++) c.MapMG[i] = -1;
        c.MapGM = (int32_t *)malloc(((size_t)g->n + 1) * 4);
        c.eCount = (uint32_t *)calloc((size_t)g->n + 1, 4);
        if (!c.MapGM || !c.eCount) {
#pragma omp atomic write
            fail = 1;
        } else {
            memset(c.MapGM, 0xff, ((size_t)g->n + 1) * 4);  /* -1 */
            tmo_query ql = q;
            ql.enum_buf = enum_buf; ql.cap = cap; ql.n_enum = &n_enum;
            c.q = &ql;
#pragma omp for schedule(dynamic, 256)
            for (uint64_t i = 0; i < nr; i++) {
                uint64_t r = roots ? roots[i] : root_lo + i;
                ql.count_slot = per_root ? per_root + i : NULL;
                mine_root(&c, r);
            }
            total += c.count;
#pragma omp critical
            {
                for (int l = 0; l < TMO_MAXL; l++) agg.nodes[l] += c.st.nodes[l];
                agg.window_sum += c.st.window_sum; agg.list_sum += c.st.list_sum;
                agg.probe_sum += c.st.probe_sum;
            }
        }
        free(c.MapGM); free(c.eCount);
    }
    if (fail) return TMO_ENOMEM;
    agg.matches = total;
    if (count) *count = total;
    if (n_total) *n_total = n_enum;
    if (stats) *stats = agg;
    return TMO_OK;
}

int tmo_max_threads(void) {
#ifdef _OPENMP
    return omp_get_max_threads();
#else
    return 1;
#endif
}
