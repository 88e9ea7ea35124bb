// Internal declarations of libtmotif (not part of the ABI).
#pragma once

#ifdef __CUDACC_RTC__
// NVRTC (tm_motif_specialise compiles mine.cuh at run time): no host headers
typedef unsigned char uint8_t;
typedef signed char int8_t;
typedef int int32_t;
typedef unsigned int uint32_t;
typedef long long int64_t;
typedef unsigned long long uint64_t;
#define INT64_MAX 9223372036854775807LL
#else
#include <cuda_runtime.h>
#include <nvtx3/nvToolsExt.h>
#include <cstdint>
#include <mutex>
#include <string>
#endif

#include "../../include/tmotif.h"

namespace tmg {

constexpr int kMaxL = TM_MAX_EDGES;      // motif edges
constexpr int kMaxV = TM_MAX_VERTICES;   // motif vertices

// Device-resident temporal graph.
//   src/dst/t : the chronologically sorted temporal edge list; edge
//               id = rank by (t, input position) (reading Q1).
//   rec       : 2(m+n)+32 packed 64-bit records (edge id << 32 | neighbour):
//               [0, m+n) out-adjacency grouped by source, [m+n, 2(m+n)) in-
//               adjacency grouped by destination; ascending edge id inside each
//               group = time order; every group is followed by a
//               sentinel record 0xFFFFFFFF'FFFFFFFF (id above every bound), so
//               scans stop by id alone; +32 records of padding (a warp's 32 consecutive
//               reads of an open window may run past the last sentinel).
//   off_out   : n+1 start positions in rec (list v = [off_out[v], off_out[v+1]-1),
//               its sentinel at off_out[v+1]-1).
//   off_in    : the same for the in-lists (values in [m+n, 2(m+n)]).
//   perm      : perm[id] = input position.
//   rank      : 4m u32, rank[var*m + e] = absolute position in rec of the first
//               record after edge e in one list touching e, var = 2*endpoint
//               + dir: 0 OUT(src e) (own), 1 IN(src e), 2 OUT(dst e),
//               3 IN(dst e) (own).  Turns the lower-bound binary search of
//               GetCandidateEdgeList into one load.
// First-record ids per list variant (k_hrank): nx[var][e] = ids of the first
// two records after e in list `var` of e (0xFFFFFFFF: none; second 0:
// unknown).  A graph property, independent of δ, allocated with the graph and
// recorded by the first query that builds window descriptors for that
// variant (from the record sector it reads anyway); later
// queries skip the record read of every window that ends before it (half of
// all windows on C4).  State per variant: 0 absent, 1 being filled, 2 ready
// (ev: the filling kernel's completion, waited on by other streams).
#ifndef __CUDACC_RTC__
struct NextIdCache {
    std::mutex mu;
    uint32_t *buf = nullptr;   // one block: nx[v] = buf + v * 2m
    uint32_t *nx[4] = {nullptr, nullptr, nullptr, nullptr};
    int state[4] = {0, 0, 0, 0};
    cudaEvent_t ev[4] = {nullptr, nullptr, nullptr, nullptr};
};
#else
struct NextIdCache;
#endif

struct DeviceGraph {
    uint64_t m = 0;
    uint32_t n = 0;
    uint32_t *src = nullptr, *dst = nullptr;
    int64_t *t = nullptr;
    uint32_t *perm = nullptr;
    uint32_t *off_out = nullptr, *off_in = nullptr;
    uint64_t *rec = nullptr;
    uint32_t *rank = nullptr;
    // skip[j] = id of rec[8j] (0xFFFFFFFF past the end; +8 entries of
    // padding), bit 31 set where a list's sentinel lies in rec(8(j-1), 8j]: one u32
    // per 8 records (66 MB on C4, L2-sized), so a window end deep in a hub's
    // list is found with one skip sector plus one record sector instead of a
    // gallop over the records, and without the list's bound (k_hrank)
    uint32_t *skip = nullptr;
    uint64_t nrec = 0;
    // pair index: prec = edge ids grouped by (src, dst) pair, ascending id in
    // each group (+8 padding); ptab = open-addressing hash table of the
    // distinct pairs, slot = {key = src << 32 | dst, start, len}, capacity a
    // power of two >= 2 x pairs, empty key = ~0.  The candidate list of a
    // motif edge whose endpoints are both mapped is exactly one pair.
    uint32_t *prec = nullptr;
    uint4 *ptab = nullptr;
    uint32_t pmask = 0;
    uint64_t npairs = 0;
    // membership filter of the pairs: one bit per hash bucket, >= 8 buckets
    // per pair (~12 % false positives), small enough to stay L2-resident, so
    // an absent pair — the common case when closing a cycle — costs one L2 hit
    uint32_t *pbits = nullptr;
    uint32_t fmask = 0;
    // id-bucketed pair filter (tm_graph_opts.pair_id_bucket_log2): one bit per
    // hash of (u, v, id >> tshift); tbits == nullptr: not built
    uint32_t *tbits = nullptr;
    uint32_t tmask = 0;
    int tshift = 0;
    // optional labels (tm_graph_set_labels): per vertex, per edge by sorted id
    int32_t *vlab = nullptr, *elab = nullptr;
    // lazily filled first-record ids (NextIdCache); owned, freed with the graph
    mutable NextIdCache *nxc = nullptr;
};

// Which motif edges with both endpoints mapped (closing edges) read
// the pair index instead of scanning a time-sorted list.
// Measured: leaves 1x time / 10x DRAM traffic; inner edges 1.2x slower once
// window ends come from the window-end ranks.  Off: the index is not built.
#ifndef TM_PAIR_LEAF
#define TM_PAIR_LEAF 0
#endif
#ifndef TM_PAIR_NONLEAF
#define TM_PAIR_NONLEAF 0
#endif
#ifndef TM_PAIR_BUILD
#define TM_PAIR_BUILD 0     // build the pair index with every graph (long closing windows use it)
#endif

#ifndef TM_BLOOM_K
#define TM_BLOOM_K 0        // 0: one bit per pair; k > 0: blocked Bloom, k bits in one 32-byte block
#endif
#ifndef TM_BLOOM_BITS
#define TM_BLOOM_BITS 8     // filter bits per distinct pair (rounded up to a power of two)
#endif

__host__ __device__ inline uint64_t pair_hash(uint64_t k) {   // splitmix64 finaliser
    k ^= k >> 30;
    k *= 0xbf58476d1ce4e5b9ull;
    k ^= k >> 27;
    k *= 0x94d049bb133111ebull;
    k ^= k >> 31;
    return k;
}

// bit of (pair u -> v, edge-id bucket b) in the id-bucketed pair filter: a
// 32-bit multiply-add combination and the murmur3 finaliser (cheap: the
// mining kernel evaluates it for every live closing leaf)
__host__ __device__ inline uint32_t pair_bucket_bit(uint32_t u, uint32_t v, uint32_t b, uint32_t mask) {
    uint32_t k = u * 0x9E3779B1u + v * 0x85EBCA77u + b * 0xC2B2AE3Du + 0x27D4EB2Fu;
    k ^= k >> 16;
    k *= 0x85EBCA6Bu;
    k ^= k >> 13;
    k *= 0xC2B2AE35u;
    k ^= k >> 16;
    return k & mask;
}

// filter bit positions of a pair hash; fmask = filter bits - 1
__host__ __device__ inline uint32_t bloom_bit(uint64_t h, uint32_t fmask, int i) {
    if (TM_BLOOM_K == 0) return (uint32_t)(h >> 32) & fmask;
    const uint32_t block = ((uint32_t)(h >> 32) & fmask) & ~255u;        // 256-bit (32-byte) block
    return block | (uint32_t)((h >> (8 * i)) & 255u);
}

#ifdef __CUDACC__
__device__ __forceinline__ bool pair_maybe(const uint32_t *bits, uint32_t fmask, uint64_t h) {
    if (TM_BLOOM_K == 0) {
        const uint32_t b = bloom_bit(h, fmask, 0);
        return (__ldg(bits + (b >> 5)) >> (b & 31)) & 1u;
    }
    const uint32_t block = bloom_bit(h, fmask, 0) & ~255u;
    const uint4 *bp = reinterpret_cast<const uint4 *>(bits + (block >> 5));
    const uint4 q0 = __ldg(bp), q1 = __ldg(bp + 1);
    const uint32_t w[8] = {q0.x, q0.y, q0.z, q0.w, q1.x, q1.y, q1.z, q1.w};
    bool ok = true;
#pragma unroll
    for (int i = 0; i < (TM_BLOOM_K > 0 ? TM_BLOOM_K : 1); i++) {
        const uint32_t b = bloom_bit(h, fmask, i) & 255u;
        uint32_t word = 0;
#pragma unroll
        for (int j = 0; j < 8; j++)
            if (j == (int)(b >> 5)) word = w[j];
        ok &= (word >> (b & 31)) & 1u;
    }
    return ok;
}
#endif

}  // namespace tmg

#ifndef __CUDACC_RTC__
struct tm_graph {
    int device = 0;
    tmg::DeviceGraph d;
};

struct tm_motif {
    uint32_t L = 0;          // motif edges
    uint32_t nv = 0;         // motif vertices
    uint8_t u[tmg::kMaxL] = {}, v[tmg::kMaxL] = {};   // relabelled by first appearance
    int64_t delta = 0;
    int64_t fine[tmg::kMaxL] = {};                    // gap i between edges i and i+1 (0-based)
    uint64_t code = 0;       // packed structure, selects the specialised kernel
    int8_t internal[64];     // caller's motif vertex label -> internal vertex (-1: not in the motif)
    // generalized query: label requirements and anti-edges
    int32_t vreq[tmg::kMaxV];                         // per internal vertex, TM_ANY_LABEL = none
    int32_t ereq[tmg::kMaxL];                         // per motif edge
    uint32_t n_anti = 0;
    uint8_t anti_u[TM_MAX_ANTI] = {}, anti_v[TM_MAX_ANTI] = {}, anti_attach[TM_MAX_ANTI] = {};
    int64_t anti_window[TM_MAX_ANTI] = {};
    bool disconnected = false;   // some edge after the first touches no earlier vertex (Q9): dfs.cu
    void *rtc_fn[2] = {nullptr, nullptr};   // tm_motif_specialise: count / enumerate kernels (CUfunction)
    int rtc_smem[2] = {0, 0};               // their shared memory per warp (bytes)
    bool constrained() const {
        if (n_anti) return true;
        for (uint32_t i = 0; i < nv; i++) if (vreq[i] != TM_ANY_LABEL) return true;
        for (uint32_t i = 0; i < L; i++) if (ereq[i] != TM_ANY_LABEL) return true;
        return false;
    }
};
#endif  // !__CUDACC_RTC__

namespace tmg {

// Modes of the mining kernel.
// kCountPfx: counting that also counts the nodes of the levels in
// MineParams::prefix_mask (prefix fusion, tm_count_multi) — a separate
// instantiation, so the plain counting kernels carry none of that code.
// kResume: counting that starts from rows of partial matches (sibling
// emission of another kernel) instead of root edges.
// kCountSib: kCountPfx plus sibling emission at level 2 (level-2 tasks keep
// every φ slot and matched id for the rows).
enum Mode : int { kCount = 0, kEnum = 1, kRoots = 2, kStats = 3, kCountPfx = 4, kResume = 5, kCountSib = 6 };
constexpr int kSibLevel = 2;   // the level kCountSib kernels emit sibling rows at

// Packed motif structure: bits 0-2 L, then per edge i: u at 3+6i, v at 6+6i.
constexpr uint64_t motif_code(int L, const uint8_t *u, const uint8_t *v) {
    uint64_t c = (uint64_t)L;
    for (int i = 0; i < L; i++) c |= ((uint64_t)u[i] << (3 + 6 * i)) | ((uint64_t)v[i] << (6 + 6 * i));
    return c;
}

// Kernel parameters of one mining launch (passed by value; lives in the
// constant bank).
struct MineParams {
    const uint32_t *src, *dst;
    const uint32_t *off_out, *off_in;
    const uint64_t *rec;
    const uint32_t *rank;              // DeviceGraph::rank
    uint32_t m;
    uint32_t split;                    // rec positions < split are out-records (m + n)
    const uint32_t *prec;              // DeviceGraph pair index
    const uint4 *ptab;
    uint32_t pmask;
    const uint32_t *pbits;
    uint32_t fmask;
    const uint32_t *tbits;
    uint32_t tmask;
    int tshift;
    const uint32_t *H;                 // H_δ  (coarse δ-horizon)
    const uint32_t *Hf[kMaxL];         // H_{δ_i} per gap i, nullptr when δ_i = ∞
    const uint4 *HW[kMaxL];            // per gap i (TM_HRANK == 3): window descriptors {start, end, H_δi, 0}
    uint32_t *HR[kMaxL];               // per gap i: window-end ranks of H_{δ_i} in the list motif edge
                                       // i+1 reads (build_hrank, or a zeroed memo of pos + 1 the kernel
                                       // fills, TM_HRANK == 2), nullptr when not applicable
    uint64_t root_lo, n_roots;         // roots root_lo + [0, n_roots) ...
    const uint64_t *roots;             // ... or roots[0, n_roots) when non-null
    unsigned long long *scratch;       // [0] root cursor, [1] count, [2] enum cursor, [8..] stats
    unsigned long long *root_counts;   // kRoots: per root slot
    uint32_t *enum_buf;
    uint64_t cap;
    uint32_t id_offset;
    // heavy-subtree sharing (tm_run_opts::share): a ring of
    // qmask+1 task records of kShareWords words and their ticket flags
    // (0 = empty, ticket+1 = filled for that ticket); tickets and the idle
    // counter live in scratch[kShareTail..kShareDone]
    int share;
    unsigned int *qflag;
    uint32_t *qrec;
    uint32_t qmask;
    uint32_t total_warps;
    // prefix fusion (tm_count_multi): bit l set -> count the search-tree nodes
    // created at level l (= the matches of this motif's l-edge prefix) into
    // scratch[kPrefixBase + l]
    uint32_t prefix_mask;
    uint32_t prefix_lv0;               // lowest set level of prefix_mask (counted per lane)
    uint32_t root_prune;               // 1: a root whose closing look-ahead window is empty is not searched
    // sibling emission (kCountPfx): at level sib_level, candidates whose
    // neighbour is φ[sib_vtx] complete a sibling motif's closing edge; their
    // rows (e_1..e_sib_level, e) go to sib_rows (cap rows), counted in
    // scratch[kSibCount]
    uint32_t sib_level, sib_vtx, sib_cap;
    uint32_t *sib_rows;
    // resume (kResume): rows of resume_level edge ids, *resume_n of them (<= sib_cap)
    const uint32_t *resume_rows;
    const unsigned long long *resume_n;
    uint32_t resume_level;
    // generalized query (PlanR only, gen != 0): labels and anti-edges
    int gen;
    const int32_t *vlab, *elab;        // graph labels (nullptr = all 0)
    int32_t vreq[kMaxV], ereq[kMaxL];  // TM_ANY_LABEL = no requirement
    uint32_t n_anti;
    uint8_t anti_u[TM_MAX_ANTI], anti_v[TM_MAX_ANTI], anti_a[TM_MAX_ANTI];
    const uint32_t *anti_hi[TM_MAX_ANTI];   // H_{δ_ij}: last id with t <= t(e) + δ_ij
    const uint32_t *tie_lo;            // first id with t == t(e): the window [t(e), ...] starts there
    // runtime plan (generic kernel)
    uint32_t L;
    uint8_t u[kMaxL], v[kMaxL];
};

constexpr int kScratchWords = 48;
// load-balance timing (globaltimer ns): max(~start) over warps, max(~drain)
// (the first warp to find the root queue empty), max(exit), Σ per-warp
// (exit - start), Σ time spent waiting for handed-over work
constexpr int kTimeStart = 40, kTimeDrain = 41, kTimeExit = 42, kTimeBusy = 43, kTimeWait = 44;
// scratch words of the sharing queue: donor tickets, receiver tickets, idle
// warps (an int in the low half), subtrees handed over
constexpr int kShareTail = 3, kShareHead = 4, kShareIdle = 5, kShareDone = 6;
constexpr int kShareWords = 32;   // u32 words per shared task record (fields + level in word 31)
constexpr int kSibCount = 45;     // scratch[45]: sibling rows emitted (all, even beyond sib_cap)
constexpr int kPrefixBase = 32;   // scratch[32 + l]: prefix matches (nodes created at level l)
constexpr int kStatsBase = 8;   // scratch[8 + l] nodes[l], [16] window, [17] list, [18] probes, [19] fast window

// Parameters of the fused 36-motif census (census.cu).
struct CensusParams {
    const uint32_t *src, *dst;
    const uint64_t *rec;
    const uint32_t *rank;
    uint32_t m;
    const uint32_t *H;              // H_δ
    const uint32_t *Hf0, *Hf1;      // H_δ1, H_δ2 or nullptr (δ_i = ∞ or >= δ)
    uint64_t root_lo, n_roots;
    unsigned long long *counts;     // 36 bins, index a * 6 + b
};

#ifndef __CUDACC_RTC__
cudaError_t launch_census36(const CensusParams &p, int grid, cudaStream_t s);
// prefix-disconnected motifs (dfs.cu): thread-per-root search, modes kCount / kEnum / kRoots
cudaError_t launch_mine_dfs(const MineParams &p, int mode, int sms, cudaStream_t s, uint32_t *grid_out);

using MineKernel = void (*)(MineParams);

struct KernelInfo {
    MineKernel fn;
    int smem_per_warp;    // bytes
};

// Runtime-specialised kernels (csrc/rtc.cu, tm_motif_specialise): a CUfunction
// of mine_kernel<PlanC<code, gen>, mode> compiled with NVRTC, and its launch.
struct RtcKernel {
    void *fn = nullptr;     // CUfunction
    int smem_per_warp = 0;  // bytes
};
tm_status rtc_kernel(uint64_t code, bool gen, int mode, RtcKernel *out);
cudaError_t rtc_set_smem(void *fn, int bytes);
cudaError_t rtc_occupancy(void *fn, int threads, size_t smem, int *per_sm);
// coop: a cooperative launch (every CTA resident at once, or the launch fails)
cudaError_t rtc_launch(void *fn, unsigned grid, int threads, size_t smem, cudaStream_t s, const MineParams &p,
                       bool coop);

// catalog lookup: specialised kernel for `code` in `mode`, else the generic one
KernelInfo lookup_kernel(uint64_t code, int mode, bool *specialised, bool generic = false);
bool is_specialised(uint64_t code);

// Device memory of the library: a per-device CUDA memory pool that keeps
// freed blocks for reuse (release threshold = max), so per-query buffers
// (horizons, scratch) and repeated graph builds cost no cudaMalloc/cudaFree.
cudaError_t dev_alloc(void **p, size_t bytes, cudaStream_t s);
void dev_free(void *p, cudaStream_t s);

// NVTX range for profilers (nsys / ncu --nvtx): host-side phase markers of
// graph build, horizons, window descriptors and each mining launch
struct NvtxRange {
    explicit NvtxRange(const char *name) { nvtxRangePushA(name); }
    ~NvtxRange() { nvtxRangePop(); }
    NvtxRange(const NvtxRange &) = delete;
    NvtxRange &operator=(const NvtxRange &) = delete;
};

// error plumbing
void set_error(const std::string &msg);
tm_status fail(tm_status st, const std::string &msg);
#endif  // !__CUDACC_RTC__

}  // namespace tmg

#ifndef __CUDACC_RTC__
#define TM_CUDA_TRY(expr)                                                                   \
    do {                                                                                     \
        cudaError_t _e = (expr);                                                             \
        if (_e != cudaSuccess)                                                               \
            return tmg::fail(_e == cudaErrorMemoryAllocation ? TM_ENOMEM : TM_ECUDA,          \
                            std::string(#expr) + ": " + cudaGetErrorString(_e));             \
    } while (0)
#endif  // !__CUDACC_RTC__
