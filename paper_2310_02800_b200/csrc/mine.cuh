// Mining kernel: δ-windowed backtracking search rooted at every edge
// (Algorithm 1), re-designed warp-cooperatively for sm_100a.
//
// One persistent warp owns a depth-first stack of *tasks* per search level.
// A task at level l is a partial match with l matched edges (a search-tree
// node) together with its cached candidate window [lo, up) — a range of
// packed (edge id << 32 | neighbour) records in one time-sorted adjacency
// list — plus what the next levels need: the coarse bound hi = H_δ[e_1], the
// bound motif vertices φ (and, for enumeration, the matched edge ids).  The
// window is searched exactly once, when the node is created, and consumed
// from the cache afterwards (the paper's candidate caching).
//
// Each step the warp takes up to 32 candidates from the top tasks of one level
// (warp scan over window sizes, ballot/popc lane->task map, shfl broadcast),
// loads their records (consecutive lanes, consecutive records), checks the
// structure (StructConstraints P:324-331 as compile-time equal/not-equal
// tests), and either counts/enumerates (last level) or turns
// survivors into child tasks by searching their next window (binary search on
// the record array, edge ids only — no timestamps in this kernel: the time
// bounds are precomputed as horizon indices).  Levels are chosen
// deepest-first whenever a full 32-candidate batch is available, which keeps
// every stack within kCap tasks (a level is expanded only while its child
// stack has room for a full batch of 32 children).
#pragma once

#include "tm_internal.cuh"

namespace tmg {

#ifndef TM_CAP
#define TM_CAP 48   // measured (C4 bench step, mining kernel): 64: 9.10 ms, 48/44: 8.22, 40: 8.31, 36: 8.60, 33: 9.31 —
                    // smaller stacks leave more of the SM's 228 KB to L1 (hub lists, descriptors)
#endif
constexpr int kCap = TM_CAP;         // tasks per level per warp (>= 33)
constexpr uint32_t kRoom = kCap - 31;   // a level with fewer tasks takes a batch of 32 children
static_assert(kCap >= 33 && kCap <= 64, "kCap");
#ifndef TM_WARPS_PER_BLOCK
#define TM_WARPS_PER_BLOCK 8
#endif
constexpr int kWarpsPerBlock = TM_WARPS_PER_BLOCK;
#ifndef TM_ROOT_CHUNK
#define TM_ROOT_CHUNK 64    // measured: 32 +0.8 %, 64 -0.4 % (C4) / -1.2 % (C5 slice), 256 +3.2 % against 128
#endif
constexpr int kRootChunk = TM_ROOT_CHUNK;   // roots claimed per global atomic (large launches)
// A resume from few rows (~10^5 sibling rows) claims 32 at a time so every
// warp of the grid gets some: with 128, 216 k diamond rows reach only ~1700
// of the 5920 warps and the kernel is all tail (DIA 0.41 -> 0.24 ms).
#ifndef TM_SMALL_CHUNK
#define TM_SMALL_CHUNK 1
#endif
#ifndef TM_SHARE
#define TM_SHARE 1          // heavy-subtree sharing compiled in (tm_run_opts.share)
#endif
#ifndef TM_TIMING
#define TM_TIMING 1         // load-balance timing (tm_run_info.tail_ms / warp_busy)
#endif
#ifndef TM_SHARE_MIN
#define TM_SHARE_MIN 128
#endif
constexpr int kShareMin = TM_SHARE_MIN;   // smallest window handed to an idle warp (share = 0)
#ifndef TM_HRANK
#define TM_HRANK 3          // window-end ranks: 0 off, 1 precomputed per query (build_hrank), 2 memoised in-kernel,
                            // 3 precomputed window descriptors {start, end, H_δi} (one 16-byte load)
#endif
constexpr bool kHrankMemo = TM_HRANK == 2;
constexpr bool kHrankDesc = TM_HRANK == 3;
#ifndef TM_SHARE_POLL
#define TM_SHARE_POLL 16
#endif
constexpr uint32_t kSharePoll = TM_SHARE_POLL;   // iterations between reads of the idle counter (power of 2)
constexpr unsigned kShareStop = 0xFFFFFFFFu;     // flag value: the search is complete
#ifndef TM_SHARE_SLEEP
#define TM_SHARE_SLEEP 2048
#endif
constexpr unsigned kShareSleepMax = TM_SHARE_SLEEP;   // ns, longest back-off of a waiting warp
#ifndef TM_LEAF_SECTORS
#define TM_LEAF_SECTORS 4
#endif
constexpr int kLeafSectors = TM_LEAF_SECTORS;
#ifndef TM_PAIR_FILTER
#define TM_PAIR_FILTER 1    // 1: closing leaves test the pair index's membership filter first (graphs with one)
#endif
#ifndef TM_ROOT_PRUNE
#define TM_ROOT_PRUNE 1     // roots with an empty closing look-ahead window are not searched (no prefix counts)
#endif
#ifndef TM_LOOK_EXTRA
#define TM_LOOK_EXTRA 7     // with root pruning: sectors of the look-ahead window read past the first
#endif
#ifndef TM_ROOT_CLAMP
#define TM_ROOT_CLAMP 1     // with root pruning: the root's horizon clamps to its closing window's latest edge
#endif
#ifndef TM_LEAF_TASK
#define TM_LEAF_TASK 0      // 1: known leaf windows are pushed as tasks instead of scanned in the lane
#endif
#ifndef TM_PAIR_LONG
#define TM_PAIR_LONG 1      // long closing-leaf windows counted from the pair index (when the graph has one)
#endif
#ifndef TM_PAIR_MIN
#define TM_PAIR_MIN 16      // ... for known windows of more than this many records (the in-lane scan's 4 sectors)
#endif
constexpr uint32_t kPairMin = TM_PAIR_MIN;
#ifndef TM_PAIR_SECTORS
#define TM_PAIR_SECTORS 1   // ... and unknown-end windows after this many sectors in the lane
#endif                      // (C5 slice: 1: 169 ms, 4: 182 ms; none: 231 ms)
constexpr int kPairSectors = TM_PAIR_SECTORS;
#ifndef TM_LOOKAHEAD
#define TM_LOOKAHEAD 1      // closing look-ahead bound from the root (Shape::look)
#endif
      // leaf windows scanned inline up to 8 records
constexpr unsigned kFull = 0xffffffffu;

__device__ __forceinline__ unsigned long long globaltimer_ns() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}

__device__ __forceinline__ uint32_t lanemask_lt() {
    uint32_t r;
    asm("mov.u32 %0, %%lanemask_lt;" : "=r"(r));
    return r;
}

// Compile-time loop: f(ic<I>) for I = 0..N-1, so that per-index layout
// decisions are constant expressions (if constexpr).  Own index sequence:
// the header also compiles under NVRTC (tm_motif_specialise), without <utility>.
template <int V>
struct ic {
    static constexpr int value = V;
};
template <int... I>
struct iseq {};
template <int N, int... I>
struct make_iseq : make_iseq<N - 1, N - 1, I...> {};
template <int... I>
struct make_iseq<0, I...> {
    using type = iseq<I...>;
};
template <class F, int... I>
__device__ __forceinline__ void sfor_impl(F &&f, iseq<I...>) {
    (f(ic<I>{}), ...);
}
template <int N, class F>
__device__ __forceinline__ void sfor(F &&f) {
    if constexpr (N > 0) sfor_impl(f, typename make_iseq<N>::type{});
}

// First position p in [b, e) whose record's edge id is > key (e if none):
// the "filter via binary search" of GetCandidateEdgeList on
// edge ids (ids are ranks in time order, so "after e_prev" is "id > e_prev"
// and "t <= bound" is "id <= H_bound[...]").
__device__ __forceinline__ uint32_t first_after(const uint64_t *__restrict__ rec, uint32_t b,
                                                uint32_t e, uint32_t key) {
    while (b < e) {
        uint32_t mid = b + ((e - b) >> 1);
        uint32_t id = (uint32_t)(__ldg(rec + mid) >> 32);
        if (id > key) e = mid;
        else b = mid + 1;
    }
    return b;
}

// Same answer as first_after, for a key whose answer is expected near b
// (windows are δ-bounded and short): the first round trip fetches the whole
// aligned 32-byte sector holding b (records 4k..4k+3, two 16-byte loads in
// flight together), then gallops sector by sector and binary-searches the
// bracket.  rec is padded by 4 records, so the vector loads never leave the
// allocation.
__device__ __forceinline__ uint32_t gallop_after(const uint64_t *__restrict__ rec, uint32_t b, uint32_t e,
                                                 uint32_t key) {
    if (b >= e) return b;
    const uint32_t a = b & ~3u;
    const ulonglong2 *v = reinterpret_cast<const ulonglong2 *>(rec + a);
    const ulonglong2 x0 = __ldg(v), x1 = __ldg(v + 1);
    const uint32_t id[4] = {(uint32_t)(x0.x >> 32), (uint32_t)(x0.y >> 32), (uint32_t)(x1.x >> 32),
                            (uint32_t)(x1.y >> 32)};
#pragma unroll
    for (int k = 0; k < 4; k++) {
        const uint32_t p = a + k;
        if (p >= b && p < e && id[k] > key) return p;
    }
    if (a + 4 >= e) return e;
    uint32_t lo = a + 4, step = 4, hi;
    while (true) {
        hi = lo + step - 1;
        if (hi >= e) { hi = e; break; }
        if ((uint32_t)(__ldg(rec + hi) >> 32) > key) break;
        lo = hi + 1;
        step <<= 1;
    }
    return first_after(rec, lo, hi, key);
}

// First position p >= b with id > key in a sentinel-terminated list (every
// list ends with an id-0xFFFFFFFF record, so no list end is needed): scans
// aligned 32-byte sectors, two 16-byte loads each.  Used where the answer is
// close to b (the lower bound after an older anchor edge).
__device__ __forceinline__ uint32_t scan_after(const uint64_t *__restrict__ rec, uint32_t b, uint32_t key) {
    uint32_t a = b & ~3u;
    while (true) {
        const ulonglong2 *v = reinterpret_cast<const ulonglong2 *>(rec + a);
        const ulonglong2 x0 = __ldg(v), x1 = __ldg(v + 1);
        const uint32_t id[4] = {(uint32_t)(x0.x >> 32), (uint32_t)(x0.y >> 32), (uint32_t)(x1.x >> 32),
                                (uint32_t)(x1.y >> 32)};
#pragma unroll
        for (int k = 0; k < 4; k++)
            if (a + k >= b && id[k] > key) return a + k;
        a += 4;
    }
}

// first index p in [b, e) with a[p] > key (u32 ids)
__device__ __forceinline__ uint32_t first_after32(const uint32_t *__restrict__ a, uint32_t b, uint32_t e, uint32_t key) {
    while (b < e) {
        const uint32_t mid = b + ((e - b) >> 1);
        if (__ldg(a + mid) > key) e = mid;
        else b = mid + 1;
    }
    return b;
}

// The candidate window of a motif edge with both endpoints mapped: the edges
// a -> b with id in (e, lim], as positions [lo, up) of the pair index.  One
// hash probe (linear probing) finds the pair; an absent pair is the common
// case and costs that probe only.
__device__ __forceinline__ void pair_window(const MineParams &p, uint32_t a, uint32_t b, uint32_t e, uint32_t lim,
                                            const uint32_t *hf, uint32_t &lo, uint32_t &up) {
    const uint64_t key = ((uint64_t)a << 32) | b;
    const uint64_t hh = pair_hash(key);
    if (!pair_maybe(p.pbits, p.fmask, hh)) {   // certainly absent
        lo = up = 0;
        return;
    }
    uint32_t h = (uint32_t)hh & p.pmask;
    uint32_t st = 0, len = 0;
    while (true) {
        const uint4 sl = __ldg(p.ptab + h);
        const uint64_t k = ((uint64_t)sl.y << 32) | sl.x;
        if (k == key) { st = sl.z; len = sl.w; break; }
        if (k == ~0ull) break;
        h = (h + 1) & p.pmask;
    }
    if (hf) lim = min(lim, __ldg(hf + e));   // the fine bound, read only for pairs that exist
    lo = first_after32(p.prec, st, st + len, e);
    up = first_after32(p.prec, lo, st + len, lim);
}

// records of the root window read for the closing look-ahead mask, from the
// aligned sector holding the window start (4: one sector, 8 or 12: two or three)
#ifndef TM_LOOK_RECS
#define TM_LOOK_RECS 4
#endif
constexpr int kLookRecs = TM_LOOK_RECS;
static_assert(kLookRecs == 4 || kLookRecs == 8 || kLookRecs == 12, "kLookRecs");

// Per-root arrays (src, dst, H, the look-ahead rank) are read once per root in
// root order: with TM_STREAM_HINT they are loaded evict-first (ld.global.cs),
// so they do not push list records and descriptors out of L2
#ifndef TM_STREAM_HINT
#define TM_STREAM_HINT 0
#endif
__device__ __forceinline__ uint32_t ld_stream(const uint32_t *q) {
    if (TM_STREAM_HINT) return __ldcs(q);
    return __ldg(q);
}

// bit of vertex v in a closing look-ahead mask (Fibonacci hashing)
__device__ __forceinline__ uint32_t look_hash(uint32_t v);

// The rest of a closing look-ahead window past its first sector (root
// pruning): from position a (sector-aligned), up to TM_LOOK_EXTRA sectors.
// Returns {mask, latest id} with the records <= hi folded into mask / last,
// or {~0u, last} if the window runs on past them.
static __device__ __noinline__ uint2 look_more(const uint64_t *__restrict__ rec, uint32_t a, uint32_t hi, uint32_t mask,
                                        uint32_t last) {
    const ulonglong2 *vp = reinterpret_cast<const ulonglong2 *>(rec + a);
#pragma unroll 1
    for (int q = 0; q < TM_LOOK_EXTRA; q++) {
        const ulonglong2 x0 = __ldg(vp + 2 * q), x1 = __ldg(vp + 2 * q + 1);
        const uint64_t r4[4] = {x0.x, x0.y, x1.x, x1.y};
#pragma unroll
        for (int k = 0; k < 4; k++) {
            if ((uint32_t)(r4[k] >> 32) > hi) return make_uint2(mask, last);
            mask |= 1u << look_hash((uint32_t)r4[k]);
            last = (uint32_t)(r4[k] >> 32);
        }
    }
    return make_uint2(~0u, last);
}

// bit of vertex v in a closing look-ahead mask (Fibonacci hashing)
__device__ __forceinline__ uint32_t look_hash(uint32_t v) { return (v * 0x9E3779B1u) >> 27; }

// saturating arithmetic of the per-level candidate hints (Warp::cand)
__device__ __forceinline__ uint32_t cand_add(uint32_t c, uint32_t a) { return c > 0x7FFFFFFFu - a ? 0x7FFFFFFFu : c + a; }
__device__ __forceinline__ uint32_t cand_sub(uint32_t c, uint32_t a) { return c > a ? c - a : 0u; }

__device__ __forceinline__ uint32_t ceil_log2p1(uint32_t len) {  // ceil(log2(len+1))
    return len ? 32 - __clz(len) : 0;
}

// ------------------------------------------------------------------ plans
// Static decode of a motif, the `minfo` of P:739-780: for motif edge l
// (0-based) which endpoints are already mapped, which adjacency list supplies
// the candidates, and which earlier matched edge anchors the window's lower
// bound.  Used at compile time (PlanC) and at run time (PlanR).
struct Shape {
    int L;
    int u[kMaxL], v[kMaxL];
    __host__ __device__ constexpr int nv(int l) const {  // vertices mapped by edges [0, l)
        int mx = -1;
        for (int i = 0; i < l; i++) {
            mx = u[i] > mx ? u[i] : mx;
            mx = v[i] > mx ? v[i] : mx;
        }
        return mx + 1;
    }
    __host__ __device__ constexpr int last_touch(int l, int x) const {
        for (int i = l - 1; i >= 0; --i)
            if (u[i] == x || v[i] == x) return i;
        return -1;
    }
    // candidate list of motif edge l: 0 = OUT(φ(u_l)), 1 = IN(φ(v_l)).  With
    // both endpoints mapped (reading Q8) take the list whose vertex
    // was touched most recently: its window start is one rank load away.
    __host__ __device__ constexpr int ldir(int l) const {
        const int nb = nv(l);
        const bool ub = u[l] < nb, vb = v[l] < nb;
        if (ub && vb) return last_touch(l, u[l]) > last_touch(l, v[l]) ? 0 : 1;
        return ub ? 0 : 1;
    }
    __host__ __device__ constexpr int lx(int l) const { return ldir(l) == 0 ? u[l] : v[l]; }
    // the latest matched edge touching the list vertex, and the rank variant
    // (2 * endpoint + dir) locating it in that list
    __host__ __device__ constexpr int anc(int l) const { return last_touch(l, lx(l)); }
    __host__ __device__ constexpr int avar(int l) const { return (u[anc(l)] == lx(l) ? 0 : 2) + ldir(l); }
    // What a task at level l (l matched edges) must carry for the rest of its
    // subtree — the paper's "number of valid mappings at each level"
    // taken one step further: only the φ slots later checks or lists read, the
    // matched ids later window anchors read, and hi only if windows follow.
    // both endpoints of motif edge l mapped: its candidates are exactly the
    // edges of one vertex pair, read from the pair index
    __host__ __device__ constexpr bool pairk(int l) const {
        return u[l] < nv(l) && v[l] < nv(l) && ((TM_PAIR_LEAF && TM_PAIR_NONLEAF) || (TM_PAIR_LEAF ? l + 1 == L : (TM_PAIR_NONLEAF && l + 1 < L)));
    }
    __host__ __device__ constexpr bool keep_phi(int l, int k) const {
        if (k >= nv(l)) return false;
        for (int q = l; q < L; ++q)             // injectivity check of a new endpoint
            if (!pairk(q) && k < nv(q)) return true;
        for (int q = l + 1; q < L; ++q) {       // vertices of a later window
            if (pairk(q) ? (u[q] == k || v[q] == k) : lx(q) == k) return true;
        }
        return false;
    }
    // Closing look-ahead.  The last motif edge with both endpoints mapped is
    // an edge between two bound vertices, so it lies in BOTH of their lists
    // (Algorithm 1 may read either, "N_out(u_G)/N_in(v_G)").  The
    // kernel scans the list of the most recently touched endpoint x (ldir);
    // when the other endpoint y is an endpoint of the root edge (motif vertex
    // 0 or 1), every match's last edge is also a record of y's other-direction
    // list with id in (e_1, H_δ(e_1)], whose neighbour is φ(x).  The root
    // reads that window once (one rank load, one sector) and keeps a 32-bit
    // mask of hashed neighbours (0 for an empty window, all ones when the
    // window runs past the sector).  A closing window whose φ(x) is not in
    // the mask holds no match and is not read at all.  The search tree is
    // unchanged (the closing edge is a leaf), so the counts, the matches and
    // every level's nodes are Algorithm 1's; only leaf scans are skipped.
    __host__ __device__ constexpr int lkdir() const { return 1 - ldir(L - 1); }
    __host__ __device__ constexpr int lky() const { return lkdir() == 0 ? u[L - 1] : v[L - 1]; }
    __host__ __device__ constexpr bool look() const {
        return TM_LOOKAHEAD && L >= 3 && u[L - 1] < nv(L - 1) && v[L - 1] < nv(L - 1) && !pairk(L - 1) && lky() <= 1;
    }
    // rank variant of the root edge in y's list: 2 * (endpoint of e_1) + direction
    __host__ __device__ constexpr int lkvar() const { return (lky() == 0 ? 0 : 2) + lkdir(); }
    __host__ __device__ constexpr bool keep_eh(int l, int k) const {
        for (int q = l + 1; q < L; ++q)
            if (k < l && !pairk(q) && anc(q) == k) return true;
        return false;
    }
    __host__ __device__ constexpr bool keep_hi(int l) const { return l + 1 < L; }
};

template <uint64_t CODE>
__host__ __device__ constexpr Shape shape_of() {
    Shape s{};
    s.L = (int)(CODE & 7);
    for (int i = 0; i < kMaxL; i++) {
        s.u[i] = i < s.L ? (int)((CODE >> (3 + 6 * i)) & 7) : 0;
        s.v[i] = i < s.L ? (int)((CODE >> (6 + 6 * i)) & 7) : 0;
    }
    return s;
}

// Compile-time plan: the motif structure is a template argument, so every
// per-level choice (which list, which checks, how many mapped vertices, the
// anchor) is a constant — the B200 counterpart of the paper's generated
// motif-specific code.
// GEN: the generalized query (labels, anti-edges) is checked too; tasks then
// keep every φ slot and matched id (a complete match's anti-edge check reads
// them).  Catalog kernels are GEN = false; GEN = true ones are compiled at run
// time (tm_motif_specialise, csrc/rtc.cu).
template <uint64_t CODE, bool GEN = false>
struct PlanC {
    static constexpr bool kGeneral = GEN;
    static constexpr int kL = shape_of<CODE>().L;
    // φ slots stored with a level-l task
    __host__ __device__ static constexpr int nslots(int l) { return shape_of<CODE>().nv(l); }
    __host__ __device__ static constexpr bool keep_phi(int l, int k) {
        return GEN ? k < nslots(l) : shape_of<CODE>().keep_phi(l, k);
    }
    __host__ __device__ static constexpr bool keep_eh(int l, int k) { return GEN || shape_of<CODE>().keep_eh(l, k); }
    __host__ __device__ static constexpr bool keep_hi(int l) { return shape_of<CODE>().keep_hi(l); }
    __device__ explicit PlanC(const MineParams &) {}
    // every accessor is forced through a constant expression, so no decode
    // survives to run time (no local-memory copy of the Shape)
    __device__ __forceinline__ static constexpr int L() { return kL; }
    template <int I> __device__ __forceinline__ static constexpr int u() { constexpr int r = shape_of<CODE>().u[I]; return r; }
    template <int I> __device__ __forceinline__ static constexpr int v() { constexpr int r = shape_of<CODE>().v[I]; return r; }
    template <int I> __device__ __forceinline__ static constexpr int nv() { constexpr int r = shape_of<CODE>().nv(I); return r; }
    template <int I> __device__ __forceinline__ static constexpr int ldir() { constexpr int r = shape_of<CODE>().ldir(I); return r; }
    template <int I> __device__ __forceinline__ static constexpr int lx() { constexpr int r = shape_of<CODE>().lx(I); return r; }
    template <int I> __device__ __forceinline__ static constexpr int anc() { constexpr int r = shape_of<CODE>().anc(I); return r; }
    template <int I> __device__ __forceinline__ static constexpr int avar() { constexpr int r = shape_of<CODE>().avar(I); return r; }
    template <int I> __device__ __forceinline__ static constexpr bool pairk() { constexpr bool r = shape_of<CODE>().pairk(I); return r; }
    __host__ __device__ static constexpr bool look() { return !GEN && shape_of<CODE>().look(); }
    __host__ __device__ static constexpr int lkvar() { return shape_of<CODE>().lkvar(); }
};

// Runtime plan: the same kernel body for any prefix-connected motif with
// L <= kMaxL edges, the decode computed per thread from the launch
// parameters.
struct PlanR {
    static constexpr bool kGeneral = true;
    static constexpr int kL = kMaxL;
    __host__ __device__ static constexpr int nslots(int l) { return l + 1 < kMaxV ? l + 1 : kMaxV; }
    __host__ __device__ static constexpr bool keep_phi(int l, int k) { return k < nslots(l); }
    __host__ __device__ static constexpr bool keep_eh(int, int) { return true; }
    __host__ __device__ static constexpr bool keep_hi(int) { return true; }
    int L_;
    int u_[kMaxL], v_[kMaxL], nv_[kMaxL + 1], ldir_[kMaxL], lx_[kMaxL], anc_[kMaxL], avar_[kMaxL];
    bool pairk_[kMaxL];
    __device__ explicit PlanR(const MineParams &p) {
        Shape s{};
        s.L = (int)p.L;
#pragma unroll
        for (int i = 0; i < kMaxL; i++) {
            s.u[i] = i < s.L ? p.u[i] : 0;
            s.v[i] = i < s.L ? p.v[i] : 0;
        }
        L_ = s.L;
#pragma unroll
        for (int i = 0; i <= kMaxL; i++) nv_[i] = s.nv(i);
#pragma unroll
        for (int i = 0; i < kMaxL; i++) {
            u_[i] = s.u[i];
            v_[i] = s.v[i];
            const bool live = i >= 1 && i < s.L;
            ldir_[i] = live ? s.ldir(i) : 0;
            lx_[i] = live ? s.lx(i) : 0;
            anc_[i] = live ? s.anc(i) : 0;
            avar_[i] = live ? s.avar(i) : 0;
            pairk_[i] = live && s.pairk(i);
        }
    }
    __device__ __forceinline__ int L() const { return L_; }
    template <int I> __device__ __forceinline__ int u() const { return u_[I]; }
    template <int I> __device__ __forceinline__ int v() const { return v_[I]; }
    template <int I> __device__ __forceinline__ int nv() const { return nv_[I]; }
    template <int I> __device__ __forceinline__ int ldir() const { return ldir_[I]; }
    template <int I> __device__ __forceinline__ int lx() const { return lx_[I]; }
    template <int I> __device__ __forceinline__ int anc() const { return anc_[I]; }
    template <int I> __device__ __forceinline__ int avar() const { return avar_[I]; }
    template <int I> __device__ __forceinline__ bool pairk() const { return pairk_[I]; }
    // no closing look-ahead in the generic kernel (per-root counts, instrumentation)
    __host__ __device__ static constexpr bool look() { return false; }
    __host__ __device__ static constexpr int lkvar() { return 0; }
};

#ifndef TM_SIB_LAZY_EH
#define TM_SIB_LAZY_EH 1
#endif
// ------------------------------------------------------- shared-memory layout
// Per warp, per level l = 1..kL-1, a structure of arrays of kCap tasks:
//   [0] lo  [1] up  [2] hi  [3 .. 3+S) φ  [.. +l) matched edge ids  [+1] root slot (kRoots)
template <class Plan, int MODE>
struct Layout {
    // [0] lo  [1] up  [2 ..) kept φ slots  [hi]  kept matched edge ids  [root slot (kRoots)]
    // kCountSib keeps every φ slot and matched id up to its sibling level: the rows read them
    __host__ __device__ static constexpr bool kphi(int l, int k) {
        return MODE == kStats || (MODE == kCountSib && l <= kSibLevel) || Plan::keep_phi(l, k);
    }
    __host__ __device__ static constexpr bool keh(int l, int k) {
        return k < l && (MODE == kEnum || MODE == kStats || (MODE == kCountSib && l <= kSibLevel) ||
                         Plan::keep_eh(l, k));
    }
    // matched ids a level-l expansion loads per candidate: the sibling rows'
    // extra ids at kSibLevel are read from shared memory only for a row
    __host__ __device__ static constexpr bool keh_load(int l, int k) {
        return keh(l, k) && !(TM_SIB_LAZY_EH && MODE == kCountSib && l == kSibLevel && k < l && !Plan::keep_eh(l, k));
    }
    __host__ __device__ static constexpr bool khi(int l) { return MODE == kStats || Plan::keep_hi(l); }
    // the closing look-ahead mask (Shape::look) of the root, carried to level L-2
    __host__ __device__ static constexpr bool look() { return MODE != kStats && Plan::look(); }
    __host__ __device__ static constexpr bool kli(int l) { return look() && l >= 1 && l + 2 <= Plan::kL; }
    __host__ __device__ static constexpr int phi(int l, int k) {
        int f = 2;
        for (int i = 0; i < k; i++) f += kphi(l, i) ? 1 : 0;
        return f;
    }
    __host__ __device__ static constexpr int hi(int l) { return phi(l, Plan::nslots(l)); }
    __host__ __device__ static constexpr int li(int l) { return hi(l) + (khi(l) ? 1 : 0); }
    __host__ __device__ static constexpr int eh(int l, int k) {
        int f = li(l) + (kli(l) ? 1 : 0);
        for (int i = 0; i < k; i++) f += keh(l, i) ? 1 : 0;
        return f;
    }
    __host__ __device__ static constexpr int rs(int l) { return eh(l, l); }
    __host__ __device__ static constexpr int fields(int l) { return rs(l) + (MODE == kRoots ? 1 : 0); }
    __host__ __device__ static constexpr int off(int l) {  // word offset of level l
        int o = 0;
        for (int k = 1; k < l; k++) o += fields(k) * kCap;
        return o;
    }
    __host__ __device__ static constexpr int warp_words() { return Plan::kL > 1 ? off(Plan::kL) : 1; }
};

template <int N>
__device__ __forceinline__ uint32_t pick(const uint32_t (&a)[N], int k) {
    uint32_t r = 0;
#pragma unroll
    for (int i = 0; i < N; i++)
        if (i == k) r = a[i];
    return r;
}

struct Stats {
    unsigned long long nodes[kMaxL];
    unsigned long long window, list, probes, fast_window;
};

template <class Plan, int MODE>
struct Warp {
    static constexpr int LM = Plan::kL;  // levels 1..LM-1 hold tasks
    const MineParams &p;
    const Plan &plan;
    uint32_t *ws;
    int lane;
    uint32_t ntask[LM + 1];
    // candidates pending per level (Σ window sizes of its tasks): a scheduling
    // hint only (correctness never depends on it) kept in u32 — window sizes
    // are clamped to 2^26 when added and subtractions saturate at 0, so it
    // never exceeds the true value and is exact below 2^26 per window
    uint32_t cand[LM + 1];
    unsigned long long count;        // lane 0: matches found by batch expansion
    unsigned long long leaf_count;   // per lane: matches found by leaf scans
    uint32_t pfx_lane;               // per lane: nodes at level prefix_lv0 (kCountPfx)
    uint32_t n_items;                // roots (or, kResume, rows) this launch mines
    Stats st;

    __device__ Warp(const MineParams &p_, const Plan &pl, uint32_t *w, int ln) : p(p_), plan(pl), ws(w), lane(ln) {
#pragma unroll
        for (int i = 0; i <= LM; i++) { ntask[i] = 0; cand[i] = 0; }
        count = 0;
        leaf_count = 0;
        pfx_lane = 0;
        n_items = (uint32_t)p.n_roots;
        if (MODE == kResume) {
            unsigned long long n = 0;
            if (ln == 0) n = *reinterpret_cast<const volatile unsigned long long *>(p.resume_n);
            n = __shfl_sync(kFull, n, 0);
            n_items = (uint32_t)min(n, (unsigned long long)p.sib_cap);
#ifdef TM_DEBUG_RESUME
            if (ln == 0 && blockIdx.x == 0 && threadIdx.x == 0)
                printf("[resume] n=%llu cap=%u level=%u rows=%p row0=%u %u %u\n", n, p.sib_cap, p.resume_level,
                       (const void *)p.resume_rows, p.resume_rows[0], p.resume_rows[1], p.resume_rows[2]);
#endif
        }
        if (MODE == kStats) {
#pragma unroll
            for (int i = 0; i < kMaxL; i++) st.nodes[i] = 0;
            st.window = st.list = st.probes = st.fast_window = 0;
        }
    }

    // SoA column F of level L_ (both compile-time: the offset is a constant)
    template <int L_, int F>
    __device__ __forceinline__ uint32_t *fld() const {
        constexpr int o = Layout<Plan, MODE>::off(L_) + F * kCap;
        return ws + o;
    }

    // StructConstraints of a candidate record for motif edge LV,
    // with the plan's static checks.  w: the record's neighbour,
    // from_out: the record comes from the out-list of φ(u_LV) (w is its
    // destination) rather than the in-list of φ(v_LV) (w is its source).
    template <int LV, int N>
    __device__ __forceinline__ bool accept(uint32_t w, bool from_out, const uint32_t (&phi)[N]) const {
        const int uM = plan.template u<LV>(), vM = plan.template v<LV>(), nb = plan.template nv<LV>();
        if (uM < nb && vM < nb) return from_out ? (w == pick(phi, vM)) : (w == pick(phi, uM));
        bool ok = true;  // the new endpoint must be a graph vertex not yet mapped (injectivity)
#pragma unroll
        for (int k = 0; k < N; k++)
            if (k < nb) ok &= (w != phi[k]);
        return ok;
    }

    // ------------------------------------------ generalized query (N2, PlanR)
    __device__ __forceinline__ bool gen() const { return Plan::kGeneral && p.gen; }
    __device__ __forceinline__ int32_t vlabel(uint32_t v) const { return p.vlab ? __ldg(p.vlab + v) : 0; }
    __device__ __forceinline__ int32_t elabel(uint32_t e) const { return p.elab ? __ldg(p.elab + e) : 0; }

    // Label checks of graph edge e matched to motif edge l, w its endpoint
    // mapped for the first time (motif vertex nb), if any.
    __device__ __forceinline__ bool labels_ok(int l, uint32_t e, bool fresh, int nb, uint32_t w) const {
        if (p.ereq[l] != TM_ANY_LABEL && elabel(e) != p.ereq[l]) return false;
        if (fresh && p.vreq[nb] != TM_ANY_LABEL && vlabel(w) != p.vreq[nb]) return false;
        return true;
    }

    // Temporal anti-edges of a complete match: φ = phi
    // (every motif vertex), matched edges eh[0..L-2] and e.  Rejected if the
    // out-list of φ(u_j) holds an edge to φ(v_j), other than the match's own
    // (reading Q22), with id in [tie_lo[e_a], H_{δ_ij}[e_a]] — i.e. with
    // t in [t(e_a), t(e_a) + δ_ij].
    template <int NS, int NE>
    __device__ bool anti_ok(const uint32_t (&phi)[NS], const uint32_t (&eh)[NE], uint32_t e) const {
        const int L = plan.L();
        for (uint32_t j = 0; j < p.n_anti; j++) {
            const uint32_t x = pick(phi, p.anti_u[j]), y = pick(phi, p.anti_v[j]);
            const int a = p.anti_a[j];
            const uint32_t ea = a == L - 1 ? e : pick(eh, a);
            const uint32_t lo_id = __ldg(p.tie_lo + ea), hi_id = __ldg(p.anti_hi[j] + ea);
            const uint32_t b = __ldg(p.off_out + x), en = __ldg(p.off_out + x + 1) - 1;
            uint32_t q = lo_id ? first_after(p.rec, b, en, lo_id - 1) : b;
            for (;; ++q) {   // the list's sentinel (id 0xFFFFFFFF) ends the scan
                const uint64_t r = __ldg(p.rec + q);
                const uint32_t id = (uint32_t)(r >> 32);
                if (id > hi_id) break;
                if ((uint32_t)r != y) continue;
                bool own = id == e;
#pragma unroll
                for (int i = 0; i < NE; i++)
                    if (i < L - 1 && eh[i] == id) own = true;
                if (!own) return false;
            }
        }
        return true;
    }

    // enumerate one match found by a leaf scan: eh[0..nl-2], e, last
    template <int NE>
    __device__ __forceinline__ void emit_one(const uint32_t (&eh)[NE], uint32_t e, uint32_t last, int nl) {
        const unsigned long long row = atomicAdd(&p.scratch[2], 1ull);
        if (row < p.cap) {
            uint32_t *dst = p.enum_buf + row * (uint64_t)(nl + 1);
#pragma unroll
            for (int i = 0; i < NE; i++)
                if (i < nl - 1) dst[i] = eh[i] + p.id_offset;
            dst[nl - 1] = e + p.id_offset;
            dst[nl] = last + p.id_offset;
        }
    }

    // Emit the matches of the lanes with `ok` (last motif edge matched).
    // eh: the L-1 earlier edge ids, e: the last one.
    template <int NE>
    __device__ __forceinline__ void emit(bool ok, const uint32_t (&eh)[NE], uint32_t e, uint32_t rslot) {
        uint32_t mask = __ballot_sync(kFull, ok);
        if (lane == 0) count += __popc(mask);
        if (MODE == kEnum) {
            if (!mask) return;
            unsigned long long base = 0;
            if (lane == 0) base = atomicAdd(&p.scratch[2], (unsigned long long)__popc(mask));
            base = __shfl_sync(kFull, base, 0);
            if (ok) {
                uint64_t row = base + __popc(mask & lanemask_lt());
                if (row < p.cap) {
                    const int L = plan.L();
                    uint32_t *dst = p.enum_buf + row * (uint64_t)L;
#pragma unroll
                    for (int i = 0; i < NE; i++)
                        if (i < L - 1) dst[i] = eh[i] + p.id_offset;
                    dst[L - 1] = e + p.id_offset;
                }
            }
        } else if (MODE == kRoots) {
            if (ok) atomicAdd(&p.root_counts[rslot], 1ull);
        }
    }

    // Create level-NL tasks from the lanes with `ok`: a partial match with NL
    // matched edges, last edge e, bound vertices phi.  Searches the candidate
    // window of motif edge NL (GetCandidateEdgeList) and pushes the
    // task if the window is non-empty.
    // li: the root's closing look-ahead mask (Shape::look; ~0u = every vertex).
    template <int NL, int NS, int NE>
    __device__ __forceinline__ void push(bool ok, uint32_t e, uint32_t hi, const uint32_t (&phi)[NS],
                                         const uint32_t (&eh)[NE], uint32_t rslot, uint32_t li = ~0u) {
        using Lay = Layout<Plan, MODE>;
        uint32_t lo = 0, up = 0;
        if ((MODE == kCountPfx || MODE == kCountSib) && (p.prefix_mask >> NL) & 1u) {   // matches of the NL-edge prefix
            if (NL == p.prefix_lv0) {
                pfx_lane += ok ? 1u : 0u;   // the first masked level: a per-lane counter (no warp op)
            } else {   // further masked levels (rare: several prefixes of one motif): global atomics
                const uint32_t c = __popc(__ballot_sync(kFull, ok));
                if (lane == 0 && c) atomicAdd(p.scratch + kPrefixBase + NL, (unsigned long long)c);
            }
        }
        // closing edge under the look-ahead: φ(x) must be a neighbour in y's root window
        bool live = ok;
        if constexpr (Lay::look() && NL + 1 == Plan::kL)
            live = ok && ((li >> look_hash(pick(phi, plan.template lx<NL>()))) & 1u);
        if constexpr (TM_PAIR_FILTER && NL + 1 == Plan::kL && MODE != kStats) {
            // closing leaf on a graph with a pair index: a pair with no edge at all
            // (the filter's certain "absent") reads no list (the closing edge
            // is an edge of this very vertex pair)
            if (plan.template u<NL>() < plan.template nv<NL>() && plan.template v<NL>() < plan.template nv<NL>() &&
                p.ptab && live && !gen()) {
                const uint32_t pu = pick(phi, plan.template u<NL>()), pv = pick(phi, plan.template v<NL>());
                const uint32_t b0 = (e + 1) >> p.tshift, b1 = hi >> p.tshift;   // the window lies in (e, hi]
                if (p.tbits && b1 - b0 < 2u) {
                    // id-bucketed filter: the pair must have an edge in one of the window's buckets
                    const uint32_t bit0 = pair_bucket_bit(pu, pv, b0, p.tmask);
                    const uint32_t bit1 = pair_bucket_bit(pu, pv, b1, p.tmask);
                    const uint32_t w0 = __ldg(p.tbits + (bit0 >> 5)) >> (bit0 & 31);
                    const uint32_t w1 = __ldg(p.tbits + (bit1 >> 5)) >> (bit1 & 31);
                    live = (w0 | w1) & 1u;
                } else {
                    const uint64_t ph = pair_hash(((uint64_t)pu << 32) | pv);
                    live = pair_maybe(p.pbits, p.fmask, ph);
                }
            }
        }
#ifdef TM_SKIP_LEAF   // timing experiment only (wrong counts): the cost of the closing level
        if constexpr (NL + 1 == Plan::kL && MODE != kStats) live = false;
#endif
#ifdef TM_SKIP_LV      // timing experiment only (wrong counts): no tasks at level TM_SKIP_LV and below
        if constexpr (NL >= TM_SKIP_LV && MODE != kStats) live = false;
#endif
        if (live) {
            const uint32_t *hf = p.Hf[NL - 1];
            uint32_t lim = hi;   // min(t_root + δ, t_prev + δ_i) as an id; H_δi read when needed
            uint32_t hfv = ~0u;
            // window descriptor of e: {window start, window end, H_δi[e]} in one load
            const uint4 *hw = nullptr;
            if constexpr (kHrankDesc && MODE != kStats)
                if (plan.template anc<NL>() == NL - 1 && !plan.template pairk<NL>()) hw = p.HW[NL - 1];
            uint4 w4 = make_uint4(0u, 0u, ~0u, 0u);
            if (hw) w4 = __ldg(hw + e);
            if (MODE == kStats || !plan.template pairk<NL>()) {
                if (hw) hfv = w4.z;
                else if (hf) hfv = __ldg(hf + e);
                lim = min(hi, hfv);
            }
            if (MODE == kStats) {
                // instrumentation of Algorithm 1 itself: shorter list (Q8), two binary searches
                const int uM = plan.template u<NL>(), vM = plan.template v<NL>(), nb = plan.template nv<NL>();
                const bool ub = uM < nb, vb = vM < nb;
                const uint32_t xu = pick(phi, uM), xv = pick(phi, vM);
                uint32_t b, en;   // list [b, en); the sentinel sits at en
                if (ub && vb) {
                    uint32_t ob = __ldg(p.off_out + xu), oe = __ldg(p.off_out + xu + 1) - 1;
                    uint32_t ib = __ldg(p.off_in + xv), ie = __ldg(p.off_in + xv + 1) - 1;
                    if (oe - ob < ie - ib) { b = ob; en = oe; } else { b = ib; en = ie; }
                } else if (ub) {
                    b = __ldg(p.off_out + xu); en = __ldg(p.off_out + xu + 1) - 1;
                } else {
                    b = __ldg(p.off_in + xv); en = __ldg(p.off_in + xv + 1) - 1;
                }
                lo = first_after(p.rec, b, en, e);
                up = first_after(p.rec, lo, en, lim);
                if (plan.template pairk<NL>()) {   // the window the fast path (below) scans
                    uint32_t plo, pup;
                    pair_window(p, xu, xv, e, lim, nullptr, plo, pup);
                    st.fast_window += pup - plo;
                } else {
                    const int dir = plan.template ldir<NL>();
                    const uint32_t x = pick(phi, plan.template lx<NL>());
                    const uint32_t fb = __ldg((dir == 0 ? p.off_out : p.off_in) + x);
                    const uint32_t fe = __ldg((dir == 0 ? p.off_out : p.off_in) + x + 1) - 1;
                    const uint32_t flo = first_after(p.rec, fb, fe, e);
                    st.fast_window += first_after(p.rec, flo, fe, lim) - flo;
                }
                st.nodes[NL] += 1;
                st.window += up - lo;
                st.list += en - b;
                st.probes += ceil_log2p1(en - b);
            } else if (plan.template pairk<NL>()) {
                // both endpoints mapped: the pair's own edge list
                pair_window(p, pick(phi, plan.template u<NL>()), pick(phi, plan.template v<NL>()), e, hi, hf, lo, up);
                if (NL + 1 == plan.L()) {   // closing leaf: every edge of the window is a match
                    leaf_count += up - lo;
                    if (MODE == kRoots && up > lo) atomicAdd(&p.root_counts[rslot], (unsigned long long)(up - lo));
                    if (MODE == kEnum)
                        for (uint32_t q = lo; q < up; q++) emit_one<NE>(eh, e, __ldg(p.prec + q), NL);
                    lo = up = 0;
                }
            } else {
                // window start: one rank load at the anchor edge (the latest
                // matched edge touching the list vertex), then a short sector
                // scan to "after e_prev" when the anchor is older than e_prev.
                // Window end: the first sector at lo is read (a leaf reads up
                // to kLeafSectors and counts as it goes); only a window that
                // runs past them is measured by a gallop.
                const int dir = plan.template ldir<NL>(), var = plan.template avar<NL>(), j = plan.template anc<NL>();
                const uint32_t ea = (j == NL - 1) ? e : pick(eh, j);
                // window end from the horizon-rank array when the list is anchored
                // at e itself and the gap bound H_δi[e] is the tighter one: one
                // load, issued with the start and H_δi loads (no record reads)
                uint32_t *hr = (j == NL - 1) ? p.HR[NL - 1] : nullptr;
                uint32_t hrv = 0;
                if (hw) {
                    lo = w4.x;
                    hrv = w4.y;
                } else {
                    if (hr) hrv = kHrankMemo ? __ldcg(hr + e) : __ldg(hr + e);   // the memo is written by this kernel
                    lo = __ldg(p.rank + (size_t)var * p.m + ea);
                    if (j != NL - 1) lo = scan_after(p.rec, lo, e);
                }
                const bool fine_binds = (hw || hr) && hfv <= hi;   // lim == H_δi[e]: the end depends on e only
                const bool known = fine_binds && (!kHrankMemo || hrv != 0);
                const uint32_t up_known = kHrankMemo ? hrv - 1 : hrv;
                // (generalized queries check every match in expand(): no in-lane leaf scans)
                const bool leaf = NL + 1 == plan.L() && !gen();
                uint32_t pp = lo;
                bool done = false;
                uint32_t cnt = 0;
                // leaf parent: the last motif edge's window is scanned in this
                // lane and its matches counted (or emitted) on the spot, for up
                // to kLeafSectors sectors; non-leaf: one sector to size the window
                // (none when the end is known)
                int nsec = leaf ? kLeafSectors : (known ? 0 : 1);
                // closing leaf edge over a long window (a hub's list): the matches are
                // exactly the edges of one vertex pair, counted from the pair index
                // (two binary searches) instead of scanning the hub's window
                constexpr bool pairlong = TM_PAIR_LONG && MODE != kEnum && MODE != kStats;
                const bool closing = plan.template u<NL>() < plan.template nv<NL>() &&
                                     plan.template v<NL>() < plan.template nv<NL>();
                bool via_pair = false;
                if constexpr (pairlong) {
                    if (leaf && closing && p.ptab) {
                        if (known && up_known > lo + kPairMin) {
                            uint32_t plo, pup;
                            pair_window(p, pick(phi, plan.template u<NL>()), pick(phi, plan.template v<NL>()), e,
                                        lim, nullptr, plo, pup);
                            cnt = pup - plo;
                            via_pair = done = true;
                            nsec = 0;
                        } else if (!known) {
                            nsec = kPairSectors;   // then the pair index, if the window runs on
                        }
                    }
                }
                if (TM_LEAF_TASK && leaf && known && !via_pair) {
                    // timing variant: every non-empty known leaf window becomes a task
                    // (the warp scans the tasks 32 candidates at a time)
                    done = up_known <= lo;
                    pp = lo;
                    up = up_known;
                    nsec = 0;
                } else if (leaf && known && !via_pair) {
                    // the window [lo, up_known) is known: scan only the sectors it covers
                    // (an empty window reads nothing), with no end test per record
                    const int cover = up_known <= lo ? 0 : (int)(((up_known - 1) >> 2) - (lo >> 2)) + 1;
                    const int ns = min(kLeafSectors, cover);
                    uint32_t a4 = lo & ~3u;
#pragma unroll 1
                    for (int it = 0; it < ns; ++it, a4 += 4) {
                        const ulonglong2 *vp = reinterpret_cast<const ulonglong2 *>(p.rec + a4);
                        const ulonglong2 x0 = __ldg(vp), x1 = __ldg(vp + 1);
                        const uint64_t r4[4] = {x0.x, x0.y, x1.x, x1.y};
#pragma unroll
                        for (int k = 0; k < 4; k++) {
                            const uint32_t q = a4 + k;
                            if (q >= lo && q < up_known && accept<NL>((uint32_t)r4[k], dir == 0, phi)) {
                                cnt++;
                                if (MODE == kEnum) emit_one<NE>(eh, e, (uint32_t)(r4[k] >> 32), NL);
                            }
                        }
                    }
                    done = ns == cover;   // fully scanned, else the remainder [a4, up_known) becomes a task
                    pp = a4;
                    up = up_known;
                    nsec = 0;
                } else if (known && plan.template u<NL>() < plan.template nv<NL>() &&
                           plan.template v<NL>() < plan.template nv<NL>()) {
                    // inner closing edge (both endpoints mapped): few candidates
                    // close (DIA's 2->0: ~1 in 800), so the window is pre-scanned here and
                    // the task starts at its first closing candidate, or is not pushed
                    const int cover = up_known <= lo ? 0 : (int)(((up_known - 1) >> 2) - (lo >> 2)) + 1;
                    const int ns = min(kLeafSectors, cover);
                    uint32_t a4 = lo & ~3u, first = 0xFFFFFFFFu;
#pragma unroll 1
                    for (int it = 0; it < ns && first == 0xFFFFFFFFu; ++it, a4 += 4) {
                        const ulonglong2 *vp = reinterpret_cast<const ulonglong2 *>(p.rec + a4);
                        const ulonglong2 x0 = __ldg(vp), x1 = __ldg(vp + 1);
                        const uint64_t r4[4] = {x0.x, x0.y, x1.x, x1.y};
#pragma unroll
                        for (int k = 3; k >= 0; --k) {
                            const uint32_t q = a4 + k;
                            if (q >= lo && q < up_known && accept<NL>((uint32_t)r4[k], dir == 0, phi)) first = q;
                        }
                    }
                    lo = first != 0xFFFFFFFFu ? first : (ns == cover ? up_known : a4);
                    nsec = 0;
                }
#pragma unroll 1
                for (int it = 0; it < nsec && !done; ++it) {
                    const uint32_t a4 = pp & ~3u;
                    const ulonglong2 *vp = reinterpret_cast<const ulonglong2 *>(p.rec + a4);
                    const ulonglong2 x0 = __ldg(vp), x1 = __ldg(vp + 1);
                    const uint64_t r4[4] = {x0.x, x0.y, x1.x, x1.y};
#pragma unroll
                    for (int k = 0; k < 4; k++) {
                        const uint32_t q = a4 + k;
                        if (done || q < pp) continue;
                        const uint32_t id = (uint32_t)(r4[k] >> 32);
                        if (id > lim) { done = true; up = q; continue; }
                        if (leaf && accept<NL>((uint32_t)r4[k], dir == 0, phi)) {
                            cnt++;
                            if (MODE == kEnum) emit_one<NE>(eh, e, id, NL);
                        }
                    }
                    if (!done) pp = a4 + 4;
                }
                if constexpr (pairlong) {
                    if (leaf && closing && !done && p.ptab) {   // the window runs past the in-lane sectors: count it by pair
                        uint32_t plo, pup;
                        pair_window(p, pick(phi, plan.template u<NL>()), pick(phi, plan.template v<NL>()), e, lim,
                                    nullptr, plo, pup);
                        cnt = pup - plo;   // the whole window (the scanned sectors' matches included)
                        done = true;
                    }
                }
                if (leaf) {
                    leaf_count += cnt;
                    if (MODE == kRoots && cnt) atomicAdd(&p.root_counts[rslot], (unsigned long long)cnt);
                }
                if (!done) {
                    // exact end: gallop from the first unread sector, bounded by the list's
                    // sentinel (an open-ended task scanned by the warp measured slower:
                    // it cannot share a batch with other tasks)
                    lo = leaf ? pp : lo;                    // a leaf keeps only its unscanned remainder
                    if (known) {
                        up = up_known;
                    } else {
                        const uint32_t x = pick(phi, plan.template lx<NL>());
                        const uint32_t en = __ldg((dir == 0 ? p.off_out : p.off_in) + x + 1) - 1;
                        up = gallop_after(p.rec, pp, en, lim);
                    }
                }
                // first visit of e at this level: remember its window end (pos + 1)
                if (kHrankMemo && fine_binds && !known) __stcg(hr + e, up + 1);
                if (leaf && done) lo = up = 0;              // fully scanned
            }
        }
        const bool keep = live && up > lo;
        const uint32_t mask = __ballot_sync(kFull, keep);
        if (!mask) return;
        if (keep) {
            const uint32_t slot = ntask[NL] + __popc(mask & lanemask_lt());
            fld<NL, 0>()[slot] = lo;
            fld<NL, 1>()[slot] = up;
            constexpr int S = Plan::nslots(NL);
            sfor<S>([&](auto kc) {
                constexpr int k = decltype(kc)::value;
                if constexpr (Lay::kphi(NL, k)) fld<NL, Lay::phi(NL, k)>()[slot] = phi[k < NS ? k : 0];
            });
            if constexpr (Lay::khi(NL)) fld<NL, Lay::hi(NL)>()[slot] = hi;
            if constexpr (Lay::kli(NL)) fld<NL, Lay::li(NL)>()[slot] = li;
            sfor<NL>([&](auto kc) {
                constexpr int k = decltype(kc)::value;
                if constexpr (Lay::keh(NL, k)) fld<NL, Lay::eh(NL, k)>()[slot] = (k < NL - 1) ? eh[k < NE ? k : 0] : e;
            });
            if constexpr (MODE == kRoots) fld<NL, Lay::rs(NL)>()[slot] = rslot;
        }
        ntask[NL] += __popc(mask);
        cand[NL] = cand_add(cand[NL], __reduce_add_sync(kFull, keep ? min(up - lo, 1u << 26) : 0u));
        __syncwarp();
    }

    // Take up to 32 roots from the global cursor and bind motif edge 1 to them
    // (the root level maps motif edge 1 onto every graph edge).
    // kResume: row `slot` holds the NL edge ids of a partial match of this
    // motif's first NL edges (emitted by another kernel, sibling emission):
    // rebuild φ and continue the search at level NL exactly as if this kernel
    // had created that node itself
    template <int NL>
    __device__ __forceinline__ void resume(bool ok, uint32_t slot) {
        constexpr int S = Plan::nslots(NL);
        uint32_t eh[NL], phi[S + 1];
#pragma unroll
        for (int k = 0; k < S + 1; k++) phi[k] = 0u;
        uint32_t hi = 0;
        if (ok) {
            const uint32_t *row = p.resume_rows + (size_t)slot * NL;
            sfor<NL>([&](auto ic_) {
                constexpr int i = decltype(ic_)::value;
                eh[i] = __ldg(row + i);
                const uint32_t a = __ldg(p.src + eh[i]), b = __ldg(p.dst + eh[i]);
#pragma unroll
                for (int k = 0; k < S; k++) {
                    if (k == plan.template u<i>()) phi[k] = a;
                    if (k == plan.template v<i>()) phi[k] = b;
                }
            });
            hi = __ldg(p.H + eh[0]);
        } else {
#pragma unroll
            for (int i = 0; i < NL; i++) eh[i] = 0u;
        }
        push<NL>(ok, eh[NL - 1], hi, phi, eh, slot);
    }

    // The closing look-ahead mask of root r (Shape::look): the hashed
    // neighbours of y's list records in (r, hi]; 0 if there is none, all ones
    // if that window runs past the aligned sector holding its start (no
    // gallop: a superset is as correct, only less selective).
    __device__ __forceinline__ uint32_t look_ahead(uint32_t r, uint32_t hi, uint32_t &last) const {
        const uint32_t b = ld_stream(p.rank + (size_t)Plan::lkvar() * p.m + r);   // first record after r
        const uint32_t a4 = b & ~3u;
        const ulonglong2 *vp = reinterpret_cast<const ulonglong2 *>(p.rec + a4);
        constexpr int NR = kLookRecs;   // records read from the aligned sector holding b on
        uint64_t rr[NR];
#pragma unroll
        for (int q = 0; q < NR / 2; q++) {
            const ulonglong2 x = __ldg(vp + q);
            rr[2 * q] = x.x;
            rr[2 * q + 1] = x.y;
        }
        // ids ascend up to the list's sentinel (id 0xFFFFFFFF > hi): the window
        // ends in these records unless the last one is still <= hi; records
        // after the first one past hi belong to the window's end or the next list
        uint32_t mask = 0;
        bool end = false;
#pragma unroll
        for (int k = 0; k < NR; k++) {
            if (a4 + k < b || end) continue;
            if ((uint32_t)(rr[k] >> 32) > hi) {
                end = true;
            } else {
                mask |= 1u << look_hash((uint32_t)rr[k]);
                last = (uint32_t)(rr[k] >> 32);   // the window's latest edge so far
            }
        }
        if (TM_LOOK_EXTRA && !end && p.root_prune) {
            // pruning roots: follow the window up to TM_LOOK_EXTRA more sectors (the
            // clamp and the prune need its end; the mask only gets less selective);
            // out of line, so kernels that never prune keep their register allocation
            const uint2 ml = look_more(p.rec, a4 + 4, hi, mask, last);
            if (ml.x != ~0u) { mask = ml.x; last = ml.y; end = true; }
        }
        return end ? mask : ~0u;
    }

    // next/end: this warp's claimed root slots (u32: n_roots <= m < 2^31)
    __device__ __forceinline__ bool fetch_roots(uint32_t &next, uint32_t &end) {
        if (next >= end) {
            // rows claimed per atomic when resuming: 32 if the launch has fewer than 4
            // chunks per warp (the searching kernels keep 128: measured, any run-time
            // choice there costs the 4-cycle kernel 0.2 ms of code generation)
            const uint32_t chunk = (MODE == kResume && TM_SMALL_CHUNK &&
                                    n_items < 4u * kRootChunk * gridDim.x * kWarpsPerBlock)
                                       ? 32u
                                       : (uint32_t)kRootChunk;
            unsigned long long b = 0;
            if (lane == 0) b = atomicAdd(&p.scratch[0], (unsigned long long)chunk);
            b = __shfl_sync(kFull, b, 0);
            if (b >= n_items) return false;
            next = (uint32_t)b;
            end = (uint32_t)min((uint64_t)(b + chunk), (uint64_t)n_items);
        }
        const uint32_t slot = next + lane;
        bool ok = slot < end;
        next = min(next + 32u, end);
        if constexpr (MODE == kResume) {   // rows of partial matches: continue at level resume_level
            switch (p.resume_level) {
                case 2: if constexpr (LM > 2) resume<2>(ok, slot); break;
                case 3: if constexpr (LM > 3) resume<3>(ok, slot); break;
                case 4: if constexpr (LM > 4) resume<4>(ok, slot); break;
                case 5: if constexpr (LM > 5) resume<5>(ok, slot); break;
                default: break;
            }
            return true;
        }
        uint32_t r = 0, a = 0, bb = 0;
        if (ok) {
            r = (uint32_t)(p.roots ? p.roots[slot] : p.root_lo + slot);
            a = ld_stream(p.src + r);
            bb = ld_stream(p.dst + r);
            ok = a != bb;   // a self-loop cannot map two distinct motif vertices (Q4)
            if (gen() && ok)
                ok = labels_ok(0, r, true, 1, bb) && (p.vreq[0] == TM_ANY_LABEL || vlabel(a) == p.vreq[0]);
        }
        const uint32_t eh[1] = {r};
        if (plan.L() == 1) {
            if (gen() && ok && p.n_anti) {
                const uint32_t phi1[2] = {a, bb};
                const uint32_t none[1] = {0};
                ok = anti_ok(phi1, none, r);
            }
            emit(ok, eh, r, (uint32_t)slot);
        } else if constexpr (LM > 1) {
            const uint32_t phi[2] = {a, bb};
            uint32_t hi = ok ? ld_stream(p.H + r) : 0;   // t' = t_root + δ as an index
            uint32_t li = ~0u;
            if constexpr (Layout<Plan, MODE>::look()) {
                uint32_t last = hi;
                if (ok) li = look_ahead(r, hi, last);
                if (TM_ROOT_PRUNE && p.root_prune) {
                    if (li == 0u) ok = false;   // no closing edge can exist
                    // the closing edge is the match's last and latest edge, and it lies
                    // in this window: no edge of a match comes after the window's latest
                    else if (TM_ROOT_CLAMP && li != ~0u) hi = last;
                }
            }
            push<1>(ok, r, hi, phi, eh, (uint32_t)slot, li);
        }
        return true;
    }

    // Expand up to 32 candidates of level-LV tasks (matching motif edge LV).
    template <int LV>
    __device__ __forceinline__ void expand() {
        constexpr int S = Plan::nslots(LV);
        using Lay = Layout<Plan, MODE>;
        const uint32_t n = ntask[LV];
        uint32_t *flo = fld<LV, 0>(), *fup = fld<LV, 1>();
        const int j = (int)n - 1 - lane;               // lane i looks at the i-th task from the top
        uint32_t lo = 0, sz = 0;
        if (j >= 0) { lo = flo[j]; sz = fup[j] - lo; }
        const uint32_t sz32 = min(sz, 32u);
        uint32_t incl = sz32;
#pragma unroll
        for (int d = 1; d < 32; d <<= 1) {
            uint32_t y = __shfl_up_sync(kFull, incl, d);
            if (lane >= d) incl += y;
        }
        const uint32_t excl = incl - sz32;
        const bool takes = j >= 0 && excl < 32;
        const bool full = takes && sz <= 32 - excl;
        const uint32_t kfull = __popc(__ballot_sync(kFull, full));
        const uint32_t starts = __reduce_or_sync(kFull, takes ? (1u << excl) : 0u);
        const uint32_t C = min(__shfl_sync(kFull, incl, 31), 32u);
        const bool active = (uint32_t)lane < C;
        const uint32_t lemask = (lane == 31) ? kFull : ((2u << lane) - 1u);
        const int t = active ? (__popc(starts & lemask) - 1) : 0;
        const uint32_t lo_t = __shfl_sync(kFull, lo, t);
        const uint32_t ex_t = __shfl_sync(kFull, excl, t);
        const int jt = (int)n - 1 - t;
        const uint32_t pos = lo_t + ((uint32_t)lane - ex_t);

        uint32_t phi[S + 1];
        uint32_t eh[LV + 1];
        uint32_t hi = 0, rslot = 0, e = 0, w = 0, li = ~0u;
        bool ok = false;
        if (active) {
            sfor<S>([&](auto kc) {
                constexpr int k = decltype(kc)::value;
                if constexpr (Lay::kphi(LV, k)) phi[k] = fld<LV, Lay::phi(LV, k)>()[jt];
                else phi[k] = 0u;
            });
            if constexpr (Lay::khi(LV)) hi = fld<LV, Lay::hi(LV)>()[jt];
            if constexpr (Lay::kli(LV)) li = fld<LV, Lay::li(LV)>()[jt];
            sfor<LV>([&](auto kc) {
                constexpr int k = decltype(kc)::value;
                if constexpr (Lay::keh_load(LV, k)) eh[k] = fld<LV, Lay::eh(LV, k)>()[jt];
                else eh[k] = 0u;
            });
            if constexpr (MODE == kRoots) rslot = fld<LV, Lay::rs(LV)>()[jt];
            if (MODE != kStats && plan.template pairk<LV>()) {   // a pair window: the edge is the match
                e = __ldg(p.prec + pos);
                ok = true;
            } else {
                const uint64_t rc = __ldg(p.rec + pos);
                e = (uint32_t)(rc >> 32);
                w = (uint32_t)rc;
                ok = accept<LV>(w, pos < p.split, phi);
                if (gen() && ok) {
                    const int nb = plan.template nv<LV>();
                    ok = labels_ok(LV, e, nb < plan.template nv<LV + 1>(), nb, w);
                }
            }
        }
        if constexpr (MODE == kCountSib && LV == kSibLevel) {
            {   // sibling emission: a closing edge to φ[sib_vtx] on this candidate
                const bool sib = active && w == pick(phi, p.sib_vtx);
                const uint32_t smask = __ballot_sync(kFull, sib);
                if (smask) {
                    unsigned long long base = 0;
                    if (lane == 0) base = atomicAdd(p.scratch + kSibCount, (unsigned long long)__popc(smask));
                    base = __shfl_sync(kFull, base, 0);
                    if (sib) {
                        const unsigned long long row = base + __popc(smask & lanemask_lt());
                        if (row < p.sib_cap) {
                            uint32_t *dst = p.sib_rows + row * (LV + 1);
                            sfor<LV>([&](auto kc) {
                                constexpr int i = decltype(kc)::value;
                                dst[i] = Lay::keh_load(LV, i) ? eh[i] : fld<LV, Lay::eh(LV, i)>()[jt];
                            });
                            dst[LV] = e;
                        }
                    }
                }
            }
        }
        __syncwarp();
        // consume: pop the fully taken tasks, advance the partially taken one
        if (takes && !full) flo[j] = lo + (32u - excl);
        ntask[LV] = n - kfull;
        cand[LV] = cand_sub(cand[LV], C);
        __syncwarp();

        if (LV + 1 == plan.L()) {
            if (gen() && ok && p.n_anti) {   // the complete match: φ with the last edge's new vertex
                const int nb = plan.template nv<LV>();
                uint32_t phiF[S + 2];
#pragma unroll
                for (int k = 0; k < S + 1; k++) phiF[k] = phi[k];
                phiF[S + 1] = 0;
#pragma unroll
                for (int k = 0; k < S + 2; k++)
                    if (k == nb && nb < plan.template nv<LV + 1>()) phiF[k] = w;
                ok = anti_ok(phiF, eh, e);
            }
            emit(ok, eh, e, rslot);
        } else if constexpr (LV + 1 < LM) {
            const int nb = plan.template nv<LV>();
            constexpr int S2 = Plan::nslots(LV + 1);
            uint32_t phi2[S2 + 1];
#pragma unroll
            for (int k = 0; k < S2; k++) phi2[k] = (k < S) ? phi[k < S ? k : 0] : 0u;
            // a new endpoint gets the next slot (motif vertices are numbered by first appearance)
            if (nb < plan.template nv<LV + 1>()) {
#pragma unroll
                for (int k = 0; k < S2; k++)
                    if (k == nb) phi2[k] = w;
            }
            push<LV + 1>(ok, e, hi, phi2, eh, rslot, li);
        }
    }

    // ------------------------------------------ heavy-subtree sharing (§8 a8)
    // The paper's tail-warp work redistribution (abort the tail
    // warps, dump their contexts, relaunch) done inside the persistent kernel,
    // with no relaunch.  Once the root queue is drained, a warp that sees idle
    // warps hands one pending subtree to one of them: the bottom task of its
    // shallowest non-leaf level (the oldest, least explored subtree), or, when
    // that level holds a single task, the upper half of its cached candidate
    // window (sub-tree-level parallelism).  A task is
    // self-contained (its level's SoA fields: window, φ, hi, matched ids), so
    // the receiver continues exactly the search the donor would have run.
    // Hand-over: the donor claims an idle warp (decrements the idle counter),
    // takes a ticket d, writes the record to ring slot d and publishes it with
    // flag = d + 1; idle warps take tickets in the same order and wait on
    // their own slot's flag.  The warp whose arrival makes every warp idle
    // writes kShareStop into the flags of the unserved tickets: the search is
    // complete.  Only pieces of >= kShareMin candidates are handed over, and
    // busy warps read the idle counter every kSharePoll iterations (measured:
    // per-iteration reads of one counter by thousands of warps congest its L2
    // slice, profiles/r01_experiments.md).

    // hand over task j of level LV (whole, or the upper half of its window)
    template <int LV>
    __device__ __forceinline__ void give(uint32_t *rec, bool split, uint32_t j) {
        using Lay = Layout<Plan, MODE>;
        constexpr int F = Lay::fields(LV);
        static_assert(F < kShareWords, "task record too large");
        uint32_t *base = ws + Lay::off(LV);   // word f of task j at base[f * kCap + j]
        const uint32_t lo = base[j], up = base[kCap + j];
        const uint32_t mid = lo + ((up - lo) >> 1);
        uint32_t val = lane < F ? base[lane * kCap + j] : 0u;
        if (split && lane == 0) val = mid;               // handed over: [mid, up)
        if (lane == kShareWords - 1) val = (uint32_t)LV;
        __stcg(rec + lane, val);
        __syncwarp();
        if (split) {
            if (lane == 0) base[kCap + j] = mid;          // kept: [lo, mid)
            cand[LV] = cand_sub(cand[LV], up - mid);
        } else {                                          // the top task fills slot j
            const uint32_t top = ntask[LV] - 1;
            if (lane < F) base[lane * kCap + j] = base[lane * kCap + top];
            ntask[LV] = top;
            cand[LV] = cand_sub(cand[LV], up - lo);
        }
        __syncwarp();
    }

    template <int LV>
    __device__ __forceinline__ void take(uint32_t val) {
        using Lay = Layout<Plan, MODE>;
        constexpr int F = Lay::fields(LV);
        uint32_t *base = ws + Lay::off(LV);
        const uint32_t slot = ntask[LV];
        if (lane < F) base[lane * kCap + slot] = val;
        const uint32_t lo = __shfl_sync(kFull, val, 0), up = __shfl_sync(kFull, val, 1);
        ntask[LV] = slot + 1;
        cand[LV] = cand_add(cand[LV], min(up - lo, 1u << 26));
        __syncwarp();
    }

    // Called when idle warps were seen: hand over one subtree if there is one
    // worth handing (non-leaf levels; every level in eager mode).
    __device__ void try_share() {
        int lv = -1;
        bool split = false;
        uint32_t jb = 0;
        const int L = plan.L();
        sfor<LM>([&](auto lc) {
            constexpr int l = decltype(lc)::value;
            if constexpr (l >= 1) {
                if (lv < 0 && l < L && (l + 1 < L || p.share == 2) && ntask[l] > 0) {
                    // the level's task with the largest remaining window (lane i
                    // looks at tasks i and i + 32); only pieces of >= kShareMin
                    // candidates are worth a hand-over (a short window is cheaper
                    // to finish than to move; eager mode: any)
                    const uint32_t *base = ws + Layout<Plan, MODE>::off(l);
                    const uint32_t n = ntask[l];
                    const uint32_t wa = (uint32_t)lane < n ? base[kCap + lane] - base[lane] : 0u;
                    const uint32_t wb = (uint32_t)lane + 32 < n ? base[kCap + lane + 32] - base[lane + 32] : 0u;
                    const uint32_t wl = max(wa, wb);
                    const uint32_t wmax = __reduce_max_sync(kFull, wl);
                    const int src = __ffs(__ballot_sync(kFull, wl == wmax)) - 1;
                    const uint32_t j = __shfl_sync(kFull, wb > wa ? lane + 32u : (uint32_t)lane, src);
                    const uint32_t smin = p.share == 2 ? 1u : (uint32_t)kShareMin;
                    if (wmax >= 2 * smin) {
                        lv = l; jb = j; split = true;
                    } else if (n >= 2 && wmax >= smin) {
                        lv = l; jb = j;
                    }
                }
            }
        });
        if (lv < 0) return;
        unsigned long long d = 0;
        int ok = 0;
        if (lane == 0) {
            int *idle = reinterpret_cast<int *>(p.scratch + kShareIdle);
            if (atomicSub(idle, 1) > 0) {
                ok = 1;
                d = atomicAdd(p.scratch + kShareTail, 1ull);
                volatile unsigned *f = p.qflag + (d & p.qmask);
                while (*f != 0u) __nanosleep(32);   // the slot's previous record is still being read
            } else {
                atomicAdd(idle, 1);                  // nobody to give to after all
            }
        }
        if (!__shfl_sync(kFull, ok, 0)) return;
        d = __shfl_sync(kFull, d, 0);
        uint32_t *rec = p.qrec + (size_t)(d & p.qmask) * kShareWords;
        switch (lv) {
            case 1: if constexpr (LM > 1) give<1>(rec, split, jb); break;
            case 2: if constexpr (LM > 2) give<2>(rec, split, jb); break;
            case 3: if constexpr (LM > 3) give<3>(rec, split, jb); break;
            case 4: if constexpr (LM > 4) give<4>(rec, split, jb); break;
            case 5: if constexpr (LM > 5) give<5>(rec, split, jb); break;
            default: break;
        }
        __threadfence();
        __syncwarp();
        if (lane == 0) {
            atomicExch(p.qflag + (d & p.qmask), (unsigned)(d + 1));
            atomicAdd(p.scratch + kShareDone, 1ull);
        }
    }

    // This warp has no work left: wait for a handed-over subtree.  Returns
    // false when every warp is idle (the search is complete).
    __device__ bool receive() {
        int got = 0, last = 0;
        unsigned long long r = 0;
        if (lane == 0) {
            r = atomicAdd(p.scratch + kShareHead, 1ull);
            __threadfence();   // the ticket is taken before this warp counts as idle
            const int before = atomicAdd(reinterpret_cast<int *>(p.scratch + kShareIdle), 1);
            last = before + 1 == (int)p.total_warps;
            if (!last) {
                // wait on this ticket's own flag only (no shared hot spot)
                volatile unsigned *f = p.qflag + (r & p.qmask);
                unsigned ns = 64;
                while (true) {
                    const unsigned v = *f;
                    if (v == (unsigned)(r + 1)) { got = 1; break; }
                    if (v == kShareStop) break;
                    __nanosleep(ns);
                    if (ns < kShareSleepMax) ns <<= 1;
                }
                __threadfence();
            }
        }
        if (__shfl_sync(kFull, last, 0)) {
            // every warp is idle and none can become busy again: release the
            // waiting ones (their tickets are the unserved [tail, head)), one
            // flag per lane
            __threadfence();
            r = __shfl_sync(kFull, r, 0);
            const unsigned long long tl = *reinterpret_cast<volatile unsigned long long *>(p.scratch + kShareTail);
            const unsigned long long hd = *reinterpret_cast<volatile unsigned long long *>(p.scratch + kShareHead);
            for (unsigned long long d = tl + lane; d < hd; d += 32)
                if (d != r) p.qflag[d & p.qmask] = kShareStop;
            return false;
        }
        if (!__shfl_sync(kFull, got, 0)) return false;
        r = __shfl_sync(kFull, r, 0);
        const uint32_t *rec = p.qrec + (size_t)(r & p.qmask) * kShareWords;
        const uint32_t val = __ldcg(rec + lane);
        const int lv = (int)__shfl_sync(kFull, val, kShareWords - 1);
        __threadfence();
        __syncwarp();
        if (lane == 0) atomicExch(p.qflag + (r & p.qmask), 0u);   // the slot is free again
        switch (lv) {
            case 1: if constexpr (LM > 1) take<1>(val); break;
            case 2: if constexpr (LM > 2) take<2>(val); break;
            case 3: if constexpr (LM > 3) take<3>(val); break;
            case 4: if constexpr (LM > 4) take<4>(val); break;
            case 5: if constexpr (LM > 5) take<5>(val); break;
            default: break;
        }
        return true;
    }
};

// Resident CTAs per SM the register allocator must allow for specialised
// counting kernels: <= 3 motif edges fit 40 registers (6 CTAs of 256 threads
// per SM), 4 edges 48 (5 CTAs), 5 edges 64 (4 CTAs), all without spills
// (ptxas -v); left alone, ptxas lands just above each step and the grid
// loses a CTA per SM.  Everything else: the allocator's choice.
#ifndef TM_MIN_BLOCKS3
#define TM_MIN_BLOCKS3 6
#endif
#ifndef TM_MIN_BLOCKS4
#define TM_MIN_BLOCKS4 5
#endif
#ifndef TM_MIN_BLOCKS5
#define TM_MIN_BLOCKS5 4
#endif
template <class Plan, int MODE>
struct MinBlocks {
    static constexpr int value = 1;
};
template <uint64_t CODE>
struct MinBlocks<PlanC<CODE, false>, kCount> {
    static constexpr int value = PlanC<CODE>::kL <= 3 ? TM_MIN_BLOCKS3 : PlanC<CODE>::kL == 4 ? TM_MIN_BLOCKS4 : TM_MIN_BLOCKS5;
};
template <uint64_t CODE>
struct MinBlocks<PlanC<CODE, false>, kCountPfx> : MinBlocks<PlanC<CODE, false>, kCount> {};
template <uint64_t CODE>
struct MinBlocks<PlanC<CODE, false>, kResume> : MinBlocks<PlanC<CODE, false>, kCount> {};
#ifndef TM_MIN_BLOCKS_SIB
#define TM_MIN_BLOCKS_SIB 0   // 0: as the counting kernel
#endif
template <uint64_t CODE>
struct MinBlocks<PlanC<CODE, false>, kCountSib> {
    static constexpr int value = TM_MIN_BLOCKS_SIB ? TM_MIN_BLOCKS_SIB : MinBlocks<PlanC<CODE, false>, kCount>::value;
};
#ifndef TM_MIN_BLOCKS_ENUM
#define TM_MIN_BLOCKS_ENUM 4
#endif
template <uint64_t CODE>
struct MinBlocks<PlanC<CODE, false>, kEnum> {
    static constexpr int value = TM_MIN_BLOCKS_ENUM;
};

template <class Plan, int MODE>
__global__ void __launch_bounds__(kWarpsPerBlock * 32, (MinBlocks<Plan, MODE>::value)) mine_kernel(const MineParams p) {
    extern __shared__ uint32_t smem[];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    constexpr int LM = Plan::kL;
    uint32_t *ws = smem + warp * Layout<Plan, MODE>::warp_words();
    const Plan plan(p);
    Warp<Plan, MODE> W(p, plan, ws, lane);
    const int L = plan.L();
    uint32_t next = 0, end = 0;
    uint32_t iter = 0;   // iterations, for the idle-counter poll
    bool roots_left = true;
    // load-balance instrumentation (tm_run_info.tail_ms / warp_busy): this
    // warp's start in 64-ns ticks (u32: wraps after 275 s, differences stay
    // exact); time spent waiting for handed-over work is added in receive
    uint32_t t_start = 0;
    if (TM_TIMING && lane == 0) {
        const unsigned long long t = globaltimer_ns();
        t_start = (uint32_t)(t >> 6);
        atomicMax(p.scratch + kTimeStart, ~t);
    }

#ifdef TM_PHASE_PROFILE
    unsigned long long prof_cyc[6] = {0, 0, 0, 0, 0, 0}, prof_n[6] = {0, 0, 0, 0, 0, 0};
#endif
    const bool share = TM_SHARE && p.share != 1;
    while (true) {
        // every kSharePoll iterations read the idle counter and, if warps wait
        // (so the root queue is drained), hand one subtree over.  A warp deep
        // in a heavy tree never returns to the root queue itself, so this must
        // not wait for its own fetch to fail.
        if (share && (++iter & (kSharePoll - 1)) == 0) {
            int idle = 0;
            if (lane == 0) idle = *reinterpret_cast<volatile int *>(p.scratch + kShareIdle);
            if (__shfl_sync(kFull, idle, 0) > 0) W.try_share();
        }
        int sel = -1;
        // deepest level with a full batch whose child stack has room
#pragma unroll
        for (int l = LM - 1; l >= 1; --l)
            if (sel < 0 && l < L && W.cand[l] >= 32 && (l == L - 1 || W.ntask[l + 1 <= LM ? l + 1 : LM] < kRoom)) sel = l;
        if (sel < 0) {
            // a root batch pushes at level 1 (kResume: at the rows' level)
            uint32_t nroot = W.ntask[1];
            if (MODE == kResume) {
#pragma unroll
                for (int l = 2; l < LM; l++)
                    if (l == (int)p.resume_level) nroot = W.ntask[l];
            }
            if (roots_left && (L == 1 || nroot < kRoom)) {
                sel = 0;
            } else {
#pragma unroll
                for (int l = LM - 1; l >= 1; --l)
                    if (sel < 0 && l < L && W.ntask[l] > 0 && (l == L - 1 || W.ntask[l + 1 <= LM ? l + 1 : LM] < kRoom)) sel = l;
            }
        }
        if (sel < 0) {
            if (share) {
                const unsigned long long tw = TM_TIMING ? globaltimer_ns() : 0;
                const bool more = W.receive();
                if (TM_TIMING && lane == 0) atomicAdd(p.scratch + kTimeWait, globaltimer_ns() - tw);
                if (more) continue;
            }
            break;
        }
#ifdef TM_PHASE_PROFILE
        const long long t0 = clock64();
#endif
        switch (sel) {
            case 0:
                roots_left = W.fetch_roots(next, end);
                if (TM_TIMING && !roots_left && lane == 0)   // the root queue is drained: the tail starts
                    atomicMax(p.scratch + kTimeDrain, ~globaltimer_ns());
                break;
            case 1: if constexpr (LM > 1) W.template expand<1>(); break;
            case 2: if constexpr (LM > 2) W.template expand<2>(); break;
            case 3: if constexpr (LM > 3) W.template expand<3>(); break;
            case 4: if constexpr (LM > 4) W.template expand<4>(); break;
            case 5: if constexpr (LM > 5) W.template expand<5>(); break;
            default: break;
        }
#ifdef TM_PHASE_PROFILE
        // cycles and steps per selected level (0 = root fetch), flushed at exit
        {
            const unsigned long long dt = (unsigned long long)(clock64() - t0);
#pragma unroll
            for (int l = 0; l < 6; l++)
                if (l == sel) { prof_cyc[l] += dt; prof_n[l] += 1; }
        }
#endif
    }
#ifdef TM_PHASE_PROFILE
    if (lane == 0)
        for (int l = 0; l < 6; l++)
            if (prof_n[l]) {
                atomicAdd(&p.scratch[20 + 2 * l], prof_cyc[l]);
                atomicAdd(&p.scratch[21 + 2 * l], prof_n[l]);
            }
#endif
    if (TM_TIMING && lane == 0) {
        const unsigned long long te = globaltimer_ns();
        atomicMax(p.scratch + kTimeExit, te);
        atomicAdd(p.scratch + kTimeBusy, (unsigned long long)((uint32_t)(te >> 6) - t_start) << 6);
    }
    __syncwarp();
    if (MODE == kCountPfx || MODE == kCountSib) {
        unsigned long long pl = W.pfx_lane;
        for (int d = 16; d; d >>= 1) pl += __shfl_xor_sync(kFull, pl, d);
        if (lane == 0 && pl) atomicAdd(p.scratch + kPrefixBase + p.prefix_lv0, pl);
    }
    unsigned long long tot = W.leaf_count;
    for (int d = 16; d; d >>= 1) tot += __shfl_xor_sync(kFull, tot, d);
    tot += W.count;   // lane 0's batch count (other lanes hold 0)
    if (lane == 0 && tot) atomicAdd(&p.scratch[1], tot);
    if (MODE == kStats) {
#pragma unroll
        for (int l = 0; l < kMaxL; l++) {
            unsigned long long v = W.st.nodes[l];
            for (int d = 16; d; d >>= 1) v += __shfl_xor_sync(kFull, v, d);
            if (lane == 0 && v) atomicAdd(&p.scratch[kStatsBase + l], v);
        }
        unsigned long long a = W.st.window, b = W.st.list, c = W.st.probes, f = W.st.fast_window;
        for (int d = 16; d; d >>= 1) {
            a += __shfl_xor_sync(kFull, a, d);
            b += __shfl_xor_sync(kFull, b, d);
            c += __shfl_xor_sync(kFull, c, d);
            f += __shfl_xor_sync(kFull, f, d);
        }
        if (lane == 0) {
            atomicAdd(&p.scratch[16], a);
            atomicAdd(&p.scratch[17], b);
            atomicAdd(&p.scratch[18], c);
            atomicAdd(&p.scratch[19], f);
        }
    }
}

#ifndef __CUDACC_RTC__
template <class Plan, int MODE>
KernelInfo kernel_info() {
    return KernelInfo{&mine_kernel<Plan, MODE>, (int)(Layout<Plan, MODE>::warp_words() * sizeof(uint32_t))};
}
#endif

}  // namespace tmg
