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
// every stack within kCap = 64 tasks.
#pragma once

#include "tm_internal.cuh"

namespace tmg {

constexpr int kCap = 64;             // tasks per level per warp
constexpr int kWarpsPerBlock = 8;
constexpr int kRootChunk = 128;      // roots claimed per global atomic
constexpr unsigned kFull = 0xffffffffu;

__device__ __forceinline__ uint32_t lanemask_lt() {
    uint32_t r;
    asm("mov.u32 %0, %%lanemask_lt;" : "=r"(r));
    return r;
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

__device__ __forceinline__ uint32_t ceil_log2p1(uint32_t len) {  // ceil(log2(len+1))
    return len ? 32 - __clz(len) : 0;
}

// Exact warp sum of values < 2^31 as u64.
__device__ __forceinline__ uint64_t warp_sum_u31(uint32_t v) {
    uint32_t lo = __reduce_add_sync(kFull, v & 0xffffu);
    uint32_t hi = __reduce_add_sync(kFull, v >> 16);
    return ((uint64_t)hi << 16) + lo;
}

// ------------------------------------------------------------------ plans
// Compile-time plan: the motif structure is a template argument, so every
// per-level choice (which list, which checks, how many mapped vertices) is a
// constant — the B200 counterpart of the paper's generated motif-specific
// code and `minfo`.
template <uint64_t CODE>
struct PlanC {
    static constexpr int kL = (int)(CODE & 7);
    __host__ __device__ static constexpr int u_(int i) { return (int)((CODE >> (3 + 6 * i)) & 7); }
    __host__ __device__ static constexpr int v_(int i) { return (int)((CODE >> (6 + 6 * i)) & 7); }
    __host__ __device__ static constexpr int nv_(int l) {
        int mx = -1;
        for (int i = 0; i < l; i++) {
            mx = u_(i) > mx ? u_(i) : mx;
            mx = v_(i) > mx ? v_(i) : mx;
        }
        return mx + 1;
    }
    // φ slots stored with a level-l task
    __host__ __device__ static constexpr int nslots(int l) { return nv_(l); }
    __device__ explicit PlanC(const MineParams &) {}
    __device__ __forceinline__ int L() const { return kL; }
    __device__ __forceinline__ int u(int i) const { return u_(i); }
    __device__ __forceinline__ int v(int i) const { return v_(i); }
    __device__ __forceinline__ int nv(int l) const { return nv_(l); }
};

// Runtime plan: the same kernel body for any prefix-connected motif with
// L <= kMaxL edges, the structure read from the launch parameters.
struct PlanR {
    static constexpr int kL = kMaxL;
    __host__ __device__ static constexpr int nslots(int l) { return l + 1 < kMaxV ? l + 1 : kMaxV; }
    int L_;
    int nv__[kMaxL + 1];
    const MineParams &p_;
    __device__ explicit PlanR(const MineParams &p) : L_((int)p.L), p_(p) {
        int mx = -1;
        nv__[0] = 0;
#pragma unroll
        for (int i = 0; i < kMaxL; i++) {
            if (i < L_) {
                mx = max(mx, (int)p.u[i]);
                mx = max(mx, (int)p.v[i]);
            }
            nv__[i + 1] = mx + 1;
        }
    }
    __device__ __forceinline__ int L() const { return L_; }
    __device__ __forceinline__ int u(int i) const { return p_.u[i]; }
    __device__ __forceinline__ int v(int i) const { return p_.v[i]; }
    __device__ __forceinline__ int nv(int l) const { return nv__[l]; }
};

// ------------------------------------------------------- shared-memory layout
// Per warp, per level l = 1..kL-1, a structure of arrays of kCap tasks:
//   [0] lo  [1] up  [2] hi  [3 .. 3+S) φ  [.. +l) matched ids (kEnum)  [+1] root slot (kRoots)
template <class Plan, int MODE>
struct Layout {
    __host__ __device__ static constexpr int eh(int l) { return 3 + Plan::nslots(l); }
    __host__ __device__ static constexpr int rs(int l) { return eh(l) + (MODE == kEnum ? l : 0); }
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
    unsigned long long window, list, probes;
};

template <class Plan, int MODE>
struct Warp {
    static constexpr int LM = Plan::kL;  // levels 1..LM-1 hold tasks
    const MineParams &p;
    const Plan &plan;
    uint32_t *ws;
    int lane;
    uint32_t ntask[LM + 1];
    uint64_t cand[LM + 1];
    unsigned long long count;   // lane 0: matches found by this warp
    Stats st;

    __device__ Warp(const MineParams &p_, const Plan &pl, uint32_t *w, int ln) : p(p_), plan(pl), ws(w), lane(ln) {
#pragma unroll
        for (int i = 0; i <= LM; i++) { ntask[i] = 0; cand[i] = 0; }
        count = 0;
        if (MODE == kStats) {
#pragma unroll
            for (int i = 0; i < kMaxL; i++) st.nodes[i] = 0;
            st.window = st.list = st.probes = 0;
        }
    }

    __device__ __forceinline__ uint32_t *field(int l, int f) { return ws + Layout<Plan, MODE>::off(l) + f * kCap; }

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
    template <int NL, int NS, int NE>
    __device__ __forceinline__ void push(bool ok, uint32_t e, uint32_t hi, const uint32_t (&phi)[NS],
                                         const uint32_t (&eh)[NE], uint32_t rslot) {
        uint32_t lo = 0, up = 0;
        if (ok) {
            const int uM = plan.u(NL), vM = plan.v(NL), nb = plan.nv(NL);
            const bool ub = uM < nb, vb = vM < nb;
            const uint32_t xu = pick(phi, uM), xv = pick(phi, vM);
            uint32_t b, en;
            if (ub && vb) {  // both endpoints mapped: scan the shorter list (reading Q8)
                uint32_t ob = __ldg(p.off_out + xu), oe = __ldg(p.off_out + xu + 1);
                uint32_t ib = __ldg(p.off_in + xv), ie = __ldg(p.off_in + xv + 1);
                if (oe - ob < ie - ib) { b = ob; en = oe; } else { b = ib; en = ie; }
            } else if (ub) {
                b = __ldg(p.off_out + xu); en = __ldg(p.off_out + xu + 1);
            } else {
                b = __ldg(p.off_in + xv); en = __ldg(p.off_in + xv + 1);
            }
            uint32_t lim = hi;
            const uint32_t *hf = p.Hf[NL - 1];
            if (hf) lim = min(lim, __ldg(hf + e));
            lo = first_after(p.rec, b, en, e);
            up = first_after(p.rec, lo, en, lim);
            if (MODE == kStats) {
                st.nodes[NL] += 1;
                st.window += up - lo;
                st.list += en - b;
                st.probes += ceil_log2p1(en - b);
            }
        }
        const bool keep = ok && up > lo;
        const uint32_t mask = __ballot_sync(kFull, keep);
        if (!mask) return;
        if (keep) {
            const uint32_t slot = ntask[NL] + __popc(mask & lanemask_lt());
            field(NL, 0)[slot] = lo;
            field(NL, 1)[slot] = up;
            field(NL, 2)[slot] = hi;
            constexpr int S = Plan::nslots(NL);
#pragma unroll
            for (int k = 0; k < S; k++) field(NL, 3 + k)[slot] = phi[k < NS ? k : 0];
            if (MODE == kEnum) {
#pragma unroll
                for (int k = 0; k < NL; k++) field(NL, Layout<Plan, MODE>::eh(NL) + k)[slot] = (k < NL - 1) ? eh[k < NE ? k : 0] : e;
            }
            if (MODE == kRoots) field(NL, Layout<Plan, MODE>::rs(NL))[slot] = rslot;
        }
        ntask[NL] += __popc(mask);
        cand[NL] += warp_sum_u31(keep ? up - lo : 0u);
        __syncwarp();
    }

    // Take up to 32 roots from the global cursor and bind motif edge 1 to them
    // (the root level maps motif edge 1 onto every graph edge).
    __device__ __forceinline__ bool fetch_roots(uint64_t &next, uint64_t &end) {
        if (next >= end) {
            unsigned long long b = 0;
            if (lane == 0) b = atomicAdd(&p.scratch[0], (unsigned long long)kRootChunk);
            b = __shfl_sync(kFull, b, 0);
            if (b >= p.n_roots) return false;
            next = b;
            end = min((uint64_t)(b + kRootChunk), (uint64_t)p.n_roots);
        }
        const uint64_t slot = next + lane;
        bool ok = slot < end;
        next = min((uint64_t)(next + 32), end);
        uint32_t r = 0, a = 0, bb = 0;
        if (ok) {
            r = (uint32_t)(p.roots ? p.roots[slot] : p.root_lo + slot);
            a = __ldg(p.src + r);
            bb = __ldg(p.dst + r);
            ok = a != bb;   // a self-loop cannot map two distinct motif vertices (Q4)
        }
        const uint32_t eh[1] = {r};
        if (plan.L() == 1) {
            emit(ok, eh, r, (uint32_t)slot);
        } else if constexpr (LM > 1) {
            const uint32_t phi[2] = {a, bb};
            const uint32_t hi = ok ? __ldg(p.H + r) : 0;   // t' = t_root + δ as an index
            push<1>(ok, r, hi, phi, eh, (uint32_t)slot);
        }
        return true;
    }

    // Expand up to 32 candidates of level-LV tasks (matching motif edge LV).
    template <int LV>
    __device__ __forceinline__ void expand() {
        constexpr int S = Plan::nslots(LV);
        const uint32_t n = ntask[LV];
        uint32_t *flo = field(LV, 0), *fup = field(LV, 1);
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
        uint32_t hi = 0, rslot = 0, e = 0, w = 0;
        bool ok = false;
        if (active) {
#pragma unroll
            for (int k = 0; k < S; k++) phi[k] = field(LV, 3 + k)[jt];
            hi = field(LV, 2)[jt];
            if (MODE == kEnum) {
#pragma unroll
                for (int k = 0; k < LV; k++) eh[k] = field(LV, Layout<Plan, MODE>::eh(LV) + k)[jt];
            }
            if (MODE == kRoots) rslot = field(LV, Layout<Plan, MODE>::rs(LV))[jt];
            const uint64_t rc = __ldg(p.rec + pos);
            e = (uint32_t)(rc >> 32);
            w = (uint32_t)rc;
            // StructConstraints with the plan's static checks
            const int uM = plan.u(LV), vM = plan.v(LV), nb = plan.nv(LV);
            const bool ub = uM < nb, vb = vM < nb;
            if (ub && vb) {
                // record from the out-list of φ(u): w is the destination; from the in-list of φ(v): the source
                ok = (pos < p.m) ? (w == pick(phi, vM)) : (w == pick(phi, uM));
            } else {
                ok = true;  // the new endpoint must be a graph vertex not yet mapped (injectivity)
#pragma unroll
                for (int k = 0; k < S; k++)
                    if (k < nb) ok &= (w != phi[k]);
            }
        }
        __syncwarp();
        // consume: pop the fully taken tasks, advance the partially taken one
        if (takes && !full) flo[j] = lo + (32u - excl);
        ntask[LV] = n - kfull;
        cand[LV] -= C;
        __syncwarp();

        if (LV + 1 == plan.L()) {
            emit(ok, eh, e, rslot);
        } else if constexpr (LV + 1 < LM) {
            const int nb = plan.nv(LV);
            constexpr int S2 = Plan::nslots(LV + 1);
            uint32_t phi2[S2 + 1];
#pragma unroll
            for (int k = 0; k < S2; k++) phi2[k] = (k < S) ? phi[k < S ? k : 0] : 0u;
            // a new endpoint gets the next slot (motif vertices are numbered by first appearance)
            if (nb < plan.nv(LV + 1)) {
#pragma unroll
                for (int k = 0; k < S2; k++)
                    if (k == nb) phi2[k] = w;
            }
            push<LV + 1>(ok, e, hi, phi2, eh, rslot);
        }
    }
};

template <class Plan, int MODE>
__global__ void __launch_bounds__(kWarpsPerBlock * 32) mine_kernel(const MineParams p) {
    extern __shared__ uint32_t smem[];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    constexpr int LM = Plan::kL;
    uint32_t *ws = smem + warp * Layout<Plan, MODE>::warp_words();
    const Plan plan(p);
    Warp<Plan, MODE> W(p, plan, ws, lane);
    const int L = plan.L();
    uint64_t next = 0, end = 0;
    bool roots_left = true;

    while (true) {
        int sel = -1;
        // deepest level with a full batch whose child stack has room
#pragma unroll
        for (int l = LM - 1; l >= 1; --l)
            if (sel < 0 && l < L && W.cand[l] >= 32 && (l == L - 1 || W.ntask[l + 1 <= LM ? l + 1 : LM] < 32)) sel = l;
        if (sel < 0) {
            if (roots_left && (L == 1 || W.ntask[1] < 32)) {
                sel = 0;
            } else {
#pragma unroll
                for (int l = LM - 1; l >= 1; --l)
                    if (sel < 0 && l < L && W.ntask[l] > 0 && (l == L - 1 || W.ntask[l + 1 <= LM ? l + 1 : LM] < 32)) sel = l;
            }
        }
        if (sel < 0) break;
        switch (sel) {
            case 0: roots_left = W.fetch_roots(next, end); break;
            case 1: if constexpr (LM > 1) W.template expand<1>(); break;
            case 2: if constexpr (LM > 2) W.template expand<2>(); break;
            case 3: if constexpr (LM > 3) W.template expand<3>(); break;
            case 4: if constexpr (LM > 4) W.template expand<4>(); break;
            case 5: if constexpr (LM > 5) W.template expand<5>(); break;
            default: break;
        }
    }
    if (lane == 0 && W.count) atomicAdd(&p.scratch[1], W.count);
    if (MODE == kStats) {
#pragma unroll
        for (int l = 0; l < kMaxL; l++) {
            unsigned long long v = W.st.nodes[l];
            for (int d = 16; d; d >>= 1) v += __shfl_xor_sync(kFull, v, d);
            if (lane == 0 && v) atomicAdd(&p.scratch[kStatsBase + l], v);
        }
        unsigned long long a = W.st.window, b = W.st.list, c = W.st.probes;
        for (int d = 16; d; d >>= 1) {
            a += __shfl_xor_sync(kFull, a, d);
            b += __shfl_xor_sync(kFull, b, d);
            c += __shfl_xor_sync(kFull, c, d);
        }
        if (lane == 0) {
            atomicAdd(&p.scratch[16], a);
            atomicAdd(&p.scratch[17], b);
            atomicAdd(&p.scratch[18], c);
        }
    }
}

template <class Plan, int MODE>
KernelInfo kernel_info() {
    return KernelInfo{&mine_kernel<Plan, MODE>, (int)(Layout<Plan, MODE>::warp_words() * sizeof(uint32_t))};
}

}  // namespace tmg
