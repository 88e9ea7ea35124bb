// Fused census of the 36 two/three-node three-edge motifs (SURVEY.md §8(f)
// N1; config C2): every δ-temporal motif M_ab = (0→1, E[a], E[b]) with
// E = [0→1, 1→0, 0→2, 2→0, 1→2, 2→1] counted in ONE traversal instead of 36
// queries.  The matches of all 36 motifs rooted at edge r = (u→v) are
// exactly the chains r < e2 < e3 with t(e3) - t(r) <= δ, each e_i
// touching the vertices bound so far, over at most one new vertex w
// (injectivity).  Every such e2 and e3 is an edge of u or v — all six
// types of E touch vertex 0 or vertex 1 — so both levels read only the four
// time-sorted lists OUT(u), IN(u), OUT(v), IN(v), and each type
// is read from exactly one of them:
//     0→1 OUT(u)   1→0 OUT(v)   0→2 OUT(u)   2→0 IN(u)   1→2 OUT(v)   2→1 IN(v)
// The level-2 windows (after r) are shared by all 36 motifs, the level-3
// windows (after e2) by the six motifs with the same e2 type: the binning by
// (edge-2 type, edge-3 type) of SURVEY.md N1.
//
// census36_warp_kernel (default): lanes find the level-2 windows of 32 roots,
// then the warp walks their flattened level-2 candidates 32 at a time; the
// thread-per-root census36_kernel is kept as TM_CENSUS_WARP=0.  36 u64 bins
// per CTA in shared memory, one global atomic per bin per CTA.  Window bounds are edge ids from the δ-horizons:
// e2 <= min(H_δ[r], H_δ1[r]), e3 <= min(H_δ[r], H_δ2[e2]).
#include "tm_internal.cuh"

namespace tmg {
namespace {

// Type of a candidate record of list X (0 OUT(u), 1 IN(u), 2 OUT(v), 3
// IN(v)) with neighbour x, given the bound vertices u, v and, if bound
// (w != kNoVertex), the third vertex w; -1 if it matches no E type or belongs
// to another list.
constexpr uint32_t kNoVertex = 0xFFFFFFFFu;

__device__ __forceinline__ int edge_type(int X, uint32_t x, uint32_t u, uint32_t v, uint32_t w) {
    const bool free_w = w == kNoVertex;
    switch (X) {
        case 0: return x == v ? 0 : (x == u ? -1 : (free_w || x == w ? 2 : -1));   // u→x
        case 1: return (x == u || x == v) ? -1 : (free_w || x == w ? 3 : -1);      // x→u (v→u: OUT(v))
        case 2: return x == u ? 1 : (x == v ? -1 : (free_w || x == w ? 4 : -1));   // v→x
        default: return (x == u || x == v) ? -1 : (free_w || x == w ? 5 : -1);     // x→v (u→v: OUT(u))
    }
}

__global__ void __launch_bounds__(256) census36_kernel(const CensusParams p) {
    __shared__ unsigned long long bins[36];
    for (int i = threadIdx.x; i < 36; i += blockDim.x) bins[i] = 0;
    __syncthreads();
    const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
    for (uint64_t k = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; k < p.n_roots; k += stride) {
        const uint32_t r = (uint32_t)(p.root_lo + k);
        const uint32_t u = __ldg(p.src + r), v = __ldg(p.dst + r);
        if (u == v) continue;   // a self-loop maps no two distinct motif vertices (Q4)
        const uint32_t hi = __ldg(p.H + r);
        const uint32_t lim2 = p.Hf0 ? min(hi, __ldg(p.Hf0 + r)) : hi;
        uint32_t s[4];           // first record after r in OUT(u), IN(u), OUT(v), IN(v)
#pragma unroll
        for (int X = 0; X < 4; X++) s[X] = __ldg(p.rank + (size_t)X * p.m + r);
#pragma unroll
        for (int X = 0; X < 4; X++) {
            uint32_t c[4];       // per list: first record after the current e2 (moves forward)
#pragma unroll
            for (int Y = 0; Y < 4; Y++) c[Y] = s[Y];
            for (uint32_t q = s[X];; ++q) {
                const uint64_t rc = __ldg(p.rec + q);
                const uint32_t e2 = (uint32_t)(rc >> 32);
                if (e2 > lim2) break;   // the list's sentinel (id 0xFFFFFFFF) stops it too
                const int a = edge_type(X, (uint32_t)rc, u, v, kNoVertex);
                if (a < 0) continue;
                const uint32_t w = a >= 2 ? (uint32_t)rc : kNoVertex;
                const uint32_t lim3 = p.Hf1 ? min(hi, __ldg(p.Hf1 + e2)) : hi;
#pragma unroll
                for (int Y = 0; Y < 4; Y++) {
                    if (Y == X) {
                        c[Y] = q + 1;
                    } else {
                        while ((uint32_t)(__ldg(p.rec + c[Y]) >> 32) <= e2) ++c[Y];
                    }
                    for (uint32_t z = c[Y];; ++z) {
                        const uint64_t r3 = __ldg(p.rec + z);
                        if ((uint32_t)(r3 >> 32) > lim3) break;
                        const int b = edge_type(Y, (uint32_t)r3, u, v, w);
                        if (b >= 0) atomicAdd(&bins[a * 6 + b], 1ull);
                    }
                }
            }
        }
    }
    __syncthreads();
    for (int i = threadIdx.x; i < 36; i += blockDim.x)
        if (bins[i]) atomicAdd(p.counts + i, bins[i]);
}

// Warp-cooperative variant: lanes find the level-2 windows of 32 roots, then
// the warp walks the flattened list of all their level-2 candidates 32 at a
// time (lane -> owner root by a 5-step search over the lanes' prefix sums), so
// a burst at one root spreads over the warp instead of serialising one lane.
// Each lane then scans the four level-3 windows of its e2.
__global__ void __launch_bounds__(256) census36_warp_kernel(const CensusParams p) {
    __shared__ unsigned long long bins[36];
    for (int i = threadIdx.x; i < 36; i += blockDim.x) bins[i] = 0;
    __syncthreads();
    const unsigned full = 0xffffffffu;
    const int lane = threadIdx.x & 31;
    const uint64_t warps = (uint64_t)gridDim.x * (blockDim.x >> 5);
    const uint64_t wid = (uint64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
    for (uint64_t base = wid * 32; base < p.n_roots; base += warps * 32) {
        const uint64_t k = base + lane;
        uint32_t u = 0, v = 0, hi = 0, s[4] = {0, 0, 0, 0}, nx[4] = {0, 0, 0, 0};
        if (k < p.n_roots) {
            const uint32_t r = (uint32_t)(p.root_lo + k);
            u = __ldg(p.src + r);
            v = __ldg(p.dst + r);
            if (u != v) {   // a self-loop maps no two distinct motif vertices (Q4)
                hi = __ldg(p.H + r);
                const uint32_t lim2 = p.Hf0 ? min(hi, __ldg(p.Hf0 + r)) : hi;
#pragma unroll
                for (int X = 0; X < 4; X++) {
                    s[X] = __ldg(p.rank + (size_t)X * p.m + r);
                    uint32_t q = s[X];
                    while ((uint32_t)(__ldg(p.rec + q) >> 32) <= lim2) ++q;   // sentinel-bounded
                    nx[X] = q - s[X];
                }
            }
        }
        const uint32_t c = nx[0] + nx[1] + nx[2] + nx[3];
        uint32_t incl = c;
#pragma unroll
        for (int d = 1; d < 32; d <<= 1) {
            const uint32_t y = __shfl_up_sync(full, incl, d);
            if (lane >= d) incl += y;
        }
        const uint32_t excl = incl - c, total = __shfl_sync(full, incl, 31);
        for (uint32_t b0 = 0; b0 < total; b0 += 32) {
            const uint32_t kk = b0 + lane;
            // owner: the last lane whose exclusive prefix is <= kk
            int o = 0;
#pragma unroll
            for (int st = 16; st; st >>= 1) {
                const uint32_t ex = __shfl_sync(full, excl, o + st);
                if (o + st < 32 && ex <= kk) o += st;
            }
            const uint32_t ex_o = __shfl_sync(full, excl, o);
            const uint32_t uo = __shfl_sync(full, u, o), vo = __shfl_sync(full, v, o), hio = __shfl_sync(full, hi, o);
            uint32_t so[4], no[4];
#pragma unroll
            for (int X = 0; X < 4; X++) {
                so[X] = __shfl_sync(full, s[X], o);
                no[X] = __shfl_sync(full, nx[X], o);
            }
            if (kk >= total) continue;
            uint32_t q = kk - ex_o;
            int X = 0;
#pragma unroll
            for (int x = 0; x < 3; x++)
                if (X == x && q >= no[x]) { q -= no[x]; X = x + 1; }
            uint32_t pos = 0;
#pragma unroll
            for (int x = 0; x < 4; x++)
                if (X == x) pos = so[x] + q;
            const uint64_t rc = __ldg(p.rec + pos);
            const uint32_t e2 = (uint32_t)(rc >> 32);
            const int a = edge_type(X, (uint32_t)rc, uo, vo, kNoVertex);
            if (a < 0) continue;
            const uint32_t w = a >= 2 ? (uint32_t)rc : kNoVertex;
            const uint32_t lim3 = p.Hf1 ? min(hio, __ldg(p.Hf1 + e2)) : hio;
#pragma unroll
            for (int Y = 0; Y < 4; Y++) {
                uint32_t z;
                if (Y == X) {
                    z = pos + 1;
                } else {
                    z = so[Y];
                    while ((uint32_t)(__ldg(p.rec + z) >> 32) <= e2) ++z;
                }
                for (;; ++z) {
                    const uint64_t r3 = __ldg(p.rec + z);
                    if ((uint32_t)(r3 >> 32) > lim3) break;
                    const int bb = edge_type(Y, (uint32_t)r3, uo, vo, w);
                    if (bb >= 0) atomicAdd(&bins[a * 6 + bb], 1ull);
                }
            }
        }
    }
    __syncthreads();
    for (int i = threadIdx.x; i < 36; i += blockDim.x)
        if (bins[i]) atomicAdd(p.counts + i, bins[i]);
}

}  // namespace

#ifndef TM_CENSUS_WARP
#define TM_CENSUS_WARP 1
#endif
cudaError_t launch_census36(const CensusParams &p, int grid, cudaStream_t s) {
    if (TM_CENSUS_WARP)
        census36_warp_kernel<<<grid, 256, 0, s>>>(p);
    else
        census36_kernel<<<grid, 256, 0, s>>>(p);
    return cudaGetLastError();
}

}  // namespace tmg
