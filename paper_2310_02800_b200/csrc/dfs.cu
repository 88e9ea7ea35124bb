// Prefix-disconnected motifs (reading Q9): a motif edge
// that touches no earlier motif vertex takes its candidates from ALL later
// edges of the time-sorted edge list (Alg. 1's "Both u_G, v_G not mapped"
// branch).  Such a level binds two new vertices at once, which the
// warp-cooperative mine_kernel's task layout (one new vertex per level) does
// not express, so these motifs run this kernel instead: one thread per root,
// an explicit depth-first search over the levels of Algorithm 1.
//
// Candidates of level l (after e_{l-1}, ids <= lim = min(H_δ[root],
// H_{δ_l}[e_{l-1}])):
//   u_l or v_l bound : the out-list of φ(u_l) (else the in-list of φ(v_l)),
//                      from its first record after e_{l-1} (binary search on
//                      the record ids, which are time order), neighbour
//                      checked against φ;
//   neither bound    : edge ids e_{l-1}+1 .. lim themselves (AllEdges), both
//                      endpoints new and distinct.
// A vertex is bound at level l iff it occurs in motif edges 0..l-1, a static
// property, so φ entries never need clearing on backtrack.
#include "tm_internal.cuh"

namespace tmg {
namespace {

struct DfsPlan {
    int L;
    uint8_t u[kMaxL], v[kMaxL];
    uint8_t first[kMaxV];   // level at which each motif vertex first occurs
};

__device__ __forceinline__ uint32_t first_after(const uint64_t *rec, uint32_t lo, uint32_t hi, uint32_t prev) {
    // first position in rec[lo, hi) whose id > prev (hi = the list's sentinel)
    while (lo < hi) {
        const uint32_t mid = lo + ((hi - lo) >> 1);
        if ((uint32_t)(rec[mid] >> 32) > prev) hi = mid; else lo = mid + 1;
    }
    return lo;
}

template <int MODE>
__global__ void __launch_bounds__(256) mine_dfs_kernel(const MineParams p, const DfsPlan pl) {
    unsigned long long total = 0;
    const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
    for (uint64_t k = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; k < p.n_roots; k += stride) {
        const uint32_t r = (uint32_t)(p.roots ? p.roots[k] : p.root_lo + k);
        const uint32_t a0 = p.src[r], b0 = p.dst[r];
        if (a0 == b0) continue;   // a self-loop maps no two distinct motif vertices (Q4)
        uint32_t phi[kMaxV], eh[kMaxL], pos[kMaxL], lim[kMaxL];
        uint8_t kind[kMaxL];      // 0: out-list, 1: in-list, 2: all edges
        phi[pl.u[0]] = a0;
        phi[pl.v[0]] = b0;
        eh[0] = r;
        unsigned long long found = 0;
        const uint32_t hr = pl.L > 1 ? p.H[r] : 0u;
        auto emit = [&]() {
            found++;
            if (MODE == kEnum) {
                const unsigned long long row = atomicAdd(p.scratch + 2, 1ull);
                if (row < p.cap)
                    for (int i = 0; i < pl.L; i++) p.enum_buf[row * pl.L + i] = eh[i] + p.id_offset;
            }
        };
        auto bound = [&](int x, int l) { return pl.first[x] < l; };
        // a new vertex's image must differ from every bound vertex's
        auto fresh = [&](uint32_t w, int l) {
            bool ok = true;
            for (int x = 0; x < kMaxV; x++)
                if (pl.first[x] < l && phi[x] == w) ok = false;
            return ok;
        };
        // open level l below the match eh[0..l-1]
        auto open = [&](int l) {
            const uint32_t prev = eh[l - 1];
            uint32_t hi = hr;
            if (p.Hf[l - 1]) hi = min(hi, p.Hf[l - 1][prev]);
            lim[l] = hi;
            const int ul = pl.u[l], vl = pl.v[l];
            if (bound(ul, l)) {
                const uint32_t x = phi[ul];
                kind[l] = 0;
                pos[l] = first_after(p.rec, p.off_out[x], p.off_out[x + 1] - 1, prev);
            } else if (bound(vl, l)) {
                const uint32_t x = phi[vl];
                kind[l] = 1;
                pos[l] = first_after(p.rec, p.off_in[x], p.off_in[x + 1] - 1, prev);
            } else {
                kind[l] = 2;
                pos[l] = prev + 1;
            }
        };
        if (pl.L == 1) {
            emit();
        } else {
            int l = 1;
            open(1);
            while (l >= 1) {
                // next candidate of level l that passes the checks, if any
                bool got = false;
                const int ul = pl.u[l], vl = pl.v[l];
                while (true) {
                    uint32_t e, a, b;
                    if (kind[l] == 2) {
                        e = pos[l];
                        if (e > lim[l]) break;   // lim <= m - 1
                        a = p.src[e];
                        b = p.dst[e];
                    } else {
                        const uint64_t rc = p.rec[pos[l]];
                        e = (uint32_t)(rc >> 32);
                        if (e > lim[l]) break;   // the sentinel's id 0xFFFFFFFF stops it too
                        const uint32_t x = phi[kind[l] == 0 ? ul : vl];
                        a = kind[l] == 0 ? x : (uint32_t)rc;
                        b = kind[l] == 0 ? (uint32_t)rc : x;
                    }
                    pos[l]++;
                    if (a == b) continue;
                    const bool bu = bound(ul, l), bv = bound(vl, l);
                    if (bu && phi[ul] != a) continue;
                    if (bv && phi[vl] != b) continue;
                    if (!bu && !fresh(a, l)) continue;
                    if (!bv && !fresh(b, l)) continue;
                    phi[ul] = a;
                    phi[vl] = b;
                    eh[l] = e;
                    got = true;
                    break;
                }
                if (!got) {
                    l--;   // Backtrack
                    continue;
                }
                if (l == pl.L - 1) {
                    emit();
                } else {
                    l++;   // NextLevel
                    open(l);
                }
            }
        }
        if (MODE == kRoots && found) atomicAdd(&p.root_counts[k], found);
        total += found;
    }
    // warp reduce, one atomic per warp
    for (int o = 16; o; o >>= 1) total += __shfl_down_sync(0xffffffffu, total, o);
    if ((threadIdx.x & 31) == 0 && total && MODE != kEnum) atomicAdd(p.scratch + 1, total);
}

}  // namespace

cudaError_t launch_mine_dfs(const MineParams &p, int mode, int sms, cudaStream_t s, uint32_t *grid_out) {
    DfsPlan pl{};
    pl.L = (int)p.L;
    for (int x = 0; x < kMaxV; x++) pl.first[x] = kMaxL;
    for (int i = (int)p.L - 1; i >= 0; i--) {
        pl.u[i] = p.u[i];
        pl.v[i] = p.v[i];
        pl.first[p.u[i]] = (uint8_t)i;
        pl.first[p.v[i]] = (uint8_t)i;
    }
    const uint64_t want = (p.n_roots + 255) / 256;
    const uint32_t grid = (uint32_t)std::max<uint64_t>(1, std::min<uint64_t>(want, (uint64_t)sms * 8));
    *grid_out = grid;
    switch (mode) {
        case kCount: mine_dfs_kernel<kCount><<<grid, 256, 0, s>>>(p, pl); break;
        case kEnum: mine_dfs_kernel<kEnum><<<grid, 256, 0, s>>>(p, pl); break;
        case kRoots: mine_dfs_kernel<kRoots><<<grid, 256, 0, s>>>(p, pl); break;
        default: return cudaErrorInvalidValue;
    }
    return cudaGetLastError();
}

}  // namespace tmg
