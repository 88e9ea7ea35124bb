// Device graph construction: stable order by
// (t, input position), the bidirectional time-sorted CSR of packed 64-bit
// records, and the per-query δ-horizon arrays.
#include <cub/cub.cuh>

#include <mutex>
#include <vector>

#include "tm_internal.cuh"

namespace tmg {

namespace {

__global__ void k_validate(const uint32_t *src, const uint32_t *dst, const int64_t *t, uint64_t m, uint32_t n,
                           unsigned long long *flags) {
    // flags[0]: bad id, flags[1]: negative t, flags[2]: not sorted by t
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < m; i += (uint64_t)gridDim.x * blockDim.x) {
        if (src[i] >= n || dst[i] >= n) flags[0] = 1;
        if (t[i] < 0) flags[1] = 1;
        if (i + 1 < m && t[i] > t[i + 1]) flags[2] = 1;
    }
}

// the id checks of k_validate only (flags[0]); flags[1], flags[2] from k_validate_t
__global__ void k_validate_ids(const uint32_t *src, const uint32_t *dst, uint64_t m, uint32_t n,
                               unsigned long long *flags) {
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < m; i += (uint64_t)gridDim.x * blockDim.x)
        if (src[i] >= n || dst[i] >= n) flags[0] = 1;
}

__global__ void k_validate_t(const int64_t *t, uint64_t m, unsigned long long *flags) {
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < m; i += (uint64_t)gridDim.x * blockDim.x) {
        if (t[i] < 0) flags[1] = 1;
        if (i + 1 < m && t[i] > t[i + 1]) flags[2] = 1;
    }
}

__global__ void k_iota(uint32_t *a, uint64_t m) {
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < m; i += (uint64_t)gridDim.x * blockDim.x)
        a[i] = (uint32_t)i;
}

__global__ void k_gather(const uint32_t *perm, const uint32_t *src, const uint32_t *dst, const int64_t *t,
                         uint64_t m, uint32_t *os, uint32_t *od, int64_t *ot) {
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < m; i += (uint64_t)gridDim.x * blockDim.x) {
        uint32_t j = perm[i];
        os[i] = src[j];
        od[i] = dst[j];
        ot[i] = t[j];
    }
}

// H_d[e] = max{ j : T[j] <= T[e] + d }  (>= e; m-1 when d = ∞ or saturated).
// The δ-window t' = t_root + δ of Algorithm 1 and the
// fine-grained bound t_prev + δ_i become edge-id limits.
// H is monotone, so a block of kHB consecutive edges has all its answers in
// [H(e0), H(e_last)]: two threads find those ends in global memory, the
// block stages T over that range in shared memory (coalesced) and every
// thread binary-searches there.  Bursty stretches whose range exceeds the
// stage fall back to a per-thread gallop in global memory.
#ifndef TM_HB
#define TM_HB 512
#endif
constexpr int kHB = TM_HB;          // edges per block
#ifndef TM_HLIN
#define TM_HLIN 0   // single steps before the gallop from the previous answer (0: gallop only)
#endif
#ifndef TM_HEPT
#define TM_HEPT 4
#endif
#ifndef TM_HSTAGE
#define TM_HSTAGE 4
#endif
constexpr int kHEpt = TM_HEPT;      // consecutive edges per thread (4 or 8)
static_assert(kHEpt == 4 || kHEpt == 8, "kHEpt");

__device__ __forceinline__ uint64_t horizon_one(const int64_t *__restrict__ T, uint64_t m, int64_t d, uint64_t e) {
    const int64_t te = T[e];
    if (d == TM_DELTA_INF || te > INT64_MAX - d) return m - 1;
    const int64_t key = te + d;
    uint64_t lo = e + 1, step = 1, hi;
    while (true) {       // gallop from e, then binary search: first j > e with T[j] > key
        hi = lo + step - 1;
        if (hi >= m) { hi = m; break; }
        if (T[hi] > key) break;
        lo = hi + 1;
        step <<= 1;
    }
    while (lo < hi) {
        uint64_t mid = lo + ((hi - lo) >> 1);
        if (T[mid] > key) hi = mid; else lo = mid + 1;
    }
    return lo - 1;
}

// H at the first and last edge of every kHB block, per horizon (one thread each)
__global__ void k_horizon_ends(const int64_t *__restrict__ T, uint64_t m, int64_t d0, int64_t d1, int nh,
                               uint64_t *__restrict__ ends) {
    const uint64_t nb = (m + kHB - 1) / kHB;
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < 2 * nb * nh;
         i += (uint64_t)gridDim.x * blockDim.x) {
        const uint64_t h = i / (2 * nb), r = i - h * 2 * nb, b = r >> 1;
        const uint64_t e = (r & 1) ? min((b + 1) * kHB, m) - 1 : b * kHB;
        ends[i] = horizon_one(T, m, h ? d1 : d0, e);
    }
}

// Up to two horizons in one pass (the query's δ and its gap bound δ_i share
// the timestamp reads).  A block takes kHB consecutive edges, kHEpt
// consecutive edges per thread (one 32-byte load of T, one 16-byte store of
// H per horizon).  The answer range [H(e0), H(elast)] of each horizon comes
// from k_horizon_ends (all blocks' gallops in parallel); the block stages T over that range
// in shared memory (coalesced), and every thread binary-searches its first
// edge there and walks forward to the next ones (answers are monotone in e:
// usually a step or two).  Bursty blocks whose range exceeds the stage fall
// back to the global gallop per edge.
constexpr int kHThreads = kHB / kHEpt;
constexpr int kHStage = TM_HSTAGE * kHB;   // staged timestamps per horizon, as u32 offsets from the range's first (8 KB; 6 x kHB measured 0.07 ms slower: occupancy)

template <int NH>
#ifndef TM_H_MINB
#define TM_H_MINB 14   // 14 blocks of 128 threads per SM (32 registers, no spills): -0.02 ms
#endif
__global__ void __launch_bounds__(kHThreads, TM_H_MINB) k_horizon(const int64_t *__restrict__ T, uint64_t m, int64_t d0,
                                                       int64_t d1, const uint64_t *__restrict__ gends,
                                                       uint32_t *__restrict__ H0, uint32_t *__restrict__ H1) {
    __shared__ uint32_t st[NH][kHStage];
    __shared__ uint64_t ends[NH][2];
    const uint64_t e0 = (uint64_t)blockIdx.x * kHB;
    const uint64_t elast = min(e0 + kHB, m) - 1;
    if (threadIdx.x < 2 * NH) {
        const int h = threadIdx.x >> 1;
        ends[h][threadIdx.x & 1] = gends[(uint64_t)h * 2 * gridDim.x + 2 * blockIdx.x + (threadIdx.x & 1)];
    }
    const uint64_t eb = e0 + (uint64_t)threadIdx.x * kHEpt;   // this thread's first edge
    int64_t te[kHEpt];
    if (eb + kHEpt - 1 <= elast) {
        const longlong2 *v = reinterpret_cast<const longlong2 *>(T + eb);
#pragma unroll
        for (int q = 0; q < kHEpt / 2; q++) {   // 32-byte loads
            const longlong2 a = v[q];
            te[2 * q] = a.x;
            te[2 * q + 1] = a.y;
        }
    } else {
#pragma unroll
        for (int j = 0; j < kHEpt; j++) te[j] = eb + j <= elast ? T[eb + j] : 0;
    }
    __syncthreads();
    // staged: the range fits the stage and spans < 2^32 - 1 time units (u32 offsets)
    bool staged[NH];
    int64_t base[NH];
#pragma unroll
    for (int h = 0; h < NH; h++) {
        const uint64_t lo = ends[h][0], span = ends[h][1] - lo + 1;
        base[h] = T[lo];
        staged[h] = span <= kHStage && T[ends[h][1]] - base[h] < (int64_t)0xFFFFFFFF;
        if (staged[h]) {   // 32-bit indexing: span <= kHStage
            const int64_t *Tl = T + lo;
            const uint32_t sp = (uint32_t)span;
            for (uint32_t i = threadIdx.x; i < sp; i += kHThreads) st[h][i] = (uint32_t)(Tl[i] - base[h]);
        }
    }
    __syncthreads();
#pragma unroll
    for (int h = 0; h < NH; h++) {
        const int64_t d = h ? d1 : d0;
        uint32_t *H = h ? H1 : H0;
        const uint64_t lo = ends[h][0], span = ends[h][1] - lo + 1;
        uint32_t out[kHEpt];
        if (staged[h]) {
            const uint32_t *sh = st[h];
            uint32_t pos = 0;   // last index with sh[pos] <= key; sh[0] = T[H(e0)] <= every key
#pragma unroll
            for (int j = 0; j < kHEpt; j++) {
                const int64_t kf = (d == TM_DELTA_INF || te[j] > INT64_MAX - d) ? INT64_MAX : te[j] + d;
                // key as an offset from base (>= 0: T[lo] <= key); every staged offset
                // is < 2^32 - 1, so a key capped there still compares exactly
                const uint32_t key = (uint32_t)min(kf - base[h], (int64_t)0xFFFFFFFF);
                // first edge: binary search of [0, span); next ones: gallop from the
                // previous answer (answers are monotone and usually a step or two apart)
                uint32_t len;
                if (j == 0) {
                    len = (uint32_t)span;
                } else {
                    uint32_t step = 1;
                    int it = 0;
#if TM_HLIN
                    // consecutive answers are usually 0-2 apart: up to TM_HLIN single
                    // steps, then the gallop
                    while (it < TM_HLIN && pos + 1 < span && sh[pos + 1] <= key) { ++pos; ++it; }
#endif
                    if (TM_HLIN && it < TM_HLIN) {
                        len = 1;   // stopped: sh[pos + 1] > key (or the range ends)
                    } else {
                        while (pos + step < span && sh[pos + step] <= key) { pos += step; step <<= 1; }
                        len = min(step, (uint32_t)span - pos);   // answer in [pos, pos + len)
                    }
                }
                while (len > 1) {
                    const uint32_t half = len >> 1;
                    if (sh[pos + half] <= key) pos += half;
                    len -= half;
                }
                out[j] = (uint32_t)(kf == INT64_MAX ? m - 1 : lo + pos);
            }
        } else {
#pragma unroll
            for (int j = 0; j < kHEpt; j++) out[j] = eb + j <= elast ? (uint32_t)horizon_one(T, m, d, eb + j) : 0u;
        }
        if (eb + kHEpt - 1 <= elast) {
#pragma unroll
            for (int q = 0; q < kHEpt / 4; q++)
                reinterpret_cast<uint4 *>(H + eb)[q] = make_uint4(out[4 * q], out[4 * q + 1], out[4 * q + 2], out[4 * q + 3]);
        } else {
#pragma unroll
            for (int j = 0; j < kHEpt; j++)
                if (eb + j <= elast) H[eb + j] = out[j];
        }
    }
}

// Both CSR directions and the rank arrays from one stable sort of the 2m
// (vertex, edge) incidences: entry 2e is e's out-incidence at src(e), entry
// 2e+1 its in-incidence at dst(e).  A stable sort by vertex lists, for every
// vertex, all edges touching it in id (= time) order; a scan of "is an
// out-incidence" flags then counts, at every entry, the out- and in-edges of
// that vertex that come earlier — exactly the list positions and the ranks.
// value = incidence id << 32 | the other endpoint: the sort carries each
// record's neighbour, so the scatter after it gathers nothing
__global__ void k_incidences(const uint32_t *src, const uint32_t *dst, uint64_t m, uint32_t *key, uint64_t *val) {
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < 2 * m; i += (uint64_t)gridDim.x * blockDim.x) {
        const uint64_t e = i >> 1;
        const uint32_t a = src[e], b = dst[e];
        key[i] = (i & 1) ? b : a;
        val[i] = (i << 32) | ((i & 1) ? a : b);
    }
}

// start[u] = first sorted incidence of vertex u (2m past the last; vertices
// without incidences share the next vertex's start)
__global__ void k_vertex_starts(const uint32_t *kout, uint64_t n2, uint32_t n, uint32_t *start) {
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i <= n2; i += (uint64_t)gridDim.x * blockDim.x) {
        const int64_t kv = i < n2 ? (int64_t)kout[i] : (int64_t)n;
        const int64_t kp = i == 0 ? -1 : (int64_t)kout[i - 1];
        for (int64_t u = kp + 1; u <= kv; u++) start[u] = (uint32_t)i;
    }
}

// list starts from the runs of the merged incidence sort: before vertex v's
// run come outb[start v] out-incidences and the rest are in-incidences
// (plain offset + v for the out-lists' sentinels, in-lists further shifted by m + n)
__global__ void k_offsets_from_runs(const uint32_t *start, const uint32_t *outb, uint32_t n, uint64_t m,
                                    uint32_t *off_out, uint32_t *off_in) {
    for (uint32_t v = blockIdx.x * blockDim.x + threadIdx.x; v <= n; v += gridDim.x * blockDim.x) {
        const uint32_t sv = start[v], ob = outb[sv];
        off_out[v] = ob + v;
        off_in[v] = (sv - ob) + (uint32_t)(m + n) + v;
    }
}

__global__ void k_outflag(const uint64_t *val, uint64_t n2, uint32_t *flag) {
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i <= n2; i += (uint64_t)gridDim.x * blockDim.x)
        flag[i] = i < n2 && ((val[i] >> 32) & 1u) == 0 ? 1u : 0u;
}

// off_out / off_in hold the sentinel-adjusted list starts (plain offset + v,
// in-lists further shifted by m + n); the plain offsets are recovered here.
// Records go to rec[] in place (consecutive incidences of a vertex are
// consecutive positions); the two rank values of the incidence go to rk[i]
// in incidence order and reach rank[] through a radix sort by incidence id
// (k_rank_from_sorted): scattering them directly as 4-byte random writes
// measured 12 ms of a 21 ms build on C4.
__global__ void k_scatter_csr(const uint32_t *key, const uint64_t *val, const uint32_t *outb,
                              const uint32_t *off_out, const uint32_t *off_in, uint64_t m, uint32_t n, uint64_t *rec,
                              unsigned long long *rk, uint32_t *inc) {
    const uint32_t split = (uint32_t)(m + n);
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < 2 * m; i += (uint64_t)gridDim.x * blockDim.x) {
        const uint64_t vv = val[i];
        const uint32_t v = key[i], ent = (uint32_t)(vv >> 32), e = ent >> 1, nbr = (uint32_t)vv;
        inc[i] = ent;
        const uint32_t so = off_out[v], si = off_in[v];                 // list starts in rec
        const uint64_t seg = (uint64_t)(so - v) + (si - split - v);      // first incidence of v
        const uint32_t ob = outb[i] - outb[seg];                        // out-incidences of v before i
        const uint32_t ib = (uint32_t)(i - seg) - ob;                   // in-incidences of v before i
        uint32_t a, b;
        if ((ent & 1u) == 0) {            // e in OUT(v), v = src(e)
            const uint32_t pos = so + ob;
            const uint32_t w = nbr;
            rec[pos] = ((uint64_t)e << 32) | w;
            a = pos + 1;                          // var 0: OUT(src e)
            b = si + ib + (v == w ? 1u : 0u);     // var 1: IN(src e), ids <= e
        } else {                          // e in IN(v), v = dst(e)
            const uint32_t pos = si + ib;
            rec[pos] = ((uint64_t)e << 32) | nbr;
            a = pos + 1;                          // var 3: IN(dst e)
            b = so + ob;                          // var 2: OUT(dst e), ids <= e
        }
        rk[i] = ((unsigned long long)a << 32) | b;
    }
}

// rk sorted by incidence id 2e + dir: the rank values of edge e, coalesced
__global__ void k_rank_from_sorted(const unsigned long long *rk, uint64_t m, uint32_t *rank) {
    for (uint64_t j = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; j < 2 * m; j += (uint64_t)gridDim.x * blockDim.x) {
        const uint64_t e = j >> 1;
        const unsigned long long v = rk[j];
        if ((j & 1) == 0) {
            rank[e] = (uint32_t)(v >> 32);         // var 0
            rank[m + e] = (uint32_t)v;             // var 1
        } else {
            rank[3 * m + e] = (uint32_t)(v >> 32); // var 3
            rank[2 * m + e] = (uint32_t)v;         // var 2
        }
    }
}

__global__ void k_sentinels(const uint32_t *off_out, const uint32_t *off_in, uint32_t n, uint64_t *rec) {
    for (uint32_t v = blockIdx.x * blockDim.x + threadIdx.x; v < n; v += gridDim.x * blockDim.x) {
        rec[off_out[v + 1] - 1] = ~0ull;
        rec[off_in[v + 1] - 1] = ~0ull;
    }
}

__global__ void k_pair_keys(const uint32_t *src, const uint32_t *dst, uint64_t m, int nb, uint64_t *key, uint32_t *val) {
    for (uint64_t e = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; e < m; e += (uint64_t)gridDim.x * blockDim.x) {
        key[e] = ((uint64_t)src[e] << nb) | dst[e];
        val[e] = (uint32_t)e;
    }
}

// one thread per pair start: insert {key, start, len} (linear probing)
__global__ void k_pair_insert(const uint64_t *skey, uint64_t m, int nb, uint4 *tab, uint32_t mask, uint32_t *bits,
                              uint32_t fmask) {
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < m; i += (uint64_t)gridDim.x * blockDim.x) {
        const uint64_t k = skey[i];
        if (i > 0 && skey[i - 1] == k) continue;
        uint64_t j = i + 1;
        while (j < m && skey[j] == k) j++;
        const uint64_t src = k >> nb, dst = k & ((1ull << nb) - 1);
        const uint64_t key = (src << 32) | dst;
        uint32_t h = (uint32_t)pair_hash(key) & mask;
        while (true) {
            unsigned long long *slot = reinterpret_cast<unsigned long long *>(tab + h);
            if (atomicCAS(slot, ~0ull, (unsigned long long)key) == ~0ull) {
            const uint64_t hh = pair_hash(key);
            for (int k = 0; k < (TM_BLOOM_K > 0 ? TM_BLOOM_K : 1); k++) {
                const uint32_t b = bloom_bit(hh, fmask, k);
                atomicOr(bits + (b >> 5), 1u << (b & 31));
            }
                tab[h].z = (uint32_t)i;
                tab[h].w = (uint32_t)(j - i);
                break;
            }
            h = (h + 1) & mask;
        }
    }
}

// id-bucketed pair filter: the bit of (src e, dst e, e >> shift) for every edge
__global__ void k_pair_time_bits(const uint32_t *src, const uint32_t *dst, uint64_t m, int shift, uint32_t *bits,
                                 uint32_t mask) {
    for (uint64_t e = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; e < m; e += (uint64_t)gridDim.x * blockDim.x) {
        const uint32_t b = pair_bucket_bit(src[e], dst[e], (uint32_t)(e >> shift), mask);
        atomicOr(bits + (b >> 5), 1u << (b & 31));
    }
}

__global__ void k_count_starts(const uint64_t *skey, uint64_t m, unsigned long long *cnt) {
    unsigned long long c = 0;
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < m; i += (uint64_t)gridDim.x * blockDim.x)
        c += (i == 0 || skey[i - 1] != skey[i]) ? 1 : 0;
    for (int d = 16; d; d >>= 1) c += __shfl_xor_sync(0xffffffffu, c, d);
    if ((threadIdx.x & 31) == 0 && c) atomicAdd(cnt, c);
}

inline unsigned grid_for(uint64_t m) {
    uint64_t b = (m + 255) / 256;
    return (unsigned)std::max<uint64_t>(1, std::min<uint64_t>(b, 148ull * 32));
}

template <class T>
cudaError_t dmalloc(T **p, size_t count, cudaStream_t s) {
    return dev_alloc((void **)p, std::max<size_t>(count, 1) * sizeof(T), s);
}

void free_graph(DeviceGraph &d, cudaStream_t s) {
    for (void *q : {(void *)d.src, (void *)d.dst, (void *)d.t, (void *)d.perm, (void *)d.off_out, (void *)d.off_in,
                    (void *)d.rec, (void *)d.rank, (void *)d.skip, (void *)d.prec, (void *)d.ptab, (void *)d.pbits, (void *)d.tbits,
                    (void *)d.vlab, (void *)d.elab})
        dev_free(q, s);
    if (d.nxc) {
        dev_free(d.nxc->buf, s);
        for (int v = 0; v < 4; v++)
            if (d.nxc->ev[v]) cudaEventDestroy(d.nxc->ev[v]);
        delete d.nxc;
    }
    d = DeviceGraph{};
}

// Offsets (histogram + scan per direction), then the merged incidence sort.
cudaError_t build_csr(DeviceGraph &d, cudaStream_t s) {
    const uint64_t m = d.m;
    const uint32_t n = d.n;
    uint32_t *key = nullptr, *kout = nullptr, *flag = nullptr, *start = nullptr;
    uint64_t *val = nullptr, *vout = nullptr;
    unsigned long long *rk = nullptr, *rk2 = nullptr;
    void *tmp = nullptr;
    size_t sort_bytes = 0, scan2_bytes = 0, sort2_bytes = 0;
    cudaError_t err;
    int end_bit = 1;
    while (end_bit < 32 && (1ull << end_bit) < (uint64_t)n) end_bit++;
    const uint64_t n2 = 2 * m;
    int end_bit2 = 1;   // incidence ids 2e + dir < 2m
    while (end_bit2 < 32 && (1ull << end_bit2) < n2) end_bit2++;
#define TRY(x) do { err = (x); if (err != cudaSuccess) goto done; } while (0)
    TRY(dmalloc(&key, n2 + 1, s));
    TRY(dmalloc(&val, n2, s));
    TRY(dmalloc(&kout, n2, s));
    TRY(dmalloc(&vout, n2, s));
    TRY(dmalloc(&flag, n2 + 1, s));
    TRY(dmalloc(&start, (size_t)n + 1, s));
    TRY(cub::DeviceRadixSort::SortPairs(nullptr, sort_bytes, key, kout, val, vout, (int64_t)n2, 0, end_bit, s));
    TRY(cub::DeviceScan::ExclusiveSum(nullptr, scan2_bytes, flag, key, (int64_t)n2 + 1, s));
    TRY(dmalloc(&rk, n2, s));
    TRY(dmalloc(&rk2, n2, s));
    TRY(cub::DeviceRadixSort::SortPairs(nullptr, sort2_bytes, flag, kout, rk, rk2, (int64_t)n2, 0, end_bit2, s));
    TRY(dev_alloc(&tmp, std::max(std::max(sort_bytes, sort2_bytes), scan2_bytes), s));
    // one stable sort of the 2m incidences by vertex (value: incidence id and
    // neighbour); the out-flag scan over it gives every list position, rank
    // value and — at the runs' starts — both offset arrays (no degree pass)
    if (m) {
        k_incidences<<<grid_for(n2), 256, 0, s>>>(d.src, d.dst, m, key, val);
        TRY(cub::DeviceRadixSort::SortPairs(tmp, sort_bytes, key, kout, val, vout, (int64_t)n2, 0, end_bit, s));
    }
    k_outflag<<<grid_for(n2 + 1), 256, 0, s>>>(vout, n2, flag);
    TRY(cub::DeviceScan::ExclusiveSum(tmp, scan2_bytes, flag, key, (int64_t)n2 + 1, s));  // key: free after the sort
    k_vertex_starts<<<grid_for(n2 + 1), 256, 0, s>>>(kout, n2, n, start);
    k_offsets_from_runs<<<grid_for((uint64_t)n + 1), 256, 0, s>>>(start, key, n, m, d.off_out, d.off_in);
    k_sentinels<<<grid_for(n), 256, 0, s>>>(d.off_out, d.off_in, n, d.rec);
    if (m) {
        k_scatter_csr<<<grid_for(n2), 256, 0, s>>>(kout, vout, key, d.off_out, d.off_in, m, n, d.rec, rk, flag);
        // back to incidence order (flag holds the incidence ids, kout is free)
        TRY(cub::DeviceRadixSort::SortPairs(tmp, sort2_bytes, flag, kout, rk, rk2, (int64_t)n2, 0, end_bit2, s));
        k_rank_from_sorted<<<grid_for(n2), 256, 0, s>>>(rk2, m, d.rank);
    }
    TRY(cudaGetLastError());
    TRY(cudaStreamSynchronize(s));
done:
#undef TRY
    for (void *q : {(void *)key, (void *)val, (void *)kout, (void *)vout, (void *)flag, (void *)start, (void *)rk,
                    (void *)rk2, tmp})
        dev_free(q, s);
    return err;
}

// Pair index: stable radix sort of the edges by (src, dst), distinct pairs
// counted, then inserted into the hash table.
cudaError_t build_pairs(DeviceGraph &d, cudaStream_t s, int bucket_log2) {
    const uint64_t m = d.m;
    uint64_t *key = nullptr, *skey = nullptr;
    uint32_t *val = nullptr;
    unsigned long long *cnt = nullptr, hcnt = 0;
    void *tmp = nullptr;
    size_t bytes = 0;
    cudaError_t err;
    int nb = 1;
    while (nb < 32 && (1ull << nb) < (uint64_t)d.n) nb++;
#define TRY(x) do { err = (x); if (err != cudaSuccess) goto done; } while (0)
    TRY(dmalloc(&d.prec, m + 8, s));
    TRY(cudaMemsetAsync(d.prec, 0xff, (m + 8) * 4, s));
    TRY(dmalloc(&key, m, s));
    TRY(dmalloc(&skey, m, s));
    TRY(dmalloc(&val, m, s));
    TRY(dmalloc(&cnt, 1, s));
    TRY(cub::DeviceRadixSort::SortPairs(nullptr, bytes, key, skey, val, d.prec, (int64_t)m, 0, 2 * nb, s));
    TRY(dev_alloc(&tmp, std::max<size_t>(bytes, 1), s));
    TRY(cudaMemsetAsync(cnt, 0, 8, s));
    if (m) {
        k_pair_keys<<<grid_for(m), 256, 0, s>>>(d.src, d.dst, m, nb, key, val);
        TRY(cub::DeviceRadixSort::SortPairs(tmp, bytes, key, skey, val, d.prec, (int64_t)m, 0, 2 * nb, s));
        k_count_starts<<<grid_for(m), 256, 0, s>>>(skey, m, cnt);
    }
    TRY(cudaMemcpyAsync(&hcnt, cnt, 8, cudaMemcpyDeviceToHost, s));
    TRY(cudaStreamSynchronize(s));
    d.npairs = hcnt;
    {
        uint64_t cap = 16;
        while (cap < 2 * hcnt) cap <<= 1;
        d.pmask = (uint32_t)(cap - 1);
        TRY(dmalloc(&d.ptab, cap, s));
        TRY(cudaMemsetAsync(d.ptab, 0xff, cap * sizeof(uint4), s));
        uint64_t fb = 1024;
        while (fb < (uint64_t)TM_BLOOM_BITS * hcnt) fb <<= 1;
        d.fmask = (uint32_t)(fb - 1);
        TRY(dmalloc(&d.pbits, fb / 32, s));
        TRY(cudaMemsetAsync(d.pbits, 0, fb / 8, s));
    }
    if (m) k_pair_insert<<<grid_for(m), 256, 0, s>>>(skey, m, nb, d.ptab, d.pmask, d.pbits, d.fmask);
    if (m && bucket_log2 > 0) {   // the id-bucketed filter: TM_BLOOM_BITS bits per edge
        uint64_t tb = 1024;   // bits, a power of two <= 2^32 (32-bit hash)
        while (tb < (uint64_t)TM_BLOOM_BITS * m && tb < (1ull << 32)) tb <<= 1;
        d.tmask = (uint32_t)(tb - 1);
        d.tshift = std::min(bucket_log2, 31);
        TRY(dmalloc(&d.tbits, tb / 32, s));
        TRY(cudaMemsetAsync(d.tbits, 0, tb / 8, s));
        k_pair_time_bits<<<grid_for(m), 256, 0, s>>>(d.src, d.dst, m, d.tshift, d.tbits, d.tmask);
    }
    TRY(cudaGetLastError());
    TRY(cudaStreamSynchronize(s));
done:
#undef TRY
    for (void *q : {(void *)key, (void *)skey, (void *)val, (void *)cnt, tmp}) dev_free(q, s);
    return err;
}

}  // namespace

// H_delta for one or two horizons (H1 = nullptr: one), one launch.
// H arrays are 16-byte aligned (pool allocations of m words, m % 4 == 0 or the tail is scalar).
cudaError_t build_horizons(const DeviceGraph &d, int64_t d0, int64_t d1, uint32_t *H0, uint32_t *H1, cudaStream_t s) {
    if (!d.m) return cudaSuccess;
    const unsigned nb = (unsigned)((d.m + kHB - 1) / kHB);
    const int nh = H1 ? 2 : 1;
    uint64_t *ends = nullptr;
    cudaError_t err = dmalloc(&ends, (size_t)2 * nb * nh, s);
    if (err != cudaSuccess) return err;
    k_horizon_ends<<<grid_for((uint64_t)2 * nb * nh), 256, 0, s>>>(d.t, d.m, d0, d1, nh, ends);
    if (H1) k_horizon<2><<<nb, kHThreads, 0, s>>>(d.t, d.m, d0, d1, ends, H0, H1);
    else k_horizon<1><<<nb, kHThreads, 0, s>>>(d.t, d.m, d0, d0, ends, H0, nullptr);
    err = cudaGetLastError();
    dev_free(ends, s);
    return err;
}

namespace {
// Window-end ranks of one horizon: R[e] = the position of the
// first record in list `var` of edge e (0 OUT(src e), 1 IN(src e), 2 OUT(dst
// e), 3 IN(dst e)) whose edge id exceeds H[e] — i.e. the end of the
// candidate window (e, H[e]] in that list.  A search node whose list is
// anchored at its own last edge e_prev and whose tighter bound is the gap
// horizon H_δi[e_prev] then knows its window end from one load; computed once
// per edge and query instead of once per search node (on C4 every edge is
// e_prev of ~11 nodes).  Gallop from the window start rank[var][e]: windows
// are δ-short and every list ends in an id-0xFFFFFFFF sentinel.
// Window end of an edge whose window runs past the first sector: the first
// position p >= a (a: the first unread, sector-aligned position) with id >
// lim.  The skip entries 8j >= a are read a sector (8 entries = 64 records)
// at a time until one stops the scan: its id exceeds lim, or its mark bit
// says a list's sentinel lies in (8 (j - 1), 8 j] (k_skip_marks) — so the
// scan never needs the list's bound.  The answer is then within the 8
// records before it: one skip sector + two record sectors, issued one after
// the other, for any window up to 64 records past the first sector.  A mark
// at the first entry can belong to the previous list (its sentinel before
// a): no record of the window exceeds lim there, and the scan goes on.
__device__ __noinline__ uint32_t hrank_long(const uint64_t *__restrict__ rec, const uint32_t *__restrict__ skip,
                                            uint32_t a, uint32_t lim) {
    constexpr uint32_t kMark = 0x80000000u, kId = 0x7FFFFFFFu;   // ids < 2^31 (TM_MAX_M)
    uint32_t j = (a + 7) >> 3;
    for (;;) {
        uint32_t jf, svf = 0;
        for (;;) {
            const uint32_t jb = j & ~7u;
            const uint4 s0 = __ldg(reinterpret_cast<const uint4 *>(skip + jb));
            const uint4 s1 = __ldg(reinterpret_cast<const uint4 *>(skip + jb) + 1);
            const uint32_t sv[8] = {s0.x, s0.y, s0.z, s0.w, s1.x, s1.y, s1.z, s1.w};
            jf = ~0u;
#pragma unroll
            for (int k = 7; k >= 0; --k)
                if (jb + k >= j && ((sv[k] & kId) > lim || (sv[k] & kMark))) { jf = jb + k; svf = sv[k]; }
            if (jf != ~0u) break;
            j = jb + 8;
        }
        // rec[8 (jf - 1)] is not past the window (or precedes a)
        const uint32_t lo = max(a, 8 * (jf - 1)), hi = 8 * jf;
        const uint32_t a4 = lo & ~3u;
        const ulonglong2 *v = reinterpret_cast<const ulonglong2 *>(rec + a4);
        const ulonglong2 y0 = __ldg(v), y1 = __ldg(v + 1), y2 = __ldg(v + 2), y3 = __ldg(v + 3);
        const uint64_t r8[8] = {y0.x, y0.y, y1.x, y1.y, y2.x, y2.y, y3.x, y3.y};
        uint32_t ans = ~0u;
#pragma unroll
        for (int k = 7; k >= 0; --k)
            if (a4 + k >= lo && a4 + k < hi && (uint32_t)(r8[k] >> 32) > lim) ans = a4 + k;
        if (ans != ~0u) return ans;
        if ((svf & kId) > lim) return hi;   // rec[8 jf] itself (a sentinel reads 0x7FFFFFFF)
        j = jf + 1;                         // a mark of the previous list's sentinel
    }
}

#ifndef TM_HR_UNROLL
#define TM_HR_UNROLL 2
#endif
constexpr int kHrUnroll = TM_HR_UNROLL;   // edges per thread in flight (independent load chains)
#ifndef TM_NEXT_IDS
#define TM_NEXT_IDS 2   // record / use the first-record ids (NextIdCache): 1 the first, 2 the first two
#endif
constexpr bool kNx2 = TM_NEXT_IDS == 2;
constexpr bool kNx4 = TM_NEXT_IDS == 4;
#ifndef TM_HR_STREAM
#define TM_HR_STREAM 0   // evict-first loads of the per-edge inputs and stores of the descriptors
#endif

// R: window-end ranks (u32 per edge), or W: window descriptors {start, end,
// H[e], 0} (uint4 per edge) when W != nullptr.
// nxr: the first-record ids of this list variant (NextIdCache), if recorded:
// a window that ends before its first record (nx[e] > H[e], half of all
// windows on C4) is written without reading any record.  nxw: record them
// (the id of the record at the window start, from the sector read anyway).
#ifndef TM_HR_MINB
#define TM_HR_MINB 5   // 5 resident 256-thread blocks per SM (48 registers, no spills): passes -0.07 ms; 6: +0.28 ms
#endif
__global__ void __launch_bounds__(256, TM_HR_MINB) k_hrank(const uint64_t *__restrict__ rec, const uint32_t *__restrict__ skip,
                                               const uint32_t *__restrict__ rank, const uint32_t *__restrict__ H,
                                               uint64_t m, uint32_t *__restrict__ R, uint4 *__restrict__ W,
                                               const uint32_t *__restrict__ nxr, uint32_t *__restrict__ nxw) {
    const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
    for (uint64_t e0 = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; e0 < m; e0 += stride * kHrUnroll) {
        uint32_t lim[kHrUnroll], b[kHrUnroll];
        bool need[kHrUnroll];
        uint32_t b1[kHrUnroll];   // known window length when no read is needed (0 or 1)
#pragma unroll
        for (int u = 0; u < kHrUnroll; u++) b1[u] = 0u;
        ulonglong2 x0[kHrUnroll], x1[kHrUnroll];
#pragma unroll
        for (int u = 0; u < kHrUnroll; u++) {
            const uint64_t e = e0 + u * stride;
            lim[u] = e < m ? (TM_HR_STREAM ? __ldcs(H + e) : H[e]) : 0u;
            b[u] = e < m ? (TM_HR_STREAM ? __ldcs(rank + e) : rank[e]) : 0u;   // first record after e
            need[u] = e < m;
            if (nxr && e < m) {
                if (kNx4) {   // the first four record ids: windows of length 0..3 need no read
                    const uint4 q = __ldg(reinterpret_cast<const uint4 *>(nxr) + e);
                    // ids ascend up to the list's sentinel (> lim); anything after the
                    // first id past lim is not in the window (unknown ids read 0: in it)
                    const bool i1 = q.x <= lim[u], i2 = i1 && q.y <= lim[u], i3 = i2 && q.z <= lim[u];
                    need[u] = i3 && q.w <= lim[u];
                    b1[u] = (uint32_t)i1 + (uint32_t)i2 + (uint32_t)i3;
                } else if (kNx2) {   // the first two record ids: windows of length 0 and 1 need no read
                    const uint2 q = TM_HR_STREAM ? __ldcs(reinterpret_cast<const uint2 *>(nxr) + e)
                                                 : __ldg(reinterpret_cast<const uint2 *>(nxr) + e);
                    need[u] = q.x <= lim[u] && q.y <= lim[u];
                    if (q.x <= lim[u] && q.y > lim[u]) b1[u] = 1u;
                } else {
                    need[u] = __ldg(nxr + e) <= lim[u];
                }
            }
        }
        // the aligned 32-byte sector (4 records) holding the window start:
        // windows are δ_i-short, so it usually holds the end too
#pragma unroll
        for (int u = 0; u < kHrUnroll; u++) {
            if (need[u]) {
                const ulonglong2 *v = reinterpret_cast<const ulonglong2 *>(rec + (b[u] & ~3u));
                x0[u] = __ldg(v);
                x1[u] = __ldg(v + 1);
            }
        }
#pragma unroll
        for (int u = 0; u < kHrUnroll; u++) {
            const uint64_t e = e0 + u * stride;
            if (e >= m) break;
            uint32_t ans = b[u] + b1[u];   // a window of known length 0 or 1 (nx)
            if (need[u]) {
                const uint32_t a = b[u] & ~3u;
                const uint32_t id[4] = {(uint32_t)(x0[u].x >> 32), (uint32_t)(x0[u].y >> 32),
                                        (uint32_t)(x1[u].x >> 32), (uint32_t)(x1[u].y >> 32)};
                ans = 0xFFFFFFFFu;
#pragma unroll
                for (int k = 3; k >= 0; --k)
                    if (a + k >= b[u] && id[k] > lim[u]) ans = a + k;
                if (nxw) {
                    const uint32_t o = b[u] & 3u;
                    const uint32_t f = o == 0 ? id[0] : o == 1 ? id[1] : o == 2 ? id[2] : id[3];
                    if (kNx4)   // ids past the sector unknown (0)
                        reinterpret_cast<uint4 *>(nxw)[e] =
                            make_uint4(f, o == 0 ? id[1] : o == 1 ? id[2] : o == 2 ? id[3] : 0u,
                                       o == 0 ? id[2] : o == 1 ? id[3] : 0u, o == 0 ? id[3] : 0u);
                    else if (kNx2)   // second id unknown (0) when it lies in the next sector
                        reinterpret_cast<uint2 *>(nxw)[e] = make_uint2(f, o == 0 ? id[1] : o == 1 ? id[2] : o == 2 ? id[3] : 0u);
                    else
                        nxw[e] = f;
                }
                if (ans == 0xFFFFFFFFu) ans = hrank_long(rec, skip, a + 4, lim[u]);
            }
            if (W) {
                if (TM_HR_STREAM) __stcs(W + e, make_uint4(b[u], ans, lim[u], 0u));
                else W[e] = make_uint4(b[u], ans, lim[u], 0u);
            } else {
                R[e] = ans;
            }
        }
    }
}

// skip[j] = id of rec[8j] (Ids past the records: 0xFFFFFFFF)
__global__ void k_skip(const uint64_t *__restrict__ rec, uint64_t nrec, uint64_t nskip, uint32_t *__restrict__ skip) {
    for (uint64_t j = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; j < nskip; j += (uint64_t)gridDim.x * blockDim.x)
        skip[j] = 8 * j < nrec ? (uint32_t)(rec[8 * j] >> 32) : 0xFFFFFFFFu;
}

// mark bit (bit 31; ids are < 2^31) of skip[j] where a list's sentinel lies in
// (8 (j - 1), 8 j]: a scan of the skip entries then stops in the list it started in
__global__ void k_skip_marks(const uint32_t *__restrict__ off_out, const uint32_t *__restrict__ off_in, uint32_t n,
                             uint32_t *__restrict__ skip) {
    for (uint32_t v = blockIdx.x * blockDim.x + threadIdx.x; v < n; v += gridDim.x * blockDim.x) {
        atomicOr(skip + ((off_out[v + 1] - 1 + 7) >> 3), 0x80000000u);
        atomicOr(skip + ((off_in[v + 1] - 1 + 7) >> 3), 0x80000000u);
    }
}
}  // namespace

namespace {
// S[e] = the first edge id with the same timestamp as e: the anti-edge
// window [t(e), t(e) + δ_ij] starts there in id order (reading Q1
// orders equal timestamps by input position, so a witness may precede e).
__global__ void k_tie_lo(const int64_t *__restrict__ T, uint64_t m, uint32_t *__restrict__ S) {
    const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
    for (uint64_t e = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; e < m; e += stride) {
        const int64_t te = T[e];
        if (e == 0 || T[e - 1] < te) { S[e] = (uint32_t)e; continue; }
        uint64_t lo = 0, hi = e;   // first j in [0, e] with T[j] == te
        while (lo < hi) {
            const uint64_t mid = lo + ((hi - lo) >> 1);
            if (T[mid] < te) lo = mid + 1;
            else hi = mid;
        }
        S[e] = (uint32_t)lo;
    }
}

__global__ void k_gather_i32(const int32_t *__restrict__ in, const uint32_t *__restrict__ perm, uint64_t m,
                             int32_t *__restrict__ out) {
    const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
    for (uint64_t e = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; e < m; e += stride) out[e] = in[perm[e]];
}
}  // namespace

cudaError_t build_tie_lo(const DeviceGraph &d, uint32_t *S, cudaStream_t s) {
    if (!d.m) return cudaSuccess;
    k_tie_lo<<<grid_for(d.m), 256, 0, s>>>(d.t, d.m, S);
    return cudaGetLastError();
}

// tm_graph_set_labels: vertex labels as given, edge labels permuted from the
// caller's input order into edge-id order (perm[id] = input position).
tm_status set_labels(DeviceGraph &d, const int32_t *vl, const int32_t *el, bool on_device) {
    cudaStream_t s = nullptr;
    const cudaMemcpyKind kind = on_device ? cudaMemcpyDeviceToDevice : cudaMemcpyHostToDevice;
    if (vl && d.n) {
        if (!d.vlab) TM_CUDA_TRY(dmalloc(&d.vlab, (size_t)d.n, s));
        TM_CUDA_TRY(cudaMemcpyAsync(d.vlab, vl, (size_t)d.n * 4, kind, s));
    }
    if (el && d.m) {
        int32_t *tmp = nullptr;
        TM_CUDA_TRY(dmalloc(&tmp, d.m, s));
        cudaError_t e = cudaMemcpyAsync(tmp, el, d.m * 4, kind, s);
        if (e == cudaSuccess && !d.elab) e = dmalloc(&d.elab, d.m, s);
        if (e == cudaSuccess) {
            k_gather_i32<<<grid_for(d.m), 256, 0, s>>>(tmp, d.perm, d.m, d.elab);
            e = cudaGetLastError();
        }
        dev_free(tmp, s);
        TM_CUDA_TRY(e);
    }
    TM_CUDA_TRY(cudaStreamSynchronize(s));
    return TM_OK;
}



cudaError_t build_hrank(const DeviceGraph &d, int var, const uint32_t *H, uint32_t *R, cudaStream_t s,
                        uint4 *W) {
    if (!d.m) return cudaSuccess;
    const uint32_t *rk = d.rank + (size_t)var * d.m;
    const uint32_t *nxr = nullptr;
    uint32_t *nxw = nullptr;
    cudaError_t err = cudaSuccess;
    if (TM_NEXT_IDS && d.nxc) {   // allocated with the graph (build_skip)
        NextIdCache &c = *d.nxc;
        std::lock_guard<std::mutex> lk(c.mu);
        if (c.state[var] == 2) {            // recorded by an earlier query (maybe on another stream)
            err = cudaStreamWaitEvent(s, c.ev[var], 0);
            if (err != cudaSuccess) return err;
            nxr = c.nx[var];
        } else if (c.state[var] == 0) {     // this query records them
            nxw = c.nx[var];
            c.state[var] = 1;
        }                                   // state 1: another query is recording them: neither
    }
    k_hrank<<<grid_for(d.m), 256, 0, s>>>(d.rec, d.skip, rk, H, d.m, R, W, nxr, nxw);
    err = cudaGetLastError();
    if (nxw) {
        std::lock_guard<std::mutex> lk(d.nxc->mu);
        if (err == cudaSuccess) err = cudaEventRecord(d.nxc->ev[var], s);
        d.nxc->state[var] = err == cudaSuccess ? 2 : 1;   // a failed recording is never used
    }
    return err;
}

cudaError_t build_skip(DeviceGraph &d, cudaStream_t s) {
    const uint64_t nskip = (d.nrec + 7) / 8 + 8;   // + a sector of padding for the 8-entry loads
    cudaError_t err = dmalloc(&d.skip, nskip, s);
    if (err != cudaSuccess) return err;
    if (TM_NEXT_IDS && d.m) {
        // the first-record-id cache: allocated here with the graph (one block for
        // the four list variants, filled by the first query that needs each one);
        // (2 GB on C4)
        d.nxc = new NextIdCache();
        const uint64_t per = d.m * (kNx4 ? 4 : kNx2 ? 2 : 1);
        err = dmalloc(&d.nxc->buf, 4 * per, s);
        if (err != cudaSuccess) return err;
        for (int v = 0; v < 4; v++) {
            d.nxc->nx[v] = d.nxc->buf + v * per;
            err = cudaEventCreateWithFlags(&d.nxc->ev[v], cudaEventDisableTiming);
            if (err != cudaSuccess) return err;
        }
    }
    k_skip<<<grid_for(nskip), 256, 0, s>>>(d.rec, d.nrec, nskip, d.skip);
    if (d.n) k_skip_marks<<<grid_for(d.n), 256, 0, s>>>(d.off_out, d.off_in, d.n, d.skip);
    return cudaGetLastError();
}

tm_status graph_create(const uint32_t *src, const uint32_t *dst, const int64_t *t, uint64_t m, uint32_t n,
                       const tm_graph_opts *o, tm_graph **out) {
    NvtxRange nv("tm.graph_create");
    cudaStream_t s = o ? (cudaStream_t)o->stream : nullptr;
    const bool on_dev = o && o->input_on_device;
    tm_graph *g = new (std::nothrow) tm_graph();
    if (!g) return fail(TM_ENOMEM, "host allocation failed");
    cudaGetDevice(&g->device);
    DeviceGraph &d = g->d;
    d.m = m;
    d.n = n;
    uint32_t *isrc = nullptr, *idst = nullptr;
    int64_t *it = nullptr, *keys_tmp = nullptr;
    unsigned long long *flags = nullptr, hflags[3] = {0, 0, 0};
    void *tmp = nullptr;
    size_t tmp_bytes = 0;
    cudaError_t err = cudaSuccess;
    tm_status st = TM_OK;
    std::string what;
#define TRY(x) do { err = (x); if (err != cudaSuccess) { what = #x; goto fail_cuda; } } while (0)
    TRY(dmalloc(&d.src, m, s));
    TRY(dmalloc(&d.dst, m, s));
    TRY(dmalloc(&d.t, m, s));
    TRY(dmalloc(&d.perm, m, s));
    TRY(dmalloc(&d.off_out, (size_t)n + 1, s));
    TRY(dmalloc(&d.off_in, (size_t)n + 1, s));
    d.nrec = 2 * (m + n);
    TRY(dmalloc(&d.rec, d.nrec + 32, s));   // sentinels + padding: warp reads may run 31 records past a sentinel
    TRY(cudaMemsetAsync(d.rec, 0xff, (2 * (m + n) + 32) * sizeof(uint64_t), s));
    TRY(dmalloc(&d.rank, 4 * m, s));
    TRY(dmalloc(&flags, 3, s));
    TRY(cudaMemsetAsync(flags, 0, 3 * sizeof(unsigned long long), s));
    if (!on_dev && m) {
        // Host input, pipelined (DESIGN.md §6 "Graph build"): src/dst are copied
        // straight into place on a copy stream, then t; the CSR is built from
        // src/dst while t is still in flight, on the guess that the input is
        // already in time order (edge id = input position).  t's check then
        // confirms the guess; otherwise the edges are sorted and the CSR is
        // built again (the result is the same either way).
        cudaStream_t cs = nullptr;
        cudaEvent_t ev_sd = nullptr, ev_t = nullptr;
        struct Own {
            cudaStream_t &cs; cudaEvent_t &a, &b;
            ~Own() {   // a failed call may leave copies in flight: they finish before anything is freed
                if (cs) { cudaStreamSynchronize(cs); cudaStreamDestroy(cs); }
                if (a) cudaEventDestroy(a);
                if (b) cudaEventDestroy(b);
            }
        } own{cs, ev_sd, ev_t};
        TRY(cudaStreamCreateWithFlags(&cs, cudaStreamNonBlocking));
        TRY(cudaEventCreateWithFlags(&ev_sd, cudaEventDisableTiming));
        TRY(cudaEventCreateWithFlags(&ev_t, cudaEventDisableTiming));
        TRY(cudaEventRecord(ev_sd, s));            // the allocations above, in stream order
        TRY(cudaStreamWaitEvent(cs, ev_sd, 0));
        TRY(cudaMemcpyAsync(d.src, src, m * 4, cudaMemcpyHostToDevice, cs));
        TRY(cudaMemcpyAsync(d.dst, dst, m * 4, cudaMemcpyHostToDevice, cs));
        TRY(cudaEventRecord(ev_sd, cs));
        TRY(cudaMemcpyAsync(d.t, t, m * 8, cudaMemcpyHostToDevice, cs));
        TRY(cudaEventRecord(ev_t, cs));
        TRY(cudaStreamWaitEvent(s, ev_sd, 0));
        k_validate_ids<<<grid_for(m), 256, 0, s>>>(d.src, d.dst, m, n, flags);
        TRY(cudaGetLastError());
        TRY(cudaMemcpyAsync(hflags, flags, sizeof hflags, cudaMemcpyDeviceToHost, s));
        TRY(cudaStreamSynchronize(s));
        if (hflags[0]) { cudaStreamSynchronize(cs); st = fail(TM_EINVAL, "edge endpoint >= n_vertices"); goto fail_free; }
        k_iota<<<grid_for(m), 256, 0, s>>>(d.perm, m);
        TRY(build_csr(d, s));                        // overlaps the copy of t
        TRY(cudaStreamWaitEvent(s, ev_t, 0));
        k_validate_t<<<grid_for(m), 256, 0, s>>>(d.t, m, flags);
        TRY(cudaGetLastError());
        TRY(cudaMemcpyAsync(hflags, flags, sizeof hflags, cudaMemcpyDeviceToHost, s));
        TRY(cudaStreamSynchronize(s));
        if (hflags[1]) { st = fail(TM_EINVAL, "negative timestamp"); goto fail_free; }
        if (hflags[2]) {   // not in time order: sort below from copies of the input
            TRY(dmalloc(&isrc, m, s)); TRY(dmalloc(&idst, m, s)); TRY(dmalloc(&it, m, s));
            TRY(cudaMemcpyAsync(isrc, d.src, m * 4, cudaMemcpyDeviceToDevice, s));
            TRY(cudaMemcpyAsync(idst, d.dst, m * 4, cudaMemcpyDeviceToDevice, s));
            TRY(cudaMemcpyAsync(it, d.t, m * 8, cudaMemcpyDeviceToDevice, s));
            TRY(cudaMemsetAsync(d.rec, 0xff, (2 * (m + n) + 32) * sizeof(uint64_t), s));
        } else {
            TRY(build_skip(d, s));
            if (TM_PAIR_LEAF || TM_PAIR_NONLEAF || TM_PAIR_BUILD || (o && o->pair_index)) TRY(build_pairs(d, s, o ? o->pair_id_bucket_log2 : 0));
            TRY(cudaStreamSynchronize(s));
            dev_free(flags, s);
            *out = g;
            return TM_OK;
        }
    } else {
        if (on_dev) {
            isrc = const_cast<uint32_t *>(src); idst = const_cast<uint32_t *>(dst); it = const_cast<int64_t *>(t);
        } else {
            TRY(dmalloc(&isrc, m, s)); TRY(dmalloc(&idst, m, s)); TRY(dmalloc(&it, m, s));
        }
        if (m) k_validate<<<grid_for(m), 256, 0, s>>>(isrc, idst, it, m, n, flags);
        TRY(cudaGetLastError());
        TRY(cudaMemcpyAsync(hflags, flags, sizeof hflags, cudaMemcpyDeviceToHost, s));
        TRY(cudaStreamSynchronize(s));
        if (hflags[0]) { st = fail(TM_EINVAL, "edge endpoint >= n_vertices"); goto fail_free; }
        if (hflags[1]) { st = fail(TM_EINVAL, "negative timestamp"); goto fail_free; }
    }
    if (m) k_iota<<<grid_for(m), 256, 0, s>>>(d.perm, m);
    if (hflags[2]) {
        // stable LSD radix sort on t (t >= 0, so its bit pattern orders as u64):
        // ties keep input order -> (t, input position) (reading Q1)
        uint32_t *perm2 = nullptr;
        TRY(dmalloc(&keys_tmp, m, s));
        TRY(dmalloc(&perm2, m, s));
        const uint64_t *kin = reinterpret_cast<const uint64_t *>(it);
        uint64_t *kout = reinterpret_cast<uint64_t *>(keys_tmp);
        TRY(cub::DeviceRadixSort::SortPairs(nullptr, tmp_bytes, kin, kout, d.perm, perm2, (int64_t)m, 0, 64, s));
        TRY(dev_alloc(&tmp, tmp_bytes, s));
        TRY(cub::DeviceRadixSort::SortPairs(tmp, tmp_bytes, kin, kout, d.perm, perm2, (int64_t)m, 0, 64, s));
        std::swap(d.perm, perm2);
        dev_free(perm2, s);
    }
    if (m) k_gather<<<grid_for(m), 256, 0, s>>>(d.perm, isrc, idst, it, m, d.src, d.dst, d.t);
    TRY(cudaGetLastError());
    TRY(build_csr(d, s));
    TRY(build_skip(d, s));
    if (TM_PAIR_LEAF || TM_PAIR_NONLEAF || TM_PAIR_BUILD || (o && o->pair_index)) TRY(build_pairs(d, s, o ? o->pair_id_bucket_log2 : 0));
    TRY(cudaStreamSynchronize(s));
#undef TRY
    if (!on_dev) { dev_free(isrc, s); dev_free(idst, s); dev_free(it, s); }
    dev_free(keys_tmp, s); dev_free(tmp, s); dev_free(flags, s);
    *out = g;
    return TM_OK;
fail_cuda:
    st = fail(err == cudaErrorMemoryAllocation ? TM_ENOMEM : TM_ECUDA, what + ": " + cudaGetErrorString(err));
fail_free:
    cudaStreamSynchronize(s);
    if (!on_dev) { dev_free(isrc, s); dev_free(idst, s); dev_free(it, s); }
    dev_free(keys_tmp, s); dev_free(tmp, s); dev_free(flags, s);
    free_graph(d, s);
    cudaStreamSynchronize(s);
    delete g;
    return st;
}

void graph_destroy(tm_graph *g) {
    if (!g) return;
    int dev = 0;
    cudaGetDevice(&dev);
    cudaSetDevice(g->device);
    cudaDeviceSynchronize();   // no work of any stream may still read the graph
    free_graph(g->d, nullptr);
    // let the frees complete now: a graph built right after this one (on any
    // stream) then reuses the pool's memory instead of growing the pool
    // (measured: e2e steps of 32 ms with occasional 100-600 ms growth spikes)
    cudaStreamSynchronize(nullptr);
    cudaSetDevice(dev);
    delete g;
}

namespace {
std::mutex g_pool_mu;
cudaMemPool_t g_pool[64] = {};
}  // namespace

cudaError_t dev_alloc(void **p, size_t bytes, cudaStream_t s) {
    int dev = 0;
    cudaError_t e = cudaGetDevice(&dev);
    if (e != cudaSuccess) return e;
    cudaMemPool_t pool;
    {
        std::lock_guard<std::mutex> lk(g_pool_mu);
        if (!g_pool[dev]) {
            cudaMemPoolProps props = {};
            props.allocType = cudaMemAllocationTypePinned;
            props.location.type = cudaMemLocationTypeDevice;
            props.location.id = dev;
            e = cudaMemPoolCreate(&g_pool[dev], &props);
            if (e != cudaSuccess) return e;
            uint64_t keep = UINT64_MAX;
            cudaMemPoolSetAttribute(g_pool[dev], cudaMemPoolAttrReleaseThreshold, &keep);
        }
        pool = g_pool[dev];
    }
    return cudaMallocFromPoolAsync(p, bytes, pool, s);
}

void dev_free(void *p, cudaStream_t s) {
    if (p) cudaFreeAsync(p, s);
}

}  // namespace tmg
