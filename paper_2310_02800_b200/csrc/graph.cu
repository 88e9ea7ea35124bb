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

__global__ void k_degree(const uint32_t *v, uint64_t m, uint32_t *deg) {
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < m; i += (uint64_t)gridDim.x * blockDim.x)
        atomicAdd(deg + v[i], 1u);
}

__global__ void k_bias(uint32_t *off, uint32_t n1, uint32_t bias) {
    for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < n1; i += gridDim.x * blockDim.x) off[i] += bias;
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
constexpr int kHStage = 6 * kHB;    // staged timestamps (24 KB at 512)

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

// H at the first and last edge of every kHB block (one thread each)
__global__ void k_horizon_ends(const int64_t *__restrict__ T, uint64_t m, int64_t d, uint64_t *__restrict__ ends) {
    const uint64_t nb = (m + kHB - 1) / kHB;
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < 2 * nb; i += (uint64_t)gridDim.x * blockDim.x) {
        const uint64_t b = i >> 1;
        const uint64_t e = (i & 1) ? min((b + 1) * kHB, m) - 1 : b * kHB;
        ends[i] = horizon_one(T, m, d, e);
    }
}

// kHB / kHEpt threads per block, kHEpt edges each (strided for coalescing):
// the kHEpt branch-free binary searches of a thread are independent, so their
// shared-memory loads overlap (the kernel is bound by that latency chain).
#ifndef TM_HORIZON_EPT
#define TM_HORIZON_EPT 4
#endif
constexpr int kHEpt = TM_HORIZON_EPT;
constexpr int kHThreads = kHB / kHEpt;

__global__ void __launch_bounds__(kHThreads) k_horizon(const int64_t *__restrict__ T, uint64_t m, int64_t d,
                                                       const uint64_t *__restrict__ ends, uint32_t *__restrict__ H) {
    __shared__ int64_t st[kHStage];
    const uint64_t e0 = (uint64_t)blockIdx.x * kHB;
    const uint64_t elast = min(e0 + kHB, m) - 1;
    const uint64_t lo = ends[2 * blockIdx.x], hi = ends[2 * blockIdx.x + 1];   // answers lie in [lo, hi]
    const uint64_t span = hi - lo + 1;
    int64_t te[kHEpt];
#pragma unroll
    for (int j = 0; j < kHEpt; j++) {
        const uint64_t e = e0 + threadIdx.x + (uint64_t)j * kHThreads;
        te[j] = e <= elast ? T[e] : 0;
    }
    if (span <= kHStage) {
        for (uint64_t i = threadIdx.x; i < span; i += kHThreads) st[i] = T[lo + i];
        __syncthreads();
        // last index with st[idx] <= key; st[0] = T[H(e0)] <= key for every e >= e0
        uint32_t base[kHEpt];
        int64_t key[kHEpt];
#pragma unroll
        for (int j = 0; j < kHEpt; j++) {
            base[j] = 0;
            key[j] = (d == TM_DELTA_INF || te[j] > INT64_MAX - d) ? INT64_MAX : te[j] + d;
        }
        for (uint32_t len = (uint32_t)span; len > 1;) {
            const uint32_t half = len >> 1;
#pragma unroll
            for (int j = 0; j < kHEpt; j++)
                if (st[base[j] + half] <= key[j]) base[j] += half;
            len -= half;
        }
#pragma unroll
        for (int j = 0; j < kHEpt; j++) {
            const uint64_t e = e0 + threadIdx.x + (uint64_t)j * kHThreads;
            if (e <= elast) H[e] = (uint32_t)(key[j] == INT64_MAX ? m - 1 : lo + base[j]);
        }
    } else {
#pragma unroll
        for (int j = 0; j < kHEpt; j++) {
            const uint64_t e = e0 + threadIdx.x + (uint64_t)j * kHThreads;
            if (e <= elast) H[e] = (uint32_t)horizon_one(T, m, d, e);
        }
    }
}

// Both CSR directions and the rank arrays from one stable sort of the 2m
// (vertex, edge) incidences: entry 2e is e's out-incidence at src(e), entry
// 2e+1 its in-incidence at dst(e).  A stable sort by vertex lists, for every
// vertex, all edges touching it in id (= time) order; a scan of "is an
// out-incidence" flags then counts, at every entry, the out- and in-edges of
// that vertex that come earlier — exactly the list positions and the ranks.
__global__ void k_incidences(const uint32_t *src, const uint32_t *dst, uint64_t m, uint32_t *key, uint32_t *val) {
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < 2 * m; i += (uint64_t)gridDim.x * blockDim.x) {
        const uint64_t e = i >> 1;
        key[i] = (i & 1) ? dst[e] : src[e];
        val[i] = (uint32_t)i;
    }
}

__global__ void k_outflag(const uint32_t *val, uint64_t n2, uint32_t *flag) {
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n2; i += (uint64_t)gridDim.x * blockDim.x)
        flag[i] = (val[i] & 1u) ? 0u : 1u;
}

// off_out / off_in hold the sentinel-adjusted list starts (plain offset + v,
// in-lists further shifted by m + n); the plain offsets are recovered here.
// Records go to rec[] in place (consecutive incidences of a vertex are
// consecutive positions); the two rank values of the incidence go to rk[i]
// in incidence order and reach rank[] through a radix sort by incidence id
// (k_rank_from_sorted): scattering them directly as 4-byte random writes
// measured 12 ms of a 21 ms build on C4.
__global__ void k_scatter_csr(const uint32_t *key, const uint32_t *val, const uint32_t *outb, const uint32_t *src,
                              const uint32_t *dst, const uint32_t *off_out, const uint32_t *off_in, uint64_t m,
                              uint32_t n, uint64_t *rec, unsigned long long *rk) {
    const uint32_t split = (uint32_t)(m + n);
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < 2 * m; i += (uint64_t)gridDim.x * blockDim.x) {
        const uint32_t v = key[i], ent = val[i], e = ent >> 1;
        const uint32_t so = off_out[v], si = off_in[v];                 // list starts in rec
        const uint64_t seg = (uint64_t)(so - v) + (si - split - v);      // first incidence of v
        const uint32_t ob = outb[i] - outb[seg];                        // out-incidences of v before i
        const uint32_t ib = (uint32_t)(i - seg) - ob;                   // in-incidences of v before i
        uint32_t a, b;
        if ((ent & 1u) == 0) {            // e in OUT(v), v = src(e)
            const uint32_t pos = so + ob;
            const uint32_t w = dst[e];
            rec[pos] = ((uint64_t)e << 32) | w;
            a = pos + 1;                          // var 0: OUT(src e)
            b = si + ib + (v == w ? 1u : 0u);     // var 1: IN(src e), ids <= e
        } else {                          // e in IN(v), v = dst(e)
            const uint32_t pos = si + ib;
            rec[pos] = ((uint64_t)e << 32) | src[e];
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

// plain exclusive-scan offsets -> sentinel-adjusted list starts
__global__ void k_adjust_offsets(uint32_t *off_out, uint32_t *off_in, uint32_t n, uint64_t m) {
    for (uint32_t v = blockIdx.x * blockDim.x + threadIdx.x; v <= n; v += gridDim.x * blockDim.x) {
        off_out[v] += v;
        off_in[v] += (uint32_t)(m + n) + v;
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
                    (void *)d.rec, (void *)d.rank, (void *)d.prec, (void *)d.ptab, (void *)d.pbits,
                    (void *)d.vlab, (void *)d.elab})
        dev_free(q, s);
    d = DeviceGraph{};
}

// Offsets (histogram + scan per direction), then the merged incidence sort.
cudaError_t build_csr(DeviceGraph &d, cudaStream_t s) {
    const uint64_t m = d.m;
    const uint32_t n = d.n;
    uint32_t *deg = nullptr, *key = nullptr, *val = nullptr, *kout = nullptr, *vout = nullptr, *flag = nullptr;
    unsigned long long *rk = nullptr, *rk2 = nullptr;
    void *tmp = nullptr;
    size_t sort_bytes = 0, scan_bytes = 0, scan2_bytes = 0, sort2_bytes = 0;
    cudaError_t err;
    int end_bit = 1;
    while (end_bit < 32 && (1ull << end_bit) < (uint64_t)n) end_bit++;
    const uint64_t n2 = 2 * m;
    int end_bit2 = 1;   // incidence ids 2e + dir < 2m
    while (end_bit2 < 32 && (1ull << end_bit2) < n2) end_bit2++;
#define TRY(x) do { err = (x); if (err != cudaSuccess) goto done; } while (0)
    TRY(dmalloc(&deg, 2 * ((size_t)n + 1), s));
    TRY(dmalloc(&key, n2 + 1, s));
    TRY(dmalloc(&val, n2, s));
    TRY(dmalloc(&kout, n2, s));
    TRY(dmalloc(&vout, n2, s));
    TRY(dmalloc(&flag, n2 + 1, s));
    TRY(cub::DeviceRadixSort::SortPairs(nullptr, sort_bytes, key, kout, val, vout, (int64_t)n2, 0, end_bit, s));
    TRY(cub::DeviceScan::ExclusiveSum(nullptr, scan_bytes, deg, d.off_out, (int64_t)n + 1, s));
    TRY(cub::DeviceScan::ExclusiveSum(nullptr, scan2_bytes, flag, key, (int64_t)n2 + 1, s));
    TRY(dmalloc(&rk, n2, s));
    TRY(dmalloc(&rk2, n2, s));
    TRY(cub::DeviceRadixSort::SortPairs(nullptr, sort2_bytes, vout, val, rk, rk2, (int64_t)n2, 0, end_bit2, s));
    TRY(dev_alloc(&tmp, std::max(std::max(sort_bytes, sort2_bytes), std::max(scan_bytes, scan2_bytes)), s));
    TRY(cudaMemsetAsync(deg, 0, 2 * ((size_t)n + 1) * 4, s));
    if (m) {
        k_degree<<<grid_for(m), 256, 0, s>>>(d.src, m, deg);
        k_degree<<<grid_for(m), 256, 0, s>>>(d.dst, m, deg + n + 1);
    }
    TRY(cub::DeviceScan::ExclusiveSum(tmp, scan_bytes, deg, d.off_out, (int64_t)n + 1, s));
    TRY(cub::DeviceScan::ExclusiveSum(tmp, scan_bytes, deg + n + 1, d.off_in, (int64_t)n + 1, s));
    k_adjust_offsets<<<grid_for((uint64_t)n + 1), 256, 0, s>>>(d.off_out, d.off_in, n, m);
    k_sentinels<<<grid_for(n), 256, 0, s>>>(d.off_out, d.off_in, n, d.rec);
    if (m) {
        k_incidences<<<grid_for(n2), 256, 0, s>>>(d.src, d.dst, m, key, val);
        TRY(cub::DeviceRadixSort::SortPairs(tmp, sort_bytes, key, kout, val, vout, (int64_t)n2, 0, end_bit, s));
        k_outflag<<<grid_for(n2), 256, 0, s>>>(vout, n2, flag);
        TRY(cudaMemsetAsync(flag + n2, 0, 4, s));
        TRY(cub::DeviceScan::ExclusiveSum(tmp, scan2_bytes, flag, key, (int64_t)n2 + 1, s));  // key: free after the sort
        k_scatter_csr<<<grid_for(n2), 256, 0, s>>>(kout, vout, key, d.src, d.dst, d.off_out, d.off_in, m, n,
                                                   d.rec, rk);
        // back to incidence order (val is free after the first sort)
        TRY(cub::DeviceRadixSort::SortPairs(tmp, sort2_bytes, vout, val, rk, rk2, (int64_t)n2, 0, end_bit2, s));
        k_rank_from_sorted<<<grid_for(n2), 256, 0, s>>>(rk2, m, d.rank);
    }
    TRY(cudaGetLastError());
    TRY(cudaStreamSynchronize(s));
done:
#undef TRY
    for (void *q : {(void *)deg, (void *)key, (void *)val, (void *)kout, (void *)vout, (void *)flag, (void *)rk,
                    (void *)rk2, tmp})
        dev_free(q, s);
    return err;
}

// Pair index: stable radix sort of the edges by (src, dst), distinct pairs
// counted, then inserted into the hash table.
cudaError_t build_pairs(DeviceGraph &d, cudaStream_t s) {
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
    TRY(cudaGetLastError());
    TRY(cudaStreamSynchronize(s));
done:
#undef TRY
    for (void *q : {(void *)key, (void *)skey, (void *)val, (void *)cnt, tmp}) dev_free(q, s);
    return err;
}

}  // namespace

size_t horizon_scratch_words(uint64_t m) { return 2 * ((m + kHB - 1) / kHB) + 1; }

// H_delta for every edge: two launches (block ends, then the staged search).
// scratch: horizon_scratch_words(m) u64 of device memory.
cudaError_t build_horizon(const DeviceGraph &d, int64_t delta, uint32_t *H, uint64_t *scratch, cudaStream_t s) {
    if (!d.m) return cudaSuccess;
    const uint64_t nb = (d.m + kHB - 1) / kHB;
    k_horizon_ends<<<grid_for(2 * nb), 256, 0, s>>>(d.t, d.m, delta, scratch);
    k_horizon<<<(unsigned)nb, kHThreads, 0, s>>>(d.t, d.m, delta, scratch, H);
    return cudaGetLastError();
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
// window end of edge e when it lies beyond the first sector: gallop from
// a (the first unread position), capped at the list's sentinel
#ifndef TM_HR_STEP0
#define TM_HR_STEP0 4   // first gallop step (records)
#endif
__device__ __noinline__ uint32_t hrank_long(const uint64_t *__restrict__ rec, const uint32_t *__restrict__ vtx,
                                            const uint32_t *__restrict__ offs, uint64_t e, uint32_t a, uint32_t lim) {
    const uint32_t last = __ldg(offs + vtx[e] + 1) - 1;
    uint32_t lo = a, step = TM_HR_STEP0, hi = min(lo + TM_HR_STEP0 - 1, last);
    while ((uint32_t)(__ldg(rec + hi) >> 32) <= lim) {
        lo = hi + 1;
        step <<= 1;
        hi = min(lo + step - 1, last);
    }
    while (lo < hi) {   // first id > lim in [lo, hi]; rec[hi] qualifies
        const uint32_t mid = lo + ((hi - lo) >> 1);
        if ((uint32_t)(__ldg(rec + mid) >> 32) > lim) hi = mid;
        else lo = mid + 1;
    }
    return lo;
}

#ifndef TM_HR_UNROLL
#define TM_HR_UNROLL 4
#endif
constexpr int kHrUnroll = TM_HR_UNROLL;   // edges per thread in flight (independent load chains)

// Warp-cooperative long path (TM_HRANK_WARP_LONG): the lanes whose window
// runs past the first sector are served one at a time by the whole warp,
// 32 records per coalesced load, up to kHrWarpIters loads, then the gallop.
// Must be reached by all 32 lanes (no lane may have left the loop).
#ifndef TM_HRANK_2PHASE
#define TM_HRANK_2PHASE 0   // measured slower: 4.71 vs 2.56 ms (profiles/r01_experiments.md)
#endif
#ifndef TM_HRANK_WARP_LONG
#define TM_HRANK_WARP_LONG 0   // measured slower: 3.86 vs 2.66 ms (profiles/r01_experiments.md)
#endif
constexpr int kHrWarpIters = 4;
__device__ __forceinline__ uint32_t hrank_long_warp(const uint64_t *__restrict__ rec, const uint32_t *__restrict__ vtx,
                                                    const uint32_t *__restrict__ offs, uint64_t e, uint32_t a,
                                                    uint32_t lim, uint32_t ans) {
    const int lane = threadIdx.x & 31;
    unsigned need = __ballot_sync(0xffffffffu, ans == 0xFFFFFFFFu);
    while (need) {
        const int src = __ffs(need) - 1;
        need &= need - 1;
        const uint64_t es = __shfl_sync(0xffffffffu, e, src);
        const uint32_t as = __shfl_sync(0xffffffffu, a, src), ls = __shfl_sync(0xffffffffu, lim, src);
        const uint32_t last = __ldg(offs + vtx[es] + 1) - 1;   // the list's sentinel
        uint32_t res = 0xFFFFFFFFu, pos = as;
        for (int it = 0; it < kHrWarpIters && res == 0xFFFFFFFFu; it++, pos += 32) {
            const uint32_t q = pos + lane;
            const bool over = q > last || (uint32_t)(__ldg(rec + q) >> 32) > ls;
            const unsigned m = __ballot_sync(0xffffffffu, over);
            if (m) res = pos + __ffs(m) - 1;
        }
        if (res == 0xFFFFFFFFu && lane == src) res = hrank_long(rec, vtx, offs, es, pos, ls);
        if (lane == src) ans = res;
    }
    return ans;
}

// R: window-end ranks (u32 per edge), or W: window descriptors {start, end,
// H[e], 0} (uint4 per edge) when W != nullptr
__global__ void __launch_bounds__(256) k_hrank(const uint64_t *__restrict__ rec, const uint32_t *__restrict__ rank,
                                               const uint32_t *__restrict__ vtx, const uint32_t *__restrict__ offs,
                                               const uint32_t *__restrict__ H, uint64_t m, uint32_t *__restrict__ R,
                                               uint4 *__restrict__ W, uint32_t *__restrict__ qe,
                                               unsigned long long *__restrict__ qn) {
    const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
    // warp-uniform trip count (the warp long path needs all 32 lanes)
    const uint64_t lane0 = (uint64_t)blockIdx.x * blockDim.x + (threadIdx.x & ~31u);
    for (uint64_t w0 = lane0; w0 < m; w0 += stride * kHrUnroll) {
        const uint64_t e0 = w0 + (threadIdx.x & 31u);
        uint32_t lim[kHrUnroll], b[kHrUnroll];
        ulonglong2 x0[kHrUnroll], x1[kHrUnroll];
#pragma unroll
        for (int u = 0; u < kHrUnroll; u++) {
            const uint64_t e = e0 + u * stride;
            lim[u] = e < m ? H[e] : 0u;
            b[u] = e < m ? rank[e] : 0u;   // first record after e
        }
        // the aligned 32-byte sector (4 records) holding the window start:
        // windows are δ_i-short, so it usually holds the end too
#pragma unroll
        for (int u = 0; u < kHrUnroll; u++) {
            const ulonglong2 *v = reinterpret_cast<const ulonglong2 *>(rec + (b[u] & ~3u));
            x0[u] = __ldg(v);
            x1[u] = __ldg(v + 1);
        }
#pragma unroll
        for (int u = 0; u < kHrUnroll; u++) {
            const uint64_t e = e0 + u * stride;
#if !TM_HRANK_WARP_LONG && !TM_HRANK_2PHASE
            if (e >= m) break;
#endif
            const uint32_t a = b[u] & ~3u;
            const uint32_t id[4] = {(uint32_t)(x0[u].x >> 32), (uint32_t)(x0[u].y >> 32), (uint32_t)(x1[u].x >> 32),
                                    (uint32_t)(x1[u].y >> 32)};
            uint32_t ans = 0xFFFFFFFFu;
#pragma unroll
            for (int k = 3; k >= 0; --k)
                if (a + k >= b[u] && id[k] > lim[u]) ans = a + k;
#if TM_HRANK_WARP_LONG
            if (e >= m) ans = 0;   // no edge: not a long-path request
            ans = hrank_long_warp(rec, vtx, offs, e, a + 4, lim[u], ans);
            if (e >= m) continue;
#elif TM_HRANK_2PHASE
            {   // long windows go to a queue for k_hrank_long (warp-aggregated append)
                const bool lng = e < m && ans == 0xFFFFFFFFu;
                const unsigned lm = __ballot_sync(0xffffffffu, lng);
                if (lm) {
                    const int lane = threadIdx.x & 31;
                    unsigned long long base = 0;
                    if (lane == __ffs(lm) - 1) base = atomicAdd(qn, (unsigned long long)__popc(lm));
                    base = __shfl_sync(0xffffffffu, base, __ffs(lm) - 1);
                    if (lng) qe[base + __popc(lm & ((1u << lane) - 1u))] = (uint32_t)e;
                }
            }
            if (e >= m) continue;
#else
            if (ans == 0xFFFFFFFFu) ans = hrank_long(rec, vtx, offs, e, a + 4, lim[u]);
#endif
            if (W) W[e] = make_uint4(b[u], ans, lim[u], 0u);
            else R[e] = ans;
        }
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

namespace {
// Second phase (TM_HRANK_2PHASE): the queued edges whose window runs past the
// first sector, one per lane, all lanes galloping (no lane waits for a
// neighbour's long window as in the first phase).
__global__ void __launch_bounds__(256) k_hrank_long(const uint64_t *__restrict__ rec,
                                                    const uint32_t *__restrict__ rank,
                                                    const uint32_t *__restrict__ vtx,
                                                    const uint32_t *__restrict__ offs,
                                                    const uint32_t *__restrict__ H, const uint32_t *__restrict__ qe,
                                                    const unsigned long long *__restrict__ qn,
                                                    uint32_t *__restrict__ R, uint4 *__restrict__ W) {
    const unsigned long long n = *qn;
    for (unsigned long long i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n;
         i += (uint64_t)gridDim.x * blockDim.x) {
        const uint32_t e = qe[i];
        const uint32_t ans = hrank_long(rec, vtx, offs, e, (rank[e] & ~3u) + 4, H[e]);
        if (W) reinterpret_cast<uint32_t *>(W)[4 * (uint64_t)e + 1] = ans;
        else R[e] = ans;
    }
}
}  // namespace

cudaError_t build_hrank(const DeviceGraph &d, int var, const uint32_t *H, uint32_t *R, cudaStream_t s,
                        uint4 *W) {
    if (!d.m) return cudaSuccess;
    const uint32_t *rk = d.rank + (size_t)var * d.m, *vtx = var < 2 ? d.src : d.dst;
    const uint32_t *offs = (var & 1) ? d.off_in : d.off_out;
    if (!TM_HRANK_2PHASE) {
        k_hrank<<<grid_for(d.m), 256, 0, s>>>(d.rec, rk, vtx, offs, H, d.m, R, W, nullptr, nullptr);
        return cudaGetLastError();
    }
    void *q = nullptr;
    cudaError_t err = dev_alloc(&q, d.m * sizeof(uint32_t) + 16, s);
    if (err != cudaSuccess) return err;
    unsigned long long *qn = (unsigned long long *)q;
    uint32_t *qe = (uint32_t *)((char *)q + 16);
    err = cudaMemsetAsync(qn, 0, sizeof *qn, s);
    if (err == cudaSuccess) {
        k_hrank<<<grid_for(d.m), 256, 0, s>>>(d.rec, rk, vtx, offs, H, d.m, R, W, qe, qn);
        k_hrank_long<<<grid_for(d.m), 256, 0, s>>>(d.rec, rk, vtx, offs, H, qe, qn, R, W);
        err = cudaGetLastError();
    }
    dev_free(q, s);
    return err;
}

tm_status graph_create(const uint32_t *src, const uint32_t *dst, const int64_t *t, uint64_t m, uint32_t n,
                       const tm_graph_opts *o, tm_graph **out) {
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
    TRY(dmalloc(&d.rec, 2 * (m + n) + 32, s));   // sentinels + padding: warp reads may run 31 records past a sentinel
    TRY(cudaMemsetAsync(d.rec, 0xff, (2 * (m + n) + 32) * sizeof(uint64_t), s));
    TRY(dmalloc(&d.rank, 4 * m, s));
    TRY(dmalloc(&flags, 3, s));
    if (on_dev) {
        isrc = const_cast<uint32_t *>(src); idst = const_cast<uint32_t *>(dst); it = const_cast<int64_t *>(t);
    } else {
        TRY(dmalloc(&isrc, m, s)); TRY(dmalloc(&idst, m, s)); TRY(dmalloc(&it, m, s));
        if (m) {
            TRY(cudaMemcpyAsync(isrc, src, m * 4, cudaMemcpyHostToDevice, s));
            TRY(cudaMemcpyAsync(idst, dst, m * 4, cudaMemcpyHostToDevice, s));
            TRY(cudaMemcpyAsync(it, t, m * 8, cudaMemcpyHostToDevice, s));
        }
    }
    TRY(cudaMemsetAsync(flags, 0, 3 * sizeof(unsigned long long), s));
    if (m) k_validate<<<grid_for(m), 256, 0, s>>>(isrc, idst, it, m, n, flags);
    TRY(cudaGetLastError());
    TRY(cudaMemcpyAsync(hflags, flags, sizeof hflags, cudaMemcpyDeviceToHost, s));
    TRY(cudaStreamSynchronize(s));
    if (hflags[0]) { st = fail(TM_EINVAL, "edge endpoint >= n_vertices"); goto fail_free; }
    if (hflags[1]) { st = fail(TM_EINVAL, "negative timestamp"); goto fail_free; }
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
    if (TM_PAIR_LEAF || TM_PAIR_NONLEAF) TRY(build_pairs(d, s));
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
