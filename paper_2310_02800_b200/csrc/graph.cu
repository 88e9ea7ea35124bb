// Device graph construction: stable order by
// (t, input position), the bidirectional time-sorted CSR of packed 64-bit
// records, and the per-query δ-horizon arrays.
#include <cub/cub.cuh>

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

// records of one direction: edge ids grouped by key vertex, ascending id
__global__ void k_records(const uint32_t *ids, const uint32_t *nbr, uint64_t m, uint64_t *rec) {
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < m; i += (uint64_t)gridDim.x * blockDim.x) {
        uint32_t e = ids[i];
        rec[i] = ((uint64_t)e << 32) | nbr[e];
    }
}

// H_d[e] = max{ j : T[j] <= T[e] + d }  (>= e; m-1 when d = ∞ or saturated).
// The δ-window t' = t_root + δ of Algorithm 1 and the
// fine-grained bound t_prev + δ_i become edge-id limits.
__global__ void k_horizon(const int64_t *__restrict__ T, uint64_t m, int64_t d, uint32_t *__restrict__ H) {
    for (uint64_t e = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; e < m; e += (uint64_t)gridDim.x * blockDim.x) {
        const int64_t te = T[e];
        if (d == TM_DELTA_INF || te > INT64_MAX - d) { H[e] = (uint32_t)(m - 1); continue; }
        const int64_t key = te + d;
        // gallop from e, then binary search: first j > e with T[j] > key
        uint64_t lo = e + 1, step = 1, hi = e + 1;
        while (hi < m && T[hi] <= key) { lo = hi + 1; hi = e + 1 + (step <<= 1) - 1; }
        if (hi > m) hi = m;
        while (lo < hi) {
            uint64_t mid = lo + ((hi - lo) >> 1);
            if (T[mid] > key) hi = mid; else lo = mid + 1;
        }
        H[e] = (uint32_t)(lo - 1);
    }
}

inline unsigned grid_for(uint64_t m) {
    uint64_t b = (m + 255) / 256;
    return (unsigned)std::max<uint64_t>(1, std::min<uint64_t>(b, 148ull * 32));
}

template <class T>
cudaError_t dmalloc(T **p, size_t count) { return cudaMalloc((void **)p, std::max<size_t>(count, 1) * sizeof(T)); }

void free_graph(DeviceGraph &d) {
    cudaFree(d.src); cudaFree(d.dst); cudaFree(d.t); cudaFree(d.perm);
    cudaFree(d.off_out); cudaFree(d.off_in); cudaFree(d.rec);
    d = DeviceGraph{};
}

// one direction of the CSR: sort ids by key vertex (stable, so ids stay
// ascending = chronological inside each vertex), offsets by histogram + scan
cudaError_t build_direction(const uint32_t *key, const uint32_t *nbr, uint64_t m, uint32_t n, uint32_t bias,
                            uint32_t *off, uint64_t *rec, cudaStream_t s) {
    uint32_t *ids_in = nullptr, *ids_out = nullptr, *keys_out = nullptr, *deg = nullptr;
    void *tmp = nullptr;
    size_t tmp_bytes = 0, scan_bytes = 0;
    cudaError_t err;
    int end_bit = 1;
    while (end_bit < 32 && (1ull << end_bit) < (uint64_t)n) end_bit++;
#define TRY(x) do { err = (x); if (err != cudaSuccess) goto done; } while (0)
    TRY(dmalloc(&ids_in, m));
    TRY(dmalloc(&ids_out, m));
    TRY(dmalloc(&keys_out, m));
    TRY(dmalloc(&deg, (size_t)n + 1));
    TRY(cub::DeviceRadixSort::SortPairs(nullptr, tmp_bytes, key, keys_out, ids_in, ids_out, (int64_t)m, 0, end_bit, s));
    TRY(cub::DeviceScan::ExclusiveSum(nullptr, scan_bytes, deg, off, (int64_t)n + 1, s));
    TRY(cudaMalloc(&tmp, std::max(tmp_bytes, scan_bytes)));
    if (m) {
        k_iota<<<grid_for(m), 256, 0, s>>>(ids_in, m);
        TRY(cub::DeviceRadixSort::SortPairs(tmp, tmp_bytes, key, keys_out, ids_in, ids_out, (int64_t)m, 0, end_bit, s));
    }
    TRY(cudaMemsetAsync(deg, 0, ((size_t)n + 1) * 4, s));
    if (m) k_degree<<<grid_for(m), 256, 0, s>>>(key, m, deg);
    TRY(cub::DeviceScan::ExclusiveSum(tmp, scan_bytes, deg, off, (int64_t)n + 1, s));
    if (bias) k_bias<<<grid_for((uint64_t)n + 1), 256, 0, s>>>(off, n + 1, bias);
    if (m) k_records<<<grid_for(m), 256, 0, s>>>(ids_out, nbr, m, rec);
    TRY(cudaGetLastError());
    TRY(cudaStreamSynchronize(s));
done:
#undef TRY
    cudaFree(ids_in); cudaFree(ids_out); cudaFree(keys_out); cudaFree(deg); cudaFree(tmp);
    return err;
}

}  // namespace

cudaError_t build_horizon(const DeviceGraph &d, int64_t delta, uint32_t *H, cudaStream_t s) {
    if (d.m) k_horizon<<<grid_for(d.m), 256, 0, s>>>(d.t, d.m, delta, H);
    return cudaGetLastError();
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
    TRY(dmalloc(&d.src, m));
    TRY(dmalloc(&d.dst, m));
    TRY(dmalloc(&d.t, m));
    TRY(dmalloc(&d.perm, m));
    TRY(dmalloc(&d.off_out, (size_t)n + 1));
    TRY(dmalloc(&d.off_in, (size_t)n + 1));
    TRY(dmalloc(&d.rec, 2 * m));
    TRY(dmalloc(&flags, 3));
    if (on_dev) {
        isrc = const_cast<uint32_t *>(src); idst = const_cast<uint32_t *>(dst); it = const_cast<int64_t *>(t);
    } else {
        TRY(dmalloc(&isrc, m)); TRY(dmalloc(&idst, m)); TRY(dmalloc(&it, m));
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
        TRY(dmalloc(&keys_tmp, m));
        TRY(dmalloc(&perm2, m));
        const uint64_t *kin = reinterpret_cast<const uint64_t *>(it);
        uint64_t *kout = reinterpret_cast<uint64_t *>(keys_tmp);
        TRY(cub::DeviceRadixSort::SortPairs(nullptr, tmp_bytes, kin, kout, d.perm, perm2, (int64_t)m, 0, 64, s));
        TRY(cudaMalloc(&tmp, tmp_bytes));
        TRY(cub::DeviceRadixSort::SortPairs(tmp, tmp_bytes, kin, kout, d.perm, perm2, (int64_t)m, 0, 64, s));
        std::swap(d.perm, perm2);
        TRY(cudaStreamSynchronize(s));
        cudaFree(perm2);
    }
    if (m) k_gather<<<grid_for(m), 256, 0, s>>>(d.perm, isrc, idst, it, m, d.src, d.dst, d.t);
    TRY(cudaGetLastError());
    TRY(build_direction(d.src, d.dst, m, n, 0, d.off_out, d.rec, s));
    TRY(build_direction(d.dst, d.src, m, n, (uint32_t)m, d.off_in, d.rec + m, s));
    TRY(cudaStreamSynchronize(s));
#undef TRY
    if (!on_dev) { cudaFree(isrc); cudaFree(idst); cudaFree(it); }
    cudaFree(keys_tmp); cudaFree(tmp); cudaFree(flags);
    *out = g;
    return TM_OK;
fail_cuda:
    st = fail(err == cudaErrorMemoryAllocation ? TM_ENOMEM : TM_ECUDA, what + ": " + cudaGetErrorString(err));
fail_free:
    cudaStreamSynchronize(s);
    if (!on_dev) { cudaFree(isrc); cudaFree(idst); cudaFree(it); }
    cudaFree(keys_tmp); cudaFree(tmp); cudaFree(flags);
    free_graph(d);
    delete g;
    return st;
}

void graph_destroy(tm_graph *g) {
    if (!g) return;
    int dev = 0;
    cudaGetDevice(&dev);
    cudaSetDevice(g->device);
    free_graph(g->d);
    cudaSetDevice(dev);
    delete g;
}

}  // namespace tmg
