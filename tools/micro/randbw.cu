// Random-access bandwidth probe (B200): N independent gathers of G bytes
// (G = 4, 16, 32, 64) at hashed positions of a 1 GiB array, one coalesced 16 B
// write per gather — the access pattern of k_hrank (one random 32 B record
// sector per edge + a coalesced descriptor write).  Reports gathers/s and the
// implied bytes/s.  nvcc -O3 -gencode arch=compute_100a,code=sm_100a randbw.cu -o randbw
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ uint64_t mix(uint64_t x) {
    x ^= x >> 33; x *= 0xff51afd7ed558ccdull; x ^= x >> 33; x *= 0xc4ceb9fe1a85ec53ull; x ^= x >> 33;
    return x;
}

template <int G>
__global__ void gather(const uint4 *__restrict__ a, uint64_t nvec, uint64_t n, uint4 *__restrict__ out) {
    const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n; i += stride * 4) {
        uint4 acc[4];
#pragma unroll
        for (int u = 0; u < 4; u++) {
            const uint64_t j = i + u * stride;
            const uint64_t p = (mix(j) % (nvec / 4)) * 4;   // 64 B aligned slot
            uint4 v = make_uint4(0, 0, 0, 0);
            if (j < n) {
                if (G == 4) v.x = reinterpret_cast<const uint32_t *>(a + p)[0];
                else {
                    v = __ldg(a + p);
                    if (G >= 32) { uint4 w = __ldg(a + p + 1); v.x ^= w.x; v.y ^= w.y; }
                    if (G >= 64) { uint4 w = __ldg(a + p + 2), z = __ldg(a + p + 3); v.z ^= w.z ^ z.z; v.w ^= w.w ^ z.w; }
                }
            }
            acc[u] = v;
        }
#pragma unroll
        for (int u = 0; u < 4; u++) {
            const uint64_t j = i + u * stride;
            if (j < n) out[j] = acc[u];
        }
    }
}

template <int G>
void run(const uint4 *a, uint64_t nvec, uint64_t n, uint4 *out) {
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0); cudaEventCreate(&e1);
    for (int rep = 0; rep < 4; rep++) {
        cudaEventRecord(e0);
        gather<G><<<148 * 16, 256>>>(a, nvec, n, out);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
    }
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    printf("{\"gather_bytes\": %d, \"n\": %llu, \"ms\": %.4f, \"Ggathers_per_s\": %.3f, \"gather_GBps\": %.1f, "
           "\"write_GBps\": %.1f}\n", G, (unsigned long long)n, ms, n / ms / 1e6, (double)n * G / ms / 1e6,
           (double)n * 16 / ms / 1e6);
}

int main() {
    const uint64_t bytes = 1ull << 30, nvec = bytes / 16, n = 63497050;
    uint4 *a, *out;
    cudaMalloc(&a, bytes);
    cudaMalloc(&out, n * 16);
    cudaMemset(a, 1, bytes);
    run<4>(a, nvec, n, out);
    run<16>(a, nvec, n, out);
    run<32>(a, nvec, n, out);
    run<64>(a, nvec, n, out);
    return 0;
}
