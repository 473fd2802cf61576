// Ceiling for the dedup probe pattern: random 32-byte-sector reads from a table much
// larger than L2, U independent loads in flight per thread.  Prints sectors/ns and GB/s.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/rpb tools/random_probe_bench.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
template <int U>
__global__ void probe(const uint4* __restrict__ table, uint64_t mask, uint64_t n_per_thread, uint32_t* out) {
    uint32_t acc = 0;
    uint64_t x = (blockIdx.x * (uint64_t)blockDim.x + threadIdx.x) * 0x9E3779B97F4A7C15ull + 12345;
    for (uint64_t i = 0; i < n_per_thread; i += U) {
        uint4 v[U];
#pragma unroll
        for (int u = 0; u < U; ++u) {
            x ^= x << 13; x ^= x >> 7; x ^= x << 17;
            v[u] = __ldcg(table + ((x & mask) << 1));  // 32-byte slots, read the first 16 bytes
        }
#pragma unroll
        for (int u = 0; u < U; ++u) acc += v[u].x ^ v[u].w;
    }
    if (acc == 0x12345678u) out[0] = acc;
}
template <int U>
void run(const uint4* t, uint64_t slots, int blocks, int threads, uint32_t* out) {
    uint64_t per = 4096;
    cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
    probe<U><<<blocks, threads>>>(t, slots - 1, 256, out);
    cudaEventRecord(a);
    probe<U><<<blocks, threads>>>(t, slots - 1, per, out);
    cudaEventRecord(b); cudaEventSynchronize(b);
    float ms; cudaEventElapsedTime(&ms, a, b);
    double n = (double)blocks * threads * per;
    printf("slots=%llu (%.0f MB) U=%d blocks=%d thr=%d: %.2f sectors/ns  %.0f GB/s (32B/probe)\n",
           (unsigned long long)slots, slots * 32.0 / 1e6, U, blocks, threads, n / (ms * 1e6), n * 32 / (ms * 1e6));
}
int main() {
    uint32_t* out; cudaMalloc(&out, 4);
    for (uint64_t slots : {1ull << 22, 1ull << 26, 1ull << 28}) {
        uint4* t; cudaMalloc(&t, slots * 32); cudaMemset(t, 1, slots * 32);
        run<1>(t, slots, 148 * 8, 256, out);
        run<2>(t, slots, 148 * 8, 256, out);
        run<4>(t, slots, 148 * 8, 256, out);
        run<8>(t, slots, 148 * 8, 256, out);
        run<16>(t, slots, 148 * 4, 256, out);
        run<4>(t, slots, 148 * 2, 256, out);
        cudaFree(t);
    }
    return 0;
}
