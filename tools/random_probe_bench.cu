// Ceiling for the dedup probe pattern: random 32-byte-slot reads (one 256-bit load each) from a
// table far larger than L2, U independent loads in flight per thread, for several table sizes and
// occupancies.  Prints probes/ns.  This is the denominator the direct kernel's probe rate should be
// compared with (the HBM copy bandwidth is not: every probe moves one sector of a random DRAM page).
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/random_probe_bench tools/random_probe_bench.cu
#include <cstdio>
#include <cstdint>
#include <cstdlib>
#include <cuda_runtime.h>
typedef unsigned long long u64;

__device__ __forceinline__ void ld256(const void* p, uint4& a, uint4& b) {
    asm volatile("ld.relaxed.gpu.global.v8.u32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                 : "=r"(a.x), "=r"(a.y), "=r"(a.z), "=r"(a.w), "=r"(b.x), "=r"(b.y), "=r"(b.z), "=r"(b.w) : "l"(p) : "memory");
}

template <int U>
__global__ void __launch_bounds__(128) probe(const uint4* __restrict__ table, u64 mask, u64 n_per_thread, uint32_t* out) {
    uint32_t acc = 0;
    u64 x = (blockIdx.x * (u64)blockDim.x + threadIdx.x) * 0x9E3779B97F4A7C15ull + 12345;
    for (u64 i = 0; i < n_per_thread; i += U) {
        uint4 a[U], b[U];
#pragma unroll
        for (int u = 0; u < U; ++u) {
            x ^= x << 13; x ^= x >> 7; x ^= x << 17;
            const u64 h = (x * 0xD6E8FEB86659FD93ull) >> 20;
            ld256(table + ((h & mask) << 1), a[u], b[u]);
        }
#pragma unroll
        for (int u = 0; u < U; ++u) acc += a[u].x ^ b[u].w;
    }
    if (acc == 0x12345678u) out[0] = acc;
}

template <int U>
void run(const uint4* t, u64 slots, int ctas_per_sm, uint32_t* out) {
    const int blocks = 148 * ctas_per_sm, threads = 128;
    const u64 per = 2048;
    cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
    probe<U><<<blocks, threads>>>(t, slots - 1, 256, out);
    cudaEventRecord(a);
    probe<U><<<blocks, threads>>>(t, slots - 1, per, out);
    cudaEventRecord(b); cudaEventSynchronize(b);
    float ms; cudaEventElapsedTime(&ms, a, b);
    const double n = (double)blocks * threads * per;
    printf("table %6.0f MB  U=%2d  %d CTAs/SM (%4d loads in flight/SM): %6.1f probes/ns\n", slots * 32.0 / 1048576, U, ctas_per_sm,
           U * ctas_per_sm * threads, n / (ms * 1e6));
}

int main(int argc, char** argv) {
    uint32_t* out; cudaMalloc(&out, 4);
    if (argc > 1) {  // one table size (MiB, rounded up to a power of two), two occupancies
        u64 slots = 1;
        while (slots * 32 < (u64)atoll(argv[1]) << 20) slots <<= 1;
        uint4* t;
        if (cudaMalloc(&t, slots * 32) != cudaSuccess) return 1;
        cudaMemset(t, 1, slots * 32);
        run<4>(t, slots, 4, out);
        run<8>(t, slots, 8, out);
        return 0;
    }
    for (u64 slots : {1ull << 22, 1ull << 24, 1ull << 25, 1ull << 26, 1ull << 27, 1ull << 28}) {
        uint4* t;
        if (cudaMalloc(&t, slots * 32) != cudaSuccess) break;
        cudaMemset(t, 1, slots * 32);
        run<4>(t, slots, 4, out);
        run<4>(t, slots, 8, out);
        run<8>(t, slots, 8, out);
        run<16>(t, slots, 8, out);
        run<8>(t, slots, 16, out);
        cudaFree(t);
    }
    printf("%s\n", cudaGetErrorString(cudaDeviceSynchronize()));
    return 0;
}
