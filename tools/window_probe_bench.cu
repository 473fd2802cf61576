// Go/no-go microbenchmark for radix-partitioned dedup probing: records (16-byte key + 4-byte
// ordinal) are streamed from HBM in bucket order; every record probes one random 32-byte slot
// inside its bucket's table window.  Windows of <= ~64 MB should stay L2 resident while the
// record stream passes through with evict-first loads.  Prints records/ns for several window
// sizes, next to the same loop probing the whole table (no partitioning).
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/wpb tools/window_probe_bench.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
typedef unsigned long long u64;

__device__ __forceinline__ uint4 ld_stream(const uint4* p) { return __ldcs(p); }

__global__ void fill(uint4* keys, u64 n) {
    for (u64 i = blockIdx.x * (u64)blockDim.x + threadIdx.x; i < n; i += (u64)gridDim.x * blockDim.x) {
        u64 x = i * 0x9E3779B97F4A7C15ull + 777;
        x ^= x >> 29; x *= 0xBF58476D1CE4E5B9ull; x ^= x >> 32;
        u64 y = x * 0x94D049BB133111EBull; y ^= y >> 31;
        keys[i] = make_uint4((uint32_t)x, (uint32_t)(x >> 32), (uint32_t)y, (uint32_t)(y >> 32));
    }
}

// chunk = 32 * U * 4 records per warp-ticket; records [0, n) belong to window (i * n_windows / n)
template <int U, bool CAS>
__global__ void __launch_bounds__(128, 4) probe(const uint4* __restrict__ keys, u64 n, uint4* table, u64 table_slots,
                                     u64 window_slots, u64* ticket, uint32_t* out) {
    const int lane = threadIdx.x & 31;
    const u64 chunk = 32ull * U * 8;
    const u64 n_windows = table_slots / window_slots;
    uint32_t acc = 0;
    for (;;) {
        u64 t = 0;
        if (lane == 0) t = atomicAdd(ticket, 1ull);
        t = __shfl_sync(0xFFFFFFFFu, t, 0);
        const u64 r0 = t * chunk;
        if (r0 >= n) break;
        const u64 w = (r0 / (n / n_windows));  // window of this chunk
        const u64 wbase = (w < n_windows ? w : n_windows - 1) * window_slots;
        for (int it = 0; it < 8; ++it) {
            uint4 k[U], s[U];
            uint32_t v[U];
#pragma unroll
            for (int u = 0; u < U; ++u) k[u] = ld_stream(keys + r0 + (u64)(it * U + u) * 32 + lane);
#pragma unroll
            for (int u = 0; u < U; ++u) {
                const u64 slot = wbase + ((k[u].x ^ k[u].z) & (window_slots - 1));
                s[u] = __ldcg(table + slot * 2);
                v[u] = __ldcg(reinterpret_cast<const uint32_t*>(table + slot * 2 + 1) + 1);
            }
#pragma unroll
            for (int u = 0; u < U; ++u) {
                acc += s[u].x ^ s[u].w ^ v[u];
                if (CAS && (k[u].y & 7u) == 0u) {  // ~12% of the records also write their slot
                    const u64 slot = wbase + ((k[u].x ^ k[u].z) & (window_slots - 1));
                    atomicCAS(reinterpret_cast<u64*>(table + slot * 2 + 1), 0x0101010101010101ull, (u64)k[u].w);
                }
            }
        }
    }
    if (acc == 0x12345678u) out[0] = acc;
}

int main() {
    const u64 n = 96ull << 20;  // 96 Mi records = 1.5 GiB of keys
    const u64 table_slots = 1ull << 25;  // 1 GiB of 32-byte slots
    uint4 *keys, *table; u64* ticket; uint32_t* out;
    cudaMalloc(&keys, n * 16); cudaMalloc(&table, table_slots * 32); cudaMalloc(&ticket, 8); cudaMalloc(&out, 4);
    fill<<<148 * 8, 256>>>(keys, n);
    cudaMemset(table, 1, table_slots * 32);
    cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
    for (int cas = 0; cas < 2; ++cas)
    for (u64 wmb : {1024ull, 256ull, 128ull, 64ull, 32ull, 16ull, 8ull}) {
        const u64 window_slots = (wmb << 20) / 32;
        for (int rep = 0; rep < 2; ++rep) {
            cudaMemset(ticket, 0, 8);
            cudaEventRecord(a);
            if (cas) probe<4, true><<<148 * 4, 128>>>(keys, n, table, table_slots, window_slots, ticket, out);
            else probe<4, false><<<148 * 4, 128>>>(keys, n, table, table_slots, window_slots, ticket, out);
            cudaEventRecord(b); cudaEventSynchronize(b);
        }
        float ms; cudaEventElapsedTime(&ms, a, b);
        printf("cas=%d window=%4llu MB: %.3f ms  %.1f records/ns  (stream %.0f GB/s)\n", cas, wmb, ms, n / (ms * 1e6), n * 16 / (ms * 1e6));
    }
    printf("%s\n", cudaGetErrorString(cudaDeviceSynchronize()));
    return 0;
}
