// inst.cu -- instantiates the enumeration kernels of ONE lane width (see launch.h).
//
//   nvcc -DLTLB200_INST_LW=8|16|32|64 -DLTLB200_INST_WIDE=0|1 -c inst.cu     (LW=1, WIDE=1: the regex grammar)
//
// INST_WIDE=0: narrow.cuh (CMs of one uint4), INST_WIDE=1: wide2.cuh (multi-vector CMs).
#include <mutex>

#include "launch.h"
#if LTLB200_INST_WIDE
#include "wide2_tiny.cuh"
#else
#include "narrow_tiny.cuh"
#endif

#ifndef LTLB200_INST_LW
#error "compile with -DLTLB200_INST_LW=<lane bits>"
#endif

#define LTLB200_CAT_(a, b) a##b
#define LTLB200_CAT(a, b) LTLB200_CAT_(a, b)

namespace ltlb200 {

constexpr int LW = LTLB200_INST_LW;

#if !LTLB200_INST_WIDE

// one launch per operator: the fused construct + probe kernel, or (ROUTE) the kernel that routes to hash owners
template <bool ROUTE, int OP>
static void launch_one(const NarrowParams &P, int grid, cudaStream_t st) {
    if constexpr (ROUTE) narrow_route_kernel<LW, OP><<<grid, CTA_THREADS, 0, st>>>(P);
    else narrow_level_kernel<LW, OP><<<grid, CTA_THREADS, 0, st>>>(P);
}

template <bool ROUTE>
static void launch_by_operator(int op, const NarrowParams &P, int grid, cudaStream_t st) {
    switch (op) {
        case OP_ATOM: launch_one<ROUTE, OP_ATOM>(P, grid, st); break;
        case OP_NOT: launch_one<ROUTE, OP_NOT>(P, grid, st); break;
        case OP_NEXT: launch_one<ROUTE, OP_NEXT>(P, grid, st); break;
        case OP_FUTURE: launch_one<ROUTE, OP_FUTURE>(P, grid, st); break;
        case OP_GLOBALLY: launch_one<ROUTE, OP_GLOBALLY>(P, grid, st); break;
        case OP_AND: launch_one<ROUTE, OP_AND>(P, grid, st); break;
        case OP_UNTIL: launch_one<ROUTE, OP_UNTIL>(P, grid, st); break;
        default: launch_one<ROUTE, OP_OR>(P, grid, st); break;
    }
}

void LTLB200_CAT(narrow_launch_, LTLB200_INST_LW)(int kind, int op, const NarrowParams &P, int grid, cudaStream_t st) {
    if (kind == LK_SMALL) narrow_small_level_kernel<LW><<<grid, CTA_THREADS, 0, st>>>(P);
    else if (kind == LK_GUARDED) narrow_guarded_level_kernel<LW><<<grid, CTA_THREADS, 0, st>>>(P);
    else if (kind == LK_ROUTE) launch_by_operator<true>(op, P, grid, st);
    else launch_by_operator<false>(op, P, grid, st);
}

void LTLB200_CAT(narrow_probe_, LTLB200_INST_LW)(const NarrowParams &P, const void *rows, const void *ords, unsigned long long n,
                                                 int grid, cudaStream_t st) {
    narrow_probe_kernel<LW><<<grid, CTA_THREADS, 0, st>>>(P, (const uint4 *)rows, (const u64 *)ords, n);
}

void LTLB200_CAT(narrow_tiny_, LTLB200_INST_LW)(const TinyParams &T, int device, cudaStream_t st) {
    constexpr size_t smem = sizeof(WarpSharedTiny) * TINY_WARPS;
    {   // opt in to > 48 KB of dynamic shared memory: a per-device attribute of the kernel
        static std::mutex mu;
        static unsigned long long seen = 0;
        std::lock_guard<std::mutex> lock(mu);
        if (!(seen >> (device & 63) & 1ull)) {
            cudaFuncSetAttribute(narrow_tiny_levels_kernel<LW>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
            seen |= 1ull << (device & 63);
        }
    }
    narrow_tiny_levels_kernel<LW><<<1, TINY_THREADS, smem, st>>>(T);
}

int LTLB200_CAT(narrow_occupancy_, LTLB200_INST_LW)() {
    int occ = 0;
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, narrow_level_kernel<LW, OP_UNTIL>, CTA_THREADS, 0) != cudaSuccess) {
        cudaGetLastError();
        occ = 1;
    }
    return occ > 1 ? occ : 1;
}

#else  // wide

static size_t max_smem() { return LW == LW_REGEX ? kMaxDynamicSmem : wide2_warp_vecs(MAX_NVEC) * sizeof(uint4) * WARPS_PER_CTA; }

// cudaFuncAttributeMaxDynamicSharedMemorySize is a per-DEVICE attribute of a kernel: a process that drives
// several GPUs (synthesize_dnc(devices=[0, 1]), one store per device) must opt in on each of them.
template <typename Kernel>
static void opt_in(Kernel kernel, int device, unsigned long long &seen, std::mutex &mu) {
    std::lock_guard<std::mutex> lock(mu);
    const unsigned long long bit = 1ull << (device & 63);
    if (seen & bit) return;
    cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)max_smem());
    seen |= bit;
}

template <int OP>
static void launch_operator(const WideParams &P, int grid, size_t smem, int device, cudaStream_t st) {
    static unsigned long long seen = 0;
    static std::mutex mu;
    opt_in(wide2_level_kernel<LW, OP>, device, seen, mu);
    wide2_level_kernel<LW, OP><<<grid, CTA_THREADS, smem, st>>>(P);
}

template <int OP>
static void launch_route(const WideParams &P, int grid, size_t smem, int device, cudaStream_t st) {
    static unsigned long long seen = 0;
    static std::mutex mu;
    opt_in(wide2_route_kernel<LW, OP>, device, seen, mu);
    wide2_route_kernel<LW, OP><<<grid, CTA_THREADS, smem, st>>>(P);
}

void LTLB200_CAT(wide2_launch_, LTLB200_INST_LW)(int kind, int op, const WideParams &P, int grid, size_t smem, int device,
                                                 cudaStream_t st) {
    if (kind == LK_SMALL) {
        static unsigned long long seen = 0;
        static std::mutex mu;
        opt_in(wide2_small_level_kernel<LW>, device, seen, mu);
        wide2_small_level_kernel<LW><<<grid, CTA_THREADS, smem, st>>>(P);
        return;
    }
    if (kind == LK_GUARDED) {
        static unsigned long long seen = 0;
        static std::mutex mu;
        opt_in(wide2_guarded_level_kernel<LW>, device, seen, mu);
        wide2_guarded_level_kernel<LW><<<grid, CTA_THREADS, smem, st>>>(P);
        return;
    }
#if LTLB200_INST_LW == 1  // the regex front-end's operators (regex_ops.cuh, wide2_regex.cuh)
    if (kind == LK_ROUTE) {
        switch (op) {
            case OP_ATOM: launch_route<OP_ATOM>(P, grid, smem, device, st); break;
            case OP_RE_QUESTION: launch_route<OP_RE_QUESTION>(P, grid, smem, device, st); break;
            case OP_RE_STAR: launch_route<OP_RE_STAR>(P, grid, smem, device, st); break;
            case OP_RE_CONCAT: launch_route<OP_RE_CONCAT>(P, grid, smem, device, st); break;
            default: launch_route<OP_OR>(P, grid, smem, device, st); break;
        }
        return;
    }
    switch (op) {
        case OP_ATOM: launch_operator<OP_ATOM>(P, grid, smem, device, st); break;
        case OP_RE_QUESTION: launch_operator<OP_RE_QUESTION>(P, grid, smem, device, st); break;
        case OP_RE_STAR: launch_operator<OP_RE_STAR>(P, grid, smem, device, st); break;
        case OP_RE_CONCAT: launch_operator<OP_RE_CONCAT>(P, grid, smem, device, st); break;
        default: launch_operator<OP_OR>(P, grid, smem, device, st); break;
    }
#else
    if (kind == LK_ROUTE) {
        switch (op) {
            case OP_ATOM: launch_route<OP_ATOM>(P, grid, smem, device, st); break;
            case OP_NOT: launch_route<OP_NOT>(P, grid, smem, device, st); break;
            case OP_NEXT: launch_route<OP_NEXT>(P, grid, smem, device, st); break;
            case OP_FUTURE: launch_route<OP_FUTURE>(P, grid, smem, device, st); break;
            case OP_AND: launch_route<OP_AND>(P, grid, smem, device, st); break;
            case OP_UNTIL: launch_route<OP_UNTIL>(P, grid, smem, device, st); break;
            case OP_GLOBALLY: launch_route<OP_GLOBALLY>(P, grid, smem, device, st); break;
            default: launch_route<OP_OR>(P, grid, smem, device, st); break;
        }
    } else {
        switch (op) {
            case OP_ATOM: launch_operator<OP_ATOM>(P, grid, smem, device, st); break;
            case OP_NOT: launch_operator<OP_NOT>(P, grid, smem, device, st); break;
            case OP_NEXT: launch_operator<OP_NEXT>(P, grid, smem, device, st); break;
            case OP_FUTURE: launch_operator<OP_FUTURE>(P, grid, smem, device, st); break;
            case OP_AND: launch_operator<OP_AND>(P, grid, smem, device, st); break;
            case OP_UNTIL: launch_operator<OP_UNTIL>(P, grid, smem, device, st); break;
            case OP_GLOBALLY: launch_operator<OP_GLOBALLY>(P, grid, smem, device, st); break;
            default: launch_operator<OP_OR>(P, grid, smem, device, st); break;
        }
    }
#endif
}

void LTLB200_CAT(wide2_tiny_, LTLB200_INST_LW)(const WideTinyParams &T, int warps, size_t smem, int device, cudaStream_t st) {
    static unsigned long long seen = 0;
    static std::mutex mu;
    {
        std::lock_guard<std::mutex> lock(mu);
        const unsigned long long bit = 1ull << (device & 63);
        if (!(seen & bit)) {  // (less than the 227 KB of a CTA: the kernel has ~14 KB of static shared memory)
            cudaFuncSetAttribute(wide2_tiny_levels_kernel<LW>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)(kMaxDynamicSmem - 16 * 1024));
            seen |= bit;
        }
    }
    wide2_tiny_levels_kernel<LW><<<1, 32 * warps, smem, st>>>(T);
}

int LTLB200_CAT(wide2_occupancy_, LTLB200_INST_LW)(int nvec, int device, int guide_smem_words) {
    static unsigned long long seen = 0;
    static std::mutex mu;
    constexpr int kHeaviest = LW == LW_REGEX ? (int)OP_RE_CONCAT : (int)OP_UNTIL;
    opt_in(wide2_level_kernel<LW, kHeaviest>, device, seen, mu);
    int occ = 0;
    const size_t smem = wide2_warp_vecs(nvec, LW == LW_REGEX) * sizeof(uint4) * WARPS_PER_CTA + (size_t)guide_smem_words * sizeof(uint32_t);
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, wide2_level_kernel<LW, kHeaviest>, CTA_THREADS, smem) != cudaSuccess) {
        cudaGetLastError();
        occ = 1;
    }
    return occ > 1 ? occ : 1;
}

#endif

}  // namespace ltlb200
