// launch.h -- host-side entry points of the enumeration kernels, one set per lane width.
//
// The construction + dedup kernels are templates over (lane width, operator); instantiating all of
// them in one translation unit took four minutes of nvcc.  inst.cu is compiled once per
// (lane width, narrow | wide) with -DLTLB200_INST_LW / -DLTLB200_INST_WIDE and exports the plain
// functions below; engine.cu dispatches on the lane width at run time.
#pragma once
#include <cuda_runtime.h>

#include <cstddef>

namespace ltlb200 {

struct NarrowParams;
struct WideParams;
struct TinyParams;
struct WideTinyParams;

// which kernel of a (lane width) set: one launch per operator (big levels), one launch for every
// operator (levels up to kSmallLevel candidates), the guarded kernel (scan pass / dead ranges), and -- one search
// sharded over several GPUs -- the kernel that routes candidates to their hash owners instead of probing them
enum : int { LK_OPERATOR = 0, LK_SMALL = 1, LK_GUARDED = 2, LK_ROUTE = 3 };
constexpr size_t kMaxDynamicSmem = 227 * 1024;  // per CTA on sm_100

#define LTLB200_DECLARE_WIDE(LW)                                                                                   \
    void wide2_launch_##LW(int kind, int op, const WideParams &P, int grid, size_t smem, int device, cudaStream_t st); \
    int wide2_occupancy_##LW(int nvec, int device, int guide_smem_words);                                             \
    void wide2_tiny_##LW(const WideTinyParams &T, int warps, size_t smem, int device, cudaStream_t st); /* several tiny levels in one launch */
#define LTLB200_DECLARE_LW(LW)                                                                                     \
    void narrow_launch_##LW(int kind, int op, const NarrowParams &P, int grid, cudaStream_t st);                    \
    int narrow_occupancy_##LW();                                                                                    \
    void narrow_tiny_##LW(const TinyParams &T, int device, cudaStream_t st); /* several tiny levels in one launch */ \
    void narrow_probe_##LW(const NarrowParams &P, const void *rows, const void *ords, unsigned long long n, int grid, \
                           cudaStream_t st);                                                                         \
    LTLB200_DECLARE_WIDE(LW)

LTLB200_DECLARE_WIDE(1)  // the regex grammar's bitset CS (wide2_regex.cuh): the multi-vector kernels only
LTLB200_DECLARE_LW(8)
LTLB200_DECLARE_LW(16)
LTLB200_DECLARE_LW(32)
LTLB200_DECLARE_LW(64)
#undef LTLB200_DECLARE_WIDE
#undef LTLB200_DECLARE_LW

}  // namespace ltlb200
