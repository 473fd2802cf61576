// cm_ops.cuh -- bit-parallel LTLf connectives on packed characteristic matrices.
//
// A CM is stored as consecutive uint4 (16-byte) vectors holding the T trace lanes
// back to back (lane width LW = 8/16/32/64 bits, little endian) -- the byte image of
// the reference's numpy row, zero-padded to 16 bytes.  Every connective is lane
// local, so each uint4 of a CM is computed independently of the others.
//
// The reference (pkg/src/ltlsynth/kernels.py) runs numpy ufuncs on separate array
// elements, where `x >> s` zero-fills every lane.  In a packed word the same shift
// would pull the low bits of the next lane into this lane's top bits, so every
// shift here is followed by a compile-time lane mask that clears the top s bits of
// each lane (SWAR).  With that the sequences below are bit-identical to:
//   op_not    kernels.py:29-31     (~x) & masks
//   op_next   kernels.py:42-44     x >> 1
//   op_future kernels.py:47-57     for s in 1,2,4..: x |= x >> s
//   op_until  kernels.py:60-73     r=b,q=a; for s: r |= q & (r>>s); q &= q>>s; r & masks
//   separates kernels.py:102-105   ((x & 1) == target).all()
#pragma once
#include <cstdint>

namespace ltlb200 {

typedef unsigned long long u64;

// word with the low (LW - s) bits of every LW-bit lane set
template <int LW>
__host__ __device__ constexpr uint32_t lane_keep_mask32(int s) {
    return LW >= 32 ? (0xFFFFFFFFu >> s)
                    : (uint32_t)(((LW == 8 ? 0xFFu : 0xFFFFu) >> s) * (LW == 8 ? 0x01010101u : 0x00010001u));
}

template <int LW>
__host__ __device__ constexpr uint32_t lane_bit0_32() {
    return LW == 8 ? 0x01010101u : (LW == 16 ? 0x00010001u : 1u);
}

// per-lane logical right shift of a packed vector (s is a compile-time constant after unrolling)
template <int LW>
__device__ __forceinline__ uint4 lanes_shr(uint4 x, int s) {
    if constexpr (LW == 64) {
        u64 lo = ((u64)x.y << 32 | x.x) >> s;
        u64 hi = ((u64)x.w << 32 | x.z) >> s;
        return make_uint4((uint32_t)lo, (uint32_t)(lo >> 32), (uint32_t)hi, (uint32_t)(hi >> 32));
    } else {
        const uint32_t m = lane_keep_mask32<LW>(s);
        return make_uint4((x.x >> s) & m, (x.y >> s) & m, (x.z >> s) & m, (x.w >> s) & m);
    }
}

__device__ __forceinline__ uint4 v_and(uint4 a, uint4 b) { return make_uint4(a.x & b.x, a.y & b.y, a.z & b.z, a.w & b.w); }
__device__ __forceinline__ uint4 v_or(uint4 a, uint4 b) { return make_uint4(a.x | b.x, a.y | b.y, a.z | b.z, a.w | b.w); }
__device__ __forceinline__ uint4 v_andnot(uint4 m, uint4 x) { return make_uint4(m.x & ~x.x, m.y & ~x.y, m.z & ~x.z, m.w & ~x.w); }
__device__ __forceinline__ bool v_eq(uint4 a, uint4 b) {
    return ((a.x ^ b.x) | (a.y ^ b.y) | (a.z ^ b.z) | (a.w ^ b.w)) == 0u;
}

template <int LW>
__device__ __forceinline__ uint4 cm_not(uint4 x, uint4 valid) { return v_andnot(valid, x); }

template <int LW>
__device__ __forceinline__ uint4 cm_next(uint4 x) { return lanes_shr<LW>(x, 1); }

template <int LW>
__device__ __forceinline__ uint4 cm_future(uint4 x) {
#pragma unroll
    for (int s = 1; s < LW; s <<= 1) x = v_or(x, lanes_shr<LW>(x, s));
    return x;
}

template <int LW>
__device__ __forceinline__ uint4 cm_until(uint4 a, uint4 b, uint4 valid) {
    uint4 r = b, q = a;
#pragma unroll
    for (int s = 1; s < LW; s <<= 1) {
        r = v_or(r, v_and(q, lanes_shr<LW>(r, s)));
        q = v_and(q, lanes_shr<LW>(q, s));
    }
    return v_and(r, valid);
}

// word-wise "position-0 bit of every lane differs from the target" (0 when this vector agrees).
// LW == 1 is the regex front-end's bitset (regex_ops.cuh): `valid` = the bits of the example strings (positives and
// negatives), `target` = the bits of the positives; a CS separates when it agrees with the target on those bits.
template <int LW>
__device__ __forceinline__ uint32_t cm_sep_diff(uint4 x, uint4 target, uint4 valid) {
    if constexpr (LW == 1) {
        return ((x.x & valid.x) ^ target.x) | ((x.y & valid.y) ^ target.y) | ((x.z & valid.z) ^ target.z) | ((x.w & valid.w) ^ target.w);
    } else if constexpr (LW == 64) {
        return ((x.x & 1u) ^ target.x) | target.y | ((x.z & 1u) ^ target.z) | target.w;
    } else {
        const uint32_t b = lane_bit0_32<LW>();
        return ((x.x & b) ^ target.x) | ((x.y & b) ^ target.y) | ((x.z & b) ^ target.z) | ((x.w & b) ^ target.w);
    }
}

// OP_GLOBALLY is an EXTENSION beyond the reference's tags (engine.py:42 ends at OP_OR; SPEC.md:211 lists G as a
// non-goal): G x = x at every position from here to the end of the trace = !F!x, one more masked cascade.
enum : int { OP_ATOM = 0, OP_NOT = 1, OP_NEXT = 2, OP_FUTURE = 3, OP_AND = 4, OP_UNTIL = 5, OP_OR = 6, OP_GLOBALLY = 7 };

template <int LW>
__device__ __forceinline__ uint4 cm_globally(uint4 x, uint4 valid) {
    return v_andnot(valid, cm_future<LW>(v_andnot(valid, x)));
}

template <int LW, int OP>
__device__ __forceinline__ uint4 cm_apply(uint4 a, uint4 b, uint4 valid) {
    if constexpr (OP == OP_ATOM) return a;
    else if constexpr (OP == OP_NOT) return cm_not<LW>(a, valid);
    else if constexpr (OP == OP_NEXT) return cm_next<LW>(a);
    else if constexpr (OP == OP_FUTURE) return cm_future<LW>(a);
    else if constexpr (OP == OP_AND) return v_and(a, b);
    else if constexpr (OP == OP_OR) return v_or(a, b);
    else if constexpr (OP == OP_GLOBALLY) return cm_globally<LW>(a, valid);
    else return cm_until<LW>(a, b, valid);
}

// 32-bit mix of a 16-byte vector (four multiply / xor-shift rounds, one per word); `seed`
// chains the vectors of a wide key.  Hash sets here have < 2^32 slots, so 32 bits suffice,
// and 32-bit IMADs are single instructions where a 64-bit multiply costs four.
__device__ __forceinline__ uint32_t hash_vec(uint4 k, uint32_t seed) {
    uint32_t h = (k.x ^ seed) * 0x9E3779B1u + k.y;
    h ^= h >> 15;
    h = h * 0x85EBCA77u + k.z;
    h ^= h >> 13;
    h = h * 0xC2B2AE3Du + k.w;
    h ^= h >> 16;
    h *= 0x27D4EB2Fu;
    h ^= h >> 15;
    return h;
}

}  // namespace ltlb200
