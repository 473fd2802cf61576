// regex_ops.cuh -- characteristic-sequence operators of the REGEX front-end (first slice).
//
// NOT in the reference (SPEC.md:11 scopes regular-expression synthesis out; PAPER.md:81-113 only motivates it), so
// there is no reference line to cite and parity is unpinned; the CPU oracle is oracle/regex_oracle.py, whose
// membership semantics are pinned to Python's `re.fullmatch`.
//
// A CS (characteristic sequence) has one bit per INFIX of the example strings, infixes sorted by (length, text):
// bit k = "infix k is in the language".  Bit 0 is the empty word.  On such bitsets
//   union        r | s   = CS(r) | CS(s)                                   (the engine's OP_OR)
//   question     r?      = CS(r) | bit 0
//   concatenation r s    : bit w = OR over the splits w = u v of  CS(r)[u] & CS(s)[v]
//   star         r*      : bit 0, and bit w = OR over the splits w = u v, u non-empty, of  CS(r)[u] & CS(r*)[v]
//                          (v is shorter than w and infixes are sorted by length: one pass in index order)
// The splits come from the GUIDE TABLE the host precomputes: offsets[w] .. offsets[w+1] index entries (u | v << 16)
// of infix indices.  CSs of up to 128 bits are one uint4 and take the operators below (narrow kernels; the table is
// read through the read-only cache, a few KB shared by every candidate); wider ones (up to 4096 bits) are handled 32
// candidates at a time on bit-sliced rows (wide2_regex.cuh) with the same table regrouped by Engine::set_regex.
#pragma once
#include "cm_ops.cuh"

namespace ltlb200 {

constexpr int LW_REGEX = 1;  // "lane width" of the regex instantiation of the narrow kernels
enum : int { OP_RE_QUESTION = 8, OP_RE_STAR = 9, OP_RE_CONCAT = 10 };

__device__ __forceinline__ uint32_t cs_bit(uint4 x, uint32_t k) {
    const uint32_t w = k < 64u ? (k < 32u ? x.x : x.y) : (k < 96u ? x.z : x.w);
    return (w >> (k & 31u)) & 1u;
}

__device__ __forceinline__ void cs_set(uint4 &x, uint32_t k) {
    const uint32_t m = 1u << (k & 31u);
    if (k < 64u) {
        if (k < 32u) x.x |= m;
        else x.y |= m;
    } else {
        if (k < 96u) x.z |= m;
        else x.w |= m;
    }
}

// guide[0 .. n_bits] = entry offsets, guide[n_bits + 1 ...] = entries (u | v << 16)
__device__ __forceinline__ uint4 re_concat(const uint32_t *guide, int n_bits, uint4 a, uint4 b) {
    uint4 out = make_uint4(0, 0, 0, 0);
    const uint32_t *entries = guide + n_bits + 1;
    uint32_t e = __ldg(guide);
#pragma unroll 1
    for (int w = 0; w < n_bits; ++w) {
        const uint32_t e_end = __ldg(guide + w + 1);
        uint32_t hit = 0;
#pragma unroll 1
        for (; e < e_end && !hit; ++e) {
            const uint32_t uv = __ldg(entries + e);
            hit = cs_bit(a, uv & 0xFFFFu) & cs_bit(b, uv >> 16);
        }
        e = e_end;
        if (hit) cs_set(out, (uint32_t)w);
    }
    return out;
}

__device__ __forceinline__ uint4 re_star(const uint32_t *guide, int n_bits, uint4 a) {
    uint4 out = make_uint4(1u, 0, 0, 0);  // the empty word
    const uint32_t *entries = guide + n_bits + 1;
    uint32_t e = __ldg(guide + 1);
#pragma unroll 1
    for (int w = 1; w < n_bits; ++w) {
        const uint32_t e_end = __ldg(guide + w + 1);
        uint32_t hit = 0;
#pragma unroll 1
        for (; e < e_end && !hit; ++e) {
            const uint32_t uv = __ldg(entries + e);
            const uint32_t u = uv & 0xFFFFu;
            hit = (u != 0u) & cs_bit(a, u) & cs_bit(out, uv >> 16);
        }
        e = e_end;
        if (hit) cs_set(out, (uint32_t)w);
    }
    return out;
}


template <int OP>
__device__ __forceinline__ uint4 re_apply(const uint32_t *guide, int n_bits, uint4 a, uint4 b) {
    if constexpr (OP == OP_ATOM) return a;
    else if constexpr (OP == OP_OR) return v_or(a, b);
    else if constexpr (OP == OP_RE_QUESTION) return make_uint4(a.x | 1u, a.y, a.z, a.w);
    else if constexpr (OP == OP_RE_STAR) return re_star(guide, n_bits, a);
    else return re_concat(guide, n_bits, a, b);
}

}  // namespace ltlb200
