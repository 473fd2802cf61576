// tiny_plan.cuh -- what the two kernels that build SEVERAL TINY LEVELS PER LAUNCH share (narrow_tiny.cuh for one-vector
// CMs, wide2_tiny.cuh for multi-vector ones): the limits of a launch, how it reports its levels, and the planning of
// a level on the device (Engine::plan_level's blocks, in the same order, with the same ordinals; reference
// _tasks_for_level, engine.py:219-266).
#pragma once
#include "narrow.cuh"

namespace ltlb200 {

constexpr uint32_t TINY_MAX_CANDIDATES = 1u << 15;  // winners bitmap of a level: 4 KiB of shared memory
constexpr int TINY_MAX_BLOCKS = 64;
constexpr int TINY_MAX_LEVELS = 24;

// status of one level: not built (the host builds it the usual way) / built
enum : unsigned long long { TINY_NOT_BUILT = 0ull, TINY_BUILT = 1ull };
// why the launch ended before cost_last (results[TINY_MAX_LEVELS].status): the next level is too big for one CTA or
// for the set as it is; the claim arrays / the set overflowed; an exhaustive level holds a separating candidate
enum : unsigned long long { TINY_END_NONE = 0ull, TINY_END_BIG = 1ull, TINY_END_OVERFLOW = 2ull, TINY_END_SEPARATOR = 3ull };

struct TinyLevelResult {
    u64 status, n_new, sep_ord, sep_rank;
    u64 ns;  // device time of the level (LTLB200_DEBUG prints it)
};


// one block of the level's canonical order; tiles are small so that sixteen warps share even a tiny block
__device__ __forceinline__ void tiny_push(BlockDesc *blocks, int &n_blocks, u64 &constructed, u64 &n_tiles, BlockDesc b, int tile_s_cap) {
    if (b.size == 0) return;
    if (n_blocks >= TINY_MAX_BLOCKS) {
        constructed = ~0ull;  // too many blocks: the host builds this level
        return;
    }
    if (b.kind == BK_UNARY) {
        b.tile_s = 4;
        b.vg = 1;
        b.tiles_v = (b.na + (u64)TILE_V * 4 - 1) / ((u64)TILE_V * 4);
        b.tiles_s = 1;
    } else {
        const u64 n_vec = b.vec_is_b ? b.nb : b.na, n_sc = b.vec_is_b ? b.na : b.nb;
        b.tile_s = (uint32_t)(n_sc < (u64)tile_s_cap ? n_sc : (u64)tile_s_cap);
        b.tiles_s = (n_sc + b.tile_s - 1) / b.tile_s;
        b.vg = 1;
        b.tiles_v = (n_vec + TILE_V - 1) / TILE_V;
    }
    b.ord0 = constructed;
    b.tile0 = n_tiles;
    constructed += b.size;
    n_tiles += b.tiles_v * b.tiles_s;
    blocks[n_blocks++] = b;
}

// Engine::plan_level on the device (same blocks, same order, same ordinals; tile geometry is private to a launch)
__device__ inline void tiny_plan(uint32_t op_mask, int n_atoms, const int *w, int tile_s_cap, BlockDesc *blocks, int cost, const u64 *level_tab,
                                 int &n_blocks, u64 &constructed, u64 &n_tiles) {
    n_blocks = 0;
    constructed = 0;
    n_tiles = 0;
    auto n_of = [&](int c) { return level_tab[2 * c]; };
    auto base_of = [&](int c) { return level_tab[2 * c + 1]; };
    if (cost == w[OP_ATOM]) {
        BlockDesc b{};
        b.op = OP_ATOM;
        b.kind = BK_UNARY;
        b.from_atoms = 1;
        b.na = (u64)n_atoms;
        b.size = b.na;
        tiny_push(blocks, n_blocks, constructed, n_tiles, b, tile_s_cap);
    }
    // (the regex operators -- question, star unary; concatenation, non-commutative, before union = OP_OR -- are only
    // ever enabled on a handle with the regex grammar, where none of the LTL tags is: Engine::plan_level)
    const int unary_tags[6] = {OP_NOT, OP_NEXT, OP_FUTURE, OP_GLOBALLY, OP_RE_QUESTION, OP_RE_STAR};
    const int binary_tags[4] = {OP_AND, OP_UNTIL, OP_RE_CONCAT, OP_OR};
    for (int k = 0; k < 6; ++k) {
        const int tag = unary_tags[k];
        if (!(op_mask >> tag & 1u) || cost - w[tag] < 1) continue;
        const int src = cost - w[tag];
        if (n_of(src) == 0) continue;
        BlockDesc b{};
        b.op = (uint32_t)tag;
        b.kind = BK_UNARY;
        b.a_off = base_of(src);
        b.na = n_of(src);
        b.size = b.na;
        tiny_push(blocks, n_blocks, constructed, n_tiles, b, tile_s_cap);
        if (constructed == ~0ull) return;
    }
    for (int k = 0; k < 4; ++k) {
        const int tag = binary_tags[k];
        if (!(op_mask >> tag & 1u)) continue;
        const bool commutative = tag == OP_AND || tag == OP_OR;
        for (int c1 = 1; c1 < cost - w[tag]; ++c1) {
            const int c2 = cost - w[tag] - c1;
            if (commutative && c1 > c2) break;
            const u64 na = n_of(c1), nb = n_of(c2);
            if (na == 0 || nb == 0) continue;
            BlockDesc b{};
            b.op = (uint32_t)tag;
            b.a_off = base_of(c1);
            b.na = na;
            b.b_off = base_of(c2);
            b.nb = nb;
            if (commutative && c1 == c2) {
                b.kind = BK_TRI;
                b.vec_is_b = 1;
                b.size = na * (na + 1) / 2;
            } else {
                b.kind = BK_RECT;
                b.vec_is_b = nb >= na;
                b.size = na * nb;
            }
            b.c_left = (uint32_t)c1;
            tiny_push(blocks, n_blocks, constructed, n_tiles, b, tile_s_cap);
            if (constructed == ~0ull) return;
        }
    }
}

}  // namespace ltlb200
