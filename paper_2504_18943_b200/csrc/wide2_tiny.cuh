// wide2_tiny.cuh -- the tiny levels of a search over multi-vector CMs, SEVERAL LEVELS IN ONE LAUNCH.
//
// narrow_tiny.cuh for the wide path (see there for why: a level of a few thousand candidates is ~90 us of launches,
// host planning and one synchronisation around ~30 us of device work; a BASELINE configs[0]-sized regex search spent
// 1.05 ms on twelve such levels).  ONE CTA, level after level: plan the level's blocks on the device (tiny_plan.cuh),
// enumerate with the tiles and passes of wide2.cuh / wide2_regex.cuh (mode W2_TINY: counters, tickets and the block
// list in shared memory; rows and the row directory read with ld.cg, because this kernel wrote them), finalise in
// shared memory (winners bitmap -> ranks -> loc[] and ordinals; the rows stay where they were staged, at the tail
// of the row log, which moves on by the staging entries the level reserved).  The launch ends when a level would be
// too big, holds the separator, or needs the host -- as in narrow_tiny.cuh -- and the host hands the levels out one
// expand_level call at a time (Engine::tiny_*), replaying the planning; results are bit-identical.
#pragma once
#include "tiny_plan.cuh"
#include "wide2.cuh"

namespace ltlb200 {

constexpr int W2_TINY_MAX_WARPS = 8;  // (256 threads: the passes of wide2_batch keep their registers)
constexpr int W2_TINY_TILE_S = 16;    // scalar rows per tile here: small tiles, so that the warps share even a tiny block

struct WideTinyLevelResult {
    u64 status, n_new, sep_ord, sep_rank;
    u64 ns;        // device time of the level (LTLB200_DEBUG prints it)
    u64 n_staged;  // staging entries the level reserved = log entries it takes
};

struct WideTinyParams {
    WideParams P;          // blocks / counters are replaced by shared memory; total_before / stage_rows / stage_cap move on level by level
    uint4 *store;          // writable alias of P.store (the row log)
    u64 *loc, *ords;       // writable: log index and winning ordinal of every entry of the cache
    const u64 *level_tab;  // [2c] = n(c), [2c + 1] = base(c) by cost c >= 1: the stored levels (cost < cost_first)
    WideTinyLevelResult *results;  // [cost - cost_first]; [TINY_MAX_LEVELS].status = why the launch ended
    u64 total;             // entries of the cache before cost_first
    u64 log_tail, log_cap; // log entries in use before cost_first / rows the log has room for
    u64 table_slots;
    u64 max_candidates;    // a level beyond this is left to the launches that spread over the whole device
    uint32_t op_mask;
    int n_atoms, cost_first, cost_last, exhaustive;
    int weights[16];
};

struct WideTinyControl {  // CTA-wide decisions of thread 0
    int go, stop_after;
    u64 constructed, base, log_tail;
    u64 n_staged, ord_limit, sep_ord;
    u64 t0;
};

template <int LW>
__global__ void __launch_bounds__(32 * W2_TINY_MAX_WARPS, 1) wide2_tiny_levels_kernel(const __grid_constant__ WideTinyParams T) {
    extern __shared__ __align__(16) uint4 s_w2[];
    __shared__ WideParams sQ;
    __shared__ WideTinyControl ctl;
    __shared__ BlockDesc s_blocks[TINY_MAX_BLOCKS];
    __shared__ u64 s_tab[2 * 64];
    __shared__ uint32_t s_bitmap[TINY_MAX_CANDIDATES / 32];
    __shared__ uint32_t s_sbrank[TINY_MAX_CANDIDATES / 1024 + 1];
    __shared__ u64 s_counters[CTR_COUNT];
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, n_threads = blockDim.x, n_warps = n_threads >> 5;
    constexpr bool kRegex = LW == LW_REGEX;
    if (tid == 0) {
        sQ = T.P;
        sQ.blocks = s_blocks;
        sQ.counters = s_counters;
        sQ.guide_smem_words = 0;  // (the tables stay in global memory here)
        ctl.base = T.total;
        ctl.log_tail = T.log_tail;
    }
    for (int k = tid; k < 2 * 64; k += n_threads) s_tab[k] = k < 2 * T.cost_first ? T.level_tab[k] : 0ull;
    __syncthreads();
    const Wide2Warp W = wide2_carve<LW>(sQ, s_w2);
    const int tile_s_cap = min(W2_TINY_TILE_S, wide2_tile_s(T.P.nvec, kRegex));
    for (int cost = T.cost_first; cost <= T.cost_last; ++cost) {
        // ---- plan (thread 0) and reset the level's counters
        if (tid == 0) {
            int n_blocks;
            u64 constructed, n_tiles;
            ctl.t0 = global_timer_ns();
            tiny_plan(T.op_mask, T.n_atoms, T.weights, tile_s_cap, s_blocks, cost, s_tab, n_blocks, constructed, n_tiles);
            ctl.go = 1;
            // staging entries: one per candidate at most, plus what the warps may have reserved and not used
            const u64 room = T.log_cap - ctl.log_tail;
            const u64 stage_cap = room < T.P.stage_cap ? room : T.P.stage_cap;
            if (constructed == ~0ull || constructed > T.max_candidates || 2 * (ctl.base + constructed) > T.table_slots ||
                constructed + (u64)n_warps * CLAIM_CHUNK > stage_cap) {
                ctl.go = 0;
                T.results[TINY_MAX_LEVELS].status = TINY_END_BIG;
            }
            ctl.constructed = constructed;
            for (int i = 0; i < CTR_COUNT; ++i) s_counters[i] = (i == CTR_SEP || i == CTR_STOPAT || i == CTR_SPECIAL) ? VAL_EMPTY : 0ull;
            sQ.block_begin = 0;
            sQ.block_end = n_blocks;
            sQ.tile_begin = 0;
            sQ.tile_end = n_tiles;
            sQ.ticket = CTR_TICKET0;
            sQ.total_before = ctl.log_tail;
            sQ.stage_rows = T.store + ctl.log_tail * (u64)T.P.nvec;
            sQ.stage_cap = stage_cap;
        }
        __syncthreads();
        if (!ctl.go) break;
        if (ctl.constructed == 0) {  // an empty level (e.g. below the atoms' weight)
            if (tid == 0) {
                s_tab[2 * cost] = 0;
                s_tab[2 * cost + 1] = ctl.base;
                T.results[cost - T.cost_first] = WideTinyLevelResult{TINY_BUILT, 0, VAL_EMPTY, VAL_EMPTY, 0, 0};
            }
            __syncthreads();
            continue;
        }
        // ---- enumerate: the warps draw the level's tiles
        {
            Wide2State st;
            while (wide2_next_tile(sQ, W)) wide2_run_tile_any<LW, W2_TINY>(sQ, W, st);
        }
        __threadfence();
        __syncthreads();
        // ---- does the host have to take over?
        if (tid == 0) {
            const u64 sep = s_counters[CTR_SEP];
            ctl.n_staged = s_counters[CTR_CLAIMED];
            ctl.sep_ord = sep;
            ctl.go = 1;
            if (s_counters[CTR_OVERFLOW] || ctl.n_staged > sQ.stage_cap) {
                ctl.go = 0;
                T.results[TINY_MAX_LEVELS].status = TINY_END_OVERFLOW;
            }
            // an exhaustive level with a separating candidate reports "the first chunk whose first separating
            // candidate is fresh" (engine.py:331,425-433): chunk schedule and batch size are the host's business
            if (T.exhaustive && s_counters[CTR_SEPCOUNT]) {
                ctl.go = 0;
                T.results[TINY_MAX_LEVELS].status = TINY_END_SEPARATOR;
            }
            ctl.ord_limit = (!T.exhaustive && sep != VAL_EMPTY) ? sep : VAL_EMPTY - 1;
            ctl.stop_after = (!T.exhaustive && sep != VAL_EMPTY) ? 1 : 0;
        }
        __syncthreads();
        if (!ctl.go) break;  // (the host rebuilds the set: this level's claims are in it)
        // ---- finalise in shared memory: winners bitmap -> ranks -> row directory and ordinals
        const u64 n_bits = ctl.constructed, n_words = (n_bits + 31) >> 5, n_sb = (n_words + 31) >> 5;
        const u64 n_staged = ctl.n_staged, ord_limit = ctl.ord_limit, base = ctl.base, log_tail = ctl.log_tail;
        for (u64 w = tid; w < n_sb * 32; w += n_threads) s_bitmap[w] = 0u;
        __syncthreads();
        for (u64 t = tid; t < n_staged; t += n_threads) {
            const u64 ord = __ldcg(&T.P.stage_ord[t]);
            if (ord <= ord_limit) atomicOr(&s_bitmap[ord >> 5], 1u << (ord & 31));
        }
        __syncthreads();
        if (warp == 0) {  // exclusive popcount prefix per 1024-bit superblock (at most 32 of them)
            uint32_t v = 0;
            if ((u64)lane < n_sb)
                for (int k = 0; k < 32; ++k) v += __popc(s_bitmap[lane * 32 + k]);
            uint32_t incl = v;
#pragma unroll
            for (int d = 1; d < 32; d <<= 1) {
                const uint32_t t = __shfl_up_sync(0xFFFFFFFFu, incl, d);
                if (lane >= d) incl += t;
            }
            s_sbrank[lane] = incl - v;
        }
        __syncthreads();
        for (u64 t = tid; t < n_staged; t += n_threads) {
            const u64 ord = __ldcg(&T.P.stage_ord[t]);
            if (ord <= ord_limit) {  // (else: unused entry, or ordered after the separator)
                const u64 gid = base + ordinal_rank(s_bitmap, s_sbrank, ord);
                T.loc[gid] = log_tail + t;
                T.ords[gid] = ord;
            }
            T.P.stage_ord[t] = VAL_EMPTY;  // clean for the next level
        }
        if (tid == 0) {
            const u64 winners = ordinal_rank(s_bitmap, s_sbrank, n_bits - 1) + ((s_bitmap[(n_bits - 1) >> 5] >> ((n_bits - 1) & 31)) & 1u);
            const u64 sep = ctl.sep_ord;
            s_tab[2 * cost] = winners;
            s_tab[2 * cost + 1] = base;
            T.results[cost - T.cost_first] =
                WideTinyLevelResult{TINY_BUILT, winners, sep, sep < n_bits ? ordinal_rank(s_bitmap, s_sbrank, sep) : VAL_EMPTY,
                                    global_timer_ns() - ctl.t0, n_staged};
            ctl.base = base + winners;
            ctl.log_tail = log_tail + n_staged;
        }
        __threadfence();
        __syncthreads();
        if (ctl.stop_after) break;
    }
}

}  // namespace ltlb200
