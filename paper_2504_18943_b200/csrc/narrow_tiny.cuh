// narrow_tiny.cuh -- the tiny levels of a search, SEVERAL LEVELS IN ONE LAUNCH.
//
// The first levels of every search hold tens to thousands of candidates.  Built one expand_level call at a time
// each of them costs ~75 us of launches and one host synchronisation around ~10 us of work: 1 ms of the 6.3 ms of
// the paper's 7+7 example, and nearly all of a small search (a divide-and-conquer leaf, BASELINE configs[0]).
// The host needs nothing from a level but its size to plan the next one -- and the device can do that planning
// itself.  This kernel is ONE CTA that, level after level,
//
//   plans      the canonical block list of the level from the sizes of the stored levels (the same blocks, in
//              the same order, with the same ordinals as Engine::plan_level on the host, which replays the
//              planning afterwards from the sizes reported here; reference _tasks_for_level, engine.py:219-266),
//   enumerates it with the tile runners and insert_batch of the big kernels, its warps drawing tiles,
//   finalises  it in shared memory (winners bitmap -> ranks -> rows and ordinals appended to the cache),
//
// until a level would exceed TINY_MAX_CANDIDATES candidates, finds a separator, or needs the host (hash set or claim
// arrays too small; an exhaustive level that holds a separating candidate, whose reported separator depends on the
// reference's chunk schedule).  The host hands the levels out one expand_level call at a time (Engine::tiny_*),
// so callers see no difference -- results are bit-identical, which every parity test checks, since every search
// starts here.
#pragma once
#include "narrow.cuh"
#include "tiny_plan.cuh"

namespace ltlb200 {

constexpr int TINY_WARPS = 16;  // measured on spec2 level 8 (13.9 K candidates): 8 warps 172 us, 16 warps 125 us, 32 warps 153 us (64 registers)
constexpr int TINY_TILE_S = 32;  // scalar rows per tile here (the big kernels stage up to TILE_S = 128)
constexpr int TINY_THREADS = 32 * TINY_WARPS;
struct TinyParams {
    NarrowParams P;      // ords = nullptr (no pruning); blocks is replaced by the kernel's shared-memory block list
    uint4 *store;        // writable alias of P.store
    u64 *store_ords;     // winning ordinal of every entry of the cache
    const u64 *level_tab;  // [2c] = n(c), [2c + 1] = base(c) by cost c >= 1: the stored levels (cost < cost_first)
    TinyLevelResult *results;  // [cost - cost_first]
    u64 total;           // entries of the cache before cost_first
    u64 table_slots;
    u64 max_candidates;  // a level beyond this is left to the launches that spread over the whole device
    u64 store_cap;       // entries the cache arrays have room for
    uint32_t op_mask;
    int n_atoms, cost_first, cost_last, exhaustive;
    int weights[16];
};

// per-warp shared state with the row area of a tiny tile: 6 KB instead of 8.3 KB, so that 32 warps fit one SM
struct __align__(16) WarpSharedTiny {
    Parked queue[QUEUE_CAP];
    uint4 rows[TINY_TILE_S];
    u64 term[TINY_TILE_S];
    BlockDesc block;
    u64 ticket, sep_now;
};

// tile runners instantiated with this sink read operand rows with ld.cg: the rows of a level are written by this
// very kernel, which rules out the read-only path
struct TinySink {
    static constexpr bool kCoherentRows = true;
    const NarrowParams &P;
    WarpSharedTiny &ws;
    WarpState &st;
    template <int LW, typename OrdOf>
    __device__ __forceinline__ void emit(const uint4 (&cand)[PROBE_BATCH], const bool (&live)[PROBE_BATCH],
                                         const bool (&known)[PROBE_BATCH], OrdOf ord_of) {
        insert_batch<LW>(P, ws.queue, st, cand, live, known, ord_of);
    }
};

// fetch_tile for counters that live in shared memory (volatile generic loads instead of ld.global.cg)
__device__ __forceinline__ TileFetch tiny_fetch_tile(const NarrowParams &P) {
    TileFetch f;
    if ((threadIdx.x & 31) == 0) {
        f.ovf = *(volatile u64 *)&P.counters[CTR_OVERFLOW];
        f.t = atomicAdd(&P.counters[P.ticket], 1ull);
        if (P.prune_after_sep) f.sep = *(volatile u64 *)&P.counters[CTR_SEP];
    }
    return f;
}

struct TinyControl {  // CTA-wide decisions of thread 0
    int go;           // build this level
    int n_blocks;
    u64 constructed, n_tiles, base;
    u64 n_claimed, ord_limit, sep_ord;
    int stop_after;
    u64 t0;
};

template <int LW>
__global__ void __launch_bounds__(TINY_THREADS, 1) narrow_tiny_levels_kernel(const TinyParams T) {
    extern __shared__ __align__(16) unsigned char s_tiny_raw[];
    WarpSharedTiny *s_warp = reinterpret_cast<WarpSharedTiny *>(s_tiny_raw);
    __shared__ NarrowParams sQ;
    __shared__ TinyControl ctl;
    __shared__ BlockDesc s_blocks[TINY_MAX_BLOCKS];  // the level's block list (planned here, read by open_tile)
    __shared__ u64 s_tab[2 * 64];                    // n(c), base(c) of every level so far
    __shared__ uint32_t s_bitmap[TINY_MAX_CANDIDATES / 32];
    __shared__ uint32_t s_sbrank[TINY_MAX_CANDIDATES / 1024 + 1];
    __shared__ u64 s_counters[CTR_COUNT];  // the level's counters live in shared memory here: every claim-index chunk, tile
                                           // ticket and separator update is a shared-memory atomic, not a trip to the L2
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    WarpSharedTiny &ws = s_warp[warp];
    u64 *counters = s_counters;
    if (tid == 0) {
        sQ = T.P;
        sQ.blocks = s_blocks;
        sQ.counters = s_counters;
        s_counters[CTR_SPECIAL] = T.P.counters[CTR_SPECIAL];  // the all-ones key's register persists across levels and launches
        ctl.base = T.total;
    }
    for (int k = tid; k < 2 * 64; k += TINY_THREADS) s_tab[k] = k < 2 * T.cost_first ? T.level_tab[k] : 0ull;
    __syncthreads();
    for (int cost = T.cost_first; cost <= T.cost_last; ++cost) {
        // ---- plan (thread 0) and reset the level's counters
        if (tid == 0) {
            int n_blocks;
            u64 constructed, n_tiles;
            ctl.t0 = global_timer_ns();
            tiny_plan(T.op_mask, T.n_atoms, T.weights, TINY_TILE_S, s_blocks, cost, s_tab, n_blocks, constructed, n_tiles);
            ctl.go = 1;
            // the host builds levels that are too big for one CTA, or for the set / the claim arrays as they are
            if (constructed == ~0ull || constructed > T.max_candidates || 2 * (ctl.base + constructed) > T.table_slots ||
                constructed + (u64)TINY_WARPS * CLAIM_CHUNK > T.P.claim_cap || ctl.base + constructed > T.store_cap) {
                ctl.go = 0;
                T.results[TINY_MAX_LEVELS].status = TINY_END_BIG;
            }
            ctl.n_blocks = n_blocks;
            ctl.constructed = constructed;
            ctl.n_tiles = n_tiles;
            for (int i = 0; i < CTR_COUNT; ++i)
                if (i != CTR_SPECIAL) counters[i] = (i == CTR_SEP || i == CTR_STOPAT) ? VAL_EMPTY : 0ull;
            sQ.block_begin = 0;
            sQ.block_end = n_blocks;
            sQ.tile_begin = 0;
            sQ.tile_end = n_tiles;
            sQ.ticket = CTR_TICKET0;
            sQ.epoch = (u64)cost << EPOCH_SHIFT;
        }
        __syncthreads();
        if (!ctl.go) break;
        if (ctl.constructed == 0) {  // an empty level (e.g. below the atoms' weight)
            if (tid == 0) {
                s_tab[2 * cost] = 0;
                s_tab[2 * cost + 1] = ctl.base;
                T.results[cost - T.cost_first] = TinyLevelResult{TINY_BUILT, 0, VAL_EMPTY, VAL_EMPTY, 0};
            }
            __syncthreads();
            continue;
        }
        // ---- enumerate: the warps draw the level's tiles
        {
            WarpState st;
            TinySink sink{sQ, ws, st};
            TileFetch next = tiny_fetch_tile(sQ);
            for (;;) {
                const TileFetch cur = next;
                if (!open_tile(sQ, ws, cur)) break;
                next = tiny_fetch_tile(sQ);
                if (run_tile_any<LW>(sQ, ws, sink)) break;
            }
            if (*(volatile u64 *)&counters[CTR_OVERFLOW] == 0ull)
                while (st.qfill > 0u) drain_round(sQ, ws.queue, st);
        }
        __threadfence();
        __syncthreads();
        // ---- does the host have to take over?
        if (tid == 0) {
            const u64 sep = counters[CTR_SEP];
            ctl.n_claimed = counters[CTR_CLAIMED];
            ctl.sep_ord = sep;
            ctl.go = 1;
            if (counters[CTR_OVERFLOW] || ctl.n_claimed > T.P.claim_cap) {
                ctl.go = 0;
                T.results[TINY_MAX_LEVELS].status = TINY_END_OVERFLOW;
            }
            // an exhaustive level with a separating candidate reports "the first chunk whose first separating
            // candidate is fresh" (engine.py:331,425-433): chunk schedule and batch size are the host's business
            if (T.exhaustive && counters[CTR_SEPCOUNT]) {
                ctl.go = 0;
                T.results[TINY_MAX_LEVELS].status = TINY_END_SEPARATOR;
            }
            ctl.ord_limit = (!T.exhaustive && sep != VAL_EMPTY) ? sep : VAL_EMPTY - 1;
            ctl.stop_after = (!T.exhaustive && sep != VAL_EMPTY) ? 1 : 0;
        }
        __syncthreads();
        if (!ctl.go) break;  // (the host rebuilds the set: this level's claims are in it)
        // ---- finalise in shared memory: winners bitmap -> ranks -> append
        const u64 n_bits = ctl.constructed, n_words = (n_bits + 31) >> 5, n_sb = (n_words + 31) >> 5;
        const u64 n_claimed = ctl.n_claimed, ord_limit = ctl.ord_limit, base = ctl.base;
        for (u64 w = tid; w < n_sb * 32; w += TINY_THREADS) s_bitmap[w] = 0u;
        __syncthreads();
        for (u64 t = tid; t < n_claimed; t += TINY_THREADS) {
            const u64 ord = __ldcg(&T.P.claim_ord[t]);
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
        for (u64 t = tid; t < n_claimed; t += TINY_THREADS) {
            const u64 ord = __ldcg(&T.P.claim_ord[t]);
            if (ord > ord_limit) continue;  // unused index, or ordered after the separator
            const u64 gid = base + ordinal_rank(s_bitmap, s_sbrank, ord);
            T.store[gid] = __ldcg(&T.P.claim_key[t]);
            T.store_ords[gid] = ord;
        }
        for (u64 t = tid; t < n_claimed; t += TINY_THREADS) T.P.claim_ord[t] = VAL_EMPTY;  // clean for the next level
        if (tid == 0) {
            const u64 winners = ordinal_rank(s_bitmap, s_sbrank, n_bits - 1) + ((s_bitmap[(n_bits - 1) >> 5] >> ((n_bits - 1) & 31)) & 1u);
            const u64 sep = ctl.sep_ord;
            s_tab[2 * cost] = winners;
            s_tab[2 * cost + 1] = base;
            T.results[cost - T.cost_first] =
                TinyLevelResult{TINY_BUILT, winners, sep, sep < n_bits ? ordinal_rank(s_bitmap, s_sbrank, sep) : VAL_EMPTY,
                                global_timer_ns() - ctl.t0};
            ctl.base = base + winners;
        }
        __threadfence();
        __syncthreads();
        if (ctl.stop_after) break;
    }
    if (tid == 0) T.P.counters[CTR_SPECIAL] = s_counters[CTR_SPECIAL];
}

}  // namespace ltlb200
