// narrow.cuh -- construction + dedup kernels for CMs that fit one uint4 (<= 16 bytes).
//
// Replaces, for one cost level, the reference's _tasks_for_level / _build_chunk /
// _first_occurrence_indices / expand_level merge loop (engine.py:219-451):
//
//   * every candidate of the level has a level-local ORDINAL = its position in the
//     reference's canonical generation order;
//   * the kernel builds candidates tile by tile, checks separation, and inserts
//     (CM -> min ordinal) into an open-addressing hash set in HBM whose slot is one
//     32-byte sector {uint4 key, u64 val}; the key is claimed with ONE 128-bit
//     atomicCAS, so the full CM is compared, never a fingerprint;
//   * val < 2^62  : global id of a CM finalised at an earlier level (immutable)
//     val >= 2^62 : LEVEL_FLAG | ordinal of the best constructor seen so far this level
//     so "first construction wins" is atomicMin on val, and duplicates of old CMs
//     (the common case) cost one sector read and no atomic;
//   * newly claimed slots are appended to a list through per-warp shared-memory
//     buffers (one global atomic per 32 claims) for the finalisation kernels.
#pragma once
#include "cm_ops.cuh"

namespace ltlb200 {

constexpr int CTA_THREADS = 256;
constexpr int TILE_S = 64;      // scalar-dimension rows of a binary tile (staged in shared memory)
#ifndef LTLB200_PROBE_BATCH
#define LTLB200_PROBE_BATCH 4
#endif
#ifndef LTLB200_MIN_CTAS
#define LTLB200_MIN_CTAS 3
#endif
constexpr int PROBE_BATCH = LTLB200_PROBE_BATCH;  // hash probes each thread keeps in flight
constexpr int UNARY_ITEMS = 8;  // candidates per thread in a unary tile
constexpr u64 LEVEL_FLAG = 1ull << 62;
constexpr u64 VAL_EMPTY = ~0ull;
constexpr uint32_t SLOT_SPECIAL = 0xFFFFFFFFu;  // pseudo slot of the all-ones key
constexpr int WARP_BUF = 32 + 32 * PROBE_BATCH;

struct __align__(32) Slot16 {
    uint4 key;  // all ones = empty
    u64 val;
    u64 pad;
};

// kinds of candidate blocks inside a level
enum : uint32_t { BK_UNARY = 0, BK_RECT = 1, BK_TRI = 2 };

struct BlockDesc {
    uint32_t op;
    uint32_t kind;
    uint32_t vec_is_b;  // binary blocks: thread dimension walks the right operand (j) if 1, else the left (i)
    uint32_t from_atoms;  // unary source rows come from the atom table (cost 1)
    u64 a_off, na;      // first global id and count of the left operand level (unary: the source level)
    u64 b_off, nb;      // right operand level
    u64 ord0;           // level-local ordinal of the block's first candidate
    u64 size;           // candidates in the block
    u64 tile0;          // first tile index of the block in the level's flattened tile space
    u64 tiles_v, tiles_s;
};

struct NarrowParams {
    const uint4 *store;  // finalised CMs by global id
    const uint4 *atoms;
    Slot16 *slots;
    u64 slot_mask;
    uint32_t *new_list;
    u64 new_list_cap;
    u64 *counters;  // [0] tile ticket, [1] claimed slots, [2] separator ordinal (min), [3] special-key val, [4] overflow flag
    const BlockDesc *blocks;
    int block_begin, block_end;  // this launch's blocks (all of one operator)
    u64 tile_begin, tile_end;    // their tiles in the level's flattened tile space
    int ticket;                  // index of this launch's ticket counter
    uint4 valid;   // Layout.masks packed
    uint4 target;  // Layout.target packed
    int prune_after_sep;  // non-exhaustive: skip work ordered after the best separator so far
    int special_possible;
    u64 claim_limit;
    u64 *sep_list;  // exhaustive runs: ordinals of every separating candidate (NULL otherwise)
    u64 sep_list_cap;
};

// [5] winners (summary), [6] rank of the separator (summary), [7] separating candidates recorded
// [8..14] one tile ticket per operator launch
enum : int { CTR_UNUSED = 0, CTR_CLAIMED = 1, CTR_SEP = 2, CTR_SPECIAL = 3, CTR_OVERFLOW = 4, CTR_WINNERS = 5, CTR_SEPRANK = 6, CTR_SEPCOUNT = 7, CTR_TICKET0 = 8, CTR_COUNT = 16 };

__device__ __forceinline__ uint4 ld_cg_u4(const uint4 *p) { return __ldcg(p); }

__device__ __forceinline__ uint4 cas128(uint4 *addr, uint4 expect, uint4 desired) {
    u64 e0 = (u64)expect.y << 32 | expect.x, e1 = (u64)expect.w << 32 | expect.z;
    u64 d0 = (u64)desired.y << 32 | desired.x, d1 = (u64)desired.w << 32 | desired.z;
    u64 o0, o1;
    asm volatile(
        "{\n\t"
        ".reg .b128 e, d, o;\n\t"
        "mov.b128 e, {%2, %3};\n\t"
        "mov.b128 d, {%4, %5};\n\t"
        "atom.global.relaxed.gpu.cas.b128 o, [%6], e, d;\n\t"
        "mov.b128 {%0, %1}, o;\n\t"
        "}"
        : "=l"(o0), "=l"(o1)
        : "l"(e0), "l"(e1), "l"(d0), "l"(d1), "l"(addr)
        : "memory");
    return make_uint4((uint32_t)o0, (uint32_t)(o0 >> 32), (uint32_t)o1, (uint32_t)(o1 >> 32));
}

__device__ __forceinline__ bool key_is_empty(uint4 k) { return (k.x & k.y & k.z & k.w) == 0xFFFFFFFFu; }

struct WarpClaims {
    uint32_t *buf;   // WARP_BUF entries of this warp
    uint32_t *fill;  // this warp's fill counter
};

__device__ __forceinline__ void claims_push(const WarpClaims &wc, uint32_t slot) {
    uint32_t pos = atomicAdd(wc.fill, 1u);
    wc.buf[pos] = slot;
}

// warp-collective: move full groups of 32 claims (all of them when `all`) to the global list
__device__ __forceinline__ void claims_flush(const NarrowParams &P, const WarpClaims &wc, bool all) {
    __syncwarp();
    const int lane = threadIdx.x & 31;
    uint32_t fill = *(volatile uint32_t *)wc.fill;
    while (fill >= 32u || (all && fill > 0u)) {
        uint32_t n = fill >= 32u ? 32u : fill;
        u64 base = 0;
        if (lane == 0) base = atomicAdd(&P.counters[CTR_CLAIMED], (u64)n);
        base = __shfl_sync(0xFFFFFFFFu, base, 0);
        if (base + n > P.claim_limit || base + n > P.new_list_cap) {
            if (lane == 0) atomicExch(&P.counters[CTR_OVERFLOW], 1ull);
        } else if ((uint32_t)lane < n) {
            P.new_list[base + lane] = wc.buf[fill - n + lane];
        }
        fill -= n;
    }
    __syncwarp();
    if (lane == 0) *(volatile uint32_t *)wc.fill = fill;
    __syncwarp();
}

// ---- deferred slow path -------------------------------------------------------------
// The hot loop only decides, per candidate, between "duplicate of a CM finalised at an
// earlier level" (the common case: nothing to write) and "needs work".  The latter are
// parked in a per-warp shared-memory queue and drained by the whole warp after each
// batch, one parked candidate per lane: the claim / atomicMin / separator code then runs
// with full lanes and outside the hot loop's register budget.

struct __align__(16) Parked {
    uint4 key;
    u64 ord;
    uint32_t slot;   // where the probe stopped (empty slot or the slot holding `key`)
    uint32_t flags;  // PK_*
};
enum : uint32_t { PK_SEP = 1u, PK_OLD = 2u, PK_SPECIAL = 4u };
constexpr int WARP_QUEUE = 32 * PROBE_BATCH;

struct WarpCtx {
    uint32_t *claim_buf;   // WARP_BUF newly claimed slots waiting for a flush
    uint32_t *claim_fill;
    Parked *queue;         // WARP_QUEUE parked candidates
    uint32_t *queue_fill;
};

__device__ __forceinline__ void park(const WarpCtx &w, uint4 key, u64 ord, u64 slot, uint32_t flags) {
    const uint32_t pos = atomicAdd(w.queue_fill, 1u);
    Parked e;
    e.key = key;
    e.ord = ord;
    e.slot = (uint32_t)slot;
    e.flags = flags;
    w.queue[pos] = e;
}

// Insert (key -> min val) starting at `slot`; returns true when the CM was not stored by
// an earlier level (fresh for this level).
__device__ __forceinline__ bool table_claim(const NarrowParams &P, const WarpCtx &w, uint4 key, u64 val, u64 slot) {
    const uint4 empty = make_uint4(~0u, ~0u, ~0u, ~0u);
    const WarpClaims wc{w.claim_buf, w.claim_fill};
    uint4 k0 = ld_cg_u4(&P.slots[slot].key);
    u64 v0 = __ldcg(&P.slots[slot].val);
    for (int probes = 0;; ++probes) {
        if (v_eq(k0, key)) {
            if (v0 > val) atomicMin(&P.slots[slot].val, val);
            return v0 >= LEVEL_FLAG;
        }
        if (key_is_empty(k0)) {
            uint4 old = cas128(&P.slots[slot].key, empty, key);
            if (key_is_empty(old)) {
                atomicMin(&P.slots[slot].val, val);
                claims_push(wc, (uint32_t)slot);
                return true;
            }
            if (v_eq(old, key)) {
                atomicMin(&P.slots[slot].val, val);
                return true;  // claimed this level by a concurrent constructor
            }
        }
        if (probes > (1 << 16)) {  // table saturated: give up, the host regrows and redoes the level
            atomicExch(&P.counters[CTR_OVERFLOW], 1ull);
            return false;
        }
        slot = (slot + 1) & P.slot_mask;
        k0 = ld_cg_u4(&P.slots[slot].key);
        v0 = __ldcg(&P.slots[slot].val);
    }
}

// warp-collective: resolve every parked candidate, then flush full groups of claims
__device__ __forceinline__ void drain_parked(const NarrowParams &P, const WarpCtx &w) {
    __syncwarp();
    const int lane = threadIdx.x & 31;
    const uint32_t n = *(volatile uint32_t *)w.queue_fill;
    for (uint32_t idx = lane; idx < n; idx += 32) {
        const Parked e = w.queue[idx];
        const u64 val = LEVEL_FLAG | e.ord;
        bool fresh = false;
        if (e.flags & PK_SPECIAL) {
            const u64 old = atomicMin(&P.counters[CTR_SPECIAL], val);
            if (old == VAL_EMPTY) claims_push(WarpClaims{w.claim_buf, w.claim_fill}, SLOT_SPECIAL);
            fresh = old >= LEVEL_FLAG;
        } else if (!(e.flags & PK_OLD)) {
            fresh = table_claim(P, w, e.key, val, e.slot);
        }
        if (e.flags & PK_SEP) {
            if (fresh) atomicMin(&P.counters[CTR_SEP], e.ord);
            if (P.sep_list) {  // exhaustive runs keep every separating ordinal (chunk-exact separator id)
                const u64 pos = atomicAdd(&P.counters[CTR_SEPCOUNT], 1ull);
                if (pos < P.sep_list_cap) P.sep_list[pos] = e.ord;
            }
        }
    }
    __syncwarp();
    if (lane == 0) *(volatile uint32_t *)w.queue_fill = 0;
    claims_flush(P, WarpClaims{w.claim_buf, w.claim_fill}, false);
}

// Probe up to PROBE_BATCH candidates of one thread; all first probes are issued before
// any is consumed so that a warp keeps 32*PROBE_BATCH sectors in flight.  Only the high
// word of a slot's val is read: it alone tells "finalised at an earlier level" (< 2^62).
// `known[r]`: the candidate equals one of its operands, i.e. a CM that is already in the
// cache -- a duplicate by construction, no probe needed.  `ord_of(r)` recomputes the
// ordinal for the few candidates that get parked, so ordinals hold no registers here.
template <int LW, typename OrdOf>
__device__ __forceinline__ void insert_batch(const NarrowParams &P, const WarpCtx &w,
                                             const uint4 (&cand)[PROBE_BATCH], const bool (&live)[PROBE_BATCH],
                                             const bool (&known)[PROBE_BATCH], OrdOf ord_of) {
    constexpr uint32_t FLAG_HI = (uint32_t)(LEVEL_FLAG >> 32);
    const uint32_t mask32 = (uint32_t)P.slot_mask;
    uint32_t slot[PROBE_BATCH];
    uint4 k0[PROBE_BATCH];
    uint32_t vhi[PROBE_BATCH];
#pragma unroll
    for (int r = 0; r < PROBE_BATCH; ++r) {
        slot[r] = (uint32_t)hash_vec(cand[r], 0) & mask32;
        if (live[r] && !known[r]) {
            k0[r] = ld_cg_u4(&P.slots[slot[r]].key);
            vhi[r] = __ldcg(reinterpret_cast<const uint32_t *>(&P.slots[slot[r]].val) + 1);
        }
    }
#pragma unroll
    for (int r = 0; r < PROBE_BATCH; ++r) {
        if (!live[r]) continue;
        uint32_t flags = cm_sep_diff<LW>(cand[r], P.target) == 0u ? PK_SEP : 0u;
        uint32_t s = slot[r];
        if (known[r]) {
            flags |= PK_OLD;
        } else if (P.special_possible && key_is_empty(cand[r])) {
            flags |= PK_SPECIAL;
        } else {
            uint4 k = k0[r];
            uint32_t v = vhi[r];
            while (!v_eq(k, cand[r]) && !key_is_empty(k)) {  // linear probing past other CMs
                s = (s + 1) & mask32;
                k = ld_cg_u4(&P.slots[s].key);
                v = __ldcg(reinterpret_cast<const uint32_t *>(&P.slots[s].val) + 1);
            }
            if (v_eq(k, cand[r]) && v < FLAG_HI) flags |= PK_OLD;  // duplicate of an earlier level
        }
        if (flags != PK_OLD) park(w, cand[r], ord_of(r), s, flags);
    }
    drain_parked(P, w);
}

template <int LW, int OP>
__device__ __forceinline__ void run_unary_tile(const NarrowParams &P, const WarpCtx &wc, const BlockDesc &B,
                                               u64 tile_local, u64 sep_now) {
    const uint4 *src = B.from_atoms ? P.atoms : P.store + B.a_off;
    const u64 first = tile_local * (u64)(CTA_THREADS * UNARY_ITEMS) + threadIdx.x;
    const u64 ord0 = B.ord0;
#pragma unroll 1
    for (int g = 0; g < UNARY_ITEMS; g += PROBE_BATCH) {
        uint4 cand[PROBE_BATCH];
        bool live[PROBE_BATCH], known[PROBE_BATCH];
        uint4 x[PROBE_BATCH];
        auto ord_of = [&](int r) { return ord0 + first + (u64)(g + r) * CTA_THREADS; };
#pragma unroll
        for (int r = 0; r < PROBE_BATCH; ++r) {
            const u64 i = first + (u64)(g + r) * CTA_THREADS;
            live[r] = i < B.na && ord0 + i <= sep_now;
            x[r] = live[r] ? __ldg(src + i) : make_uint4(0, 0, 0, 0);
        }
#pragma unroll
        for (int r = 0; r < PROBE_BATCH; ++r) {
            cand[r] = cm_apply<LW, OP>(x[r], x[r], P.valid);
            known[r] = OP != OP_ATOM && v_eq(cand[r], x[r]);
        }
        insert_batch<LW>(P, wc, cand, live, known, ord_of);
    }
}

// Binary tile: each thread keeps one row of the "vector" operand in registers and walks
// up to TILE_S rows of the "scalar" operand staged in shared memory together with the
// row's ordinal term, so that a candidate's ordinal is one 64-bit add:
//   rectangle  ord = ord0 + i*nb + j          triangle (i <= j < n)  ord = ord0 + i*n - i(i-1)/2 + (j - i)
template <int LW, int OP>
__device__ __forceinline__ void run_binary_tile(const NarrowParams &P, const WarpCtx &wc, const BlockDesc &B,
                                                u64 tile_local, uint4 *s_rows, u64 *s_term, u64 sep_now) {
    const bool tri = B.kind == BK_TRI;
    const bool vec_b = B.vec_is_b != 0;
    // tile order follows the canonical order: left operand (i) outer, right operand (j) inner
    u64 tv, ts;
    if (vec_b) { ts = tile_local / B.tiles_v; tv = tile_local % B.tiles_v; }
    else { tv = tile_local / B.tiles_s; ts = tile_local % B.tiles_s; }
    const u64 n_vec = vec_b ? B.nb : B.na, n_sc = vec_b ? B.na : B.nb;
    const u64 v0 = tv * CTA_THREADS, s0 = ts * TILE_S;
    const int s_cnt = (int)min((u64)TILE_S, n_sc - s0);
    if (tri && v0 + CTA_THREADS - 1 < s0) return;  // tile entirely below the diagonal (j < i)
    const uint4 *vec_rows = P.store + (vec_b ? B.b_off : B.a_off);
    const uint4 *sc_rows = P.store + (vec_b ? B.a_off : B.b_off);
    __syncthreads();  // previous tile's readers of the staged rows are done
    if ((int)threadIdx.x < s_cnt) {
        const u64 s = s0 + threadIdx.x;
        s_rows[threadIdx.x] = __ldg(sc_rows + s);
        // scalar-row part of the ordinal; the thread part is j (vec_b) or ord0 + i*nb (!vec_b)
        s_term[threadIdx.x] = !vec_b ? s : B.ord0 + (tri ? s * B.na - (s ? (s * (s - 1)) / 2 : 0) - s : s * B.nb);
    }
    __syncthreads();
    const u64 v = v0 + threadIdx.x;
    const bool v_ok = v < n_vec;
    const uint4 xv = v_ok ? __ldg(vec_rows + v) : make_uint4(0, 0, 0, 0);
    const u64 thread_term = vec_b ? v : B.ord0 + v * B.nb;
    // triangle: row s0+sr pairs with columns j >= i only
    const int first_bad = tri ? (v >= s0 ? (int)min((u64)s_cnt, v - s0 + 1) : 0) : s_cnt;
    const int s_live = v_ok ? first_bad : 0;
    const bool prune = sep_now != ~0ull;
#pragma unroll 1
    for (int g = 0; g < s_cnt; g += PROBE_BATCH) {
        uint4 cand[PROBE_BATCH];
        bool live[PROBE_BATCH], known[PROBE_BATCH];
        auto ord_of = [&](int r) { return s_term[min(g + r, s_cnt - 1)] + thread_term; };
#pragma unroll
        for (int r = 0; r < PROBE_BATCH; ++r) {
            const int sr = min(g + r, s_cnt - 1);
            const uint4 xs = s_rows[sr];
            live[r] = g + r < s_live && (!prune || s_term[sr] + thread_term <= sep_now);
            const uint4 a = vec_b ? xs : xv, b = vec_b ? xv : xs;
            cand[r] = cm_apply<LW, OP>(a, b, P.valid);
            known[r] = v_eq(cand[r], a) || v_eq(cand[r], b);
        }
        insert_batch<LW>(P, wc, cand, live, known, ord_of);
    }
}

// One persistent launch per (level, operator): CTAs draw tiles of the operator's blocks from
// a ticket counter in canonical order.  The operator is a template parameter so that each
// kernel holds exactly one hot loop (a single kernel switching over all operators needed
// > 240 registers); launches of one level run back to back on the stream, in canonical
// operator order, with no host synchronisation in between.
template <int LW, int OP>
__global__ void __launch_bounds__(CTA_THREADS, LTLB200_MIN_CTAS) narrow_level_kernel(const NarrowParams P) {
    __shared__ BlockDesc B;
    __shared__ uint4 s_rows[TILE_S];
    __shared__ u64 s_term[TILE_S];
    __shared__ uint32_t s_claims[(CTA_THREADS / 32) * WARP_BUF];
    __shared__ uint32_t s_fill[CTA_THREADS / 32];
    __shared__ Parked s_queue[(CTA_THREADS / 32) * WARP_QUEUE];
    __shared__ uint32_t s_qfill[CTA_THREADS / 32];
    __shared__ u64 s_ticket;
    __shared__ u64 s_sep;
    const int warp = threadIdx.x >> 5;
    const WarpCtx wc{s_claims + warp * WARP_BUF, s_fill + warp, s_queue + warp * WARP_QUEUE, s_qfill + warp};
    if ((threadIdx.x & 31) == 0) {
        s_fill[warp] = 0;
        s_qfill[warp] = 0;
    }
    __syncthreads();
    for (;;) {
        __syncthreads();
        if (threadIdx.x == 0) {
            u64 t = P.tile_end;
            if (*(volatile u64 *)&P.counters[CTR_OVERFLOW] == 0ull) t = P.tile_begin + atomicAdd(&P.counters[P.ticket], 1ull);
            s_ticket = t;
            s_sep = P.prune_after_sep ? *(volatile u64 *)&P.counters[CTR_SEP] : (u64)~0ull;
            if (t < P.tile_end) {
                int bi = P.block_begin;
                while (bi + 1 < P.block_end && t >= P.blocks[bi + 1].tile0) ++bi;
                B = P.blocks[bi];
            }
        }
        __syncthreads();
        const u64 tile = s_ticket;
        const u64 sep_now = s_sep;
        if (tile >= P.tile_end) break;
        if (B.ord0 > sep_now) continue;  // the whole block is ordered after the separator
        if constexpr (OP == OP_AND || OP == OP_OR || OP == OP_UNTIL)
            run_binary_tile<LW, OP>(P, wc, B, tile - B.tile0, s_rows, s_term, sep_now);
        else
            run_unary_tile<LW, OP>(P, wc, B, tile - B.tile0, sep_now);
    }
    claims_flush(P, WarpClaims{wc.claim_buf, wc.claim_fill}, true);
}

// ---- finalisation: order the level's winners by ordinal without a sort -------------
// A bitmap with one bit per candidate ordinal marks the winners; a popcount prefix over
// 1024-bit superblocks turns an ordinal into its rank, i.e. the entry's position in the
// level (reference order = ordinal order), and the rows are scattered straight to it.

struct FinalizeParams {
    Slot16 *slots;
    const uint32_t *new_list;
    u64 n_claimed;
    u64 *counters;
    uint32_t *bitmap;        // one bit per ordinal
    const uint32_t *sb_rank; // exclusive popcount prefix per 32-word superblock
    u64 ord_limit;           // keep ordinals <= limit (separator in a non-exhaustive run, else all ones)
    uint4 *store;
    u64 *ords;
    u64 base;                // global id of the level's first entry
};

__device__ __forceinline__ u64 claimed_val(const FinalizeParams &F, uint32_t slot) {
    return slot == SLOT_SPECIAL ? F.counters[CTR_SPECIAL] : F.slots[slot].val;
}

__global__ void __launch_bounds__(256) narrow_mark_kernel(const FinalizeParams F) {
    for (u64 t = (u64)blockIdx.x * blockDim.x + threadIdx.x; t < F.n_claimed; t += (u64)gridDim.x * blockDim.x) {
        const u64 ord = claimed_val(F, F.new_list[t]) & ~LEVEL_FLAG;
        if (ord <= F.ord_limit) atomicOr(&F.bitmap[ord >> 5], 1u << (ord & 31));
    }
}

__device__ __forceinline__ u64 ordinal_rank(const uint32_t *bitmap, const uint32_t *sb_rank, u64 ord) {
    const u64 word = ord >> 5, sb = word >> 5;
    u64 rank = sb_rank[sb];
    for (u64 w = sb << 5; w < word; ++w) rank += __popc(bitmap[w]);
    return rank + __popc(bitmap[word] & ((1u << (ord & 31)) - 1u));
}

__global__ void __launch_bounds__(256) narrow_scatter_kernel(const FinalizeParams F) {
    for (u64 t = (u64)blockIdx.x * blockDim.x + threadIdx.x; t < F.n_claimed; t += (u64)gridDim.x * blockDim.x) {
        const uint32_t slot = F.new_list[t];
        const u64 ord = claimed_val(F, slot) & ~LEVEL_FLAG;
        if (ord > F.ord_limit) continue;  // ordered after the separator: not part of the level
        const u64 gid = F.base + ordinal_rank(F.bitmap, F.sb_rank, ord);
        F.store[gid] = slot == SLOT_SPECIAL ? make_uint4(~0u, ~0u, ~0u, ~0u) : F.slots[slot].key;
        F.ords[gid] = ord;
        if (slot == SLOT_SPECIAL) F.counters[CTR_SPECIAL] = gid;
        else F.slots[slot].val = gid;
    }
}

// re-insert finalised rows [first, first+count) into a fresh table (regrow / rollback)
__global__ void __launch_bounds__(256) narrow_rebuild_kernel(Slot16 *slots, u64 slot_mask, const uint4 *store,
                                                             u64 first, u64 count, u64 *counters) {
    const uint4 empty = make_uint4(~0u, ~0u, ~0u, ~0u);
    for (u64 t = (u64)blockIdx.x * blockDim.x + threadIdx.x; t < count; t += (u64)gridDim.x * blockDim.x) {
        const u64 gid = first + t;
        const uint4 key = store[gid];
        if (key_is_empty(key)) {
            counters[CTR_SPECIAL] = gid;
            continue;
        }
        u64 slot = hash_vec(key, 0) & slot_mask;
        for (;;) {
            uint4 old = cas128(&slots[slot].key, empty, key);
            if (key_is_empty(old)) {
                slots[slot].val = gid;
                break;
            }
            slot = (slot + 1) & slot_mask;
        }
    }
}

}  // namespace ltlb200
