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
//   * val = [epoch:16 | claim index:48], all ones while unpublished.  The epoch is the cost
//     level that stored the CM, so "duplicate of an earlier level" (the common case) is one
//     compare on the high word of the probed sector and needs no write at all, and no slot
//     has to be rewritten when a level is finalised;
//   * this level's new CMs live in two dense arrays indexed by claim index -- claim_key
//     (the CM) and claim_ord (the smallest ordinal that built it, atomicMin) -- which
//     finalisation reads sequentially; "first construction wins" is that atomicMin.
//
// Execution shape (what the first ncu capture asked for): tiles are owned by WARPS, not
// CTAs, so there is no block barrier anywhere; the hot loop issues exactly one probe per
// candidate (PROBE_BATCH of them in flight per lane) and never loops on a probe chain;
// whatever is not settled by that one probe -- a new CM, a collision, a same-level
// duplicate, a separating candidate -- is parked in a per-warp shared-memory queue and
// resolved in ROUNDS of 32 parked candidates, one per lane, re-compacted after every
// probe step, so chains of different length never idle a warp's lanes.  Queue and claim
// positions come from warp ballots, not from shared-memory atomics.
#pragma once
#include "cm_ops.cuh"
#include "regex_ops.cuh"

namespace ltlb200 {

#ifndef LTLB200_PROBE_BATCH
#define LTLB200_PROBE_BATCH 4
#endif
// CTAs per SM of the direct kernel.  Measured on spec2 (enumerate ms per search): 3 -> 5.34,
// 4 -> 5.78, 5 -> 6.47, 6 -> 7.10: registers without spills beat resident warps.
#ifndef LTLB200_MIN_CTAS
#define LTLB200_MIN_CTAS 3
#endif
#ifndef LTLB200_TILE_S
#define LTLB200_TILE_S 128
#endif
constexpr int WARPS_PER_CTA = 4;
constexpr int CTA_THREADS = 32 * WARPS_PER_CTA;
constexpr int PROBE_BATCH = LTLB200_PROBE_BATCH;  // first probes each lane keeps in flight
constexpr int TILE_V = 32;                        // vector-dimension rows of a tile: one per lane
constexpr int TILE_S = LTLB200_TILE_S;            // scalar-dimension rows of a binary tile (staged in shared memory)
constexpr int UNARY_ITEMS = 64;                   // candidates per lane in a unary tile
constexpr int QUEUE_CAP = 32 * PROBE_BATCH + 32;
constexpr int CLAIM_CHUNK = 64;  // claim indices a warp reserves at a time
constexpr u64 VAL_EMPTY = ~0ull;
constexpr int EPOCH_SHIFT = 48;
constexpr u64 CLAIM_IDX_MASK = (1ull << EPOCH_SHIFT) - 1;

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
    uint32_t vec_is_b;    // binary blocks: lane dimension walks the right operand (j) if 1, else the left (i)
    uint32_t from_atoms;  // unary source rows come from the atom table (cost 1)
    u64 a_off, na;        // first global id and count of the left operand level (unary: the source level)
    u64 b_off, nb;        // right operand level
    u64 ord0;             // level-local ordinal of the block's first candidate
    u64 size;             // candidates in the block
    u64 tile0;            // first tile index of the block in the level's flattened tile space
    u64 tiles_v, tiles_s;
    // Associativity pruning (AND blocks of a store whose levels are all complete and were built with one
    // operator set): an operand row whose own winning ordinal lies in [lo, hi) makes the candidate a
    // duplicate by construction (run_binary_tile).  Left operand: it is itself an AND node.  Right operand:
    // it is an AND node whose left child costs less than this block's left operand.  lo == hi: no such rows.
    u64 skip_a_lo, skip_a_hi, skip_b_lo, skip_b_hi;
    uint32_t c_left;  // cost of the left operand level (0 for unary blocks)
    uint32_t vg;  // vector groups (of 32 rows) per tile; > 1 when the scalar operand has few rows
    uint32_t tile_s;  // scalar rows per tile (<= TILE_S) or, for unary blocks, candidates per lane per tile;
                      // the host shrinks tiles of small blocks so that they still spread over the whole GPU
};

struct NarrowParams {
    const uint4 *store;  // finalised CMs by global id
    const uint4 *atoms;
    Slot16 *slots;
    u64 slot_mask;
    uint4 *claim_key;  // this level's new CMs by claim index
    u64 *claim_ord;    // smallest ordinal per claim index (all ones = index reserved but unused)
    u64 claim_cap;
    u64 epoch;         // this level's epoch (= cost), already shifted into the val's high bits
    u64 *counters;     // see CTR_*
    const BlockDesc *blocks;
    int block_begin, block_end;  // this launch's blocks (all of one operator)
    u64 tile_begin, tile_end;    // their tiles in the level's flattened tile space
    u64 shard_stride, shard_offset;  // this rank takes tiles tile_begin + shard_offset + k*shard_stride (1, 0 = all)
    int ticket;                  // index of this launch's ticket counter
    uint4 valid;                 // Layout.masks packed
    uint4 target;                // Layout.target packed
    int prune_after_sep;         // non-exhaustive: skip work ordered after the best separator so far
    int special_possible;
    u64 *sep_list;  // exhaustive runs: ordinals of every separating candidate (NULL otherwise)
    u64 sep_list_cap;
    const u64 *ords;  // winning ordinal of every finalised CM by global id, or NULL: no associativity pruning
    // Non-exhaustive level over a store that already holds a separating CM: the reference truncates every chunk
    // at its first separating candidate, fresh or not (engine.py:334-335).  `dead` = dead_n sorted, disjoint
    // ordinal ranges [lo, hi) -- the rest of each such chunk -- whose candidates do not exist for this level.
    const u64 *dead;
    uint32_t dead_n;
    int scan_only;  // the pass that finds those chunks: only record the ordinal of every separating candidate
    // One search sharded over several GPUs (narrow_route_kernel): candidates are not probed here but appended as
    // records {CM, ordinal} to the region of their hash owner, route_world regions of route_cap records each.
    uint4 *route_rows;
    u64 *route_ords;
    u64 route_cap;
    u64 *route_counts;     // records appended per owner; keeps counting past route_cap (the exact need of a redo)
    uint32_t route_world;
    int route_sep_any;     // the store holds no separating CM: every separating candidate is fresh w.r.t. earlier levels
};

// [0] set when the level's deadline passed while it was being built, [15] that deadline on the device's
// nanosecond timer (all ones = none), [1] claim indices reserved, [2] separator ordinal (min), [3] special-key val (persists across levels),
// [4] overflow flag, [5] winners (summary), [6] rank of the separator (summary),
// [7] separating candidates recorded, [8..14] one tile ticket per operator launch
enum : int { CTR_TIMEOUT = 0, CTR_CLAIMED = 1, CTR_SEP = 2, CTR_SPECIAL = 3, CTR_OVERFLOW = 4, CTR_WINNERS = 5, CTR_SEPRANK = 6, CTR_SEPCOUNT = 7, CTR_TICKET0 = 8, CTR_STOPAT = 15, CTR_COUNT = 16 };

__device__ __forceinline__ u64 global_timer_ns() {
    u64 t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}

// The reference polls its deadline before every chunk of a level (engine.py:416-417); here every warp polls it
// as it draws tile tickets: past the deadline no further tile is started, what was built so far is kept
// (the reference's partial level) and the host reports "time budget exhausted".
__device__ __forceinline__ bool deadline_passed(u64 *counters) {
    const u64 stop_at = *(volatile const u64 *)&counters[CTR_STOPAT];  // (generic: the tiny-levels kernel keeps its counters in shared memory)
    if (stop_at == ~0ull || global_timer_ns() <= stop_at) return false;
    atomicExch(&counters[CTR_TIMEOUT], 1ull);
    return true;
}

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

// one 32-byte slot = one sector = one 256-bit load: key and val are a consistent snapshot.
// Relaxed gpu-scope load (LDG.E.256.STRONG.GPU): served by the L2, never by a stale L1 line.
__device__ __forceinline__ void ld_slot(const Slot16 *p, uint4 &key, u64 &val) {
    uint32_t v0, v1, pad0, pad1;
    asm volatile("ld.relaxed.gpu.global.v8.u32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                 : "=r"(key.x), "=r"(key.y), "=r"(key.z), "=r"(key.w), "=r"(v0), "=r"(v1), "=r"(pad0), "=r"(pad1)
                 : "l"(p)
                 : "memory");
    (void)pad0;
    (void)pad1;
    val = (u64)v1 << 32 | v0;
}

// hash owner of a CM in a sharded search: independent of the slot hash
__device__ __forceinline__ uint32_t key_owner(uint4 key, uint32_t owners) {
    return hash_vec(key, 0x5BD1E995u) % owners;
}

// ---- per-warp state -------------------------------------------------------------------

struct __align__(16) Parked {
    uint4 key;
    u64 ord;
    uint32_t slot;   // slot to look at next
    uint32_t flags;  // PK_*
};
// PK_OLD: known duplicate of an earlier level (parked only because it separates)
// PK_EMPTY: the first probe saw this slot empty, go straight to the CAS
enum : uint32_t { PK_SEP = 1u, PK_OLD = 2u, PK_SPECIAL = 4u, PK_EMPTY = 8u };

struct __align__(16) WarpShared {
    Parked queue[QUEUE_CAP];
    uint4 rows[TILE_S];  // scalar-operand rows of the current binary tile
    u64 term[TILE_S];    // their ordinal terms
    BlockDesc block;
    u64 ticket, sep_now;
};

struct WarpState {  // warp-uniform registers
    uint32_t qfill = 0;
    u64 chunk_next = 0, chunk_end = 0;  // claim indices reserved for this warp
};

__device__ __forceinline__ uint32_t lanemask_lt() {
    uint32_t m;
    asm("mov.u32 %0, %%lanemask_lt;" : "=r"(m));
    return m;
}

// Lanes with `attempt` set reserve one claim index each (ballot ranks, no atomics); indices come
// from the warp's current chunk, and when it runs out mid-way the tail continues in a freshly
// reserved chunk (nothing is abandoned).  Warp-uniform control flow; every lane must call.
__device__ __forceinline__ u64 reserve_claims(const NarrowParams &P, WarpState &st, bool attempt) {
    const uint32_t ma = __ballot_sync(0xFFFFFFFFu, attempt);
    const uint32_t n_att = __popc(ma);
    if (n_att == 0u) return 0;
    const uint32_t rem = (uint32_t)(st.chunk_end - st.chunk_next);
    u64 fresh_chunk = 0;
    if (n_att > rem) {
        if ((threadIdx.x & 31) == 0) fresh_chunk = atomicAdd(&P.counters[CTR_CLAIMED], (u64)CLAIM_CHUNK);
        fresh_chunk = __shfl_sync(0xFFFFFFFFu, fresh_chunk, 0);
    }
    const uint32_t my_rank = __popc(ma & lanemask_lt());
    const u64 my_idx = my_rank < rem ? st.chunk_next + my_rank : fresh_chunk + (my_rank - rem);
    if (n_att > rem) {
        st.chunk_next = fresh_chunk + (n_att - rem);
        st.chunk_end = fresh_chunk + CLAIM_CHUNK;
    } else {
        st.chunk_next += n_att;
    }
    return my_idx;
}

// One resolution round: the top (up to) 32 parked candidates take one probe step each.
// Settled ones leave (recording separators), the rest are re-queued compacted.
__device__ __forceinline__ void drain_round(const NarrowParams &P, Parked *queue, WarpState &st) {
    const int lane = threadIdx.x & 31;
    const uint32_t lt = lanemask_lt();
    const uint32_t take = st.qfill < 32u ? st.qfill : 32u;
    const uint32_t base = st.qfill - take;
    const bool active = (uint32_t)lane < take;
    Parked e = queue[base + (active ? lane : 0)];
    __syncwarp();  // every lane holds its entry before the queue slots are reused
    const uint4 empty = make_uint4(~0u, ~0u, ~0u, ~0u);
    const bool special = active && (e.flags & PK_SPECIAL);
    const bool probing = active && !(e.flags & (PK_SPECIAL | PK_OLD));
    Slot16 *slot = &P.slots[e.slot];
    // ---- look at the slot (skipped when the first probe already saw it empty)
    uint4 k = empty;
    u64 v = VAL_EMPTY;
    if (probing && !(e.flags & PK_EMPTY)) ld_slot(slot, k, v);
    if (special) v = *(volatile u64 *)&P.counters[CTR_SPECIAL];
    // ---- lanes that will try to claim reserve their claim index first
    const bool attempt = (probing && key_is_empty(k)) || (special && v == VAL_EMPTY);
    const u64 my_idx = reserve_claims(P, st, attempt);
    bool again = false, fresh = false, settled_here = false;
    if (attempt) {
        if (my_idx >= P.claim_cap) {  // claim arrays exhausted: the host regrows and redoes the level
            atomicExch(&P.counters[CTR_OVERFLOW], 1ull);
        } else if (special) {
            const u64 old = atomicCAS(&P.counters[CTR_SPECIAL], VAL_EMPTY, P.epoch | my_idx);
            if (old == VAL_EMPTY) {
                P.claim_key[my_idx] = empty;
                atomicMin(&P.claim_ord[my_idx], e.ord);
                fresh = settled_here = true;
            } else {
                v = old;
            }
        } else {
            const uint4 old = cas128(&slot->key, empty, e.key);
            if (key_is_empty(old)) {  // claimed: publish the claim index, record key and ordinal
                __stcg(&slot->val, P.epoch | my_idx);
                P.claim_key[my_idx] = e.key;
                atomicMin(&P.claim_ord[my_idx], e.ord);
                fresh = settled_here = true;
            } else {
                k = old;
                v = VAL_EMPTY;  // whoever claimed it: their val may not be visible yet, look again next round
            }
        }
    }
    if ((probing || special) && !settled_here) {
        if (special || v_eq(k, e.key)) {
            if (v == VAL_EMPTY) {  // key is there, claim index not published yet
                again = true;
                e.flags &= ~PK_EMPTY;
            } else if (v >= P.epoch) {  // built earlier in this level: keep the smaller ordinal
                atomicMin(&P.claim_ord[v & CLAIM_IDX_MASK], e.ord);
                fresh = true;
            }  // else: stored by an earlier level
        } else {  // another CM lives here: linear probing
            again = true;
            e.slot = (e.slot + 1) & (uint32_t)P.slot_mask;
            e.flags &= ~PK_EMPTY;
        }
    }
    if (active && !again && (e.flags & PK_SEP)) {
        if (fresh) atomicMin(&P.counters[CTR_SEP], e.ord);
        if (P.sep_list) {  // exhaustive runs keep every separating ordinal (chunk-exact separator id)
            const u64 pos = atomicAdd(&P.counters[CTR_SEPCOUNT], 1ull);
            if (pos < P.sep_list_cap) P.sep_list[pos] = e.ord;
        }
    }
    const uint32_t mq = __ballot_sync(0xFFFFFFFFu, again);
    if (again) queue[base + __popc(mq & lt)] = e;
    st.qfill = base + __popc(mq);
    __syncwarp();
}

// Probe PROBE_BATCH candidates of one lane with ONE sector read each (all issued before any
// is consumed) and settle the three common outcomes on the spot:
//   * the slot holds the same CM, stored by an earlier level   -> duplicate, nothing to write;
//   * the slot holds the same CM, claimed earlier in this level -> one fire-and-forget min on its ordinal;
//   * the slot is empty -> reserve a claim index, claim the key with a 128-bit CAS (all CASes of
//     the batch in flight together), publish index / key / ordinal.
// What is left -- collisions, lost CAS races, claims whose index is not published yet, the
// all-ones key and every separating candidate -- is parked and resolved by drain_round.
// `known[r]`: the candidate equals one of its operands, i.e. a CM already in the cache -- a
// duplicate by construction, no probe.  `ord_of(r)` recomputes the ordinal where one is
// needed, so ordinals hold no registers in the hot loop.
template <int LW, typename OrdOf>
__device__ __forceinline__ void insert_batch(const NarrowParams &P, Parked *queue, WarpState &st,
                                             const uint4 (&cand)[PROBE_BATCH], const bool (&live)[PROBE_BATCH],
                                             const bool (&known_in)[PROBE_BATCH], OrdOf ord_of) {
    const uint32_t mask32 = (uint32_t)P.slot_mask;
    const uint32_t lt = lanemask_lt();
    const uint4 empty = make_uint4(~0u, ~0u, ~0u, ~0u);
    enum : uint32_t { ACT_NONE = 0u, ACT_PARK = 1u, ACT_CLAIM = 2u };
    uint32_t slot[PROBE_BATCH], flags[PROBE_BATCH], act[PROBE_BATCH];
    uint4 k0[PROBE_BATCH];
    u64 v0[PROBE_BATCH];
    bool known[PROBE_BATCH];
#pragma unroll
    for (int r = 0; r < PROBE_BATCH; ++r) {
        slot[r] = hash_vec(cand[r], 0u);
        known[r] = known_in[r];
    }
#pragma unroll
    for (int r = 0; r < PROBE_BATCH; ++r) {
        slot[r] &= mask32;
        if (live[r] && !known[r]) ld_slot(&P.slots[slot[r]], k0[r], v0[r]);
    }
#pragma unroll
    for (int r = 0; r < PROBE_BATCH; ++r) {
        const bool sep = cm_sep_diff<LW>(cand[r], P.target, P.valid) == 0u;
        flags[r] = sep ? PK_SEP : 0u;
        act[r] = ACT_NONE;
        if (!live[r]) continue;
        if (known[r]) {
            if (sep) { flags[r] |= PK_OLD; act[r] = ACT_PARK; }
        } else if (P.special_possible && key_is_empty(cand[r])) {
            flags[r] |= PK_SPECIAL;
            act[r] = ACT_PARK;
        } else if (v_eq(k0[r], cand[r])) {
            if (v0[r] == VAL_EMPTY || sep) {
                act[r] = ACT_PARK;  // index not published yet / separating: the queue handles it
            } else if (v0[r] >= P.epoch) {
                atomicMin(&P.claim_ord[v0[r] & CLAIM_IDX_MASK], ord_of(r));  // same level: keep the smaller ordinal
            }  // else: stored by an earlier level
        } else if (key_is_empty(k0[r])) {
            if (sep) { flags[r] |= PK_EMPTY; act[r] = ACT_PARK; }
            else act[r] = ACT_CLAIM;
        } else {
            slot[r] = (slot[r] + 1) & mask32;  // collision: continue at the next slot
            act[r] = ACT_PARK;
        }
    }
    // ---- claims: indices first (warp-uniform), then every CAS of the batch in flight at once
    u64 idx[PROBE_BATCH];
#pragma unroll
    for (int r = 0; r < PROBE_BATCH; ++r) {
        idx[r] = reserve_claims(P, st, act[r] == ACT_CLAIM);
        if (act[r] == ACT_CLAIM && idx[r] >= P.claim_cap) {  // claim arrays exhausted: the host regrows and redoes the level
            atomicExch(&P.counters[CTR_OVERFLOW], 1ull);
            act[r] = ACT_NONE;
        }
    }
#pragma unroll
    for (int r = 0; r < PROBE_BATCH; ++r)
        if (act[r] == ACT_CLAIM) k0[r] = cas128(&P.slots[slot[r]].key, empty, cand[r]);
#pragma unroll
    for (int r = 0; r < PROBE_BATCH; ++r) {
        if (act[r] == ACT_CLAIM) {
            if (key_is_empty(k0[r])) {  // claimed: publish the claim index, record key and ordinal
                __stcg(&P.slots[slot[r]].val, P.epoch | idx[r]);
                P.claim_key[idx[r]] = cand[r];
                atomicMin(&P.claim_ord[idx[r]], ord_of(r));
                act[r] = ACT_NONE;
            } else {
                act[r] = ACT_PARK;  // lost the race: look at the slot again (the reserved index stays unused)
            }
        }
        const bool need = act[r] == ACT_PARK;
        const uint32_t m = __ballot_sync(0xFFFFFFFFu, need);
        if (need) {
            Parked e;
            e.key = cand[r];
            e.ord = ord_of(r);
            e.slot = slot[r];
            e.flags = flags[r];
            queue[st.qfill + __popc(m & lt)] = e;
        }
        st.qfill += __popc(m);
    }
    __syncwarp();
    while (st.qfill >= 32u) drain_round(P, queue, st);
}

// rank of an ordinal among the level's winners: bits set before it in the winners bitmap (one bit per ordinal,
// exclusive popcount prefixes per 1024-bit superblock)
__device__ __forceinline__ u64 ordinal_rank(const uint32_t *bitmap, const uint32_t *sb_rank, u64 ord) {
    const u64 word = ord >> 5, sb = word >> 5;
    u64 rank = sb_rank[sb];
    for (u64 w = sb << 5; w < word; ++w) rank += __popc(bitmap[w]);
    return rank + __popc(bitmap[word] & ((1u << (ord & 31)) - 1u));
}

// operand rows come through the read-only path, except in a kernel that writes rows itself (narrow_tiny.cuh)
template <class S, class = void>
struct sink_coherent_rows : std::false_type {};
template <class S>
struct sink_coherent_rows<S, std::void_t<decltype(S::kCoherentRows)>> : std::bool_constant<S::kCoherentRows> {};
template <class Sink>
__device__ __forceinline__ uint4 ld_row(const uint4 *p) {
    if constexpr (sink_coherent_rows<Sink>::value) return __ldcg(p);
    else return __ldg(p);
}

template <class S, class = void>
struct sink_is_guarded : std::false_type {};
template <class S>
struct sink_is_guarded<S, std::void_t<decltype(S::kGuarded)>> : std::bool_constant<S::kGuarded> {};

// true when `ord` lies in one of the level's dead ranges (see NarrowParams::dead); cold path, out of line
static __device__ __noinline__ bool ordinal_is_dead(const u64 *dead, uint32_t n, u64 ord) {
    uint32_t a = 0, b = n;  // first range whose lo is > ord
    while (a < b) {
        const uint32_t m = (a + b) >> 1;
        if (dead[2 * m] <= ord) a = m + 1;
        else b = m;
    }
    return a > 0 && ord < dead[2 * (a - 1) + 1];
}

// one connective on one-vector CMs (cm_ops.cuh)
template <int LW, int OP>
__device__ __forceinline__ uint4 apply_op(const NarrowParams &P, uint4 a, uint4 b) {
    return cm_apply<LW, OP>(a, b, P.valid);
}

// The tile runners are generic over where candidates go: `sink.emit<LW>(cand, live, known, ord_of)`
// is the direct insert (DirectSink -> insert_batch), the routing to hash owners of a sharded search (RouteSink) or
// the tiny-levels kernel's sink (narrow_tiny.cuh); WS is the warp's shared state (rows / term / block).
// Both return true when this tile AND every later tile of the launch are ordered after the
// separator (tiles follow the canonical order of their outer index), so the warp can stop
// drawing tickets instead of fetching and skipping them one by one.
template <int LW, int OP, class WS, class Sink>
__device__ __forceinline__ bool run_unary_tile(const NarrowParams &P, WS &ws, Sink &sink, u64 tile_local,
                                               u64 sep_now) {
    const BlockDesc &B = ws.block;
    const int lane = threadIdx.x & 31;
    const uint4 *src = B.from_atoms ? P.atoms : P.store + B.a_off;
    const u64 per_tile = (u64)TILE_V * B.tile_s;
    const u64 first = tile_local * per_tile + lane;
    const u64 ord0 = B.ord0, n = B.na;
    if (ord0 + tile_local * per_tile > sep_now) return true;  // this and all later tiles are ordered after the separator
    const int n_groups = (int)min((u64)B.tile_s, (n - tile_local * per_tile + TILE_V - 1) / TILE_V);
#pragma unroll 1
    for (int g = 0; g < n_groups; g += PROBE_BATCH) {
        uint4 cand[PROBE_BATCH];
        bool live[PROBE_BATCH], known[PROBE_BATCH];
        uint4 x[PROBE_BATCH];
        auto ord_of = [&](int r) { return ord0 + first + (u64)(g + r) * TILE_V; };
#pragma unroll
        for (int r = 0; r < PROBE_BATCH; ++r) {
            const u64 i = first + (u64)(g + r) * TILE_V;
            live[r] = g + r < n_groups && i < n;
            x[r] = live[r] ? ld_row<Sink>(src + i) : make_uint4(0, 0, 0, 0);
        }
#pragma unroll
        for (int r = 0; r < PROBE_BATCH; ++r) {
            cand[r] = apply_op<LW, OP>(P, x[r], x[r]);
            known[r] = OP != OP_ATOM && v_eq(cand[r], x[r]);
        }
        if (sink_is_guarded<Sink>::value && P.dead_n) {
#pragma unroll
            for (int r = 0; r < PROBE_BATCH; ++r)
                if (live[r] && ordinal_is_dead(P.dead, P.dead_n, ord_of(r))) live[r] = false;
        }
        sink.template emit<LW>(cand, live, known, ord_of);
    }
    return false;
}

// Binary tile: each lane keeps one row of the "vector" operand in registers and walks up
// to TILE_S rows of the "scalar" operand staged in the warp's shared memory together with
// the row's ordinal term, so that a candidate's ordinal is one 64-bit add:
//   rectangle  ord = ord0 + i*nb + j          triangle (i <= j < n)  ord = ord0 + i*n - i(i-1)/2 + (j - i)
// When the scalar operand has few rows (an early, small level) a tile takes B.vg groups
// of 32 vector rows against the same staged rows, so tiles stay a few thousand candidates.
// VEC_B: the lane dimension walks the right operand; irrelevant for the commutative ones.
template <int LW, int OP, bool VEC_B, class WS, class Sink>
__device__ __forceinline__ bool run_binary_tile(const NarrowParams &P, WS &ws, Sink &sink, u64 tile_local,
                                                u64 sep_now) {
    const BlockDesc &B = ws.block;
    const int lane = threadIdx.x & 31;
    const bool tri = B.kind == BK_TRI;
    const uint32_t vg_n = B.vg;
    // tile order follows the canonical order: left operand (i) outer, right operand (j) inner
    u64 tv, ts;
    if (VEC_B) { ts = tile_local / B.tiles_v; tv = tile_local % B.tiles_v; }
    else { tv = tile_local / B.tiles_s; ts = tile_local % B.tiles_s; }
    const u64 n_vec = VEC_B ? B.nb : B.na, n_sc = VEC_B ? B.na : B.nb;
    const u64 v0 = tv * (u64)(TILE_V * vg_n), s0 = ts * (u64)B.tile_s;
    const int s_cnt = (int)min((u64)B.tile_s, n_sc - s0);
    const u64 ord0 = B.ord0, na = B.na, nb = B.nb;
    // smallest ordinal of this tile's outer row of tiles (the left operand is the outer index
    // in both layouts): beyond the separator => so is everything that follows in the launch
    const u64 outer_min = ord0 + (VEC_B ? (tri ? s0 * na - (s0 ? (s0 * (s0 - 1)) / 2 : 0) : s0 * nb) : v0 * nb);
    if (outer_min > sep_now) return true;
    if (tri && v0 + (u64)TILE_V * vg_n - 1 < s0) return false;  // tile entirely below the diagonal (j < i)
    // a lower bound of the tile's ordinals: skip tiles ordered after the separator
    const u64 tile_min = outer_min + (VEC_B ? (tri ? 0 : v0) : s0);
    if (tile_min > sep_now) return false;
    const uint4 *vec_rows = P.store + (VEC_B ? B.b_off : B.a_off);
    const uint4 *sc_rows = P.store + (VEC_B ? B.a_off : B.b_off);
    // Associativity pruning.  (x & y) & r has the same CM as x & (y & r): the CM of y & r is in the cache
    // (its level is complete), at a cost that puts x & rep(y & r) either in an earlier level -- then the CM
    // is an older one -- or in this level in a block whose left operand costs cost(x) < cost(x & y), i.e.
    // at a smaller ordinal.  Either way the candidate never wins its CM: it is a duplicate by
    // construction (`known`), like one that equals an operand.  Mirrored for l & (y & z) when
    // cost(y) < cost(l).  The test is a range check on the operand row's own winning ordinal (AND blocks
    // are contiguous in a level's canonical order, by ascending left cost); bit 63 of `term` carries it
    // for the staged rows.
    constexpr u64 SKIP_BIT = 1ull << 63;
    const bool prune = (OP == OP_AND) && P.ords != nullptr;
    const u64 sc_lo = VEC_B ? B.skip_a_lo : B.skip_b_lo, sc_hi = VEC_B ? B.skip_a_hi : B.skip_b_hi;
    const u64 vec_lo = VEC_B ? B.skip_b_lo : B.skip_a_lo, vec_hi = VEC_B ? B.skip_b_hi : B.skip_a_hi;
    const u64 *sc_ords = P.ords + (VEC_B ? B.a_off : B.b_off), *vec_ords = P.ords + (VEC_B ? B.b_off : B.a_off);
    __syncwarp();
    for (int k = lane; k < s_cnt; k += 32) {
        const u64 s = s0 + k;
        ws.rows[k] = ld_row<Sink>(sc_rows + s);
        // scalar-row part of the ordinal; the lane part is j (VEC_B) or ord0 + i*nb (!VEC_B)
        u64 term = !VEC_B ? s : ord0 + (tri ? s * na - (s ? (s * (s - 1)) / 2 : 0) - s : s * nb);
        if (prune && sc_hi > sc_lo) {
            const u64 o = __ldg(sc_ords + s);
            if (o >= sc_lo && o < sc_hi) term |= SKIP_BIT;
        }
        ws.term[k] = term;
    }
    __syncwarp();
    // the vector row of the NEXT group is loaded while this group is processed
    uint4 xv_next = v0 + lane < n_vec ? ld_row<Sink>(vec_rows + v0 + lane) : make_uint4(0, 0, 0, 0);
#pragma unroll 1
    for (uint32_t vg = 0; vg < vg_n; ++vg) {
        const u64 v = v0 + (u64)vg * TILE_V + lane;
        if (v0 + (u64)vg * TILE_V >= n_vec) break;
        const bool v_ok = v < n_vec;
        const uint4 xv = xv_next;
        if (vg + 1 < vg_n && v + TILE_V < n_vec) xv_next = ld_row<Sink>(vec_rows + v + TILE_V);
        bool skip_v = false;
        if (prune && vec_hi > vec_lo && v_ok) {
            const u64 o = __ldg(vec_ords + v);
            skip_v = o >= vec_lo && o < vec_hi;
        }
        const u64 lane_term = VEC_B ? v : ord0 + v * nb;
        // triangle: row s0+sr pairs with columns j >= i only
        const int first_bad = tri ? (v >= s0 ? (int)min((u64)s_cnt, v - s0 + 1) : 0) : s_cnt;
        const int s_live = v_ok ? first_bad : 0;
#pragma unroll 1
        for (int g = 0; g < s_cnt; g += PROBE_BATCH) {
            uint4 cand[PROBE_BATCH];
            bool live[PROBE_BATCH], known[PROBE_BATCH];
            auto ord_of = [&](int r) { return (ws.term[min(g + r, s_cnt - 1)] & ~SKIP_BIT) + lane_term; };
#pragma unroll
            for (int r = 0; r < PROBE_BATCH; ++r) {
                const uint4 xs = ws.rows[min(g + r, s_cnt - 1)];
                live[r] = g + r < s_live;
                cand[r] = VEC_B ? apply_op<LW, OP>(P, xs, xv) : apply_op<LW, OP>(P, xv, xs);
                known[r] = v_eq(cand[r], xs) || v_eq(cand[r], xv);
                if (prune) known[r] = known[r] || skip_v || (ws.term[min(g + r, s_cnt - 1)] & SKIP_BIT) != 0ull;
            }
            if (sink_is_guarded<Sink>::value && P.dead_n) {
#pragma unroll
                for (int r = 0; r < PROBE_BATCH; ++r)
                    if (live[r] && ordinal_is_dead(P.dead, P.dead_n, ord_of(r))) live[r] = false;
            }
            sink.template emit<LW>(cand, live, known, ord_of);
        }
    }
    return false;
}

// scan pass (NarrowParams::scan_only): no set, no claims -- the ordinal of every separating candidate, fresh or not
template <int LW, typename OrdOf>
__device__ __noinline__ void scan_batch(const NarrowParams &P, const uint4 (&cand)[PROBE_BATCH], const bool (&live)[PROBE_BATCH],
                                        OrdOf ord_of) {
#pragma unroll
    for (int r = 0; r < PROBE_BATCH; ++r) {
        if (!live[r] || cm_sep_diff<LW>(cand[r], P.target, P.valid) != 0u) continue;
        const u64 pos = atomicAdd(&P.counters[CTR_SEPCOUNT], 1ull);
        if (pos < P.sep_list_cap) P.sep_list[pos] = ord_of(r);
    }
}

struct DirectSink {
    const NarrowParams &P;
    WarpShared &ws;
    WarpState &st;
    template <int LW, typename OrdOf>
    __device__ __forceinline__ void emit(const uint4 (&cand)[PROBE_BATCH], const bool (&live)[PROBE_BATCH],
                                         const bool (&known)[PROBE_BATCH], OrdOf ord_of) {
        insert_batch<LW>(P, ws.queue, st, cand, live, known, ord_of);
    }
};

// The sink of narrow_guarded_level_kernel: the scan pass and the enumeration with dead ranges (NarrowParams::dead)
// of a non-exhaustive level over a store that already holds a separating CM.  Only tile runners instantiated with
// a guarded sink contain that code, so the hot kernels carry none of it.
struct GuardedSink {
    static constexpr bool kGuarded = true;
    const NarrowParams &P;
    WarpShared &ws;
    WarpState &st;
    template <int LW, typename OrdOf>
    __device__ __forceinline__ void emit(const uint4 (&cand)[PROBE_BATCH], const bool (&live)[PROBE_BATCH],
                                         const bool (&known)[PROBE_BATCH], OrdOf ord_of) {
        if (P.scan_only) scan_batch<LW>(P, cand, live, ord_of);
        else insert_batch<LW>(P, ws.queue, st, cand, live, known, ord_of);
    }
};

// Tile tickets are drawn ONE TILE AHEAD: the atomicAdd for the next tile, and the reads of the
// overflow flag and of the separator bound that go with it, are issued before the current tile
// is processed and consumed after it, so their latency hides behind the tile's work (the first
// profile of the partitioned path had half of its stall samples on exactly these round trips).
// The bound is therefore one tile stale, which only makes pruning marginally later.
struct TileFetch {  // meaningful in lane 0
    u64 t = 0, sep = ~0ull, ovf = 0;
};

__device__ __forceinline__ TileFetch fetch_tile(const NarrowParams &P, const u64 *sep_extra) {
    TileFetch f;
    if ((threadIdx.x & 31) == 0) {
        f.ovf = __ldcg(&P.counters[CTR_OVERFLOW]);
        f.t = atomicAdd(&P.counters[P.ticket], 1ull);
        if (P.prune_after_sep) f.sep = __ldcg(&P.counters[CTR_SEP]);
        if (sep_extra) {
            const u64 x = __ldcg(sep_extra);
            f.sep = x < f.sep ? x : f.sep;
        }
    }
    return f;
}

// Turns a fetched ticket into the warp's current tile: finds its block (the launch's blocks are
// the (c1, c2) splits of one operator, sorted by first tile; 32 of them are tested per step, one
// per lane) and copies the descriptor to shared memory.  False when the launch has no tiles left
// (or the level overflowed).
template <class WS>
__device__ __forceinline__ bool open_tile(const NarrowParams &P, WS &ws, const TileFetch &f) {
    const int lane = threadIdx.x & 31;
    const u64 ticket = __shfl_sync(0xFFFFFFFFu, f.t, 0);
    u64 ovf = f.ovf;
    // the level's deadline, polled with every 16th ticket a warp draws (a look at it with EVERY ticket cost 4 % of
    // the kernel: one more word kept alive across the tile in a kernel at its register limit)
    if (lane == 0 && (f.t & 15ull) == 0ull && deadline_passed(P.counters)) ovf = 1ull;  // start no further tile; the claims stay valid
    ovf = __shfl_sync(0xFFFFFFFFu, ovf, 0);
    const u64 sep = __shfl_sync(0xFFFFFFFFu, f.sep, 0);
    const u64 t = ovf ? P.tile_end : P.tile_begin + P.shard_offset + ticket * P.shard_stride;
    if (t >= P.tile_end) return false;
    int bi = P.block_begin;
    for (int b0 = P.block_begin + 1; b0 < P.block_end; b0 += 32) {
        const int b = b0 + lane;
        const uint32_t m = __ballot_sync(0xFFFFFFFFu, b < P.block_end && P.blocks[b].tile0 <= t);
        bi += __popc(m);
        if (m != 0xFFFFFFFFu) break;
    }
    static_assert(sizeof(BlockDesc) % 4 == 0 && sizeof(BlockDesc) / 4 <= 64, "descriptor copied two words per lane at most");
    __syncwarp();
    for (int w = lane; w < (int)(sizeof(BlockDesc) / 4); w += 32)
        reinterpret_cast<uint32_t *>(&ws.block)[w] = reinterpret_cast<const uint32_t *>(&P.blocks[bi])[w];
    if (lane == 0) {
        ws.ticket = t;
        ws.sep_now = sep;
    }
    __syncwarp();
    return true;
}

template <int LW, int OP, class WS, class Sink>
__device__ __forceinline__ bool run_tile(const NarrowParams &P, WS &ws, Sink &sink) {
    const u64 sep_now = ws.sep_now;
    if (ws.block.ord0 > sep_now) return true;  // the whole block, and every later one, is ordered after the separator
    const u64 tile_local = ws.ticket - ws.block.tile0;
    if constexpr (OP == OP_AND || OP == OP_OR || OP == OP_UNTIL) {
        // which operand sits in the lanes changes only how the ordinal is formed, not the result
        if (ws.block.vec_is_b) return run_binary_tile<LW, OP, true>(P, ws, sink, tile_local, sep_now);
        return run_binary_tile<LW, OP, false>(P, ws, sink, tile_local, sep_now);
    } else {
        return run_unary_tile<LW, OP>(P, ws, sink, tile_local, sep_now);
    }
}

// run-time operator dispatch of the one-launch kernels
template <int LW, class WS, class Sink>
__device__ __forceinline__ bool run_tile_any(const NarrowParams &P, WS &ws, Sink &sink) {
    switch (ws.block.op) {
        case OP_ATOM: return run_tile<LW, OP_ATOM>(P, ws, sink);
        case OP_NOT: return run_tile<LW, OP_NOT>(P, ws, sink);
        case OP_NEXT: return run_tile<LW, OP_NEXT>(P, ws, sink);
        case OP_FUTURE: return run_tile<LW, OP_FUTURE>(P, ws, sink);
        case OP_GLOBALLY: return run_tile<LW, OP_GLOBALLY>(P, ws, sink);
        case OP_AND: return run_tile<LW, OP_AND>(P, ws, sink);
        case OP_UNTIL: return run_tile<LW, OP_UNTIL>(P, ws, sink);
        default: return run_tile<LW, OP_OR>(P, ws, sink);
    }
}

// One persistent launch per (level, operator): WARPS draw tiles of the operator's blocks
// from a ticket counter in canonical order.  The operator is a template parameter so that
// each kernel holds exactly one hot loop (a single kernel switching over all operators
// needed > 240 registers); launches of one level run back to back on the stream, in
// canonical operator order, with no host synchronisation in between.
template <int LW, int OP>
__global__ void __launch_bounds__(CTA_THREADS, LTLB200_MIN_CTAS) narrow_level_kernel(const NarrowParams P) {
    __shared__ WarpShared s_warp[WARPS_PER_CTA];
    WarpShared &ws = s_warp[threadIdx.x >> 5];
    WarpState st;
    DirectSink sink{P, ws, st};
    TileFetch next = fetch_tile(P, nullptr);
    for (;;) {
        const TileFetch cur = next;
        if (!open_tile(P, ws, cur)) break;
        next = fetch_tile(P, nullptr);
        if (run_tile<LW, OP>(P, ws, sink)) break;
    }
    if (*(volatile u64 *)&P.counters[CTR_OVERFLOW] == 0ull)
        while (st.qfill > 0u) drain_round(P, ws.queue, st);
}

// Small levels: ONE launch covers every operator (the operator is a run-time switch per tile).
// The per-operator kernels exist because a single hot loop needs fewer registers; a level of a
// few thousand candidates is pure launch latency instead, and five launches cost five times it.
template <int LW>
__global__ void __launch_bounds__(CTA_THREADS, 1) narrow_small_level_kernel(const NarrowParams P) {
    __shared__ WarpShared s_warp[WARPS_PER_CTA];
    WarpShared &ws = s_warp[threadIdx.x >> 5];
    WarpState st;
    DirectSink sink{P, ws, st};
    TileFetch next = fetch_tile(P, nullptr);
    for (;;) {
        const TileFetch cur = next;
        if (!open_tile(P, ws, cur)) break;
        next = fetch_tile(P, nullptr);
        if (run_tile_any<LW>(P, ws, sink)) break;
    }
    if (*(volatile u64 *)&P.counters[CTR_OVERFLOW] == 0ull)
        while (st.qfill > 0u) drain_round(P, ws.queue, st);
}

// Non-exhaustive level over a store that already holds a separating CM (rare: synthesize() stops at the first
// separator): one launch for every operator like the small-level kernel, with the guarded sink.
template <int LW>
__global__ void __launch_bounds__(CTA_THREADS, 1) narrow_guarded_level_kernel(const NarrowParams P) {
    __shared__ WarpShared s_warp[WARPS_PER_CTA];
    WarpShared &ws = s_warp[threadIdx.x >> 5];
    WarpState st;
    GuardedSink sink{P, ws, st};
    TileFetch next = fetch_tile(P, nullptr);
    for (;;) {
        const TileFetch cur = next;
        if (!open_tile(P, ws, cur)) break;
        next = fetch_tile(P, nullptr);
        if (run_tile_any<LW>(P, ws, sink)) break;
    }
    if (*(volatile u64 *)&P.counters[CTR_OVERFLOW] == 0ull)
        while (st.qfill > 0u) drain_round(P, ws.queue, st);
}

// ---- one search sharded over several GPUs: route instead of probe ----------------------------------------------
// The hash set of a sharded search is OWNER-SHARDED: rank r holds exactly the CMs with key_owner(CM) == r, of
// every level.  A rank therefore cannot decide locally whether a candidate is new; it builds its share of the
// level's pair space and appends every candidate that is not a duplicate by construction as a record
// {CM, ordinal} to the send region of the CM's owner (phase A, narrow_route_kernel).  After the all-to-all the
// owner folds what it received into its part of the set (phase B, narrow_probe_kernel = insert_batch over
// records).  Per rank and level that is C/N candidates built, (K+8)*C/N bytes streamed out and in, and C/N
// random probes into a set of 1/N of the keys: every term shrinks with the number of GPUs.
//
// Records are staged per owner in the warp's shared memory and flushed 32 at a time (one atomicAdd per 32 records
// and owner; 512 + 256 contiguous bytes per flush), so the regions are dense: no holes, exact send sizes.
constexpr int ROUTE_MAX_WORLD = 8;

struct __align__(16) WarpSharedRoute {
    uint4 skey[ROUTE_MAX_WORLD][32];
    u64 sord[ROUTE_MAX_WORLD][32];
    uint4 rows[TILE_S];
    u64 term[TILE_S];
    BlockDesc block;
    u64 ticket, sep_now;
    uint32_t fill[ROUTE_MAX_WORLD];
};

__device__ __forceinline__ void route_flush(const NarrowParams &P, WarpSharedRoute &ws, uint32_t w, uint32_t cnt) {
    const int lane = threadIdx.x & 31;
    u64 base = 0;
    if (lane == 0) base = atomicAdd(&P.route_counts[w], (u64)cnt);
    base = __shfl_sync(0xFFFFFFFFu, base, 0);
    if (base + cnt <= P.route_cap && (uint32_t)lane < cnt) {  // (past the region: only counted; the host redoes the level)
        const u64 at = (u64)w * P.route_cap + base + lane;
        P.route_rows[at] = ws.skey[w][lane];
        P.route_ords[at] = ws.sord[w][lane];
    }
}

struct RouteSink {
    const NarrowParams &P;
    WarpSharedRoute &ws;
    template <int LW, typename OrdOf>
    __device__ __forceinline__ void emit(const uint4 (&cand)[PROBE_BATCH], const bool (&live)[PROBE_BATCH],
                                         const bool (&known)[PROBE_BATCH], OrdOf ord_of) {
        const int lane = threadIdx.x & 31;
        const uint32_t lt = lanemask_lt();
#pragma unroll
        for (int r = 0; r < PROBE_BATCH; ++r) {
            if (live[r] && cm_sep_diff<LW>(cand[r], P.target, P.valid) == 0u) {
                const u64 o = ord_of(r);
                if (P.route_sep_any) atomicMin(&P.counters[CTR_SEP], o);
                if (P.sep_list) {  // exhaustive runs keep every separating ordinal (chunk-exact separator id)
                    const u64 pos = atomicAdd(&P.counters[CTR_SEPCOUNT], 1ull);
                    if (pos < P.sep_list_cap) P.sep_list[pos] = o;
                }
            }
            const bool send = live[r] && !known[r];
            const uint32_t owner = send ? key_owner(cand[r], P.route_world) : 0xFFFFFFFFu;
            uint32_t pending = __ballot_sync(0xFFFFFFFFu, send);
            while (pending) {  // one round per owner present in this batch row
                const uint32_t w = __shfl_sync(0xFFFFFFFFu, owner, __ffs(pending) - 1);
                const bool mine = owner == w;
                const uint32_t m = __ballot_sync(0xFFFFFFFFu, mine);
                pending &= ~m;
                const uint32_t n = __popc(m), fill = ws.fill[w];
                const uint32_t pos = fill + __popc(m & lt);
                if (mine && pos < 32u) {
                    ws.skey[w][pos] = cand[r];
                    ws.sord[w][pos] = ord_of(r);
                }
                uint32_t fill_after = fill + n;
                __syncwarp();
                if (fill_after >= 32u) {
                    route_flush(P, ws, w, 32u);
                    __syncwarp();
                    if (mine && pos >= 32u) {
                        ws.skey[w][pos - 32u] = cand[r];
                        ws.sord[w][pos - 32u] = ord_of(r);
                    }
                    fill_after -= 32u;
                }
                if (lane == 0) ws.fill[w] = fill_after;
                __syncwarp();
            }
        }
    }
};

template <int LW, int OP>
__global__ void __launch_bounds__(CTA_THREADS, LTLB200_MIN_CTAS) narrow_route_kernel(const NarrowParams P) {
    __shared__ WarpSharedRoute s_warp[WARPS_PER_CTA];
    WarpSharedRoute &ws = s_warp[threadIdx.x >> 5];
    const int lane = threadIdx.x & 31;
    if (lane < ROUTE_MAX_WORLD) ws.fill[lane] = 0u;
    __syncwarp();
    RouteSink sink{P, ws};
    TileFetch next = fetch_tile(P, nullptr);
    for (;;) {
        const TileFetch cur = next;
        if (!open_tile(P, ws, cur)) break;
        next = fetch_tile(P, nullptr);
        if (run_tile<LW, OP>(P, ws, sink)) break;
    }
    __syncwarp();
    for (uint32_t w = 0; w < P.route_world; ++w) {
        const uint32_t fill = ws.fill[w];
        if (fill) route_flush(P, ws, w, fill);
    }
}

#ifndef LTLB200_PROBE_CTAS
#define LTLB200_PROBE_CTAS 3  // (3 / 4 / 5 CTAs per SM: 4.83 / 5.13 / 5.82 ms on c3 to cost 15 with two ranks)
#endif
// Phase B on the owner: insert-or-min of `n` received records, PROBE_BATCH coalesced records per lane and step
// through the same insert_batch / drain_round as the single-GPU kernel.
template <int LW>
__global__ void __launch_bounds__(CTA_THREADS, LTLB200_PROBE_CTAS) narrow_probe_kernel(const NarrowParams P, const uint4 *rows,
                                                                                    const u64 *ords, u64 n) {
    __shared__ WarpShared s_warp[WARPS_PER_CTA];
    WarpShared &ws = s_warp[threadIdx.x >> 5];
    WarpState st;
    const int lane = threadIdx.x & 31;
    const u64 warp = (u64)blockIdx.x * WARPS_PER_CTA + (threadIdx.x >> 5), n_warps = (u64)gridDim.x * WARPS_PER_CTA;
    constexpr u64 STEP = 32ull * PROBE_BATCH;
    // the records of the next step are fetched before the current ones are probed (a step is two dependent trips to
    // memory otherwise: the records, then their slots), and the overflow flag is looked at every eighth step
    uint4 cand[PROBE_BATCH];
    u64 o[PROBE_BATCH];
    auto fetch = [&](u64 base) {
#pragma unroll
        for (int r = 0; r < PROBE_BATCH; ++r) {
            const u64 i = base + (u64)r * 32 + lane;
            cand[r] = i < n ? __ldcs(rows + i) : make_uint4(0, 0, 0, 0);
            o[r] = i < n ? __ldcs(ords + i) : 0ull;
        }
    };
    u64 base = warp * STEP;
    if (base < n) fetch(base);
    uint32_t step = 0;
#pragma unroll 1
    for (; base < n; base += n_warps * STEP, ++step) {
        if ((step & 7u) == 0u && *(volatile u64 *)&P.counters[CTR_OVERFLOW] != 0ull) break;
        uint4 cur[PROBE_BATCH];
        u64 cur_o[PROBE_BATCH];
        bool live[PROBE_BATCH], known[PROBE_BATCH];
#pragma unroll
        for (int r = 0; r < PROBE_BATCH; ++r) {
            cur[r] = cand[r];
            cur_o[r] = o[r];
            live[r] = base + (u64)r * 32 + lane < n;
            known[r] = false;
        }
        if (base + n_warps * STEP < n) fetch(base + n_warps * STEP);
        insert_batch<LW>(P, ws.queue, st, cur, live, known, [&](int r) { return cur_o[r]; });
    }
    if (*(volatile u64 *)&P.counters[CTR_OVERFLOW] == 0ull)
        while (st.qfill > 0u) drain_round(P, ws.queue, st);
}

}  // namespace ltlb200
