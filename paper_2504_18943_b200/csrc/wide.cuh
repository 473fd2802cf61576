// wide.cuh -- construction + dedup kernels for CMs wider than one uint4 (17..512 bytes).
//
// Same contract as narrow.cuh (canonical ordinals, first construction wins, fused
// separation check), different data layout, because a multi-vector key cannot be claimed
// with one compare-and-swap:
//
//   * a CM is `nvec` uint4 vectors; a GROUP of G = pow2 >= nvec lanes owns one candidate,
//     lane p of the group holding vector p (every connective is lane local, so the lanes
//     never exchange CM bits; only hash, equality and the separation flag are reduced
//     across the group, with ballots and xor-shuffles);
//   * the hash set holds 8-byte words  [fingerprint:24 | row index + 1 : 40]  (0 = empty).
//     The row index points either into the language cache (a CM finalised at an earlier
//     level: index < total_before) or into this level's STAGING pool of new rows;
//   * to claim a slot a group first writes its full row to a private staging entry, fences,
//     and only then publishes it with one 64-bit CAS on the slot word.  A reader that finds
//     a matching fingerprint therefore always finds a complete row behind it -- no waiting,
//     no locks -- and compares the whole CM (coalesced: G lanes x 16 bytes);
//   * per staging entry an atomicMin keeps the smallest ordinal that built the row.
//
// Finalisation ranks the staging entries by ordinal (bitmap + popcount prefix, as in the
// narrow path), copies the rows into the cache in that order and re-points the slot words
// at the final ids.
#pragma once
#include "narrow.cuh"

namespace ltlb200 {

constexpr int WIDE_ROW_VECS = 256;   // uint4 vectors of scalar-operand rows staged per warp (4 KiB)
constexpr int WIDE_TERMS = 128;      // max scalar rows per tile (G = 2)
constexpr int WIDE_CHUNK = 16;       // staging entries a group reserves at a time
// CTAs per SM of the wide kernel.  Unlike the narrow kernel it wants resident warps more than
// registers (every batch is a chain probe -> row write + fence -> CAS): c5 enumerate time per
// search with 3 / 4 / 6 / 8 / 10 CTAs per SM = 3.76 / 3.06 / 2.65 / 2.58 / 2.86 ms.
#ifndef LTLB200_WIDE_MIN_CTAS
#define LTLB200_WIDE_MIN_CTAS 6
#endif
#ifndef LTLB200_WIDE_BATCH
#define LTLB200_WIDE_BATCH 2
#endif
constexpr int WIDE_BATCH = LTLB200_WIDE_BATCH;  // candidates a group settles per phase round
constexpr u64 SLOT_IDX_MASK = (1ull << 40) - 1;
constexpr int MAX_NVEC = 32;

struct WideParams {
    const uint4 *store;  // finalised rows by global id, nvec vectors each
    const uint4 *atoms;  // atom rows, nvec vectors each
    u64 *slots;
    u64 slot_mask;
    uint4 *stage_rows;  // this level's new rows, nvec vectors each
    u64 *stage_ord;     // min ordinal per staging entry (all ones = unused)
    uint32_t *stage_slot;
    u64 stage_cap;
    u64 total_before;  // rows finalised before this level
    u64 *counters;     // CTR_*; CTR_CLAIMED counts reserved staging entries
    const BlockDesc *blocks;
    int block_begin, block_end;
    u64 tile_begin, tile_end;
    u64 shard_stride, shard_offset;
    int ticket;
    const uint4 *valid;   // Layout.masks packed, nvec vectors
    const uint4 *target;  // Layout.target packed, nvec vectors
    int nvec, log2g;
    int prune_after_sep;
    u64 *sep_list;
    u64 sep_list_cap;
    // non-exhaustive level over a store that already holds a separating CM (see NarrowParams::dead / scan_only;
    // wide2_guarded_level_kernel only)
    const u64 *dead;
    uint32_t dead_n;
    int scan_only;
};

struct __align__(16) WideWarpShared {
    uint4 rows[WIDE_ROW_VECS];  // (256 / G) scalar rows x G vectors
    u64 term[WIDE_TERMS];
    BlockDesc block;
    u64 ticket, sep_now;
};

// per-group registers (uniform inside a group)
struct GroupState {
    u64 chunk_next = 0, chunk_end = 0;  // staging entries reserved for this group
    u64 spare = ~0ull;                  // a reserved entry whose publish lost its race
};

struct GroupGeom {
    uint32_t mask;   // lanes of this group
    int base;        // first lane of the group
    int part;        // this lane's vector index inside the row
    int leader;      // base lane
    bool has_part;   // part < nvec
};

__device__ __forceinline__ u64 slot_word(uint32_t fp, u64 idx) { return ((u64)(fp & 0xFFFFFFu) << 40) | (idx + 1); }

// group-wide reductions
__device__ __forceinline__ bool group_all_zero(uint32_t diff, const GroupGeom &g) {
    return (__ballot_sync(g.mask, diff != 0u) & g.mask) == 0u;
}

// two independent 32-bit hashes of the whole row (slot index and fingerprint)
__device__ __forceinline__ void row_hash(uint4 part, const GroupGeom &g, int log2g, uint32_t &h_slot, uint32_t &h_fp) {
    uint32_t a = g.has_part ? hash_vec(part, 0x9E3779B9u * (uint32_t)(g.part + 1)) : 0u;
    uint32_t b = g.has_part ? hash_vec(part, 0x7F4A7C15u * (uint32_t)(g.part + 1) + 0x632BE5ABu) : 0u;
    for (int d = 1; d < (1 << log2g); d <<= 1) {
        a ^= __shfl_xor_sync(g.mask, a, d);
        b ^= __shfl_xor_sync(g.mask, b, d);
    }
    a ^= a >> 16;
    a *= 0x85EBCA6Bu;
    a ^= a >> 13;
    b ^= b >> 15;
    b *= 0xC2B2AE35u;
    b ^= b >> 16;
    h_slot = a;
    h_fp = b >> 8;
}

// the slot word as seen by the group's leader, broadcast to the group: every lane must act on
// the SAME value (a slot can be published by another group between two lanes' loads)
__device__ __forceinline__ u64 group_load_slot(const u64 *slot, const GroupGeom &g) {
    u64 w = 0;
    if ((int)(threadIdx.x & 31) == g.leader) w = __ldcg(slot);
    return __shfl_sync(g.mask, w, g.leader);
}

// Serial slow path: group-collective insert of one candidate row.  `w0` is the (group-uniform)
// word of slot `s`.  Returns true when the CM was not stored by an earlier level (fresh for
// this level).  Out of line on purpose: it is rare after wide_batch's phases, and inlining it
// at every call site blew the kernel past the instruction cache (25 % no-instruction stalls).
__device__ __noinline__ bool wide_insert(const WideParams &P, GroupGeom g, GroupState &gs, uint4 part, uint32_t s,
                                         uint32_t fp, u64 w0, u64 ord) {
    const int lane = threadIdx.x & 31;
    const uint32_t mask32 = (uint32_t)P.slot_mask;
    bool row_staged = false;
    u64 w = w0;
    for (;;) {
        if (w == 0ull) {
            // ---- empty slot: stage the row, then publish it with one CAS
            if (!row_staged) {
                if (gs.spare == ~0ull) {
                    if (gs.chunk_next == gs.chunk_end) {
                        u64 first = 0;
                        if (lane == g.leader) first = atomicAdd(&P.counters[CTR_CLAIMED], (u64)WIDE_CHUNK);
                        first = __shfl_sync(g.mask, first, g.leader);
                        gs.chunk_next = first;
                        gs.chunk_end = first + WIDE_CHUNK;
                    }
                    gs.spare = gs.chunk_next++;
                }
                if (gs.spare >= P.stage_cap) {  // staging pool exhausted: the host regrows and redoes the level
                    if (lane == g.leader) atomicExch(&P.counters[CTR_OVERFLOW], 1ull);
                    return false;
                }
                if (g.has_part) P.stage_rows[gs.spare * P.nvec + g.part] = part;
                __threadfence();
                row_staged = true;
            }
            __syncwarp(g.mask);
            u64 old = 0;
            if (lane == g.leader) old = atomicCAS(&P.slots[s], 0ull, slot_word(fp, P.total_before + gs.spare));
            old = __shfl_sync(g.mask, old, g.leader);
            if (old == 0ull) {
                if (lane == g.leader) {
                    atomicMin(&P.stage_ord[gs.spare], ord);
                    P.stage_slot[gs.spare] = s;
                }
                gs.spare = ~0ull;
                return true;
            }
            w = old;  // somebody else published here first: look at what they put
        }
        if ((uint32_t)(w >> 40) == (fp & 0xFFFFFFu)) {
            const u64 idx = (w & SLOT_IDX_MASK) - 1;
            const bool staged = idx >= P.total_before;
            const uint4 *row = staged ? P.stage_rows + (idx - P.total_before) * P.nvec : P.store + idx * P.nvec;
            uint32_t diff = 0;
            if (g.has_part) {
                const uint4 k = __ldcg(row + g.part);
                diff = (k.x ^ part.x) | (k.y ^ part.y) | (k.z ^ part.z) | (k.w ^ part.w);
            }
            if (group_all_zero(diff, g)) {
                if (!staged) return false;  // duplicate of an earlier level
                if (lane == g.leader) atomicMin(&P.stage_ord[idx - P.total_before], ord);
                return true;
            }
        }
        s = (s + 1) & mask32;
        w = group_load_slot(&P.slots[s], g);
    }
}

// Process WIDE_BATCH candidates of one group in lock-step PHASES, so that the latencies of a
// claim (slot probe -> row write + fence -> CAS) and of a duplicate check (slot probe -> row
// read) are paid once per batch, not once per candidate:
//   1. hash all, issue all first slot probes;
//   2. per candidate: empty slot -> reserve a staging entry and write the row;
//      fingerprint match -> issue the read of the stored row;  one fence for the whole batch;
//   3. the group leader issues all publishing CASes back to back;
//   4. settle: CAS won -> record ordinal; stored row equal -> duplicate (old) or atomicMin (this
//      level); anything else (lost race, fingerprint alias, collision) -> the serial slow path.
#ifndef LTLB200_WIDE_INLINE_BATCH
#define LTLB200_WIDE_INLINE_BATCH 1
#endif
#if LTLB200_WIDE_INLINE_BATCH
#define WIDE_BATCH_LINKAGE __forceinline__
#else
#define WIDE_BATCH_LINKAGE __noinline__  // one copy per kernel: the hot loop must fit the instruction cache
#endif
template <int LW>
__device__ WIDE_BATCH_LINKAGE void wide_batch(const WideParams &P, const GroupGeom g, GroupState &gs,
                                              const uint4 (&cand)[WIDE_BATCH], const bool (&live)[WIDE_BATCH],
                                              const bool (&known)[WIDE_BATCH], const uint4 target,
                                              const u64 (&ords)[WIDE_BATCH]) {
    const int lane = threadIdx.x & 31;
    auto ord_of = [&](int r) { return ords[r]; };
    enum : int { ST_SKIP = 0, ST_CLAIM = 1, ST_CHECK = 2, ST_SLOW = 3 };
    uint32_t slot[WIDE_BATCH], fp[WIDE_BATCH];
    u64 w[WIDE_BATCH];
    int state[WIDE_BATCH];
    // ---- 1. hashes and first probes
#pragma unroll
    for (int r = 0; r < WIDE_BATCH; ++r) {
        row_hash(cand[r], g, P.log2g, slot[r], fp[r]);
        slot[r] &= (uint32_t)P.slot_mask;
        w[r] = 0;
        if (live[r] && !known[r] && lane == g.leader) w[r] = __ldcg(&P.slots[slot[r]]);
    }
#pragma unroll
    for (int r = 0; r < WIDE_BATCH; ++r) w[r] = __shfl_sync(0xFFFFFFFFu, w[r], g.leader);  // one value per group
    // ---- 2. stage rows of the claims, start the row reads of the fingerprint matches
    uint4 stored[WIDE_BATCH];
    u64 entry[WIDE_BATCH];
    int n_claims = 0;
#pragma unroll
    for (int r = 0; r < WIDE_BATCH; ++r) {
        state[r] = ST_SKIP;
        entry[r] = 0;
        stored[r] = make_uint4(0, 0, 0, 0);
        if (!live[r] || known[r]) continue;
        if (w[r] == 0ull) {
            state[r] = ST_CLAIM;
            ++n_claims;
        } else if ((uint32_t)(w[r] >> 40) == (fp[r] & 0xFFFFFFu)) {
            state[r] = ST_CHECK;
            const u64 idx = (w[r] & SLOT_IDX_MASK) - 1;
            const uint4 *row = idx >= P.total_before ? P.stage_rows + (idx - P.total_before) * P.nvec : P.store + idx * P.nvec;
            if (g.has_part) stored[r] = __ldcg(row + g.part);
        } else {
            state[r] = ST_SLOW;
        }
    }
    if (n_claims) {  // group-uniform
        if (gs.chunk_next + (u64)n_claims > gs.chunk_end) {  // the rest of the old chunk stays unused
            u64 first = 0;
            if (lane == g.leader) first = atomicAdd(&P.counters[CTR_CLAIMED], (u64)WIDE_CHUNK);
            first = __shfl_sync(g.mask, first, g.leader);
            gs.chunk_next = first;
            gs.chunk_end = first + WIDE_CHUNK;
        }
#pragma unroll
        for (int r = 0; r < WIDE_BATCH; ++r) {
            if (state[r] != ST_CLAIM) continue;
            entry[r] = gs.chunk_next++;
            if (entry[r] >= P.stage_cap) {  // staging pool exhausted: the host regrows and redoes the level
                if (lane == g.leader) atomicExch(&P.counters[CTR_OVERFLOW], 1ull);
                state[r] = ST_SKIP;
                continue;
            }
            if (g.has_part) P.stage_rows[entry[r] * P.nvec + g.part] = cand[r];
        }
        __threadfence();
        __syncwarp(g.mask);
        // ---- 3. publish: all CASes in flight together
        u64 old[WIDE_BATCH];
#pragma unroll
        for (int r = 0; r < WIDE_BATCH; ++r) {
            old[r] = 0;
            if (state[r] == ST_CLAIM && lane == g.leader)
                old[r] = atomicCAS(&P.slots[slot[r]], 0ull, slot_word(fp[r], P.total_before + entry[r]));
        }
#pragma unroll
        for (int r = 0; r < WIDE_BATCH; ++r) {
            if (state[r] != ST_CLAIM) continue;
            w[r] = __shfl_sync(g.mask, old[r], g.leader);
            if (w[r] != 0ull) state[r] = ST_SLOW;  // lost the race: the staged entry stays unused
        }
    }
    // ---- 4. settle
#pragma unroll
    for (int r = 0; r < WIDE_BATCH; ++r) {
        if (!live[r]) continue;  // group-uniform
        const uint32_t sep_diff = g.has_part ? cm_sep_diff<LW>(cand[r], target) : 0u;
        const bool sep = group_all_zero(sep_diff, g);
        bool fresh = false;
        if (state[r] == ST_CLAIM) {
            if (lane == g.leader) {
                atomicMin(&P.stage_ord[entry[r]], ord_of(r));
                P.stage_slot[entry[r]] = slot[r];
            }
            fresh = true;
        } else if (state[r] == ST_CHECK) {
            const uint32_t diff = (stored[r].x ^ cand[r].x) | (stored[r].y ^ cand[r].y) | (stored[r].z ^ cand[r].z) | (stored[r].w ^ cand[r].w);
            if (group_all_zero(g.has_part ? diff : 0u, g)) {
                const u64 idx = (w[r] & SLOT_IDX_MASK) - 1;
                if (idx >= P.total_before) {
                    if (lane == g.leader) atomicMin(&P.stage_ord[idx - P.total_before], ord_of(r));
                    fresh = true;
                }
            } else {  // fingerprint alias: keep probing from the next slot
                const uint32_t s = (slot[r] + 1) & (uint32_t)P.slot_mask;
                fresh = wide_insert(P, g, gs, cand[r], s, fp[r], group_load_slot(&P.slots[s], g), ord_of(r));
            }
        } else if (state[r] == ST_SLOW) {
            fresh = wide_insert(P, g, gs, cand[r], slot[r], fp[r], w[r], ord_of(r));
        }
        if (sep && lane == g.leader) {
            const u64 ord = ord_of(r);
            if (fresh) atomicMin(&P.counters[CTR_SEP], ord);
            if (P.sep_list) {
                const u64 pos = atomicAdd(&P.counters[CTR_SEPCOUNT], 1ull);
                if (pos < P.sep_list_cap) P.sep_list[pos] = ord;
            }
        }
    }
}

template <int LW, int OP>
__device__ __forceinline__ void wide_unary_tile(const WideParams &P, WideWarpShared &ws, const GroupGeom &g,
                                                GroupState &gs, uint4 valid, uint4 target, u64 tile_local, u64 sep_now) {
    const BlockDesc &B = ws.block;
    const int groups = 32 >> P.log2g;
    const int gi = (threadIdx.x & 31) >> P.log2g;  // this group's index in the warp
    const uint4 *src = B.from_atoms ? P.atoms : P.store + B.a_off * P.nvec;
    const u64 per_tile = (u64)groups * B.tile_s;
    const u64 first = tile_local * per_tile + gi;
    const u64 ord0 = B.ord0, n = B.na;
    if (ord0 + tile_local * per_tile > sep_now) return;
    const int n_steps = (int)min((u64)B.tile_s, (n - tile_local * per_tile + groups - 1) / groups);
#pragma unroll 1
    for (int k = 0; k < n_steps; k += WIDE_BATCH) {
        uint4 cand[WIDE_BATCH];
        bool live[WIDE_BATCH], known[WIDE_BATCH];
        u64 ords[WIDE_BATCH];
#pragma unroll
        for (int r = 0; r < WIDE_BATCH; ++r) {
            const u64 i = first + (u64)(k + r) * groups;
            ords[r] = ord0 + i;
            live[r] = k + r < n_steps && i < n;
            const uint4 x = (live[r] && g.has_part) ? __ldg(src + i * P.nvec + g.part) : make_uint4(0, 0, 0, 0);
            cand[r] = cm_apply<LW, OP>(x, x, valid);
            const uint32_t d = (cand[r].x ^ x.x) | (cand[r].y ^ x.y) | (cand[r].z ^ x.z) | (cand[r].w ^ x.w);
            known[r] = OP != OP_ATOM && group_all_zero(d, g);
        }
        wide_batch<LW>(P, g, gs, cand, live, known, target, ords);
    }
}

template <int LW, int OP, bool VEC_B>
__device__ __forceinline__ void wide_binary_tile(const WideParams &P, WideWarpShared &ws, const GroupGeom &g,
                                                 GroupState &gs, uint4 valid, uint4 target, u64 tile_local, u64 sep_now) {
    const BlockDesc &B = ws.block;
    const int lane = threadIdx.x & 31;
    const int G = 1 << P.log2g, groups = 32 >> P.log2g, gi = lane >> P.log2g;
    const int tile_s = (int)B.tile_s;  // scalar rows per tile (<= WIDE_ROW_VECS / G)
    const bool tri = B.kind == BK_TRI;
    const uint32_t vg_n = B.vg;
    u64 tv, ts;
    if (VEC_B) { ts = tile_local / B.tiles_v; tv = tile_local % B.tiles_v; }
    else { tv = tile_local / B.tiles_s; ts = tile_local % B.tiles_s; }
    const u64 n_vec = VEC_B ? B.nb : B.na, n_sc = VEC_B ? B.na : B.nb;
    const u64 v0 = tv * (u64)(groups * vg_n), s0 = ts * (u64)tile_s;
    const int s_cnt = (int)min((u64)tile_s, n_sc - s0);
    if (tri && v0 + (u64)groups * vg_n - 1 < s0) return;
    const u64 ord0 = B.ord0, na = B.na, nb = B.nb;
    const u64 tile_min = ord0 + (VEC_B ? (tri ? s0 * na - (s0 ? (s0 * (s0 - 1)) / 2 : 0) : s0 * nb + v0) : v0 * nb + s0);
    if (tile_min > sep_now) return;
    const uint4 *vec_rows = P.store + (VEC_B ? B.b_off : B.a_off) * P.nvec;
    const uint4 *sc_rows = P.store + (VEC_B ? B.a_off : B.b_off) * P.nvec;
    __syncwarp();
    // stage the scalar rows: row k occupies vectors [k*G, k*G + nvec)
    for (int k = gi; k < s_cnt; k += groups) {
        const u64 s = s0 + k;
        if (g.has_part) ws.rows[k * G + g.part] = __ldg(sc_rows + s * P.nvec + g.part);
        if (lane == g.leader)
            ws.term[k] = !VEC_B ? s : ord0 + (tri ? s * na - (s ? (s * (s - 1)) / 2 : 0) - s : s * nb);
    }
    __syncwarp();
#pragma unroll 1
    for (uint32_t vg = 0; vg < vg_n; ++vg) {
        if (v0 + (u64)vg * groups >= n_vec) break;
        const u64 v = v0 + (u64)vg * groups + gi;
        const bool v_ok = v < n_vec;
        const uint4 xv = (v_ok && g.has_part) ? __ldg(vec_rows + v * P.nvec + g.part) : make_uint4(0, 0, 0, 0);
        const u64 lane_term = VEC_B ? v : ord0 + v * nb;
        const int first_bad = tri ? (v >= s0 ? (int)min((u64)s_cnt, v - s0 + 1) : 0) : s_cnt;
        const int s_live = v_ok ? first_bad : 0;
#pragma unroll 1
        for (int k = 0; k < s_cnt; k += WIDE_BATCH) {
            uint4 cand[WIDE_BATCH];
            bool live[WIDE_BATCH], known[WIDE_BATCH];
            u64 ords[WIDE_BATCH];
#pragma unroll
            for (int r = 0; r < WIDE_BATCH; ++r) {
                const int sr = min(k + r, s_cnt - 1);
                ords[r] = ws.term[sr] + lane_term;
                const uint4 xs = g.has_part ? ws.rows[sr * G + g.part] : make_uint4(0, 0, 0, 0);
                live[r] = k + r < s_live;
                cand[r] = VEC_B ? cm_apply<LW, OP>(xs, xv, valid) : cm_apply<LW, OP>(xv, xs, valid);
                const uint32_t da = (cand[r].x ^ xs.x) | (cand[r].y ^ xs.y) | (cand[r].z ^ xs.z) | (cand[r].w ^ xs.w);
                const uint32_t db = (cand[r].x ^ xv.x) | (cand[r].y ^ xv.y) | (cand[r].z ^ xv.z) | (cand[r].w ^ xv.w);
                const uint32_t ma = __ballot_sync(g.mask, da != 0u) & g.mask, mb = __ballot_sync(g.mask, db != 0u) & g.mask;
                known[r] = ma == 0u || mb == 0u;
            }
            wide_batch<LW>(P, g, gs, cand, live, known, target, ords);
        }
    }
}

// group geometry of the calling lane
__device__ __forceinline__ GroupGeom wide_geometry(const WideParams &P) {
    const int lane = threadIdx.x & 31;
    const int G = 1 << P.log2g;
    GroupGeom g;
    g.base = lane & ~(G - 1);
    g.part = lane & (G - 1);
    g.leader = g.base;
    g.has_part = g.part < P.nvec;
    g.mask = (G == 32 ? 0xFFFFFFFFu : ((1u << G) - 1u)) << g.base;
    return g;
}

// draws the warp's next tile (lane 0 takes a ticket) and loads its block descriptor
__device__ __forceinline__ bool wide_next_tile(const WideParams &P, WideWarpShared &ws) {
    const int lane = threadIdx.x & 31;
    __syncwarp();
    if (lane == 0) {
        u64 t = P.tile_end;
        if (*(volatile u64 *)&P.counters[CTR_OVERFLOW] == 0ull)
            t = P.tile_begin + P.shard_offset + atomicAdd(&P.counters[P.ticket], 1ull) * P.shard_stride;
        ws.ticket = t;
        ws.sep_now = P.prune_after_sep ? *(volatile u64 *)&P.counters[CTR_SEP] : (u64)~0ull;
        if (t < P.tile_end) {
            int bi = P.block_begin;
            while (bi + 1 < P.block_end && t >= P.blocks[bi + 1].tile0) ++bi;
            ws.block = P.blocks[bi];
        }
    }
    __syncwarp();
    return ws.ticket < P.tile_end;
}

template <int LW, int OP>
__device__ __forceinline__ void wide_run_tile(const WideParams &P, WideWarpShared &ws, const GroupGeom &g, GroupState &gs,
                                              uint4 valid, uint4 target) {
    const u64 sep_now = ws.sep_now;
    if (ws.block.ord0 > sep_now) return;
    const u64 tile_local = ws.ticket - ws.block.tile0;
    if constexpr (OP == OP_AND || OP == OP_OR || OP == OP_UNTIL) {
        if (ws.block.vec_is_b) wide_binary_tile<LW, OP, true>(P, ws, g, gs, valid, target, tile_local, sep_now);
        else wide_binary_tile<LW, OP, false>(P, ws, g, gs, valid, target, tile_local, sep_now);
    } else {
        wide_unary_tile<LW, OP>(P, ws, g, gs, valid, target, tile_local, sep_now);
    }
}

template <int LW, int OP>
__global__ void __launch_bounds__(CTA_THREADS, LTLB200_WIDE_MIN_CTAS) wide_level_kernel(const __grid_constant__ WideParams P) {
    __shared__ WideWarpShared s_warp[WARPS_PER_CTA];
    WideWarpShared &ws = s_warp[threadIdx.x >> 5];
    const GroupGeom g = wide_geometry(P);
    GroupState gs;
    const uint4 valid = g.has_part ? P.valid[g.part] : make_uint4(0, 0, 0, 0);
    const uint4 target = g.has_part ? P.target[g.part] : make_uint4(0, 0, 0, 0);
    while (wide_next_tile(P, ws)) wide_run_tile<LW, OP>(P, ws, g, gs, valid, target);
}

// Small levels: one launch for every operator (run-time switch per tile), as in the narrow path.
template <int LW>
__global__ void __launch_bounds__(CTA_THREADS, 1) wide_small_level_kernel(const __grid_constant__ WideParams P) {
    __shared__ WideWarpShared s_warp[WARPS_PER_CTA];
    WideWarpShared &ws = s_warp[threadIdx.x >> 5];
    const GroupGeom g = wide_geometry(P);
    GroupState gs;
    const uint4 valid = g.has_part ? P.valid[g.part] : make_uint4(0, 0, 0, 0);
    const uint4 target = g.has_part ? P.target[g.part] : make_uint4(0, 0, 0, 0);
    while (wide_next_tile(P, ws)) {
        switch (ws.block.op) {
            case OP_ATOM: wide_run_tile<LW, OP_ATOM>(P, ws, g, gs, valid, target); break;
            case OP_NOT: wide_run_tile<LW, OP_NOT>(P, ws, g, gs, valid, target); break;
            case OP_NEXT: wide_run_tile<LW, OP_NEXT>(P, ws, g, gs, valid, target); break;
            case OP_FUTURE: wide_run_tile<LW, OP_FUTURE>(P, ws, g, gs, valid, target); break;
            case OP_AND: wide_run_tile<LW, OP_AND>(P, ws, g, gs, valid, target); break;
            case OP_UNTIL: wide_run_tile<LW, OP_UNTIL>(P, ws, g, gs, valid, target); break;
            default: wide_run_tile<LW, OP_OR>(P, ws, g, gs, valid, target); break;
        }
    }
}

// ---- finalisation (wide) -------------------------------------------------------------------

struct WideFinalize {
    u64 *slots;
    const uint4 *stage_rows;
    const u64 *stage_ord;
    const uint32_t *stage_slot;
    u64 n_staged;  // staging entries reserved (some unused: ord = all ones)
    uint32_t *bitmap;
    const uint32_t *sb_rank;
    u64 ord_limit;
    uint4 *store;
    u64 *ords;
    u64 base;
    int nvec;
    u64 *stage_gid;  // final id per staging entry (written by wide_rank_kernel)
    // deferred mode (see FinalizeParams in narrow.cuh): bounds resolved on the device
    const u64 *live;
    u64 stage_cap;
    int cut_allowed;
};

__device__ __forceinline__ bool wide_finalize_bounds(const WideFinalize &F, u64 &n_staged, u64 &ord_limit) {
    n_staged = F.n_staged;
    ord_limit = F.ord_limit;
    if (F.live == nullptr) return true;
    if (F.live[CTR_OVERFLOW]) return false;
    const u64 claimed = F.live[CTR_CLAIMED], sep = F.live[CTR_SEP];
    n_staged = claimed < F.stage_cap ? claimed : F.stage_cap;
    ord_limit = (F.cut_allowed && sep != VAL_EMPTY) ? sep : VAL_EMPTY - 1;
    return true;
}

__global__ void __launch_bounds__(256) wide_mark_kernel(const WideFinalize F) {
    u64 n_staged, ord_limit;
    if (!wide_finalize_bounds(F, n_staged, ord_limit)) return;
    for (u64 t = (u64)blockIdx.x * blockDim.x + threadIdx.x; t < n_staged; t += (u64)gridDim.x * blockDim.x) {
        const u64 ord = F.stage_ord[t];
        if (ord <= ord_limit) atomicOr(&F.bitmap[ord >> 5], 1u << (ord & 31));
    }
}

// Scatter in two steps, so that the rank of an entry is computed once, not once per vector:
//   wide_rank_kernel   one thread per staging entry: final id = base + rank(ordinal); records the
//                      ordinal, re-points the entry's slot word at the final id, leaves the id in
//                      stage_gid (all ones = entry unused or ordered after the separator);
//   wide_copy_kernel   one thread per (staging entry, vector): coalesced copy of the row to its
//                      place in the cache.
__global__ void __launch_bounds__(256) wide_rank_kernel(const WideFinalize F) {
    u64 n_staged, ord_limit;
    if (!wide_finalize_bounds(F, n_staged, ord_limit)) return;
    for (u64 k = (u64)blockIdx.x * blockDim.x + threadIdx.x; k < n_staged; k += (u64)gridDim.x * blockDim.x) {
        const u64 ord = F.stage_ord[k];
        if (ord > ord_limit) {
            F.stage_gid[k] = ~0ull;
            continue;
        }
        const u64 gid = F.base + ordinal_rank(F.bitmap, F.sb_rank, ord);
        F.stage_gid[k] = gid;
        F.ords[gid] = ord;
        u64 *slot = &F.slots[F.stage_slot[k]];
        *slot = (*slot & ~SLOT_IDX_MASK) | (gid + 1);  // same fingerprint, final row id
    }
}

__global__ void __launch_bounds__(256) wide_copy_kernel(const WideFinalize F) {
    u64 n_staged, ord_limit;
    if (!wide_finalize_bounds(F, n_staged, ord_limit)) return;
    const u64 total = n_staged * (u64)F.nvec;
    for (u64 t = (u64)blockIdx.x * blockDim.x + threadIdx.x; t < total; t += (u64)gridDim.x * blockDim.x) {
        const u64 k = t / F.nvec;
        const u64 gid = F.stage_gid[k];
        if (gid == ~0ull) continue;
        F.store[gid * F.nvec + (t - k * F.nvec)] = F.stage_rows[t];
    }
}

// re-insert finalised rows [0, count) into a fresh table: rows of the cache are pairwise
// distinct, so claiming the first empty slot of the probe sequence is enough
__global__ void __launch_bounds__(256) wide_rebuild_kernel(u64 *slots, u64 slot_mask, const uint4 *store, u64 count,
                                                           int nvec, int log2g) {
    for (u64 gid = (u64)blockIdx.x * blockDim.x + threadIdx.x; gid < count; gid += (u64)gridDim.x * blockDim.x) {
        uint32_t a = 0, b = 0;
        for (int p = 0; p < nvec; ++p) {
            const uint4 part = store[gid * nvec + p];
            a ^= hash_vec(part, 0x9E3779B9u * (uint32_t)(p + 1));
            b ^= hash_vec(part, 0x7F4A7C15u * (uint32_t)(p + 1) + 0x632BE5ABu);
        }
        a ^= a >> 16;
        a *= 0x85EBCA6Bu;
        a ^= a >> 13;
        b ^= b >> 15;
        b *= 0xC2B2AE35u;
        b ^= b >> 16;
        u64 s = a & slot_mask;
        const u64 word = slot_word(b >> 8, gid);
        while (atomicCAS(&slots[s], 0ull, word) != 0ull) s = (s + 1) & slot_mask;
    }
}

// ---- exchange of a level's claims between ranks (wide rows) ----------------------------------

__device__ __forceinline__ uint32_t row_owner(const uint4 *row, int nvec, uint32_t owners) {
    uint32_t h = 0;
    for (int p = 0; p < nvec; ++p) h ^= hash_vec(row[p], 0x5BD1E995u * (uint32_t)(p + 1));
    h ^= h >> 15;
    h *= 0x2C1B3C6Du;
    h ^= h >> 13;
    return h % owners;
}

// one thread per staging entry: count per owner, or (with cursors) copy the records out grouped by owner
__global__ void __launch_bounds__(256) wide_export_kernel(const uint4 *stage_rows, const u64 *stage_ord, u64 n_staged, int nvec,
                                                          uint32_t owners, u64 *counts, u64 *cursors, uint4 *rows_out,
                                                          u64 *ords_out) {
    for (u64 t = (u64)blockIdx.x * blockDim.x + threadIdx.x; t < n_staged; t += (u64)gridDim.x * blockDim.x) {
        const u64 ord = stage_ord[t];
        if (ord == VAL_EMPTY) continue;  // reserved but never published
        const uint32_t o = row_owner(stage_rows + t * nvec, nvec, owners);
        if (cursors) {
            const u64 pos = atomicAdd(&cursors[o], 1ull);
            for (int p = 0; p < nvec; ++p) rows_out[pos * nvec + p] = stage_rows[t * nvec + p];
            ords_out[pos] = ord;
        } else {
            atomicAdd(&counts[o], 1ull);
        }
    }
}

// one group per received record: the same insert as the enumeration kernel
__global__ void __launch_bounds__(CTA_THREADS) wide_import_kernel(const __grid_constant__ WideParams P, const uint4 *rows, const u64 *ords, u64 n) {
    const int lane = threadIdx.x & 31;
    const int G = 1 << P.log2g;
    GroupGeom g;
    g.base = lane & ~(G - 1);
    g.part = lane & (G - 1);
    g.leader = g.base;
    g.has_part = g.part < P.nvec;
    g.mask = (G == 32 ? 0xFFFFFFFFu : ((1u << G) - 1u)) << g.base;
    GroupState gs;
    const u64 groups_per_block = (u64)(CTA_THREADS >> P.log2g);
    const u64 first = (u64)blockIdx.x * groups_per_block + (threadIdx.x >> P.log2g);
    for (u64 t = first; t < n; t += (u64)gridDim.x * groups_per_block) {
        const uint4 part = g.has_part ? rows[t * P.nvec + g.part] : make_uint4(0, 0, 0, 0);
        uint32_t slot, fp;
        row_hash(part, g, P.log2g, slot, fp);
        slot &= (uint32_t)P.slot_mask;
        wide_insert(P, g, gs, part, slot, fp, group_load_slot(&P.slots[slot], g), ords[t]);
    }
}

}  // namespace ltlb200
