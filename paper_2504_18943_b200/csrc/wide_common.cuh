// wide_common.cuh -- data layout and protocol of the dedup set for CMs wider than one uint4 (17..512 bytes).
//
// Same contract as narrow.cuh (canonical ordinals, first construction wins, fused separation
// check), different data layout, because a multi-vector key cannot be claimed with one
// compare-and-swap:
//
//   * a CM is `nvec` uint4 vectors;
//   * rows live in a ROW LOG in the order they were staged; the hash set holds 8-byte words
//     [fingerprint:24 | log index + 1 : 40]  (0 = empty).  An index below total_before is a row of an
//     earlier level, anything beyond is one of this level's new rows, staged at the tail of the log;
//     finalising a level leaves the rows where they are and records loc[id] = log index (no copy,
//     no slot rewrite);
//   * to claim a slot the row is first written to a private staging entry and only then
//     published with one 64-bit CAS on the slot word.  A reader that finds a matching
//     fingerprint therefore always finds a complete row behind it -- no waiting, no locks --
//     and compares the whole CM;
//   * per staging entry an atomicMin keeps the smallest ordinal that built the row.
//
// The enumeration kernel is wide2.cuh (one lane per candidate).  The group-collective insert
// below (a group of G = pow2 >= nvec lanes owns one row, lane p holding vector p) serves the
// import of records received from other ranks (wide_fin.cuh).
#pragma once
#include "narrow.cuh"

namespace ltlb200 {

constexpr int WIDE_CHUNK = 16;       // staging entries a group reserves at a time (wide_insert: the import of exchanged records)
constexpr u64 SLOT_IDX_MASK = (1ull << 40) - 1;
constexpr int MAX_NVEC = 32;

struct WideParams {
    // The ROW LOG: every row the search ever staged, in claim order, nvec vectors each.  A level's new rows are staged
    // at its tail and STAY there when the level is finalised (no copy into id order): `loc[id]` = the log index of
    // entry `id`, and a slot word's row index is a log index.
    const uint4 *store;
    const u64 *loc;      // log index of every finalised entry by global id
    const uint4 *atoms;  // atom rows, nvec vectors each
    u64 *slots;
    u64 slot_mask;
    uint4 *stage_rows;  // this level's new rows = the tail of the log (store + total_before * nvec)
    u64 *stage_ord;     // min ordinal per staging entry (all ones = unused)
    u64 stage_cap;
    u64 total_before;  // log entries before this level: a slot word pointing at or beyond it is one of this level's rows
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
    // sharded search (wide2_route_kernel; see NarrowParams): rows go to the region of their hash owner
    uint4 *route_rows;  // route_world regions of route_cap rows of nvec vectors
    u64 *route_ords;
    u64 route_cap;
    u64 *route_counts;
    uint32_t route_world;
    int route_sep_any;
    // regex grammar (LW_REGEX instantiation of wide2.cuh; wide2_regex.cuh): the guide tables laid out by
    // Engine::set_regex, bits per characteristic sequence, entries of the table, rounds of the star
    const uint32_t *guide;
    int n_bits;
    uint32_t guide_entries, guide_rounds;
    uint32_t guide_smem_words;  // > 0: the kernels stage the tables in the CTA's shared memory
};

// hash owner of a row in a sharded search (independent of the slot hash and of the fingerprint)
__device__ __forceinline__ uint32_t row_owner_mix(uint32_t h) {
    h ^= h >> 15;
    h *= 0x2C1B3C6Du;
    h ^= h >> 13;
    return h;
}
__device__ __forceinline__ uint32_t row_owner(const uint4 *row, int nvec, uint32_t owners) {
    uint32_t h = 0;
    for (int p = 0; p < nvec; ++p) h ^= hash_vec(row[p], 0x5BD1E995u * (uint32_t)(p + 1));
    return row_owner_mix(h) % owners;
}

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
static __device__ __noinline__ bool wide_insert(const WideParams &P, GroupGeom g, GroupState &gs, uint4 part, uint32_t s,
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
                if (lane == g.leader) atomicMin(&P.stage_ord[gs.spare], ord);
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

}  // namespace ltlb200
