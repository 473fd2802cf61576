// wide_fin.cuh -- finalisation, regrow and claim exchange kernels of the wide path (non-template
// kernels: included by engine.cu only, so that they exist once in the library).
#pragma once
#include "wide_common.cuh"

namespace ltlb200 {

// ---- finalisation (wide) -------------------------------------------------------------------

struct WideFinalize {
    const u64 *stage_ord;
    u64 n_staged;  // staging entries reserved (some unused: ord = all ones)
    uint32_t *bitmap;
    const uint32_t *sb_rank;
    u64 ord_limit;
    u64 *loc;      // log index per global id (written here)
    u64 *ords;
    u64 base;      // global id of the level's first entry
    u64 log_base;  // log index of staging entry 0
    // deferred mode (see FinalizeParams in narrow_fin.cuh): bounds resolved on the device
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

// small levels: narrow_fin.cuh's one-CTA finalisation (small_finalize_kernel<WideFinalize>)
__device__ __forceinline__ bool fin_bounds(const WideFinalize &F, u64 &n, u64 &ord_limit) { return wide_finalize_bounds(F, n, ord_limit); }
__device__ __forceinline__ u64 fin_ord(const WideFinalize &F, u64 t) { return F.stage_ord[t]; }
__device__ __forceinline__ void fin_place(const WideFinalize &F, u64 t, u64 gid, u64 ord) {
    F.loc[gid] = F.log_base + t;
    F.ords[gid] = ord;
}

__global__ void __launch_bounds__(256) wide_mark_kernel(const WideFinalize F) {
    u64 n_staged, ord_limit;
    if (!wide_finalize_bounds(F, n_staged, ord_limit)) return;
    for (u64 t = (u64)blockIdx.x * blockDim.x + threadIdx.x; t < n_staged; t += (u64)gridDim.x * blockDim.x) {
        const u64 ord = F.stage_ord[t];
        if (ord <= ord_limit) atomicOr(&F.bitmap[ord >> 5], 1u << (ord & 31));
    }
}

// One thread per staging entry: final id = base + rank(ordinal).  The row stays where it was staged -- the slot
// word that published it already points there -- so finalising an entry is two 8-byte stores: its place in the
// row log and the ordinal it won with.  (Round 1 copied every row into id order and rewrote every slot word:
// wide_copy_kernel + the slot read-modify-write were 12 of the 41 ms of a c5 search to cost 12.)
__global__ void __launch_bounds__(256) wide_rank_kernel(const WideFinalize F) {
    u64 n_staged, ord_limit;
    if (!wide_finalize_bounds(F, n_staged, ord_limit)) return;
    for (u64 k = (u64)blockIdx.x * blockDim.x + threadIdx.x; k < n_staged; k += (u64)gridDim.x * blockDim.x) {
        const u64 ord = F.stage_ord[k];
        if (ord > ord_limit) continue;  // unused entry, or ordered after the separator
        const u64 gid = F.base + ordinal_rank(F.bitmap, F.sb_rank, ord);
        F.loc[gid] = F.log_base + k;
        F.ords[gid] = ord;
    }
}

// re-insert finalised rows into a fresh table: rows of the cache are pairwise distinct, so claiming the first
// empty slot of the probe sequence is enough.  Entries are visited by id, their rows found through loc[]
// (owners > 1: an owner-sharded set holds only the rows whose hash owner is `rank`)
__global__ void __launch_bounds__(256) wide_rebuild_kernel(u64 *slots, u64 slot_mask, const uint4 *store, const u64 *loc, u64 count,
                                                           int nvec, int log2g, uint32_t owners, uint32_t rank) {
    for (u64 gid = (u64)blockIdx.x * blockDim.x + threadIdx.x; gid < count; gid += (u64)gridDim.x * blockDim.x) {
        const u64 at = loc[gid];
        const uint4 *row = store + at * nvec;
        if (owners > 1u && row_owner(row, nvec, owners) != rank) continue;
        uint32_t a = 0, b = 0;
        for (int p = 0; p < nvec; ++p) {
            const uint4 part = row[p];
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
        const u64 word = slot_word(b >> 8, at);
        while (atomicCAS(&slots[s], 0ull, word) != 0ull) s = (s + 1) & slot_mask;
    }
}

// rows [first, first + count) of the cache in id order, gathered from the row log (level_copy / level_device)
__global__ void __launch_bounds__(256) wide_gather_kernel(const uint4 *store, const u64 *loc, u64 first, u64 count, int nvec, uint4 *out) {
    const u64 total = count * (u64)nvec;
    for (u64 t = (u64)blockIdx.x * blockDim.x + threadIdx.x; t < total; t += (u64)gridDim.x * blockDim.x) {
        const u64 k = t / nvec;
        out[t] = store[loc[first + k] * nvec + (t - k * nvec)];
    }
}

// ---- sharded search: what an owner publishes, what every rank appends, what an owner folds in ---------------

// This owner's winners (staging entries whose smallest ordinal is <= ord_limit) as dense record arrays in ordinal
// order (see narrow_winners_kernel: the place of a winner is the rank of its ordinal among the owner's own marks);
// cursor[0] = how many.  Rows copied vector by vector.
__global__ void __launch_bounds__(256) wide_winners_kernel(const uint4 *stage_rows, const u64 *stage_ord, u64 n_staged, int nvec,
                                                           u64 ord_limit, const uint32_t *bitmap, const uint32_t *sb_rank, u64 *cursor,
                                                           uint4 *rows_out, u64 *ords_out) {
    const int lane = threadIdx.x & 31;
    const u64 n_round = (n_staged + 31) & ~31ull;
    for (u64 t = (u64)blockIdx.x * blockDim.x + threadIdx.x; t < n_round; t += (u64)gridDim.x * blockDim.x) {
        const u64 ord = t < n_staged ? stage_ord[t] : VAL_EMPTY;
        const bool keep = ord != VAL_EMPTY && ord <= ord_limit;
        const uint32_t m = __ballot_sync(0xFFFFFFFFu, keep);
        if (m == 0u) continue;
        if (lane == 0) atomicAdd(cursor, (u64)__popc(m));
        if (keep) {
            const u64 pos = ordinal_rank(bitmap, sb_rank, ord);
            for (int p = 0; p < nvec; ++p) rows_out[pos * nvec + p] = stage_rows[t * nvec + p];
            ords_out[pos] = ord;
        }
    }
}

// Appends records published by OTHER owners to the cache: the rows go to the tail of the row log (record t at
// log_at + t), and loc[] / ords[] of the id the ordinal ranks at point there.  The sources are walked in step
// (see RecordSources in narrow_fin.cuh) so that the loc / ords writes of all of them land in the same region.
__global__ void __launch_bounds__(256) wide_append_records_kernel(const uint4 *rows, const u64 *ords, const RecordSources S, int nvec,
                                                                  const uint32_t *bitmap, const uint32_t *sb_rank, uint4 *store,
                                                                  u64 log_at, u64 *loc, u64 *store_ords, u64 base) {
    const u64 total = S.longest * (u64)S.n * (u64)nvec;
    for (u64 x = (u64)blockIdx.x * blockDim.x + threadIdx.x; x < total; x += (u64)gridDim.x * blockDim.x) {
        const u64 v = x / nvec;
        const int p = (int)(x - v * nvec);
        u64 t;
        if (!interleaved_record(S, v, t)) continue;
        store[(log_at + t) * nvec + p] = rows[t * nvec + p];
        if (p == 0) {
            const u64 ord = ords[t];
            const u64 gid = base + ordinal_rank(bitmap, sb_rank, ord);
            loc[gid] = log_at + t;
            store_ords[gid] = ord;
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
