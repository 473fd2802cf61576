// narrow_fin.cuh -- finalisation, regrow and claim exchange kernels of the narrow path (non-template
// kernels: included by engine.cu only, so that they exist once in the library).
#pragma once
#include "narrow.cuh"

namespace ltlb200 {

// ---- finalisation: order the level's winners by ordinal without a sort -------------
// A bitmap with one bit per candidate ordinal marks the winners; a popcount prefix over
// 1024-bit superblocks turns an ordinal into its rank, i.e. the entry's position in the
// level (reference order = ordinal order), and the rows are scattered straight to it.

struct FinalizeParams {
    const uint4 *claim_key;
    const u64 *claim_ord;
    u64 n_claimed;  // claim indices reserved (some unused: ord = all ones)
    uint32_t *bitmap;         // one bit per ordinal
    const uint32_t *sb_rank;  // exclusive popcount prefix per 32-word superblock
    u64 ord_limit;            // keep ordinals <= limit (separator in a non-exhaustive run, else all ones - 1)
    uint4 *store;
    u64 *ords;
    u64 base;  // global id of the level's first entry
    // Deferred mode (live != NULL): the host has not read the level's counters yet -- it launched
    // the finalisation right behind the enumeration, one synchronisation per level instead of
    // two -- so the claim count, the separator and the overflow flag are read here.
    const u64 *live;
    u64 claim_cap;
    int cut_allowed;  // non-exhaustive: keep only ordinals <= the separator
};

// resolves n_claimed / ord_limit in deferred mode; false = the level overflowed and is redone
__device__ __forceinline__ bool finalize_bounds(const FinalizeParams &F, u64 &n_claimed, u64 &ord_limit) {
    n_claimed = F.n_claimed;
    ord_limit = F.ord_limit;
    if (F.live == nullptr) return true;
    if (F.live[CTR_OVERFLOW]) return false;
    const u64 claimed = F.live[CTR_CLAIMED], sep = F.live[CTR_SEP];
    n_claimed = claimed < F.claim_cap ? claimed : F.claim_cap;
    ord_limit = (F.cut_allowed && sep != VAL_EMPTY) ? sep : VAL_EMPTY - 1;
    return true;
}

__global__ void __launch_bounds__(256) narrow_mark_kernel(const FinalizeParams F) {
    u64 n_claimed, ord_limit;
    if (!finalize_bounds(F, n_claimed, ord_limit)) return;
    for (u64 t = (u64)blockIdx.x * blockDim.x + threadIdx.x; t < n_claimed; t += (u64)gridDim.x * blockDim.x) {
        const u64 ord = F.claim_ord[t];
        if (ord <= ord_limit) atomicOr(&F.bitmap[ord >> 5], 1u << (ord & 31));
    }
}

__global__ void __launch_bounds__(256) narrow_scatter_kernel(const FinalizeParams F) {
    u64 n_claimed, ord_limit;
    if (!finalize_bounds(F, n_claimed, ord_limit)) return;
    for (u64 t = (u64)blockIdx.x * blockDim.x + threadIdx.x; t < n_claimed; t += (u64)gridDim.x * blockDim.x) {
        const u64 ord = F.claim_ord[t];
        if (ord > ord_limit) continue;  // unused index, or ordered after the separator
        const u64 gid = F.base + ordinal_rank(F.bitmap, F.sb_rank, ord);
        F.store[gid] = F.claim_key[t];
        F.ords[gid] = ord;
    }
}

// Small levels: the whole finalisation in ONE CTA.  The winners bitmap of a level of up to 2^15
// candidates is 4 KiB and lives in shared memory, so mark -> superblock ranks -> summary ->
// scatter need no global bitmap, no scan launches and no separate summary launch: such a level
// is launch latency, and this is one launch instead of five.  One kernel for both key widths: what differs is where
// the ordinals come from and what placing an entry means (fin_* overloads here and in wide_fin.cuh).
constexpr int SMALL_FIN_THREADS = 1024;
constexpr u64 SMALL_FIN_MAX_BITS = 1ull << 15;

__device__ __forceinline__ bool fin_bounds(const FinalizeParams &F, u64 &n, u64 &ord_limit) { return finalize_bounds(F, n, ord_limit); }
__device__ __forceinline__ u64 fin_ord(const FinalizeParams &F, u64 t) { return F.claim_ord[t]; }
__device__ __forceinline__ void fin_place(const FinalizeParams &F, u64 t, u64 gid, u64 ord) {
    F.store[gid] = F.claim_key[t];
    F.ords[gid] = ord;
}

template <class Fin>
__global__ void __launch_bounds__(SMALL_FIN_THREADS) small_finalize_kernel(const Fin F, u64 n_bits, u64 *counters, int export_bitmap) {
    extern __shared__ uint32_t s_fin[];
    const u64 n_words = (n_bits + 31) >> 5, n_sb = (n_words + 31) >> 5;  // <= 1024 words, <= 32 superblocks
    uint32_t *bitmap = s_fin, *sb_rank = s_fin + n_sb * 32;              // bitmap padded to whole superblocks
    __shared__ uint32_t warp_tot[32];
    u64 n_claimed, ord_limit;
    if (!fin_bounds(F, n_claimed, ord_limit)) return;  // uniform: the level overflowed and is redone
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    for (u64 w = tid; w < n_sb * 32; w += SMALL_FIN_THREADS) bitmap[w] = 0u;
    __syncthreads();
    for (u64 t = tid; t < n_claimed; t += SMALL_FIN_THREADS) {
        const u64 ord = fin_ord(F, t);
        if (ord <= ord_limit) atomicOr(&bitmap[ord >> 5], 1u << (ord & 31));
    }
    __syncthreads();
    // exclusive popcount prefix per superblock (n_sb <= threads)
    uint32_t v = 0;
    if ((u64)tid < n_sb)
        for (int k = 0; k < 32; ++k) v += __popc(bitmap[tid * 32 + k]);
    uint32_t incl = v;
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
        const uint32_t t = __shfl_up_sync(0xFFFFFFFFu, incl, d);
        if (lane >= d) incl += t;
    }
    if (lane == 31) warp_tot[warp] = incl;
    __syncthreads();
    if (warp == 0) {
        const uint32_t w = warp_tot[lane];
        uint32_t wi = w;
#pragma unroll
        for (int d = 1; d < 32; d <<= 1) {
            const uint32_t t = __shfl_up_sync(0xFFFFFFFFu, wi, d);
            if (lane >= d) wi += t;
        }
        warp_tot[lane] = wi - w;
    }
    __syncthreads();
    if ((u64)tid < n_sb) sb_rank[tid] = warp_tot[warp] + incl - v;
    __syncthreads();
    if (export_bitmap) {  // exhaustive runs pick their reported separator against the winners bitmap afterwards
        for (u64 w = tid; w < n_sb * 32; w += SMALL_FIN_THREADS) F.bitmap[w] = bitmap[w];
        if ((u64)tid < n_sb) const_cast<uint32_t *>(F.sb_rank)[tid] = sb_rank[tid];
    }
    if (tid == 0) {  // winners of the level, rank of the separator
        const u64 sep_ord = counters[CTR_SEP];
        counters[CTR_WINNERS] = n_bits ? ordinal_rank(bitmap, sb_rank, n_bits - 1) + ((bitmap[(n_bits - 1) >> 5] >> ((n_bits - 1) & 31)) & 1u) : 0;
        counters[CTR_SEPRANK] = sep_ord < n_bits ? ordinal_rank(bitmap, sb_rank, sep_ord) : ~0ull;
    }
    for (u64 t = tid; t < n_claimed; t += SMALL_FIN_THREADS) {
        const u64 ord = fin_ord(F, t);
        if (ord > ord_limit) continue;
        fin_place(F, t, F.base + ordinal_rank(bitmap, sb_rank, ord), ord);
    }
}

// re-insert finalised rows [first, first+count) into a fresh table (regrow / rollback)
// (owners > 1: an owner-sharded set holds only the CMs whose hash owner is `rank`)
__global__ void __launch_bounds__(256) narrow_rebuild_kernel(Slot16 *slots, u64 slot_mask, const uint4 *store,
                                                             u64 first, u64 count, u64 *counters, uint32_t owners, uint32_t rank) {
    const uint4 empty = make_uint4(~0u, ~0u, ~0u, ~0u);
    for (u64 t = (u64)blockIdx.x * blockDim.x + threadIdx.x; t < count; t += (u64)gridDim.x * blockDim.x) {
        const u64 gid = first + t;
        const uint4 key = store[gid];
        if (owners > 1u && key_owner(key, owners) != rank) continue;
        if (key_is_empty(key)) {
            counters[CTR_SPECIAL] = gid;
            continue;
        }
        u64 slot = hash_vec(key, 0u) & slot_mask;
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

// ---- sharded search: what an owner publishes, and what every rank appends to its cache ----------------------

// This owner's winners (claims whose smallest ordinal is <= ord_limit) as dense record arrays IN ORDINAL ORDER;
// cursor[0] = how many.  `bitmap` / `sb_rank` are the owner's OWN marks, ranked (before the ranks all-reduce the
// bitmap): the rank of a winner's ordinal among them is its place in the export -- the winners up to a separator are
// a prefix of that order, so the places are dense.  Sorting here costs the owner one random store per winner it
// publishes (u C / N of them); it saves every receiver the random placement of everything it receives: records
// that arrive in ordinal order go to ascending ids (narrow_scatter_records_kernel).
__global__ void __launch_bounds__(256) narrow_winners_kernel(const uint4 *claim_key, const u64 *claim_ord, u64 n_claimed,
                                                             u64 ord_limit, const uint32_t *bitmap, const uint32_t *sb_rank,
                                                             u64 *cursor, uint4 *rows_out, u64 *ords_out) {
    const int lane = threadIdx.x & 31;
    const u64 n_round = (n_claimed + 31) & ~31ull;  // whole warps stay in the loop for the ballot
    for (u64 t = (u64)blockIdx.x * blockDim.x + threadIdx.x; t < n_round; t += (u64)gridDim.x * blockDim.x) {
        const u64 ord = t < n_claimed ? claim_ord[t] : VAL_EMPTY;
        const bool keep = ord != VAL_EMPTY && ord <= ord_limit;
        const uint32_t m = __ballot_sync(0xFFFFFFFFu, keep);
        if (m == 0u) continue;
        if (lane == 0) atomicAdd(cursor, (u64)__popc(m));
        if (keep) {
            const u64 pos = ordinal_rank(bitmap, sb_rank, ord);
            rows_out[pos] = claim_key[t];
            ords_out[pos] = ord;
        }
    }
}

// Where the records of the other owners sit in the receive buffers: source s sent counts[s] records starting at
// record offsets[s], each source's in ordinal order.  The sources are walked in step (record i of source 0, of source
// 1, ...): the i-th winners of all owners have neighbouring ordinals (owners are hash classes), so a warp's stores go
// to one neighbourhood of ids.  (With unordered records -- the first version -- the walk order made no difference:
// 4.2 vs 4.3 ms for the 54.6 M records a rank of eight receives on c3 to cost 15; tools/shard_model.py.)
struct RecordSources {
    unsigned long long offsets[8], counts[8];
    unsigned long long longest;  // max of counts
    int n;
};

__device__ __forceinline__ bool interleaved_record(const RecordSources &S, u64 v, u64 &rec) {
    const u64 i = v / (u64)S.n;
    const int s = (int)(v - i * (u64)S.n);
    if (i >= S.counts[s]) return false;
    rec = S.offsets[s] + i;
    return true;
}

// Appends records published by OTHER owners to the cache: position = rank of the ordinal in the level's global
// winners bitmap (the all-reduced union of every owner's marks), exactly as narrow_scatter_kernel places this
// owner's own claims.
__global__ void __launch_bounds__(256) narrow_scatter_records_kernel(const uint4 *rows, const u64 *ords, const RecordSources S,
                                                                     const uint32_t *bitmap, const uint32_t *sb_rank,
                                                                     uint4 *store, u64 *store_ords, u64 base) {
    const u64 total = S.longest * (u64)S.n;
    for (u64 v = (u64)blockIdx.x * blockDim.x + threadIdx.x; v < total; v += (u64)gridDim.x * blockDim.x) {
        u64 t;
        if (!interleaved_record(S, v, t)) continue;
        const u64 ord = ords[t];
        const u64 gid = base + ordinal_rank(bitmap, sb_rank, ord);
        store[gid] = rows[t];
        store_ords[gid] = ord;
    }
}

}  // namespace ltlb200
