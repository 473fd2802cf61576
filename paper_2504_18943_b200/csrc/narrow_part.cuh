// narrow_part.cuh -- radix-partitioned dedup for large levels of narrow (<= 16 byte) CMs.
//
// Why: the direct path (narrow.cuh) probes the hash set once per candidate at a random
// address of a multi-GB table.  On B200 that pattern tops out at ~17-20 sectors/ns of DRAM
// (tools/random_probe_bench.cu), and the big levels of a search run exactly at that ceiling
// (profiles/r01_s2_*).  The same probes against a table WINDOW that fits the 126 MB L2 run at
// 80-90 probes/ns including the record stream (tools/window_probe_bench.cu).  So a big level
// is done in two phases over the SAME hash set and claim arrays as the direct path:
//
//   phase A  narrow_partition_kernel<LW, OP>: builds the candidates tile by tile exactly like
//            narrow_level_kernel, but instead of probing, appends {CM, ordinal} records to the
//            bucket of the table window their home slot lies in (bucket = slot >> shift,
//            PART_NB windows).  A warp stages a few hundred records in shared memory, ranks
//            them inside their bucket with a shared-memory atomicAdd, and writes them out --
//            every lane in parallel, no sort -- into warp-private 64-record chunks drawn from
//            a global pool; a chunk belongs to one bucket.
//            The open chunk of every (warp, bucket) is carried from one operator launch to the
//            next, so a level ends with one partly filled chunk per warp and bucket, not five.
//   order    part_seal_kernel + part_order_kernel: fill of the open chunks, then the chunk ids
//            grouped by bucket (block-level counting sort on 64 counters).
//   phase B  narrow_probe_kernel<LW>: walks the chunks bucket by bucket -- all SMs are in the
//            same window at the same time, so it stays L2 resident -- and feeds the records to
//            the direct path's insert_batch / drain_round (same slots, same claims, same
//            atomicMin on the ordinal: "first construction wins" does not depend on the order
//            in which candidates reach the set).
//
// Nothing here changes what a level contains; only the order of the probes changes.
#pragma once
#include "narrow.cuh"

namespace ltlb200 {

#ifndef LTLB200_PART_STAGE
#define LTLB200_PART_STAGE 320
#endif
#ifndef LTLB200_PART_MIN_CTAS
#define LTLB200_PART_MIN_CTAS 4
#endif
#ifndef LTLB200_PROBE_MIN_CTAS
#define LTLB200_PROBE_MIN_CTAS 5
#endif
constexpr int PART_NB = 64;                      // buckets = table windows
constexpr int PART_STAGE = LTLB200_PART_STAGE;   // records a warp stages in shared memory before it writes them out
constexpr int PART_STAGE_FLUSH = PART_STAGE - 32 * PROBE_BATCH;  // written out once more than this is staged (a full batch still fits)
constexpr int PART_CHUNK = 64;                   // records per pool chunk
constexpr int PART_STASH = 128;                  // chunk ids a warp draws from the pool at a time
constexpr int PART_TICKET_CHUNKS = 8;            // chunks per phase-B ticket
constexpr int PART_WSTATE = PART_NB + 2;         // u64 words of carried state per warp slot
static_assert(PART_STAGE_FLUSH >= 32, "staging area too small");

// pcounters: [0] chunk ids drawn from the pool, [1] chunks in `order`, [2] pool overflow,
// [3] smallest ordinal of a separating candidate seen by phase A (pruning bound),
// [4] phase-B ticket, [8..8+NB) chunks per bucket, [8+NB..8+2NB) cursors of the ordering pass
enum : int { PC_POOL = 0, PC_ORDERED = 1, PC_OVERFLOW = 2, PC_SEPBOUND = 3, PC_TICKET = 4, PC_BUCKET0 = 8, PC_CURSOR0 = PC_BUCKET0 + PART_NB, PC_COUNT = PC_CURSOR0 + PART_NB };

struct PartParams {
    uint4 *pool_keys;       // record r of chunk c = pool_keys[c * PART_CHUNK + r]
    u64 *pool_ords;
    uint8_t *chunk_bucket;  // 0xFF = chunk id never used
    uint8_t *chunk_fill;    // records in the chunk (preset to PART_CHUNK; open chunks are corrected by part_seal_kernel)
    uint32_t *order;        // chunk ids grouped by bucket
    u64 *wstate;            // per warp slot: open chunk of every bucket + chunk-id stash, carried from one
                            // operator launch of the segment to the next
    u64 wstate_slots;
    u64 pool_chunks;        // capacity of the pool
    u64 *pc;                // PC_*
    int bucket_shift;       // bucket = home slot >> bucket_shift
    int sep_bound_ok;       // the cache holds no separating CM, so any separating candidate is fresh:
                            // phase A may prune tiles ordered after the smallest one it has seen
};

// Per-warp shared state of phase A.  Records are staged in arrival order together with
// {bucket, rank inside the bucket} (the rank is what a shared-memory atomicAdd on the bucket's
// counter returned), so writing them out needs no sort: record -> bucket state -> address.
struct __align__(16) WarpSharedPart {
    uint4 skey[PART_STAGE];
    u64 sord[PART_STAGE];
    uint32_t smeta[PART_STAGE];  // bucket | rank << 8
    uint4 bstate[PART_NB];       // x = next free record of the bucket's open chunk, y = records left in it,
                                 // z = (first record of the chunks drawn for this write-out) - y, w = 1 if those are usable
    uint32_t cnt[PART_NB];       // staged records per bucket
    uint4 rows[TILE_S];
    u64 term[TILE_S];
    BlockDesc block;
    u64 ticket, sep_now;
};

struct PartSink {
    const NarrowParams &P;
    const PartParams &Q;
    WarpSharedPart &ws;
    uint32_t staged = 0;                // warp-uniform
    u64 stash_next = 0, stash_end = 0;  // chunk ids drawn from the pool, warp-uniform

    // Writes the staged records to their buckets' chunks.  Lane l plans buckets l and l+32 (how
    // many new chunks each needs; ids come from the warp's stash, contiguous per bucket, so no
    // global atomic is on this path except one pool atomicAdd per PART_STASH chunks), then all
    // lanes copy records out in staging order.
    __device__ __forceinline__ void write_out() {
        const int lane = threadIdx.x & 31;
        __syncwarp();
        uint32_t n[2], k[2];
        uint4 bs[2];
#pragma unroll
        for (int h = 0; h < 2; ++h) {
            n[h] = ws.cnt[lane + 32 * h];
            bs[h] = ws.bstate[lane + 32 * h];
            k[h] = n[h] > bs[h].y ? (n[h] - bs[h].y + PART_CHUNK - 1) / PART_CHUNK : 0u;
        }
        uint32_t incl = k[0] + k[1];
#pragma unroll
        for (int d = 1; d < 32; d <<= 1) {
            const uint32_t t = __shfl_up_sync(0xFFFFFFFFu, incl, d);
            if (lane >= d) incl += t;
        }
        const uint32_t total = __shfl_sync(0xFFFFFFFFu, incl, 31);
        if ((u64)total > stash_end - stash_next) {  // refill; the few ids left in the old stash are abandoned
            const u64 grab = total > (uint32_t)PART_STASH ? total : (uint32_t)PART_STASH;
            u64 base = 0;
            if (lane == 0) base = atomicAdd(&Q.pc[PC_POOL], grab);
            base = __shfl_sync(0xFFFFFFFFu, base, 0);
            stash_next = base;
            stash_end = base + grab;
        }
        u64 first[2];
        first[0] = stash_next + (incl - k[0] - k[1]);
        first[1] = first[0] + k[0];
        stash_next += total;
#pragma unroll
        for (int h = 0; h < 2; ++h) {
            const uint32_t b = lane + 32 * h;
            bool ok = true;
            if (k[h]) {
                ok = first[h] + k[h] <= Q.pool_chunks;
                if (ok) {
                    for (uint32_t j = 0; j < k[h]; ++j) Q.chunk_bucket[first[h] + j] = (uint8_t)b;
                } else {
                    atomicExch(&Q.pc[PC_OVERFLOW], 1ull);
                }
            }
            bs[h].z = (uint32_t)(first[h] * PART_CHUNK) - bs[h].y;
            bs[h].w = ok ? 1u : 0u;
            ws.bstate[b] = bs[h];
        }
        __syncwarp();
        for (uint32_t i = lane; i < staged; i += 32) {
            const uint32_t meta = ws.smeta[i];
            const uint32_t rank = meta >> 8;
            const uint4 st = ws.bstate[meta & 0xFFu];
            const bool in_open = rank < st.y;
            const uint32_t dst = (in_open ? st.x : st.z) + rank;
            if (in_open || st.w) {
                Q.pool_keys[dst] = ws.skey[i];  // plain stores: the 16- and 8-byte pieces merge into full
                Q.pool_ords[dst] = ws.sord[i];  // lines in the L2 before they are written back
            }
        }
        __syncwarp();
#pragma unroll
        for (int h = 0; h < 2; ++h) {
            const uint32_t b = lane + 32 * h;
            if (n[h]) {
                if (n[h] <= bs[h].y) {
                    bs[h].x += n[h];
                    bs[h].y -= n[h];
                } else if (bs[h].w) {
                    const uint32_t used = n[h] - bs[h].y;  // records that went into the new chunks
                    bs[h].x = (uint32_t)(first[h] * PART_CHUNK) + used;
                    bs[h].y = k[h] * PART_CHUNK - used;
                } else {
                    bs[h].y = 0u;
                }
                ws.bstate[b] = bs[h];
                ws.cnt[b] = 0u;
            }
        }
        staged = 0;
        __syncwarp();
    }

    template <int LW, typename OrdOf>
    __device__ __forceinline__ void emit(const uint4 (&cand)[PROBE_BATCH], const bool (&live)[PROBE_BATCH],
                                         const bool (&known_in)[PROBE_BATCH], OrdOf ord_of) {
        const uint32_t lt = lanemask_lt();
        const uint32_t mask32 = (uint32_t)P.slot_mask;
        uint32_t hash[PROBE_BATCH];
        bool known[PROBE_BATCH];
#pragma unroll
        for (int r = 0; r < PROBE_BATCH; ++r) {
            hash[r] = hash_vec(cand[r], 0u);
            known[r] = known_in[r];
        }
#pragma unroll
        for (int r = 0; r < PROBE_BATCH; ++r) {
            const bool sep = cm_sep_diff<LW>(cand[r], P.target) == 0u;
            // a duplicate by construction is dropped here, unless it separates: exhaustive runs list
            // every separating ordinal, so those few take the normal route through phase B
            const bool need = live[r] && (!known[r] || sep);
            const uint32_t m = __ballot_sync(0xFFFFFFFFu, need);
            if (need) {
                const u64 ord = ord_of(r);
                const uint32_t b = (hash[r] & mask32) >> Q.bucket_shift;
                const uint32_t rank = atomicAdd(&ws.cnt[b], 1u);
                const uint32_t i = staged + __popc(m & lt);
                ws.skey[i] = cand[r];
                ws.sord[i] = ord;
                ws.smeta[i] = b | rank << 8;
                if (sep && Q.sep_bound_ok) atomicMin(&Q.pc[PC_SEPBOUND], ord);
            }
            staged += __popc(m);
        }
        if (staged > (uint32_t)PART_STAGE_FLUSH) write_out();
    }

    // start of a launch: adopt the open chunks and the stash this warp slot was left with
    __device__ __forceinline__ void adopt(u64 slot) {
        const int lane = threadIdx.x & 31;
        const u64 *w = Q.wstate + slot * PART_WSTATE;
#pragma unroll
        for (int h = 0; h < 2; ++h) {
            const u64 v = slot < Q.wstate_slots ? w[lane + 32 * h] : 0ull;
            ws.cnt[lane + 32 * h] = 0u;
            ws.bstate[lane + 32 * h] = make_uint4((uint32_t)v, (uint32_t)(v >> 32), 0u, 0u);
        }
        if (slot < Q.wstate_slots) {
            stash_next = w[PART_NB];
            stash_end = w[PART_NB + 1];
        }
        __syncwarp();
    }

    // end of a launch: write out what is staged, hand the state to the slot's next user
    __device__ __forceinline__ void finish(u64 slot) {
        const int lane = threadIdx.x & 31;
        if (staged) write_out();
        __syncwarp();
        u64 *w = Q.wstate + slot * PART_WSTATE;
        if (slot < Q.wstate_slots) {
#pragma unroll
            for (int h = 0; h < 2; ++h) {
                const uint4 bs = ws.bstate[lane + 32 * h];
                w[lane + 32 * h] = (u64)bs.y << 32 | bs.x;
            }
            if (lane == 0) {
                w[PART_NB] = stash_next;
                w[PART_NB + 1] = stash_end;
            }
        } else {  // no slot to carry the state in (cannot happen with the host's sizing): seal here
#pragma unroll
            for (int h = 0; h < 2; ++h) {
                const uint4 bs = ws.bstate[lane + 32 * h];
                if (bs.y > 0u && bs.y < (uint32_t)PART_CHUNK) Q.chunk_fill[bs.x / PART_CHUNK] = (uint8_t)(PART_CHUNK - bs.y);
            }
        }
    }
};

template <int LW, int OP>
__global__ void __launch_bounds__(CTA_THREADS, LTLB200_PART_MIN_CTAS) narrow_partition_kernel(const NarrowParams P, const PartParams Q) {
    extern __shared__ __align__(16) unsigned char s_raw[];
    WarpSharedPart &ws = reinterpret_cast<WarpSharedPart *>(s_raw)[threadIdx.x >> 5];
    const u64 slot = (u64)blockIdx.x * WARPS_PER_CTA + (threadIdx.x >> 5);
    PartSink sink{P, Q, ws};
    sink.adopt(slot);
    const u64 *bound = (Q.sep_bound_ok && P.prune_after_sep) ? &Q.pc[PC_SEPBOUND] : nullptr;
    TileFetch next = fetch_tile(P, bound);
    for (;;) {
        const TileFetch cur = next;
        if (!open_tile(P, ws, cur)) break;
        next = fetch_tile(P, bound);
        if (run_tile<LW, OP>(P, ws, sink)) break;
    }
    sink.finish(slot);
}

// After the last operator launch of a segment: record the fill of every warp slot's open
// chunks, and count the chunks of each bucket (block-level histogram, one global atomicAdd per
// block and bucket).
__global__ void __launch_bounds__(256) part_seal_kernel(const PartParams Q) {
    __shared__ uint32_t hist[PART_NB];
    if (threadIdx.x < PART_NB) hist[threadIdx.x] = 0u;
    __syncthreads();
    const u64 tid = (u64)blockIdx.x * blockDim.x + threadIdx.x, stride = (u64)gridDim.x * blockDim.x;
    for (u64 i = tid; i < Q.wstate_slots * PART_NB; i += stride) {
        const u64 v = Q.wstate[(i / PART_NB) * PART_WSTATE + (i % PART_NB)];
        const uint32_t x = (uint32_t)v, left = (uint32_t)(v >> 32);
        if (left > 0u && left < (uint32_t)PART_CHUNK) Q.chunk_fill[x / PART_CHUNK] = (uint8_t)(PART_CHUNK - left);
    }
    const u64 drawn = min(Q.pc[PC_POOL], Q.pool_chunks);
    for (u64 c = tid; c < drawn; c += stride) {
        const uint32_t b = Q.chunk_bucket[c];
        if (b != 0xFFu) atomicAdd(&hist[b], 1u);
    }
    __syncthreads();
    if (threadIdx.x < PART_NB && hist[threadIdx.x]) atomicAdd(&Q.pc[PC_BUCKET0 + threadIdx.x], (u64)hist[threadIdx.x]);
}

// Groups the chunk ids by bucket (counting sort): every block ranks its chunks inside their
// buckets in shared memory and reserves its ranges with one atomicAdd per bucket.
__global__ void __launch_bounds__(256) part_order_kernel(const PartParams Q) {
    __shared__ u64 off[PART_NB];
    __shared__ uint32_t hist[PART_NB];
    __shared__ u64 base[PART_NB];
    if (threadIdx.x == 0) {
        u64 acc = 0;
        for (int b = 0; b < PART_NB; ++b) {
            off[b] = acc;
            acc += Q.pc[PC_BUCKET0 + b];
        }
        if (blockIdx.x == 0) Q.pc[PC_ORDERED] = acc;
    }
    if (threadIdx.x < PART_NB) hist[threadIdx.x] = 0u;
    __syncthreads();
    const u64 drawn = min(Q.pc[PC_POOL], Q.pool_chunks);
    // a block owns a contiguous range of chunk ids, PER_THREAD per thread
    constexpr int PER_THREAD = 8;
    const u64 c0 = ((u64)blockIdx.x * blockDim.x + threadIdx.x) * PER_THREAD;
    uint32_t bucket[PER_THREAD], rank[PER_THREAD];
#pragma unroll
    for (int j = 0; j < PER_THREAD; ++j) {
        const u64 c = c0 + j;
        bucket[j] = c < drawn ? Q.chunk_bucket[c] : 0xFFu;
        rank[j] = bucket[j] != 0xFFu ? atomicAdd(&hist[bucket[j]], 1u) : 0u;
    }
    __syncthreads();
    if (threadIdx.x < PART_NB) base[threadIdx.x] = hist[threadIdx.x] ? off[threadIdx.x] + atomicAdd(&Q.pc[PC_CURSOR0 + threadIdx.x], (u64)hist[threadIdx.x]) : 0ull;
    __syncthreads();
#pragma unroll
    for (int j = 0; j < PER_THREAD; ++j)
        if (bucket[j] != 0xFFu) Q.order[base[bucket[j]] + rank[j]] = (uint32_t)(c0 + j);
}
constexpr int PART_ORDER_PER_BLOCK = 256 * 8;  // chunk ids per block of part_order_kernel

// Phase B: a warp takes PART_TICKET_CHUNKS chunks per ticket in bucket order and runs them,
// PROBE_BATCH/2 chunks (PROBE_BATCH records per lane) at a time, through the direct path's
// probe machinery.  The records of the next batch are loaded before the current ones are
// probed (the stream comes from HBM, the probes hit the L2-resident window).
struct ProbeBatch {
    uint4 cand[PROBE_BATCH];
    u64 ords[PROBE_BATCH];
    bool live[PROBE_BATCH];
};

struct ProbeTicket {  // lane l < PART_TICKET_CHUNKS: chunk l of the ticket
    u64 chunk = 0;
    uint32_t fill = 0;
    bool any = false;  // warp-uniform
};

__device__ __forceinline__ ProbeTicket probe_ticket(const NarrowParams &P, const PartParams &Q, u64 n_chunks) {
    const int lane = threadIdx.x & 31;
    ProbeTicket T;
    u64 t = 0;
    if (lane == 0) {
        t = ~0ull;
        if (__ldcg(&P.counters[CTR_OVERFLOW]) == 0ull) t = atomicAdd(&Q.pc[PC_TICKET], 1ull);
    }
    t = __shfl_sync(0xFFFFFFFFu, t, 0);
    T.any = t != ~0ull && t * PART_TICKET_CHUNKS < n_chunks;
    const u64 k = t * PART_TICKET_CHUNKS + lane;
    if (T.any && lane < PART_TICKET_CHUNKS && k < n_chunks) {
        T.chunk = Q.order[k];
        T.fill = Q.chunk_fill[T.chunk];
    }
    return T;
}

__device__ __forceinline__ void probe_load(const PartParams &Q, const ProbeTicket &T, int step, ProbeBatch &B) {
    constexpr int CHUNKS_PER_STEP = PROBE_BATCH / 2;
    const int lane = threadIdx.x & 31;
#pragma unroll
    for (int c = 0; c < CHUNKS_PER_STEP; ++c) {
        const u64 chunk = __shfl_sync(0xFFFFFFFFu, T.chunk, step * CHUNKS_PER_STEP + c);
        const uint32_t fill = __shfl_sync(0xFFFFFFFFu, T.fill, step * CHUNKS_PER_STEP + c);
#pragma unroll
        for (int h = 0; h < 2; ++h) {
            const int r = 2 * c + h;
            const uint32_t idx = lane + 32 * h;
            B.live[r] = idx < fill;
            B.cand[r] = B.live[r] ? __ldcs(&Q.pool_keys[chunk * PART_CHUNK + idx]) : make_uint4(0, 0, 0, 0);
            B.ords[r] = B.live[r] ? __ldcs(&Q.pool_ords[chunk * PART_CHUNK + idx]) : 0ull;
        }
    }
}

template <int LW>
__global__ void __launch_bounds__(CTA_THREADS, LTLB200_PROBE_MIN_CTAS) narrow_probe_kernel(const NarrowParams P, const PartParams Q) {
    static_assert(PROBE_BATCH == 4 || PROBE_BATCH == 2, "phase B maps chunks onto the probe batch");
    constexpr int STEPS = PART_TICKET_CHUNKS / (PROBE_BATCH / 2);
    __shared__ Parked s_queue[WARPS_PER_CTA][QUEUE_CAP];
    Parked *queue = s_queue[threadIdx.x >> 5];
    WarpState st;
    const u64 n_chunks = Q.pc[PC_ORDERED];
    ProbeTicket T = probe_ticket(P, Q, n_chunks);
    while (T.any) {
        const ProbeTicket next = probe_ticket(P, Q, n_chunks);  // consumed after this ticket's records
        ProbeBatch cur, nxt;
        probe_load(Q, T, 0, cur);
#pragma unroll 1
        for (int step = 0; step < STEPS; ++step) {
            if (step + 1 < STEPS) probe_load(Q, T, step + 1, nxt);
            const bool known[PROBE_BATCH] = {};
            auto ord_of = [&](int r) { return cur.ords[r]; };
            insert_batch<LW>(P, queue, st, cur.cand, cur.live, known, ord_of);
            cur = nxt;
        }
        T = next;
    }
    if (__ldcg(&P.counters[CTR_OVERFLOW]) == 0ull)
        while (st.qfill > 0u) drain_round(P, queue, st);
}

}  // namespace ltlb200
