// narrow_async.cuh -- the direct construction + dedup kernel with an asynchronous probe pipeline.
//
// Why: ncu on the synchronous kernel (narrow_level_kernel, profiles/r01_s2_*) shows a latency
// chain, not a bandwidth limit: a warp builds 128 candidates, loads their 128 slots, WAITS,
// claims the new ones with a CAS, WAITS, resolves the parked ones, WAITS -- 13.7 us per batch,
// 16 warps per SM (128 registers), issue slots 25 % used, ~220 probes in flight per SM where
// the memory system wants thousands.  Registers cap the loads a thread can have in flight, so
// here the slot snapshots do not go to registers at all: every probe is a cp.async (LDGSTS)
// from the hash set straight into a per-warp ring of stages in shared memory, together with
// the candidate and its ordinal.  A warp keeps ASYNC_STAGES batches (x 128 probes) in flight
// while it builds the next batch; a stage is consumed -- classified from shared memory -- only
// when its copies have landed (cp.async.wait_group), several batches later.
//
//   emit    candidate + ordinal + flags -> stage[head]; cp.async slot key (16 B) and val (8 B)
//           -> stage[head]; commit.  If the ring is full, consume the oldest stage first.
//   consume per entry: duplicate of an earlier level -> nothing; claimed earlier in this level
//           -> one fire-and-forget atomicMin on its ordinal; everything else (empty slot = new
//           CM, collision, unpublished claim, separating, all-ones key) -> parked queue, whose
//           rounds (drain_round) do the CAS / re-probe 32 at a time as before.
//
// Results are identical to the synchronous kernel: the set, the claim arrays and the
// min-ordinal rule are the same; only when a probe's answer is looked at changes.
#pragma once
#include "narrow.cuh"

namespace ltlb200 {

#ifndef LTLB200_ASYNC_STAGES
#define LTLB200_ASYNC_STAGES 3
#endif
#ifndef LTLB200_ASYNC_MIN_CTAS
#define LTLB200_ASYNC_MIN_CTAS 2
#endif
constexpr int ASYNC_STAGES = LTLB200_ASYNC_STAGES;
constexpr int STAGE_N = 32 * PROBE_BATCH;  // entries per stage: lane l owns entries l, l+32, ...

// while an entry waits in a stage the top bits of its ordinal carry its flags (ordinals are < 2^60)
constexpr u64 SF_LIVE = 1ull << 60, SF_PROBED = 1ull << 61, SF_SEP = 1ull << 62, SF_OLD = 1ull << 63;
constexpr u64 SF_ORD_MASK = SF_LIVE - 1;

struct __align__(16) AsyncStage {
    uint4 key[STAGE_N];       // the candidate
    uint4 snap_key[STAGE_N];  // its home slot as the probe found it: key ...
    u64 snap_val[STAGE_N];    // ... and val
    u64 ord[STAGE_N];         // ordinal | SF_*
};

struct __align__(16) WarpSharedAsync {
    AsyncStage stage[ASYNC_STAGES];
    Parked queue[QUEUE_CAP];
    uint4 rows[TILE_S];
    u64 term[TILE_S];
    BlockDesc block;
    u64 ticket, sep_now;
};

__device__ __forceinline__ void cp_async_16(void *smem, const void *gmem) {
    const uint32_t s = (uint32_t)__cvta_generic_to_shared(smem);
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(s), "l"(gmem) : "memory");
}
// 8-byte copies exist only with .ca (through L1).  A stale val can only read as "not published
// yet" (vals are written once and never change), which parks the entry: conservative, correct.
__device__ __forceinline__ void cp_async_8(void *smem, const void *gmem) {
    const uint32_t s = (uint32_t)__cvta_generic_to_shared(smem);
    asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(s), "l"(gmem) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() {
    asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory");
}

struct AsyncSink {
    const NarrowParams &P;
    WarpSharedAsync &ws;
    WarpState &st;
    int head = 0, inflight = 0;  // warp-uniform: stage to fill next, stages whose copies are committed

    // Classifies the entries of one landed stage.
    template <int LW>
    __device__ __forceinline__ void consume(AsyncStage &S) {
        const int lane = threadIdx.x & 31;
        const uint32_t lt = lanemask_lt();
        const uint32_t mask32 = (uint32_t)P.slot_mask;
#pragma unroll
        for (int r = 0; r < PROBE_BATCH; ++r) {
            const int i = r * 32 + lane;
            const u64 o = S.ord[i];
            const uint4 key = S.key[i];
            uint32_t flags = (o & SF_SEP) ? PK_SEP : 0u;
            uint32_t slot = hash_vec(key, 0u) & mask32;
            bool park = false;
            if (o & SF_PROBED) {
                const uint4 k0 = S.snap_key[i];
                const u64 v0 = S.snap_val[i];
                if (key_is_empty(k0)) {  // new CM (so far): the round does the CAS
                    flags |= PK_EMPTY;
                    park = true;
                } else if (v_eq(k0, key)) {
                    if (v0 == VAL_EMPTY || (o & SF_SEP)) {
                        park = true;  // index not published yet / separating: the queue handles it
                    } else if (v0 >= P.epoch) {
                        atomicMin(&P.claim_ord[v0 & CLAIM_IDX_MASK], o & SF_ORD_MASK);  // same level: keep the smaller ordinal
                    }  // else: stored by an earlier level
                } else {  // another CM lives there: linear probing
                    slot = (slot + 1) & mask32;
                    park = true;
                }
            } else if (o & SF_LIVE) {
                if (o & SF_OLD) {  // duplicate by construction: matters only if it separates (exhaustive lists)
                    if (o & SF_SEP) {
                        flags |= PK_OLD;
                        park = true;
                    }
                } else {  // the all-ones key: side register
                    flags |= PK_SPECIAL;
                    park = true;
                }
            }
            const uint32_t m = __ballot_sync(0xFFFFFFFFu, park);
            if (park) {
                Parked e;
                e.key = key;
                e.ord = o & SF_ORD_MASK;
                e.slot = slot;
                e.flags = flags;
                ws.queue[st.qfill + __popc(m & lt)] = e;
            }
            st.qfill += __popc(m);
        }
        __syncwarp();
        while (st.qfill >= 32u) drain_round(P, ws.queue, st);
    }

    template <int LW>
    __device__ __forceinline__ void consume_oldest() {
        const int tail = (head + ASYNC_STAGES - inflight) % ASYNC_STAGES;
        consume<LW>(ws.stage[tail]);
        --inflight;
    }

    template <int LW, typename OrdOf>
    __device__ __forceinline__ void emit(const uint4 (&cand)[PROBE_BATCH], const bool (&live)[PROBE_BATCH],
                                         const bool (&known)[PROBE_BATCH], OrdOf ord_of) {
        const int lane = threadIdx.x & 31;
        const uint32_t mask32 = (uint32_t)P.slot_mask;
        if (inflight == ASYNC_STAGES) {  // ring full: the oldest stage's copies must have landed
            cp_async_wait<ASYNC_STAGES - 1>();
            consume_oldest<LW>();
        }
        AsyncStage &S = ws.stage[head];
#pragma unroll
        for (int r = 0; r < PROBE_BATCH; ++r) {
            const int i = r * 32 + lane;
            const bool sep = cm_sep_diff<LW>(cand[r], P.target) == 0u;
            const bool special = P.special_possible && key_is_empty(cand[r]);
            const bool probe = live[r] && !known[r] && !special;
            u64 o = ord_of(r);
            if (live[r]) o |= SF_LIVE;
            if (probe) o |= SF_PROBED;
            if (sep) o |= SF_SEP;
            if (known[r]) o |= SF_OLD;
            S.ord[i] = live[r] ? o : 0ull;
            S.key[i] = cand[r];
            if (probe) {
                const Slot16 *slot = &P.slots[hash_vec(cand[r], 0u) & mask32];
                cp_async_16(&S.snap_key[i], &slot->key);
                cp_async_8(&S.snap_val[i], &slot->val);
            }
        }
        cp_async_commit();
        head = (head + 1) % ASYNC_STAGES;
        ++inflight;
    }

    // end of the launch: everything in flight lands and is classified, then the queue empties
    template <int LW>
    __device__ __forceinline__ void finish() {
        cp_async_wait<0>();
        while (inflight > 0) consume_oldest<LW>();
        if (__ldcg(&P.counters[CTR_OVERFLOW]) == 0ull)
            while (st.qfill > 0u) drain_round(P, ws.queue, st);
    }
};

template <int LW, int OP>
__global__ void __launch_bounds__(CTA_THREADS, LTLB200_ASYNC_MIN_CTAS) narrow_async_kernel(const NarrowParams P) {
    extern __shared__ __align__(16) unsigned char s_raw[];
    WarpSharedAsync &ws = reinterpret_cast<WarpSharedAsync *>(s_raw)[threadIdx.x >> 5];
    WarpState st;
    AsyncSink sink{P, ws, st};
    TileFetch next = fetch_tile(P, nullptr);
    for (;;) {
        const TileFetch cur = next;
        if (!open_tile(P, ws, cur)) break;
        next = fetch_tile(P, nullptr);
        if (run_tile<LW, OP>(P, ws, sink)) break;
    }
    sink.template finish<LW>();
}

}  // namespace ltlb200
