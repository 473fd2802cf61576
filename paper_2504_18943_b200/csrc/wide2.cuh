// wide2.cuh -- construction + dedup kernel for multi-vector CMs, one LANE per candidate.
//
// Round 1's first wide kernel gave a candidate to a group of G lanes (one uint4 each).  Its ncu capture on the
// LTL configuration of BASELINE.json (c5: 128-byte CMs) showed why that is slow: 96 warp
// instructions per candidate, because everything that is scalar per candidate -- hashing,
// the slot probe, the claim, the CAS -- ran with 1/G of the lanes, and every step was a
// group-wide ballot or shuffle.  Here a lane owns a whole candidate, like in the narrow path:
//
//   * a tile = 32 vector-operand rows (one per lane) x up to tile_s scalar-operand rows; both are
//     staged in the warp's shared memory, the vector rows TRANSPOSED (vec[p*32 + lane]) so that
//     the 32 lanes read 32 consecutive uint4 (no bank conflicts), the scalar rows as they are
//     (all lanes read the same address: a broadcast);
//   * a candidate is never held in registers as a whole.  Pass 1 streams over its nvec vectors:
//     build vector p, fold it into the two row hashes, the separation flag and the
//     "equals an operand" flags.  Then one 8-byte slot probe.  Then, only for the candidates that
//     need it, pass 2 streams over the vectors again: a CLAIM writes them to its staging entry,
//     a fingerprint MATCH compares them with the stored row.  Rebuilding a vector costs a few
//     dozen integer instructions; keeping 32 rows x nvec vectors in registers is impossible;
//   * the hash set, the row log and the publish protocol (row -> release-ordered 64-bit CAS on the slot word)
//     are wide_common.cuh's; the group-collective insert there serves the import of exchanged records and
//     the regrow, against the same set;
//   * the regex grammar (LW_REGEX) has its own tiles for the operators that are not vector-local
//     (wide2_regex.cuh) and shares the passes below.
#pragma once
#include "regex_ops.cuh"
#include "wide_common.cuh"

namespace ltlb200 {

// CTAs per SM: 2..6 measure the same on c5 (the big levels run at ~70 % of the random-access
// ceiling of the memory system, not at an occupancy limit); 3 leaves 168 registers for the row prefetch.
#ifndef LTLB200_WIDE2_MIN_CTAS
#define LTLB200_WIDE2_MIN_CTAS 3
#endif
#ifndef LTLB200_RE_MIN_CTAS
#define LTLB200_RE_MIN_CTAS 5  // regex tiles: one candidate per lane in the passes; 96 registers (4 and 5 CTAs measure the same on the e-mail example, 5 is 9 % faster on re-c2, 6 spills)
#endif
#ifndef LTLB200_W2_BATCH
#define LTLB200_W2_BATCH 2
#endif
constexpr int W2_BATCH = LTLB200_W2_BATCH;  // candidates a lane carries through the passes together
#ifndef LTLB200_W2_PREFETCH
#define LTLB200_W2_PREFETCH 4
#endif
constexpr int W2_PREFETCH = LTLB200_W2_PREFETCH;  // vectors of a stored row fetched ahead of the full-row compare
constexpr int W2_SC_VECS = 512;    // uint4 vectors of scalar-operand rows staged per warp (8 KiB)
constexpr int W2_TERMS = 128;      // max scalar rows per tile
// what a tile does with its candidates (wide2_batch / wide2_route_batch); W2_TINY = W2_PLAIN inside the kernel that
// builds several levels per launch (wide2_tiny.cuh): the rows and the row directory it reads were written by that
// very kernel, which rules out the read-only path
enum : int { W2_PLAIN = 0, W2_GUARD = 1, W2_ROUTE = 2, W2_TINY = 3 };

template <int MODE, typename T>
__device__ __forceinline__ T w2_ld(const T *p) {
    if constexpr (MODE == W2_TINY) return __ldcg(p);
    else return __ldg(p);
}

struct __align__(16) Wide2Fixed {  // per-warp shared state behind the row areas
    u64 term[W2_TERMS];
    BlockDesc block;
    u64 ticket, sep_now;
};

// Regex grammar (LW_REGEX, wide2_regex.cuh): fewer scalar rows per tile, and one more area per warp the size of the
// vector-row area -- the 32 vector rows BIT-SLICED (word x = bit x of every row); the vector-row area itself also
// takes the 32 result rows of the concatenation and star tiles.
constexpr int W2_RE_SC_VECS = 128;

// per-warp shared memory in uint4 units: vec rows | scalar rows | valid + target | fixed part [| bit-sliced rows]
__host__ __device__ inline size_t wide2_warp_vecs(int nvec, bool regex = false) {
    const size_t fixed = 2 * (size_t)nvec + (sizeof(Wide2Fixed) + 15) / 16;
    if (regex) return (size_t)nvec * 32 + W2_RE_SC_VECS + fixed + (size_t)nvec * 32;
    return (size_t)nvec * 32 + W2_SC_VECS + fixed;
}
__host__ __device__ inline int wide2_tile_s(int nvec, bool regex = false) {
    const int rows = (regex ? W2_RE_SC_VECS : W2_SC_VECS) / nvec;
    return rows < W2_TERMS ? rows : W2_TERMS;
}

struct Wide2Warp {
    uint4 *vec;     // [nvec][32] transposed vector-operand rows
    uint4 *sc;      // [tile_s][nvec] scalar-operand rows
    uint4 *consts;  // [0, nvec) valid masks, [nvec, 2 nvec) targets
    Wide2Fixed *fx;
    // regex grammar: the guide tables (regex_ops.cuh; staged in the CTA's shared memory on request), the vector rows
    // bit-sliced, and the result rows ([word][lane] once finished)
    const uint32_t *guide;
    uint32_t *sliced, *out;
};

struct Wide2State {  // warp-uniform registers
    u64 chunk_next = 0, chunk_end = 0;  // staging entries reserved for this warp
};

// lanes with `want` get one staging entry each (ballot ranks; one atomicAdd per CLAIM_CHUNK entries)
__device__ __forceinline__ u64 wide2_reserve(const WideParams &P, Wide2State &st, bool want) {
    const uint32_t m = __ballot_sync(0xFFFFFFFFu, want);
    const uint32_t n = __popc(m);
    if (n == 0u) return 0;
    const uint32_t rem = (uint32_t)(st.chunk_end - st.chunk_next);
    u64 fresh = 0;
    if (n > rem) {
        if ((threadIdx.x & 31) == 0) fresh = atomicAdd(&P.counters[CTR_CLAIMED], (u64)CLAIM_CHUNK);
        fresh = __shfl_sync(0xFFFFFFFFu, fresh, 0);
    }
    const uint32_t rank = __popc(m & lanemask_lt());
    const u64 mine = rank < rem ? st.chunk_next + rank : fresh + (rank - rem);
    if (n > rem) {
        st.chunk_next = fresh + (n - rem);
        st.chunk_end = fresh + CLAIM_CHUNK;
    } else {
        st.chunk_next += n;
    }
    return mine;
}

// 64-bit compare-and-swap with release semantics at gpu scope: the row written by this lane is visible to whoever
// reads the published word
__device__ __forceinline__ u64 cas64_release(u64 *addr, u64 expect, u64 desired) {
    u64 old;
    asm volatile("atom.release.gpu.global.cas.b64 %0, [%1], %2, %3;" : "=l"(old) : "l"(addr), "l"(expect), "l"(desired) : "memory");
    return old;
}

__device__ __forceinline__ uint32_t v_diff(uint4 a, uint4 b) { return (a.x ^ b.x) | (a.y ^ b.y) | (a.z ^ b.z) | (a.w ^ b.w); }

// Carries NB candidates of one lane (W2_BATCH; 1 in the regex tiles) through hash -> probe -> claim / compare.
// `gen(r, p, a, b, c)` yields the operands of candidate r's vector p in formula order and the vector itself (for the
// LTL operators c = cm_apply(a, b): a vector depends on the same vector of its operands; the regex concatenation
// and star read bits all over their operands, see the regex tiles below).
// GUARD (wide2_guarded_level_kernel): candidates whose ordinal lies in a dead range do not exist, and in the scan
// pass only the ordinal of every separating candidate is recorded (NarrowParams::dead / scan_only).
template <int LW, int OP, bool GUARD, int NB, class Gen>
__device__ __forceinline__ void wide2_batch(const WideParams &P, const Wide2Warp &W, Wide2State &st, Gen gen,
                                            const bool (&live_in)[NB], const u64 (&ords)[NB]) {
    const int nvec = P.nvec;
    const uint32_t mask32 = (uint32_t)P.slot_mask;
    bool live[NB];
#pragma unroll
    for (int r = 0; r < NB; ++r) {
        live[r] = live_in[r];
        if (GUARD && P.dead_n && live[r] && ordinal_is_dead(P.dead, P.dead_n, ords[r])) live[r] = false;
    }
    // ---- pass 1: hashes, separation flag, duplicate-by-construction flags
    uint32_t ha[NB], hb[NB], sepacc[NB], da[NB], db[NB];
#pragma unroll
    for (int r = 0; r < NB; ++r) ha[r] = hb[r] = sepacc[r] = da[r] = db[r] = 0u;
#pragma unroll 1
    for (int p = 0; p < nvec; ++p) {
        const uint4 valid = W.consts[p], target = W.consts[nvec + p];
        const uint32_t seed_a = 0x9E3779B9u * (uint32_t)(p + 1), seed_b = 0x7F4A7C15u * (uint32_t)(p + 1) + 0x632BE5ABu;
#pragma unroll
        for (int r = 0; r < NB; ++r) {
            uint4 a, b, c;
            gen(r, p, a, b, c);
            ha[r] ^= hash_vec(c, seed_a);
            hb[r] ^= hash_vec(c, seed_b);
            sepacc[r] |= cm_sep_diff<LW>(c, target, valid);
            da[r] |= v_diff(c, a);
            db[r] |= v_diff(c, b);
        }
    }
    if (GUARD && P.scan_only) {
#pragma unroll
        for (int r = 0; r < NB; ++r) {
            if (!live[r] || sepacc[r] != 0u) continue;
            const u64 pos = atomicAdd(&P.counters[CTR_SEPCOUNT], 1ull);
            if (pos < P.sep_list_cap) P.sep_list[pos] = ords[r];
        }
        return;
    }
    uint32_t slot[NB], fp[NB];
    u64 w[NB], entry[NB];
    bool active[NB], fresh[NB];
#pragma unroll
    for (int r = 0; r < NB; ++r) {  // final mix of wide_common.cuh's row_hash
        uint32_t a = ha[r], b = hb[r];
        a ^= a >> 16;
        a *= 0x85EBCA6Bu;
        a ^= a >> 13;
        b ^= b >> 15;
        b *= 0xC2B2AE35u;
        b ^= b >> 16;
        slot[r] = a & mask32;
        fp[r] = (b >> 8) & 0xFFFFFFu;
        const bool known = OP != OP_ATOM && (da[r] == 0u || db[r] == 0u);  // equals an operand: already in the cache
        active[r] = live[r] && !known;
        fresh[r] = false;
        entry[r] = ~0ull;
        w[r] = active[r] ? __ldcg(&P.slots[slot[r]]) : 0ull;
    }
    // ---- resolve: every round, claims write their row and matches compare theirs in ONE pass over the vectors
    for (;;) {
        bool claim[NB], match[NB];
        bool any = false;
#pragma unroll
        for (int r = 0; r < NB; ++r) {
            claim[r] = active[r] && w[r] == 0ull;
            match[r] = active[r] && !claim[r] && (uint32_t)(w[r] >> 40) == fp[r];
            if (active[r] && !claim[r] && !match[r]) {  // another CM lives there: linear probing
                slot[r] = (slot[r] + 1) & mask32;
                w[r] = __ldcg(&P.slots[slot[r]]);
            }
            any = any || active[r];
        }
        if (!__any_sync(0xFFFFFFFFu, any)) break;
        bool staged_row[NB];
        const uint4 *row[NB];
        uint32_t diff[NB];
#pragma unroll
        for (int r = 0; r < NB; ++r) {
            const bool want = claim[r] && entry[r] == ~0ull;  // (a lost race left this candidate its entry)
            const u64 got = wide2_reserve(P, st, want);
            if (want) entry[r] = got;
            if (claim[r] && entry[r] >= P.stage_cap) {  // staging pool exhausted: the host regrows and redoes the level
                atomicExch(&P.counters[CTR_OVERFLOW], 1ull);
                claim[r] = active[r] = false;
            }
            const u64 idx = (w[r] & SLOT_IDX_MASK) - 1;
            staged_row[r] = match[r] && idx >= P.total_before;
            row[r] = match[r] ? (staged_row[r] ? P.stage_rows + (idx - P.total_before) * nvec : P.store + idx * nvec) : nullptr;
            diff[r] = 0u;
        }
        // The stored rows of the fingerprint matches are fetched W2_PREFETCH vectors ahead of the compare: taken one
        // at a time (load, compare, next vector) a 128-byte CM costs eight dependent trips to the L2 / DRAM, and
        // the first ncu capture had a third of this kernel's stall samples on exactly that compare.
#pragma unroll 1
        for (int p0 = 0; p0 < nvec; p0 += W2_PREFETCH) {
            uint4 stored[NB][W2_PREFETCH];
#pragma unroll
            for (int r = 0; r < NB; ++r)
#pragma unroll
                for (int q = 0; q < W2_PREFETCH; ++q)
                    if (match[r] && p0 + q < nvec) stored[r][q] = __ldcg(row[r] + p0 + q);
#pragma unroll
            for (int q = 0; q < W2_PREFETCH; ++q) {
                const int p = p0 + q;
                if (p >= nvec) break;
#pragma unroll
                for (int r = 0; r < NB; ++r) {
                    if (!claim[r] && !match[r]) continue;
                    uint4 a, b, c;
                    gen(r, p, a, b, c);
                    if (claim[r]) P.stage_rows[entry[r] * nvec + p] = c;
                    else diff[r] |= v_diff(c, stored[r][q]);
                }
            }
        }
#pragma unroll
        for (int r = 0; r < NB; ++r) {
            if (claim[r]) {
                // release-ordered publish: the row this lane wrote above is visible to whoever reads the word (a warp-wide
                // __threadfence() before a relaxed CAS was 5-7 % of this kernel's stall samples; c5 to cost 12: 26.2 -> 25.6 ms)
                const u64 old = cas64_release(&P.slots[slot[r]], 0ull, slot_word(fp[r], P.total_before + entry[r]));
                if (old == 0ull) {
                    atomicMin(&P.stage_ord[entry[r]], ords[r]);
                    fresh[r] = true;
                    active[r] = false;
                } else {
                    w[r] = old;  // somebody published here first: look at what they put (the entry is kept for a retry)
                }
            } else if (match[r]) {
                if (diff[r] == 0u) {
                    if (staged_row[r]) {
                        atomicMin(&P.stage_ord[(w[r] & SLOT_IDX_MASK) - 1 - P.total_before], ords[r]);
                        fresh[r] = true;
                    }
                    active[r] = false;
                } else {  // fingerprint alias: keep probing
                    slot[r] = (slot[r] + 1) & mask32;
                    w[r] = __ldcg(&P.slots[slot[r]]);
                }
            }
        }
    }
#pragma unroll
    for (int r = 0; r < NB; ++r) {
        if (live[r] && sepacc[r] == 0u) {
            if (fresh[r]) atomicMin(&P.counters[CTR_SEP], ords[r]);
            if (P.sep_list) {
                const u64 pos = atomicAdd(&P.counters[CTR_SEPCOUNT], 1ull);
                if (pos < P.sep_list_cap) P.sep_list[pos] = ords[r];
            }
        }
    }
}

// One search sharded over several GPUs (see narrow.cuh: "route instead of probe"): the candidate is not probed
// here; its row goes to the send region of its hash owner.  Pass 1 yields the owner hash, the separation flag and
// the equals-an-operand flags; the lanes of one owner take consecutive records (one atomicAdd per owner present in
// the batch row); pass 2 writes the row -- nvec consecutive vectors per lane, whole 32-byte sectors.
template <int LW, int OP, int NB, class Gen>
__device__ __forceinline__ void wide2_route_batch(const WideParams &P, const Wide2Warp &W, Gen gen,
                                                  const bool (&live)[NB], const u64 (&ords)[NB]) {
    const int nvec = P.nvec;
    uint32_t ho[NB], sepacc[NB], da[NB], db[NB];
#pragma unroll
    for (int r = 0; r < NB; ++r) ho[r] = sepacc[r] = da[r] = db[r] = 0u;
#pragma unroll 1
    for (int p = 0; p < nvec; ++p) {
        const uint4 valid = W.consts[p], target = W.consts[nvec + p];
#pragma unroll
        for (int r = 0; r < NB; ++r) {
            uint4 a, b, c;
            gen(r, p, a, b, c);
            ho[r] ^= hash_vec(c, 0x5BD1E995u * (uint32_t)(p + 1));
            sepacc[r] |= cm_sep_diff<LW>(c, target, valid);
            da[r] |= v_diff(c, a);
            db[r] |= v_diff(c, b);
        }
    }
    u64 at[NB];
    bool send[NB];
    const uint32_t lt = lanemask_lt();
    const int lane = threadIdx.x & 31;
#pragma unroll
    for (int r = 0; r < NB; ++r) {
        if (live[r] && sepacc[r] == 0u) {
            if (P.route_sep_any) atomicMin(&P.counters[CTR_SEP], ords[r]);
            if (P.sep_list) {
                const u64 pos = atomicAdd(&P.counters[CTR_SEPCOUNT], 1ull);
                if (pos < P.sep_list_cap) P.sep_list[pos] = ords[r];
            }
        }
        const bool known = OP != OP_ATOM && (da[r] == 0u || db[r] == 0u);  // equals an operand: already in the cache
        send[r] = live[r] && !known;
        const uint32_t owner = send[r] ? row_owner_mix(ho[r]) % P.route_world : 0xFFFFFFFFu;
        at[r] = ~0ull;
        uint32_t pending = __ballot_sync(0xFFFFFFFFu, send[r]);
        while (pending) {
            const uint32_t w = __shfl_sync(0xFFFFFFFFu, owner, __ffs(pending) - 1);
            const bool mine = owner == w;
            const uint32_t m = __ballot_sync(0xFFFFFFFFu, mine);
            pending &= ~m;
            u64 base = 0;
            if (lane == __ffs(m) - 1) base = atomicAdd(&P.route_counts[w], (u64)__popc(m));
            base = __shfl_sync(0xFFFFFFFFu, base, __ffs(m) - 1);
            if (mine) {
                const u64 pos = base + __popc(m & lt);
                if (pos < P.route_cap) {  // (past the region: only counted; the host redoes the level)
                    at[r] = (u64)w * P.route_cap + pos;
                    P.route_ords[at[r]] = ords[r];
                }
            }
        }
    }
    bool any = false;
#pragma unroll
    for (int r = 0; r < NB; ++r) any = any || at[r] != ~0ull;
    if (!any) return;
#pragma unroll 1
    for (int p = 0; p < nvec; ++p) {
#pragma unroll
        for (int r = 0; r < NB; ++r) {
            if (at[r] == ~0ull) continue;
            uint4 a, b, c;
            gen(r, p, a, b, c);
            P.route_rows[at[r] * nvec + p] = c;
        }
    }
}

template <int LW, int OP, int MODE>
__device__ __forceinline__ void wide2_unary_tile(const WideParams &P, const Wide2Warp &W, Wide2State &st, u64 tile_local,
                                                 u64 sep_now) {
    const BlockDesc &B = W.fx->block;
    const int lane = threadIdx.x & 31;
    const int nvec = P.nvec;
    const u64 per_tile = (u64)32 * B.tile_s;
    const u64 first = tile_local * per_tile + lane;
    const u64 ord0 = B.ord0, n = B.na;
    if (ord0 + tile_local * per_tile > sep_now) return;
    const int n_steps = (int)min((u64)B.tile_s, (n - tile_local * per_tile + 31) / 32);
#pragma unroll 1
    for (int k = 0; k < n_steps; k += W2_BATCH) {
        bool live[W2_BATCH];
        u64 ords[W2_BATCH];
        const uint4 *rows[W2_BATCH];
#pragma unroll
        for (int r = 0; r < W2_BATCH; ++r) {
            const u64 i = first + (u64)(k + r) * 32;
            live[r] = k + r < n_steps && i < n;
            ords[r] = ord0 + i;
            // a finalised row lives where it was staged (claim order): loc[id] is its place in the row log
            rows[r] = B.from_atoms ? P.atoms + (live[r] ? i : 0) * nvec : P.store + w2_ld<MODE>(P.loc + B.a_off + (live[r] ? i : 0)) * nvec;
        }
        auto gen = [&](int r, int p, uint4 &a, uint4 &b, uint4 &c) {
            a = w2_ld<MODE>(rows[r] + p);
            b = a;
            c = cm_apply<LW, OP>(a, b, W.consts[p]);
        };
        if constexpr (MODE == W2_ROUTE) wide2_route_batch<LW, OP>(P, W, gen, live, ords);
        else wide2_batch<LW, OP, MODE == W2_GUARD>(P, W, st, gen, live, ords);
    }
}

template <int LW, int OP, bool VEC_B, int MODE>
__device__ __forceinline__ void wide2_binary_tile(const WideParams &P, const Wide2Warp &W, Wide2State &st, u64 tile_local,
                                                  u64 sep_now) {
    const BlockDesc &B = W.fx->block;
    const int lane = threadIdx.x & 31;
    const int nvec = P.nvec;
    const int tile_s = (int)B.tile_s;
    const bool tri = B.kind == BK_TRI;
    const uint32_t vg_n = B.vg;
    u64 tv, ts;
    if (VEC_B) { ts = tile_local / B.tiles_v; tv = tile_local % B.tiles_v; }
    else { tv = tile_local / B.tiles_s; ts = tile_local % B.tiles_s; }
    const u64 n_vec = VEC_B ? B.nb : B.na, n_sc = VEC_B ? B.na : B.nb;
    const u64 v0 = tv * (u64)(32 * vg_n), s0 = ts * (u64)tile_s;
    const int s_cnt = (int)min((u64)tile_s, n_sc - s0);
    if (tri && v0 + (u64)32 * vg_n - 1 < s0) return;
    const u64 ord0 = B.ord0, na = B.na, nb = B.nb;
    const u64 tile_min = ord0 + (VEC_B ? (tri ? s0 * na - (s0 ? (s0 * (s0 - 1)) / 2 : 0) : s0 * nb + v0) : v0 * nb + s0);
    if (tile_min > sep_now) return;
    // operand rows by id: a finalised row lives where it was staged (claim order), loc[id] = its place in the row log
    const u64 *vec_loc = P.loc + (VEC_B ? B.b_off : B.a_off);
    const u64 *sc_loc = P.loc + (VEC_B ? B.a_off : B.b_off);
    __syncwarp();
    // stage the scalar rows (whole rows of nvec consecutive vectors) and their ordinal terms
    for (int t = lane; t < s_cnt * nvec; t += 32) {
        const int rrow = t / nvec, p = t - rrow * nvec;
        W.sc[t] = w2_ld<MODE>(P.store + w2_ld<MODE>(sc_loc + s0 + rrow) * nvec + p);
    }
    for (int k = lane; k < s_cnt; k += 32) {
        const u64 s = s0 + k;
        W.fx->term[k] = !VEC_B ? s : ord0 + (tri ? s * na - (s ? (s * (s - 1)) / 2 : 0) - s : s * nb);
    }
#pragma unroll 1
    for (uint32_t vg = 0; vg < vg_n; ++vg) {
        const u64 vbase = v0 + (u64)vg * 32;
        if (vbase >= n_vec) break;
        __syncwarp();
        // stage 32 vector rows transposed: the warp copies row after row (coalesced reads), vec[p*32 + row]
        const int rows_here = (int)min((u64)32, n_vec - vbase);
        for (int t = lane; t < rows_here * nvec; t += 32) {
            const int rrow = t / nvec, p = t - rrow * nvec;
            const uint4 x = w2_ld<MODE>(P.store + w2_ld<MODE>(vec_loc + vbase + rrow) * nvec + p);
            if constexpr (LW == LW_REGEX) {  // word q of row i at [q][i]: the concatenation tests single bits of a lane's row
                uint32_t *vw = reinterpret_cast<uint32_t *>(W.vec) + rrow;
                vw[(p * 4) * 32] = x.x;
                vw[(p * 4 + 1) * 32] = x.y;
                vw[(p * 4 + 2) * 32] = x.z;
                vw[(p * 4 + 3) * 32] = x.w;
            } else {
                W.vec[p * 32 + rrow] = x;
            }
        }
        __syncwarp();
        const u64 v = vbase + lane;
        const bool v_ok = v < n_vec;
        const u64 lane_term = VEC_B ? v : ord0 + v * nb;
        const int first_bad = tri ? (v >= s0 ? (int)min((u64)s_cnt, v - s0 + 1) : 0) : s_cnt;
        const int s_live = v_ok ? first_bad : 0;
#pragma unroll 1
        for (int k = 0; k < s_cnt; k += W2_BATCH) {
            bool live[W2_BATCH];
            u64 ords[W2_BATCH];
            int srow[W2_BATCH];
#pragma unroll
            for (int r = 0; r < W2_BATCH; ++r) {
                srow[r] = min(k + r, s_cnt - 1);
                live[r] = k + r < s_live;
                ords[r] = W.fx->term[srow[r]] + lane_term;
            }
            auto gen = [&](int r, int p, uint4 &a, uint4 &b, uint4 &c) {
                if constexpr (LW == LW_REGEX) {  // vector rows staged word by word (see above)
                    const uint32_t *vw = reinterpret_cast<const uint32_t *>(W.vec) + lane;
                    const uint4 xv = make_uint4(vw[(p * 4) * 32], vw[(p * 4 + 1) * 32], vw[(p * 4 + 2) * 32], vw[(p * 4 + 3) * 32]);
                    const uint4 xs = W.sc[srow[r] * nvec + p];
                    a = VEC_B ? xs : xv;
                    b = VEC_B ? xv : xs;
                    c = v_or(a, b);  // union (the concatenation has its own tile, wide2_regex_concat_tile)
                } else {
                    const uint4 xv = W.vec[p * 32 + lane], xs = W.sc[srow[r] * nvec + p];
                    a = VEC_B ? xs : xv;
                    b = VEC_B ? xv : xs;
                    c = cm_apply<LW, OP>(a, b, W.consts[p]);
                }
            };
            if constexpr (MODE == W2_ROUTE) wide2_route_batch<LW, OP>(P, W, gen, live, ords);
            else wide2_batch<LW, OP, MODE == W2_GUARD>(P, W, st, gen, live, ords);
        }
    }
}

#include "wide2_regex.cuh"

template <int LW>
__device__ __forceinline__ Wide2Warp wide2_carve(const WideParams &P, uint4 *base) {
    constexpr bool kRegex = LW == LW_REGEX;
    Wide2Warp W;
    uint4 *mine = base + (threadIdx.x >> 5) * wide2_warp_vecs(P.nvec, kRegex);
    W.vec = mine;
    W.sc = W.vec + (size_t)P.nvec * 32;
    W.consts = W.sc + (kRegex ? W2_RE_SC_VECS : W2_SC_VECS);
    W.fx = reinterpret_cast<Wide2Fixed *>(W.consts + 2 * (size_t)P.nvec);
    W.guide = P.guide;
    W.sliced = W.out = nullptr;
    if constexpr (kRegex) {
        W.sliced = reinterpret_cast<uint32_t *>(mine + (size_t)P.nvec * 32 + W2_RE_SC_VECS + 2 * (size_t)P.nvec + (sizeof(Wide2Fixed) + 15) / 16);
        W.out = reinterpret_cast<uint32_t *>(W.vec);  // (the union tile stages its vector rows there, wide2_binary_tile)
        if (P.guide_smem_words) {  // the guide table behind the warps' areas: one copy per CTA
            uint32_t *g = reinterpret_cast<uint32_t *>(base + (size_t)WARPS_PER_CTA * wide2_warp_vecs(P.nvec, true));
            for (uint32_t k = threadIdx.x; k < P.guide_smem_words; k += blockDim.x) g[k] = __ldg(P.guide + k);
            W.guide = g;
            __syncthreads();
        }
    }
    const int lane = threadIdx.x & 31;
    for (int p = lane; p < P.nvec; p += 32) {
        W.consts[p] = P.valid[p];
        W.consts[P.nvec + p] = P.target[p];
    }
    __syncwarp();
    return W;
}

__device__ __forceinline__ bool wide2_next_tile(const WideParams &P, const Wide2Warp &W) {
    const int lane = threadIdx.x & 31;
    __syncwarp();
    if (lane == 0) {
        u64 t = P.tile_end;
        if (*(volatile u64 *)&P.counters[CTR_OVERFLOW] == 0ull && !deadline_passed(P.counters))
            t = P.tile_begin + P.shard_offset + atomicAdd(&P.counters[P.ticket], 1ull) * P.shard_stride;
        W.fx->ticket = t;
        W.fx->sep_now = P.prune_after_sep ? *(volatile u64 *)&P.counters[CTR_SEP] : (u64)~0ull;
        if (t < P.tile_end) {
            int bi = P.block_begin;
            while (bi + 1 < P.block_end && t >= P.blocks[bi + 1].tile0) ++bi;
            W.fx->block = P.blocks[bi];
        }
    }
    __syncwarp();
    return W.fx->ticket < P.tile_end;
}

template <int LW, int OP, int MODE = W2_PLAIN>
__device__ __forceinline__ void wide2_run_tile(const WideParams &P, const Wide2Warp &W, Wide2State &st) {
    const u64 sep_now = W.fx->sep_now;
    if (W.fx->block.ord0 > sep_now) return;
    const u64 tile_local = W.fx->ticket - W.fx->block.tile0;
    if constexpr (OP == OP_RE_CONCAT) {
        if (W.fx->block.vec_is_b) wide2_regex_concat_tile<true, MODE>(P, W, st, tile_local, sep_now);
        else wide2_regex_concat_tile<false, MODE>(P, W, st, tile_local, sep_now);
    } else if constexpr (OP == OP_AND || OP == OP_OR || OP == OP_UNTIL) {
        if (W.fx->block.vec_is_b) wide2_binary_tile<LW, OP, true, MODE>(P, W, st, tile_local, sep_now);
        else wide2_binary_tile<LW, OP, false, MODE>(P, W, st, tile_local, sep_now);
    } else if constexpr (LW == LW_REGEX) {
        wide2_regex_unary_tile<OP, MODE>(P, W, st, tile_local, sep_now);
    } else {
        wide2_unary_tile<LW, OP, MODE>(P, W, st, tile_local, sep_now);
    }
}

// the tile's operator read from its block (kernels that serve every operator in one launch)
template <int LW, int MODE>
__device__ __forceinline__ void wide2_run_tile_any(const WideParams &P, const Wide2Warp &W, Wide2State &st) {
    if constexpr (LW == LW_REGEX) {
        switch (W.fx->block.op) {
            case OP_ATOM: wide2_run_tile<LW, OP_ATOM, MODE>(P, W, st); break;
            case OP_RE_QUESTION: wide2_run_tile<LW, OP_RE_QUESTION, MODE>(P, W, st); break;
            case OP_RE_STAR: wide2_run_tile<LW, OP_RE_STAR, MODE>(P, W, st); break;
            case OP_RE_CONCAT: wide2_run_tile<LW, OP_RE_CONCAT, MODE>(P, W, st); break;
            default: wide2_run_tile<LW, OP_OR, MODE>(P, W, st); break;
        }
    } else {
        switch (W.fx->block.op) {
            case OP_ATOM: wide2_run_tile<LW, OP_ATOM, MODE>(P, W, st); break;
            case OP_NOT: wide2_run_tile<LW, OP_NOT, MODE>(P, W, st); break;
            case OP_NEXT: wide2_run_tile<LW, OP_NEXT, MODE>(P, W, st); break;
            case OP_FUTURE: wide2_run_tile<LW, OP_FUTURE, MODE>(P, W, st); break;
            case OP_AND: wide2_run_tile<LW, OP_AND, MODE>(P, W, st); break;
            case OP_UNTIL: wide2_run_tile<LW, OP_UNTIL, MODE>(P, W, st); break;
            case OP_GLOBALLY: wide2_run_tile<LW, OP_GLOBALLY, MODE>(P, W, st); break;
            default: wide2_run_tile<LW, OP_OR, MODE>(P, W, st); break;
        }
    }
}

template <int LW, int OP>
__global__ void __launch_bounds__(CTA_THREADS, LW == LW_REGEX ? LTLB200_RE_MIN_CTAS : LTLB200_WIDE2_MIN_CTAS) wide2_level_kernel(const __grid_constant__ WideParams P) {
    extern __shared__ __align__(16) uint4 s_w2[];
    const Wide2Warp W = wide2_carve<LW>(P, s_w2);
    Wide2State st;
    while (wide2_next_tile(P, W)) wide2_run_tile<LW, OP>(P, W, st);
}

// small levels: one launch for every operator
template <int LW>
__global__ void __launch_bounds__(CTA_THREADS, 1) wide2_small_level_kernel(const __grid_constant__ WideParams P) {
    extern __shared__ __align__(16) uint4 s_w2[];
    const Wide2Warp W = wide2_carve<LW>(P, s_w2);
    Wide2State st;
    while (wide2_next_tile(P, W)) {
        wide2_run_tile_any<LW, W2_PLAIN>(P, W, st);
    }
}

// non-exhaustive level over a store that already holds a separating CM (see narrow_guarded_level_kernel)
template <int LW>
__global__ void __launch_bounds__(CTA_THREADS, 1) wide2_guarded_level_kernel(const __grid_constant__ WideParams P) {
    extern __shared__ __align__(16) uint4 s_w2[];
    const Wide2Warp W = wide2_carve<LW>(P, s_w2);
    Wide2State st;
    while (wide2_next_tile(P, W)) {
        wide2_run_tile_any<LW, W2_GUARD>(P, W, st);
    }
}

// sharded search, phase A: one launch per operator like wide2_level_kernel, candidates routed to their owners
template <int LW, int OP>
__global__ void __launch_bounds__(CTA_THREADS, LTLB200_WIDE2_MIN_CTAS) wide2_route_kernel(const __grid_constant__ WideParams P) {
    extern __shared__ __align__(16) uint4 s_w2[];
    const Wide2Warp W = wide2_carve<LW>(P, s_w2);
    Wide2State st;
    while (wide2_next_tile(P, W)) wide2_run_tile<LW, OP, W2_ROUTE>(P, W, st);
}

}  // namespace ltlb200
