// wide2_regex.cuh -- the regex grammar's tiles of the wide kernels (LW_REGEX; included by wide2.cuh).
//
// NOT in the reference; see regex_ops.cuh for the operators and the guide tables.  A warp's tile is, as
// for LTL, 32 "vector" rows (one per lane) combined with one "scalar" row at a time, but concatenation and star do
// not map vector p of the operands to vector p of the result: bit w of  r s  is the OR over the splits w = u v of
// r[u] & s[v].  Walking the splits per candidate (what regex_ops.cuh does for one-vector CSs) costs thousands of
// dependent shared-memory reads per candidate on sequences of several hundred bits.  Here the 32 vector rows are
// BIT-SLICED instead: word x of the sliced area holds bit x of all 32 rows, so one 32-bit AND / OR acts on the 32
// candidates of the tile at once, the lanes work on 32 guide entries in parallel, and nothing branches on data:
//
//   concatenation  for every infix u in the scalar row (a warp-uniform walk over its set bits), for every entry
//                  (x, w) of u's group in the guide table grouped by that side:   out[w] |= sliced[x]
//                  (within a group the w are distinct: plain read-modify-write, one __syncwarp per group);
//   star           out[empty] = all ones; rounds by split depth (= infix length): for every entry (u, v) -> w of
//                  the round, u non-empty:   out[w] |= sliced[u] & out[v]   (shared-memory atomicOr: several
//                  entries of a round share their w);
//
// then 32 x 32 bit transposes (five shuffle rounds per 32 infixes) turn `out` back into one row per lane, in place,
// which the hashing / probe / claim / compare passes of wide2_batch read from shared memory (a row is built once;
// the LTL vectors are cheap enough to be rebuilt in pass 2 instead).
#pragma once
// (included by wide2.cuh inside namespace ltlb200, between the batch passes and the tile dispatch)

// lane r holds row r of a 32 x 32 bit matrix (bit c = column c); returns column `lane` (bit r = row r).
// Five butterfly rounds, s = 16, 8, 4, 2, 1: a lane keeps the half of its word that stays and takes the other half from
// lane ^ s, shifted by s towards it.  The sender rotates (left by s if its bit s is set, right otherwise: the bits that
// wrap around land where the receiver's mask drops them), so a round is one funnel shift, one shuffle and one LOP3.
__device__ __forceinline__ uint32_t transpose32(uint32_t x) {
    const int lane = threadIdx.x & 31;
#pragma unroll
    for (int s = 16; s >= 1; s >>= 1) {
        const uint32_t m = s == 16 ? 0x0000FFFFu : s == 8 ? 0x00FF00FFu : s == 4 ? 0x0F0F0F0Fu : s == 2 ? 0x33333333u : 0x55555555u;
        const bool up = (lane & s) != 0;
        const uint32_t y = __shfl_xor_sync(0xFFFFFFFFu, __funnelshift_l(x, x, up ? s : 32 - s), s);
        const uint32_t keep = up ? ~m : m;
        x = (x & keep) | (y & ~keep);
    }
    return x;
}

// rows [word][lane] -> bit-sliced [infix] (and back: the transpose is its own inverse), 32 infixes per step
__device__ __forceinline__ void regex_slice(const uint32_t *rows, uint32_t *sliced, int n_words) {
    const int lane = threadIdx.x & 31;
#pragma unroll 2
    for (int q = 0; q < n_words; ++q) sliced[q * 32 + lane] = transpose32(rows[q * 32 + lane]);
}

struct RegexGuide {  // the tables of Engine::set_regex (global memory or the CTA's staged copy)
    const uint32_t *off, *uv, *w_of;          // sorted by result infix: offsets, entries u | v << 16, result infix per entry
    const uint32_t *left_off, *left_ent;      // grouped by the LEFT part u:  entries v | w << 16
    const uint32_t *right_off, *right_ent;    // grouped by the RIGHT part v: entries u | w << 16
    const uint32_t *rounds;                   // entry offsets of the star's rounds (split depth), n_rounds + 1 values
};

__device__ __forceinline__ RegexGuide regex_guide(const WideParams &P, const uint32_t *base) {
    RegexGuide G;
    const uint32_t n = (uint32_t)P.n_bits, E = P.guide_entries;
    G.off = base;
    G.uv = base + n + 1;
    G.w_of = G.uv + E;
    G.left_off = G.w_of + E;
    G.left_ent = G.left_off + n + 1;
    G.right_off = G.left_ent + E;
    G.right_ent = G.right_off + n + 1;
    G.rounds = G.right_ent + E;
    return G;
}

// bit j of the result = rows `x` and `y` (both bit-sliced) differ in candidate j somewhere in the first n_bits infixes
__device__ __forceinline__ uint32_t sliced_diff(const uint32_t *x, const uint32_t *y, int n_bits) {
    uint32_t d = 0;
    for (int k = threadIdx.x & 31; k < n_bits; k += 32) d |= x[k] ^ y[k];
    return __reduce_or_sync(0xFFFFFFFFu, d);
}

// wide2_batch takes "the operands" of a candidate only to spot one that equals an operand (such a CM is in the cache
// already).  The regex tiles decide that on the bit-sliced rows, 32 candidates at a time, and hand the verdict over
// as operands that do / do not equal the result.
__device__ __forceinline__ uint4 regex_operand_stub(uint4 c, bool equals) { return equals ? c : make_uint4(~c.x, ~c.y, ~c.z, ~c.w); }

// literal, question, star.  The lanes' rows are staged word by word ([word][lane]) in the row area, which is also
// where the finished rows end up; the star works on their bit-sliced copy.
template <int OP, int MODE>
__device__ __forceinline__ void wide2_regex_unary_tile(const WideParams &P, const Wide2Warp &W, Wide2State &st, u64 tile_local,
                                                       u64 sep_now) {
    const BlockDesc &B = W.fx->block;
    const int lane = threadIdx.x & 31;
    const int nvec = P.nvec, n_words = nvec * 4;
    const u64 per_tile = (u64)32 * B.tile_s;
    const u64 first = tile_local * per_tile + lane;
    const u64 ord0 = B.ord0, n = B.na;
    if (ord0 + tile_local * per_tile > sep_now) return;
    const int n_steps = (int)min((u64)B.tile_s, (n - tile_local * per_tile + 31) / 32);
    const RegexGuide G = regex_guide(P, W.guide);
    uint32_t *ow = W.out + lane;
#pragma unroll 1
    for (int k = 0; k < n_steps; ++k) {
        const u64 i = first + (u64)k * 32;
        const bool live[1] = {i < n};
        const u64 ords[1] = {ord0 + i};
        const uint4 *row = B.from_atoms ? P.atoms + (live[0] ? i : 0) * nvec : P.store + w2_ld<MODE>(P.loc + B.a_off + (live[0] ? i : 0)) * nvec;
        __syncwarp();
        for (int p = 0; p < nvec; ++p) {  // every lane its own row, word by word into its own bank
            const uint4 x = w2_ld<MODE>(row + p);
            ow[(p * 4) * 32] = x.x;
            ow[(p * 4 + 1) * 32] = x.y;
            ow[(p * 4 + 2) * 32] = x.z;
            ow[(p * 4 + 3) * 32] = x.w;
        }
        bool same = false;  // the result equals the operand
        if constexpr (OP == OP_RE_QUESTION) {
            same = (ow[0] & 1u) != 0u;
            ow[0] |= 1u;
        }
        if constexpr (OP == OP_RE_STAR) {
            __syncwarp();
            regex_slice(W.out, W.sliced, n_words);
            __syncwarp();
            for (int q = 0; q < n_words; ++q) W.out[q * 32 + lane] = 0u;
            __syncwarp();
            if (lane == 0) W.out[0] = 0xFFFFFFFFu;  // the empty word, in every row
            __syncwarp();
            uint32_t e_lo = G.rounds[1];
#pragma unroll 1
            for (uint32_t r = 1; r < P.guide_rounds; ++r) {
                const uint32_t e_hi = G.rounds[r + 1];
                // four entries per lane and step, their table words loaded together: with sequences of thousands of
                // bits few warps fit an SM and nothing else hides the latency of the loads
                for (uint32_t e0 = e_lo; e0 < e_hi; e0 += 128) {
                    uint32_t uv[4], w[4];
#pragma unroll
                    for (int t = 0; t < 4; ++t) {
                        const uint32_t e = e0 + (uint32_t)t * 32u + lane;
                        uv[t] = e < e_hi ? G.uv[e] : 0u;  // (u = 0: skipped below)
                        w[t] = e < e_hi ? G.w_of[e] : 0u;
                    }
                    uint32_t val[4];
#pragma unroll
                    for (int t = 0; t < 4; ++t) val[t] = (uv[t] & 0xFFFFu) ? (W.sliced[uv[t] & 0xFFFFu] & W.out[uv[t] >> 16]) : 0u;
#pragma unroll
                    for (int t = 0; t < 4; ++t)
                        if (val[t]) atomicOr(&W.out[w[t]], val[t]);
                }
                e_lo = e_hi;
                __syncwarp();
            }
            same = ((sliced_diff(W.out, W.sliced, P.n_bits) >> lane) & 1u) == 0u;
            regex_slice(W.out, W.out, n_words);  // back to one row per lane, in place
        }
        __syncwarp();
        auto gen = [&](int r, int p, uint4 &a, uint4 &b, uint4 &c) {
            c = make_uint4(ow[(p * 4) * 32], ow[(p * 4 + 1) * 32], ow[(p * 4 + 2) * 32], ow[(p * 4 + 3) * 32]);
            a = b = regex_operand_stub(c, same);
        };
        if constexpr (MODE == W2_ROUTE) wide2_route_batch<LW_REGEX, OP>(P, W, gen, live, ords);
        else wide2_batch<LW_REGEX, OP, MODE == W2_GUARD>(P, W, st, gen, live, ords);
    }
}

// concatenation  left . right;  VEC_B: the lanes' rows are the RIGHT operands, the scalar row is the left one
template <bool VEC_B, int MODE>
__device__ __forceinline__ void wide2_regex_concat_tile(const WideParams &P, const Wide2Warp &W, Wide2State &st, u64 tile_local,
                                                        u64 sep_now) {
    const BlockDesc &B = W.fx->block;
    const int lane = threadIdx.x & 31;
    const int nvec = P.nvec, n_words = nvec * 4;
    const int tile_s = (int)B.tile_s;
    const uint32_t vg_n = B.vg;
    u64 tv, ts;
    if (VEC_B) { ts = tile_local / B.tiles_v; tv = tile_local % B.tiles_v; }
    else { tv = tile_local / B.tiles_s; ts = tile_local % B.tiles_s; }
    const u64 n_vec = VEC_B ? B.nb : B.na, n_sc = VEC_B ? B.na : B.nb;
    const u64 v0 = tv * (u64)(32 * vg_n), s0 = ts * (u64)tile_s;
    const int s_cnt = (int)min((u64)tile_s, n_sc - s0);
    const u64 ord0 = B.ord0, nb = B.nb;
    if (ord0 + (VEC_B ? s0 * nb + v0 : v0 * nb + s0) > sep_now) return;
    const u64 *vec_loc = P.loc + (VEC_B ? B.b_off : B.a_off);
    const u64 *sc_loc = P.loc + (VEC_B ? B.a_off : B.b_off);
    const RegexGuide G = regex_guide(P, W.guide);
    // the table grouped by the scalar row's side: its entries name the bit of the lanes' rows and the result bit
    const uint32_t *g_off = VEC_B ? G.left_off : G.right_off, *g_ent = VEC_B ? G.left_ent : G.right_ent;
    const int sc_words = (P.n_bits + 31) >> 5;
    uint32_t *ow = W.out + lane;
    __syncwarp();
    for (int t = lane; t < s_cnt * nvec; t += 32) {
        const int rrow = t / nvec, p = t - rrow * nvec;
        W.sc[t] = w2_ld<MODE>(P.store + w2_ld<MODE>(sc_loc + s0 + rrow) * nvec + p);
    }
#pragma unroll 1
    for (uint32_t vg = 0; vg < vg_n; ++vg) {
        const u64 vbase = v0 + (u64)vg * 32;
        if (vbase >= n_vec) break;
        __syncwarp();
        // the 32 vector rows: staged [word][row] in the row area, bit-sliced from there (the row area then takes the results)
        const int rows_here = (int)min((u64)32, n_vec - vbase);
        for (int t = lane; t < 32 * nvec; t += 32) {  // (rows past the end of the level: zero)
            const int rrow = t / nvec, p = t - rrow * nvec;
            const uint4 x = rrow < rows_here ? w2_ld<MODE>(P.store + w2_ld<MODE>(vec_loc + vbase + rrow) * nvec + p) : make_uint4(0, 0, 0, 0);
            uint32_t *col = W.out + rrow;
            col[(p * 4) * 32] = x.x;
            col[(p * 4 + 1) * 32] = x.y;
            col[(p * 4 + 2) * 32] = x.z;
            col[(p * 4 + 3) * 32] = x.w;
        }
        __syncwarp();
        regex_slice(W.out, W.sliced, n_words);
        const u64 v = vbase + lane;
        const bool v_ok = v < n_vec;
#pragma unroll 1
        for (int k = 0; k < s_cnt; ++k) {
            const uint32_t *sw = reinterpret_cast<const uint32_t *>(W.sc + k * nvec);
            __syncwarp();
            for (int q = 0; q < n_words; ++q) W.out[q * 32 + lane] = 0u;
            __syncwarp();
            // (the offsets and the first 32 entries of the NEXT infix's group are fetched while this one is applied)
            int q = 0;
            uint32_t word = 0;
            auto next_infix = [&]() -> uint32_t {  // the same for every lane; ~0u = the row is done
                while (word == 0u) {
                    if (q >= sc_words) return ~0u;
                    word = sw[q++];
                }
                const uint32_t s = (uint32_t)(q - 1) * 32u + (uint32_t)(__ffs(word) - 1);
                word &= word - 1u;
                return s;
            };
            uint32_t s = next_infix();
            uint32_t lo = 0, hi = 0, ent0 = 0;
            if (s != ~0u) {
                lo = g_off[s];
                hi = g_off[s + 1];
                ent0 = lo + lane < hi ? g_ent[lo + lane] : 0u;
            }
            while (s != ~0u) {
                const uint32_t s_next = next_infix();
                uint32_t lo_n = 0, hi_n = 0, ent_n = 0;
                if (s_next != ~0u) {
                    lo_n = g_off[s_next];
                    hi_n = g_off[s_next + 1];
                    ent_n = lo_n + lane < hi_n ? g_ent[lo_n + lane] : 0u;
                }
                if (lo + lane < hi) W.out[ent0 >> 16] |= W.sliced[ent0 & 0xFFFFu];
                for (uint32_t e = lo + 32 + lane; e < hi; e += 32) {
                    const uint32_t ent = g_ent[e];
                    W.out[ent >> 16] |= W.sliced[ent & 0xFFFFu];
                }
                __syncwarp();
                s = s_next;
                lo = lo_n;
                hi = hi_n;
                ent0 = ent_n;
            }
            // a candidate that equals one of its operands is in the cache already: decided here, on the sliced rows
            uint32_t differs_vec = 0, differs_sc = 0;
            for (int x = lane; x < P.n_bits; x += 32) {
                const uint32_t o = W.out[x];
                differs_vec |= o ^ W.sliced[x];
                differs_sc |= o ^ (((sw[x >> 5] >> (x & 31)) & 1u) ? 0xFFFFFFFFu : 0u);
            }
            const uint32_t differs = __reduce_or_sync(0xFFFFFFFFu, differs_vec) & __reduce_or_sync(0xFFFFFFFFu, differs_sc);
            const bool same = ((differs >> lane) & 1u) == 0u;
            __syncwarp();
            regex_slice(W.out, W.out, sc_words);  // one row per lane, in place (the words past the last infix stay zero)
            __syncwarp();
            const bool live[1] = {v_ok};
            const u64 ords[1] = {ord0 + (VEC_B ? (s0 + k) * nb + v : v * nb + (s0 + k))};
            auto gen = [&](int r, int p, uint4 &a, uint4 &b, uint4 &c) {
                c = make_uint4(ow[(p * 4) * 32], ow[(p * 4 + 1) * 32], ow[(p * 4 + 2) * 32], ow[(p * 4 + 3) * 32]);
                a = b = regex_operand_stub(c, same);
            };
            if constexpr (MODE == W2_ROUTE) wide2_route_batch<LW_REGEX, OP_RE_CONCAT>(P, W, gen, live, ords);
            else wide2_batch<LW_REGEX, OP_RE_CONCAT, MODE == W2_GUARD>(P, W, st, gen, live, ords);
        }
    }
}
