/*
 * ltlsynth_b200.h -- C ABI of the B200 enumeration engine.
 *
 * The reference (ltlsynth 0.1.0, pure Python + numpy) has no FFI of its own: its
 * seam is the Python API of pkg/src/ltlsynth/engine.py.  Each entry point below
 * states the reference interface it replaces (file:line under
 * /root/reference/pkg/src/ltlsynth).  INTEGRATION.md shows the ctypes binding a
 * reference maintainer would add; paper_2504_18943_b200/_native.py is that
 * binding as shipped here.
 *
 * Plain C types only.  All host pointers are caller-owned.  The engine owns all
 * device memory behind the handle (language cache, hash set, scratch) until
 * ltlb200_destroy.  One handle is used by one host thread at a time.  There is
 * no CPU fallback: every entry point fails (NULL / negative status) when no
 * sm_100 device is usable, and ltlb200_last_error() says why.
 *
 * Vocabulary: a CM (characteristic matrix) is T lanes of `lane_bits` bits, one
 * lane per example trace, bit j of lane t = "the formula holds at position j of
 * trace t".  Row byte image = the T lanes little-endian, back to back, exactly
 * numpy's `cms.tobytes()` for the reference's lane dtype.
 */
#ifndef LTLSYNTH_B200_H
#define LTLSYNTH_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define LTLB200_ABI_VERSION 2

/* operator tags == reference engine.py:42 (OP_ATOM..OP_OR) */
enum {
    LTLB200_OP_ATOM = 0,
    LTLB200_OP_NOT = 1,
    LTLB200_OP_NEXT = 2,
    LTLB200_OP_FUTURE = 3,
    LTLB200_OP_AND = 4,
    LTLB200_OP_UNTIL = 5,
    LTLB200_OP_OR = 6,
    /* EXTENSION, not a reference tag: G ("globally"; SPEC.md:211 lists it as a non-goal).  Enabled only when bit 7
     * of op_mask is set, which the Python face does only for EngineConfig(extended_grammar=True). */
    LTLB200_OP_GLOBALLY = 7
};

/* status of ltlb200_expand_level; 1 and 2 are the reference's two _BudgetExceeded
 * messages (engine.py:416-417, 443-444), which are outcomes, not errors */
enum {
    LTLB200_OK = 0,
    LTLB200_TIME_BUDGET = 1,
    LTLB200_MEMORY_BUDGET = 2,
    LTLB200_ERR_ARGUMENT = -1,
    LTLB200_ERR_CUDA = -2,
    LTLB200_ERR_UNSUPPORTED = -3
};

typedef struct ltlb200_engine ltlb200_engine;

/* counters of one handle since creation */
typedef struct ltlb200_stats {
    uint64_t constructed;        /* candidates built, pre-dedup (RunStats.constructed, engine.py:85) */
    uint64_t unique;             /* stored CMs (RunStats.unique, engine.py:86) */
    uint64_t kernel_launches;    /* CUDA kernels launched by this handle */
    double enumerate_ms;         /* device time of the construction+dedup kernels (CUDA events) */
    double finalize_ms;          /* device time of the per-level compaction kernels */
    uint64_t enumerate_launches; /* launches of the construction+dedup kernel */
    uint64_t enumerate_candidates; /* candidates covered by those launches */
    uint64_t table_slots;        /* hash-set capacity now */
    uint64_t table_rebuilds;     /* times the hash set was regrown */
    uint64_t device_bytes;       /* device memory held now */
    uint64_t h2d_bytes;          /* bytes copied host->device since creation */
    uint64_t d2h_bytes;          /* bytes copied device->host since creation */
    uint32_t row_bytes;          /* CM bytes (T * lane_bits / 8) */
    uint32_t key_bytes;          /* CM bytes as stored in HBM (row_bytes padded to 16) */
    double alloc_ms;             /* host time spent in device allocations */
    double rebuild_host_ms;      /* host time spent issuing hash-set regrows */
    double create_ms;            /* host time of ltlb200_create */
    double route_ms;             /* sharded search: device time of the route kernels (phase A; also in enumerate_ms) */
    double probe_ms;             /* sharded search: device time of the owner-side insert-or-min (phase B; also in enumerate_ms) */
    uint64_t routed_records;     /* records this handle sent to hash owners */
    uint64_t received_records;   /* records this handle folded into its part of the set */
    double tiny_ms;              /* device time of the launches that build several tiny levels each (plan + enumerate +
                                    finalise; not part of enumerate_ms / finalize_ms) */
} ltlb200_stats;

/* ABI version of the loaded library (== LTLB200_ABI_VERSION it was built with). */
int ltlb200_abi_version(void);

/* Last error message of the calling thread ("" when none). */
const char *ltlb200_last_error(void);

/* Number of usable sm_100 devices; 0 (and an error message) when there is none. */
int ltlb200_device_count(void);

/*
 * Replaces CandidateStore.__init__ (engine.py:121-131).
 *   trace_count, lane_bits (8/16/32/64 = smallest_lane_dtype, traces.py:168)
 *   masks[T], target[T]   = Layout.masks / Layout.target as uint64 (traces.py:196-199)
 *   atoms[n_atoms*T]      = atom_bitvectors as uint64, row-major (traces.py:217-230)
 *   device                = CUDA device ordinal
 *   hbm_budget_bytes      = cap on device memory held by the handle (0 = 90% of what is free now)
 *   cuda_stream           = cudaStream_t to launch on, or NULL for an engine-owned stream
 * Returns NULL on failure.
 */
ltlb200_engine *ltlb200_create(int32_t trace_count, int32_t lane_bits, const uint64_t *masks,
                               const uint64_t *target, const uint64_t *atoms, int32_t n_atoms,
                               int32_t device, uint64_t hbm_budget_bytes, void *cuda_stream);

/*
 * EXTENSION (no reference counterpart: formulas.py:65-71 counts every node as 1; SPEC.md:315 calls the weights
 * "config-extensible" without implementing them).  weights[k] = cost of one node of operator tag k (weights[0] = an
 * atom), each in 1..64; cost level c then holds the formulas whose node weights add up to c.  Before the first
 * level only.  All ones (the default) is the reference's cost.
 */
int ltlb200_set_weights(ltlb200_engine *e, const int32_t *weights);

/*
 * REGEX FRONT-END.  Not in the reference (SPEC.md:11 scopes regular-expression
 * synthesis out; PAPER.md:81-113 only motivates it): no reference interface to cite, PARITY UNPINNED; the CPU
 * oracle is oracle/regex_oracle.py (membership pinned to Python's re.fullmatch).
 *
 * The same engine enumerates regular expressions when its rows are characteristic sequences (CS: one bit per infix
 * of the example strings, infixes sorted by (length, text), bit 0 = the empty word).  Create the handle with the CS
 * bitsets as byte rows -- ltlb200_create(trace_count = max(17, ceil(n_bits / 8)), lane_bits = 8, masks = the bits of all
 * example strings, target = the bits of the positive ones, atoms = the CSs of the empty word and of the letters) --
 * then, before the first level, hand over the infix-split guide table: the splits w = u v of infix w are entries
 * offsets[w] .. offsets[w + 1] - 1, each (index of u) | (index of v) << 16.  Levels are then built with
 *   op_mask bits  LTLB200_OP_RE_QUESTION  r?      LTLB200_OP_RE_STAR  r*
 *                 LTLB200_OP_RE_CONCAT    r s     LTLB200_OP_OR       r | s  (union)
 * and the five cost parameters (literal, ?, *, concatenation, union) are ltlb200_set_weights on the tags
 * 0, 8, 9, 10, 6.  CSs of up to 4096 bits; the rows must be wider than 16 bytes (the regex operators exist in the
 * multi-vector kernels only: pad short sequences with zero lanes) and the infixes sorted by length (the right part of
 * a split comes before the whole).  A sharded search (ltlb200_route_begin ...) works as for LTL.
 */
enum { LTLB200_OP_RE_QUESTION = 8, LTLB200_OP_RE_STAR = 9, LTLB200_OP_RE_CONCAT = 10 };
int ltlb200_set_regex(ltlb200_engine *e, int32_t n_bits, const uint32_t *offsets, const uint32_t *entries, uint64_t n_entries);

/* Frees every device allocation of the handle. */
void ltlb200_destroy(ltlb200_engine *e);

/* Empties the store (a fresh CandidateStore on the same specification) while keeping the
 * handle's device buffers, so that repeated searches do not re-allocate. */
int ltlb200_reset(ltlb200_engine *e);

/*
 * Replaces expand_level (engine.py:367-451) together with _tasks_for_level (:219-266),
 * _build_chunk (:269-350) and _first_occurrence_indices (:185-205): builds every
 * candidate of cost `cost` on the device, keeps the canonical-order-first constructor
 * of each CM not seen before, appends them as level `cost`.
 *   cost              must be (number of levels built so far) + 1
 *   op_mask           bit k set <=> operator tag k enabled (normalize_operators, :52-58)
 *   exhaustive        EngineConfig.exhaustive (:69)
 *   batch_size        EngineConfig.batch_size (:67); only the `constructed` counter of the
 *                     level that holds the separator depends on it
 *   memory_budget_bytes  EngineConfig.memory_budget_mb << 20, applied to the reference's own
 *                     estimate (rows + n*(key_words*8+80), :442-444); 0 = unlimited
 *   deadline_s        absolute CLOCK_MONOTONIC seconds (see ltlb200_now), < 0 = none.  The reference polls it
 *                     before every chunk (:416-417); the device polls it with every tile of candidates a warp
 *                     starts, so a level stops within a tile of the deadline, keeps what it built until then
 *                     (the reference's partial level) and the call returns LTLB200_TIME_BUDGET
 * Outputs: *n_new entries appended, *sep_gid id of the level's first fresh separating
 * entry or -1, *constructed_delta the reference's `stats.constructed` increment.
 * A level is appended on every status >= 0 (the reference's `finally: flush()`).
 */
int ltlb200_expand_level(ltlb200_engine *e, int32_t cost, uint32_t op_mask, int32_t exhaustive,
                         int64_t batch_size, uint64_t memory_budget_bytes, double deadline_s,
                         int64_t *n_new, int64_t *sep_gid, int64_t *constructed_delta);

/*
 * One search sharded over several GPUs.  The language cache is replicated on every rank; the dedup set
 * is OWNER-SHARDED (rank r holds the CMs whose hash owner is r), so its capacity grows with the number of GPUs and
 * every rank probes 1/N of the level's candidates.  The reference has no counterpart: its only parallelism is a
 * thread pool inside expand_level (engine.py:386-391) whose results must not depend on the thread count
 * (tests/test_engine.py:162-175) -- the contract kept here: N ranks == 1 rank, bit for bit.
 *
 * One level (the collectives in brackets are the caller's: NCCL through torch.distributed in dist.py; all
 * buffers are DEVICE memory owned by the handle, records are {CM row of ltlb200_key_bytes bytes, ordinal u64}):
 *
 *   ltlb200_route_begin     builds this rank's tile-strided share of the pair space; every candidate that is not
 *                           a duplicate by construction is appended to the send region of its hash owner.
 *                           Outputs, per owner o: send_counts[o] records starting at record send_offsets[o] of
 *                           *rows_dev / *ords_dev; the smallest ordinal of a separating candidate this rank built
 *                           (all ones = none) and how many separating ordinals it recorded (exhaustive runs,
 *                           ltlb200_seps_copy).
 *   [all-to-all]            into the buffers ltlb200_exchange_recv hands out (source-major, dense)
 *   ltlb200_owner_reduce    insert-or-min of the first n_records received records into the owned part of the set;
 *                           marks this owner's winners in the level's bitmap (one bit per candidate ordinal of the
 *                           whole level; *bitmap_words 32-bit words at *bitmap_dev)
 *   [all-reduce SUM]        of the bitmaps (the owners' bits are disjoint, so the sum is the union); min of the
 *                           separator ordinal
 *   ltlb200_winners_export  this owner's winners with ordinal <= sep_ord, as dense records in ordinal order
 *   [all-gather]            every rank receives the winners of the OTHER owners (ltlb200_exchange_recv again)
 *   ltlb200_level_commit    ids from the global bitmap; own winners and the received records appended to the
 *                           cache (recv_counts[k], k < n_sources <= 8: how many records each source sent, in the
 *                           order they sit in the receive buffers); outputs as ltlb200_expand_level (`seps`: every
 *                           separating ordinal of the level, host array, exhaustive runs).
 *
 * A non-exhaustive level over a store that already holds a separating CM is refused (the reference's chunk
 * truncation, engine.py:334-335, needs the whole set): build it with ltlb200_expand_level on every rank.
 * ltlb200_expand_level on a sharded handle rebuilds the full set first, and vice versa.
 */
int ltlb200_route_begin(ltlb200_engine *e, int32_t cost, uint32_t op_mask, int32_t exhaustive, double deadline_s, int32_t rank,
                        int32_t world, uint64_t *send_counts, uint64_t *send_offsets, void **rows_dev, void **ords_dev,
                        uint64_t *sep_ord, uint64_t *n_seps);
int ltlb200_exchange_recv(ltlb200_engine *e, uint64_t n_records, void **rows_dev, void **ords_dev);
int ltlb200_owner_reduce(ltlb200_engine *e, uint64_t n_records, uint64_t *n_claimed, void **bitmap_dev, uint64_t *bitmap_words);
int ltlb200_winners_export(ltlb200_engine *e, uint64_t sep_ord, uint64_t *n_winners, void **rows_dev, void **ords_dev);
int ltlb200_level_commit(ltlb200_engine *e, uint64_t sep_ord, const uint64_t *seps, uint64_t n_seps, const uint64_t *recv_counts,
                         int32_t n_sources, int64_t batch_size, uint64_t memory_budget_bytes, int64_t *n_new, int64_t *sep_gid,
                         int64_t *constructed_delta);
/* Ends the pending routed level empty: another rank ran out of its time or memory budget (statuses 1 / 2 of
 * ltlb200_route_begin / ltlb200_owner_reduce), and every rank stops or none does. */
int ltlb200_level_abort(ltlb200_engine *e);
/* Copies the separating ordinals recorded by ltlb200_route_begin (exhaustive runs); returns how many. */
int64_t ltlb200_seps_copy(ltlb200_engine *e, uint64_t *out, uint64_t cap);
/* Bytes of one CM row as stored on the device and in exchange records (16 * vectors). */
int32_t ltlb200_key_bytes(const ltlb200_engine *e);

/* CLOCK_MONOTONIC now, in seconds (time base of deadline_s). */
double ltlb200_now(void);

/* _Level.n / _Level.base (engine.py:101-111).  cost is 1-based. */
int ltlb200_level_info(const ltlb200_engine *e, int32_t cost, int64_t *n, int64_t *base);

/*
 * Number of candidates the next level (cost = levels built + 1) constructs when it is built in full: the sum of
 * the chunk sizes of _tasks_for_level (engine.py:219-266), a closed form of the stored level sizes.  Identical
 * on every rank of a sharded search, which is what lets the ranks agree without communication to build a
 * small level redundantly instead of sharding it (dist.py).
 */
int ltlb200_level_candidates(ltlb200_engine *e, int32_t cost, uint32_t op_mask, int64_t *n);

/*
 * 1 when some stored CM separates the examples (a level found a separator, or an exhaustive level recorded a
 * separating candidate).  A NON-exhaustive expand_level on such a store follows the reference's chunk truncation
 * (engine.py:334-335), which only ltlb200_expand_level reproduces: a sharded search builds such a level on every rank.
 */
int32_t ltlb200_holds_separator(const ltlb200_engine *e);

/* Number of levels built (len(store.levels)). */
int32_t ltlb200_num_levels(const ltlb200_engine *e);

/*
 * Copies _Level.cms / .op / .left / .right (engine.py:103-106) of one level to host
 * buffers: cms = n * row_bytes bytes (numpy byte image), op = n bytes, left/right = n
 * int64 each.  Any output pointer may be NULL.  `first`/`count` select a row range.
 */
int ltlb200_level_copy(ltlb200_engine *e, int32_t cost, int64_t first, int64_t count, uint8_t *cms,
                       uint8_t *op, int64_t *left, int64_t *right);

/*
 * _Level.cms where it lives: DEVICE pointers to the level's rows (ltlb200_key_bytes bytes each: the numpy row image
 * zero padded to 16-byte vectors) and to the ordinal each entry won with, for consumers that stay on the GPU.
 * Valid until the next level is built or the handle is reset / destroyed; NULL for an empty level.  (Multi-vector
 * CMs live in claim order on the device -- finalising a level does not move them -- so for those the rows pointer
 * is the level's range of an id-ordered image gathered on demand.)
 */
int ltlb200_level_device(ltlb200_engine *e, int32_t cost, void **rows_dev, void **ords_dev);

/* CandidateStore.entry (engine.py:140-145): provenance of one global id. */
int ltlb200_entry(ltlb200_engine *e, int64_t gid, int32_t *op, int64_t *left, int64_t *right);

/* Returns the device blocks cached by destroyed / regrown handles on `device` to the driver. */
void ltlb200_trim(int32_t device);

/* approx_bytes of the reference's accounting (engine.py:131,442). */
uint64_t ltlb200_approx_bytes(const ltlb200_engine *e);

int ltlb200_get_stats(ltlb200_engine *e, ltlb200_stats *out);

#ifdef __cplusplus
}
#endif
#endif /* LTLSYNTH_B200_H */
