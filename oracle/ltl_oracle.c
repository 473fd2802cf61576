/*
 * ltl_oracle.c -- CPU restatement of the reference enumerator.  TEST INFRASTRUCTURE ONLY.
 *
 * This file restates, in plain scalar C, the algorithm of the reference's
 * enumeration hot path (reference = /root/reference/pkg/src/ltlsynth, pure
 * Python + numpy).  It exists so that the CUDA engine can be compared with the
 * reference's results on a machine where the Python reference is not present
 * (the GPU box).  Only tests/, __graft_entry__.smoke() and bench.py's
 * cpu_baseline / --impl reference legs may load it; the product package never
 * does, and has no CPU path of its own.
 *
 * Parity pin: tests/test_oracle_golden.py checks this restatement against
 * the JSON files under tests/golden, which tests/golden/make_golden.py produced by running the
 * UNMODIFIED reference in the build container (per-level counts, sha256 of every
 * level's cms/op/left/right arrays, constructed counters, separator ids, formula
 * text) and against the known-answer values of the reference's own tests.
 *
 * Deliberately naive: characteristic matrices are handled lane by lane (one
 * 64-bit integer per trace), exactly like numpy's element-wise ufuncs, with no
 * packed-word (SWAR) tricks, so it shares no bit-twiddling with the CUDA kernels.
 * Candidates are visited strictly in the reference's canonical order and the
 * first constructor of a CM wins, which is what the reference's chunked
 * sort-dedup + seen-set computes.
 *
 * Each function cites the reference lines it follows.
 *
 * EXTENSION, not in the reference (SPEC.md:211 lists G as a non-goal, SPEC.md:315 calls the
 * operator weights "config-extensible" without implementing them): OP_GLOBALLY and per-operator cost weights
 * (orc_set_weights).  With the default weights (all 1) and G disabled every code path below is the restatement of
 * the reference; with them the level structure generalises as "operator of weight w over operands whose costs add
 * up to cost - w".  PARITY UNPINNED for the extension: no reference output exists; tests pin it to the semantic
 * identity G x = !F!x and to a brute-force search over weighted formula trees.
 */
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#include <time.h>

enum { OP_ATOM = 0, OP_NOT, OP_NEXT, OP_FUTURE, OP_AND, OP_UNTIL, OP_OR, OP_GLOBALLY /* extension */ }; /* engine.py:42 */
enum { ST_OK = 0, ST_TIME = 1, ST_MEMORY = 2, ST_BAD = -1 };

typedef struct {
    int64_t n, base;
    uint8_t *op;
    int64_t *left, *right;
    int64_t row0; /* index of the level's first row in the global row store (== base) */
} level_t;

typedef struct {
    int T, w, lane_bytes, row_bytes, key_words; /* engine.py:121-128 */
    uint64_t *masks, *target;                   /* traces.py:196-199 */
    int n_atoms;
    uint64_t *atoms; /* n_atoms x T lanes, traces.py:217-230 */
    /* global row store: rows in id order, lane dtype, little endian (numpy tobytes image) */
    uint8_t *rows;
    int64_t total, rows_cap;
    level_t *levels;
    int n_levels, levels_cap;
    int64_t dup_hist[64]; /* analysis only: candidates of the last level by the cost level of the entry they
                             duplicate ([0] = new CM, [c] = duplicate of a CM stored at cost c) */
    int64_t last_match;   /* id matched by the last seen_add that returned 0 */
    /* seen set (engine.py:130): open addressing over row ids, keyed by the row bytes */
    int64_t *slots; /* id+1, 0 = empty */
    int64_t n_slots;
    int64_t approx_bytes; /* engine.py:131,442 */
    /* scratch */
    uint64_t *la, *lb, *lc;
    uint8_t *packed;
    int weights[8]; /* extension: cost of one node of every operator tag ([0] = an atom); all 1 = the reference */
} oracle_t;

static double now_s(void) {
    struct timespec ts;
    clock_gettime(CLOCK_MONOTONIC, &ts);
    return (double)ts.tv_sec + 1e-9 * (double)ts.tv_nsec;
}

static inline uint64_t lane_trunc(const oracle_t *o, uint64_t x) {
    return o->w == 64 ? x : (x & ((1ULL << o->w) - 1ULL));
}

static void load_row(const oracle_t *o, int64_t id, uint64_t *lanes) {
    const uint8_t *p = o->rows + (size_t)id * (size_t)o->row_bytes;
    for (int t = 0; t < o->T; t++) {
        uint64_t v = 0;
        memcpy(&v, p + (size_t)t * o->lane_bytes, (size_t)o->lane_bytes);
        lanes[t] = v;
    }
}

static void pack_row(const oracle_t *o, const uint64_t *lanes, uint8_t *out) {
    for (int t = 0; t < o->T; t++) memcpy(out + (size_t)t * o->lane_bytes, &lanes[t], (size_t)o->lane_bytes);
}

/* kernels.py:24-26 : shifts 1,2,4,... while < lane width */
static int shift_schedule(int w, int *out) {
    int n = 0;
    for (int s = 1; s < w; s <<= 1) out[n++] = s;
    return n;
}

/* kernels.py:29-31 */
static void k_not(const oracle_t *o, const uint64_t *x, uint64_t *r) {
    for (int t = 0; t < o->T; t++) r[t] = lane_trunc(o, ~x[t]) & o->masks[t];
}
/* kernels.py:42-44 : plain per-lane shift, no mask */
static void k_next(const oracle_t *o, const uint64_t *x, uint64_t *r) {
    for (int t = 0; t < o->T; t++) r[t] = x[t] >> 1;
}
/* kernels.py:47-57 */
static void k_future(const oracle_t *o, const uint64_t *x, uint64_t *r) {
    int sh[8], ns = shift_schedule(o->w, sh);
    for (int t = 0; t < o->T; t++) {
        uint64_t v = x[t];
        for (int k = 0; k < ns; k++) v |= v >> sh[k];
        r[t] = v;
    }
}
/* extension (not in the reference): G x = "x at every position from here to the end" = !F!x */
static void k_globally(const oracle_t *o, const uint64_t *x, uint64_t *r) {
    int sh[8], ns = shift_schedule(o->w, sh);
    for (int t = 0; t < o->T; t++) {
        uint64_t v = lane_trunc(o, ~x[t]) & o->masks[t];
        for (int k = 0; k < ns; k++) v |= v >> sh[k];
        r[t] = lane_trunc(o, ~v) & o->masks[t];
    }
}
/* kernels.py:60-73 */
static void k_until(const oracle_t *o, const uint64_t *a, const uint64_t *b, uint64_t *out) {
    int sh[8], ns = shift_schedule(o->w, sh);
    for (int t = 0; t < o->T; t++) {
        uint64_t r = b[t], q = a[t];
        for (int k = 0; k < ns; k++) {
            r |= q & (r >> sh[k]);
            q &= q >> sh[k];
        }
        out[t] = r & o->masks[t];
    }
}
/* engine.py:330 (== kernels.py:102-105) */
static int k_separates(const oracle_t *o, const uint64_t *c) {
    for (int t = 0; t < o->T; t++)
        if ((c[t] & 1ULL) != o->target[t]) return 0;
    return 1;
}

/* ---- seen set ---------------------------------------------------------- */
static uint64_t hash_bytes(const uint8_t *p, int n) {
    uint64_t h = 1469598103934665603ULL;
    for (int i = 0; i < n; i++) {
        h ^= p[i];
        h *= 1099511628211ULL;
    }
    h ^= h >> 29;
    h *= 0xBF58476D1CE4E5B9ULL;
    h ^= h >> 32;
    return h;
}

static void set_grow(oracle_t *o) {
    int64_t ncap = o->n_slots ? o->n_slots * 2 : 1024;
    int64_t *ns = (int64_t *)calloc((size_t)ncap, sizeof(int64_t));
    for (int64_t id = 0; id < o->total; id++) {
        uint64_t h = hash_bytes(o->rows + (size_t)id * o->row_bytes, o->row_bytes);
        int64_t s = (int64_t)(h & (uint64_t)(ncap - 1));
        while (ns[s]) s = (s + 1) & (ncap - 1);
        ns[s] = id + 1;
    }
    free(o->slots);
    o->slots = ns;
    o->n_slots = ncap;
}

/* returns 1 and appends the row when the key was not seen (engine.py:421-424), else 0 */
static int seen_add(oracle_t *o, const uint8_t *row) {
    if ((o->total + 1) * 2 > o->n_slots) set_grow(o);
    uint64_t h = hash_bytes(row, o->row_bytes);
    int64_t s = (int64_t)(h & (uint64_t)(o->n_slots - 1));
    while (o->slots[s]) {
        int64_t id = o->slots[s] - 1;
        if (memcmp(o->rows + (size_t)id * o->row_bytes, row, (size_t)o->row_bytes) == 0) {
            o->last_match = id;
            return 0;
        }
        s = (s + 1) & (o->n_slots - 1);
    }
    if (o->total == o->rows_cap) {
        o->rows_cap = o->rows_cap ? o->rows_cap * 2 : 1024;
        o->rows = (uint8_t *)realloc(o->rows, (size_t)o->rows_cap * o->row_bytes);
    }
    memcpy(o->rows + (size_t)o->total * o->row_bytes, row, (size_t)o->row_bytes);
    o->slots[s] = o->total + 1;
    o->total++;
    return 1;
}

/* ---- public API -------------------------------------------------------- */

/* CandidateStore.__init__, engine.py:121-131.  masks/target/atoms are given as uint64 lanes. */
oracle_t *orc_create(int T, int lane_bits, const uint64_t *masks, const uint64_t *target,
                     const uint64_t *atoms, int n_atoms) {
    if (T < 1 || (lane_bits != 8 && lane_bits != 16 && lane_bits != 32 && lane_bits != 64)) return NULL;
    oracle_t *o = (oracle_t *)calloc(1, sizeof(oracle_t));
    o->T = T;
    o->w = lane_bits;
    o->lane_bytes = lane_bits / 8;
    o->row_bytes = T * o->lane_bytes;
    o->key_words = (o->row_bytes + 7) / 8;
    o->masks = (uint64_t *)malloc(sizeof(uint64_t) * T);
    o->target = (uint64_t *)malloc(sizeof(uint64_t) * T);
    memcpy(o->masks, masks, sizeof(uint64_t) * T);
    memcpy(o->target, target, sizeof(uint64_t) * T);
    o->n_atoms = n_atoms;
    o->atoms = (uint64_t *)malloc(sizeof(uint64_t) * (size_t)T * (size_t)(n_atoms > 0 ? n_atoms : 1));
    memcpy(o->atoms, atoms, sizeof(uint64_t) * (size_t)T * (size_t)n_atoms);
    o->la = (uint64_t *)malloc(sizeof(uint64_t) * T);
    o->lb = (uint64_t *)malloc(sizeof(uint64_t) * T);
    o->lc = (uint64_t *)malloc(sizeof(uint64_t) * T);
    o->packed = (uint8_t *)malloc((size_t)o->row_bytes);
    for (int k = 0; k < 8; k++) o->weights[k] = 1;
    return o;
}

/* extension: cost of one node per operator tag (weights[0] = an atom), before the first level */
int orc_set_weights(oracle_t *o, const int *weights) {
    if (!o || o->n_levels) return ST_BAD;
    for (int k = 0; k < 8; k++) {
        if (weights[k] < 1) return ST_BAD;
        o->weights[k] = weights[k];
    }
    return ST_OK;
}

void orc_destroy(oracle_t *o) {
    if (!o) return;
    for (int i = 0; i < o->n_levels; i++) {
        free(o->levels[i].op);
        free(o->levels[i].left);
        free(o->levels[i].right);
    }
    free(o->levels);
    free(o->rows);
    free(o->slots);
    free(o->masks);
    free(o->target);
    free(o->atoms);
    free(o->la);
    free(o->lb);
    free(o->lc);
    free(o->packed);
    free(o);
}

/* accumulators of one expand_level call (engine.py:393-397) */
typedef struct {
    oracle_t *o;
    level_t lv;
    int64_t cap;
    int64_t n_new, sep_gid, constructed;
    int exhaustive;
    int64_t mem_limit;
    double deadline;
    int status, stop;
} run_t;

static void lv_push(run_t *r, int tag, int64_t left, int64_t right) {
    if (r->lv.n == r->cap) {
        r->cap = r->cap ? r->cap * 2 : 256;
        r->lv.op = (uint8_t *)realloc(r->lv.op, (size_t)r->cap);
        r->lv.left = (int64_t *)realloc(r->lv.left, sizeof(int64_t) * (size_t)r->cap);
        r->lv.right = (int64_t *)realloc(r->lv.right, sizeof(int64_t) * (size_t)r->cap);
    }
    r->lv.op[r->lv.n] = (uint8_t)tag;
    r->lv.left[r->lv.n] = left;
    r->lv.right[r->lv.n] = right;
    r->lv.n++;
}

/* One chunk = _build_chunk (engine.py:269-350) followed by the merge step of
 * expand_level (engine.py:415-446).  The chunk's candidates are k = 0..count-1;
 * `gen` yields candidate k's operands.  Scanning k upwards and asking the global
 * seen set is the same as "chunk-local first occurrences, then seen filter"
 * (a later chunk-local duplicate would be found in `seen` anyway). */
typedef struct {
    int kind; /* 0 atoms, 1 unary, 2 rect, 3 tri, 4 trij */
    int tag;
    int64_t a_base, b_base; /* global ids of operand rows */
    int64_t i0, i1, j0, j1, n; /* ranges local to the operand levels; n = level size (tri) */
} chunk_t;

static int64_t chunk_count(const chunk_t *c) {
    switch (c->kind) {
    case 0: return c->i1;
    case 1: return c->i1 - c->i0;
    case 2: return (c->i1 - c->i0) * (c->j1 - c->j0);
    case 3: { /* rows i0..i1-1 of the triangle, row i has n-i entries (engine.py:312) */
        int64_t a = c->n - c->i0, b = c->n - c->i1; /* lengths n-i0 ... n-i1+1 */
        return (a * (a + 1) - b * (b + 1)) / 2;
    }
    default: return c->j1 - c->j0;
    }
}

static void do_chunk(run_t *r, const chunk_t *c) {
    oracle_t *o = r->o;
    if (r->deadline >= 0 && now_s() > r->deadline) { /* engine.py:416-417 */
        r->status = ST_TIME;
        r->stop = 1;
        return;
    }
    int64_t count = chunk_count(c);
    r->constructed += count; /* engine.py:418 */
    int64_t fresh_in_chunk = 0, fresh_bytes_rows = 0;
    int have_sep = 0;
    /* tri iteration state (engine.py:312-315: row-major over i0 <= i < i1, i <= j < n) */
    int64_t ti = c->i0, tj = c->i0;
    for (int64_t k = 0; k < count; k++) {
        int64_t left, right;
        const uint64_t *res;
        switch (c->kind) {
        case 0: /* engine.py:274-278 */
            memcpy(o->lc, o->atoms + (size_t)k * o->T, sizeof(uint64_t) * o->T);
            left = k;
            right = -1;
            break;
        case 1: /* engine.py:279-291 */
            left = c->a_base + c->i0 + k;
            right = -1;
            load_row(o, left, o->la);
            if (c->tag == OP_NOT) k_not(o, o->la, o->lc);
            else if (c->tag == OP_NEXT) k_next(o, o->la, o->lc);
            else if (c->tag == OP_GLOBALLY) k_globally(o, o->la, o->lc);
            else k_future(o, o->la, o->lc);
            break;
        case 2: { /* engine.py:292-307 */
            int64_t nb = c->j1 - c->j0;
            left = c->a_base + c->i0 + k / nb;
            right = c->b_base + c->j0 + k % nb;
            break;
        }
        case 3: /* engine.py:308-319 */
            left = c->a_base + ti;
            right = c->a_base + tj;
            if (++tj == c->n) {
                ti++;
                tj = ti;
            }
            break;
        default: /* engine.py:320-327 */
            left = c->a_base + c->i0;
            right = c->a_base + c->j0 + k;
            break;
        }
        if (c->kind >= 2) {
            load_row(o, left, o->la);
            load_row(o, right, o->lb);
            if (c->tag == OP_UNTIL) k_until(o, o->la, o->lb, o->lc);
            else if (c->tag == OP_AND)
                for (int t = 0; t < o->T; t++) o->lc[t] = o->la[t] & o->lb[t];
            else
                for (int t = 0; t < o->T; t++) o->lc[t] = o->la[t] | o->lb[t];
        }
        res = o->lc;
        int sep = k_separates(o, res); /* engine.py:330-331 */
        pack_row(o, res, o->packed);
        int fresh = seen_add(o, o->packed); /* engine.py:333,421-424 */
        if (fresh) {
            o->dup_hist[0]++;
        } else { /* analysis only: which cost level holds the duplicated entry */
            int cost_of = o->n_levels + 1; /* the level being built */
            if (o->last_match < r->lv.base) {
                cost_of = o->n_levels;
                while (cost_of > 1 && o->last_match < o->levels[cost_of - 1].base) cost_of--;
            }
            if (cost_of < 64) o->dup_hist[cost_of]++;
        }
        if (fresh) {
            lv_push(r, c->tag, left, right); /* engine.py:434-441 */
            fresh_in_chunk++;
            fresh_bytes_rows += o->row_bytes;
        }
        if (sep && !have_sep) {
            /* first separating candidate of the chunk: sep_raw (engine.py:331) */
            have_sep = 1;
            if (r->sep_gid < 0 && fresh) /* engine.py:425-433 */
                r->sep_gid = r->lv.base + r->n_new + fresh_in_chunk - 1;
            if (!r->exhaustive) break; /* kept = kept[kept <= sep_raw], engine.py:334-335 */
        }
    }
    r->n_new += fresh_in_chunk;
    if (fresh_in_chunk) { /* engine.py:442-444 */
        o->approx_bytes += fresh_bytes_rows + fresh_in_chunk * ((int64_t)o->key_words * 8 + 80);
        if (o->approx_bytes > r->mem_limit) {
            r->status = ST_MEMORY;
            r->stop = 1;
            return;
        }
    }
    if (r->sep_gid >= 0 && !r->exhaustive) r->stop = 1; /* engine.py:445-446 */
}

/*
 * expand_level (engine.py:367-451) driven by the chunk schedule of
 * _tasks_for_level (engine.py:219-266).
 *   op_mask bit k set <=> operator tag k enabled (OP_NOT..OP_OR)
 *   deadline_s < 0: no deadline, else seconds on CLOCK_MONOTONIC (see orc_now)
 * Outputs: n_new, sep_gid (-1 = None), constructed_delta.  Returns ST_*.
 * The (possibly partial) level is always appended (the `finally: flush()`).
 */
int orc_expand_level(oracle_t *o, int cost, unsigned op_mask, int exhaustive, int64_t batch,
                     int64_t mem_limit_bytes, double deadline_s, int64_t *n_new, int64_t *sep_gid,
                     int64_t *constructed_delta) {
    if (!o || cost != o->n_levels + 1 || batch < 1) return ST_BAD;
    memset(o->dup_hist, 0, sizeof(o->dup_hist));
    run_t r;
    memset(&r, 0, sizeof(r));
    r.o = o;
    r.lv.base = o->total;
    r.lv.row0 = o->total;
    r.sep_gid = -1;
    r.exhaustive = exhaustive;
    r.mem_limit = mem_limit_bytes;
    r.deadline = deadline_s;
    chunk_t c;
    memset(&c, 0, sizeof(c));

    const int *w = o->weights; /* all 1 in the reference: cost - w - ... below is then engine.py's cost - 1 - ... */
    if (cost == w[OP_ATOM]) { /* engine.py:221-223 */
        c.kind = 0;
        c.tag = OP_ATOM;
        c.i1 = o->n_atoms;
        do_chunk(&r, &c);
    }
    if (cost > 1) {
        static const int unary_tags[4] = {OP_NOT, OP_NEXT, OP_FUTURE, OP_GLOBALLY}; /* engine.py:44 (+ extension) */
        static const int binary_tags[3] = {OP_AND, OP_UNTIL, OP_OR};                /* engine.py:45 */
        for (int u = 0; u < 4 && !r.stop; u++) { /* engine.py:225-229 */
            int tag = unary_tags[u];
            if (!(op_mask >> tag & 1) || cost - w[tag] < 1) continue;
            const level_t *prev = &o->levels[cost - w[tag] - 1];
            if (prev->n == 0) continue;
            for (int64_t i0 = 0; i0 < prev->n && !r.stop; i0 += batch) {
                c.kind = 1;
                c.tag = tag;
                c.a_base = prev->base;
                c.i0 = i0;
                c.i1 = i0 + batch < prev->n ? i0 + batch : prev->n;
                do_chunk(&r, &c);
            }
        }
        for (int b = 0; b < 3 && !r.stop; b++) { /* engine.py:230-266 */
            int tag = binary_tags[b];
            if (!(op_mask >> tag & 1)) continue;
            int commutative = (tag == OP_AND || tag == OP_OR); /* engine.py:46 */
            for (int c1 = 1; c1 < cost - w[tag] && !r.stop; c1++) {
                int c2 = cost - w[tag] - c1;
                if (commutative && c1 > c2) break;
                const level_t *la = &o->levels[c1 - 1], *lb = &o->levels[c2 - 1];
                int64_t na = la->n, nb = lb->n;
                if (na == 0 || nb == 0) continue;
                c.tag = tag;
                c.a_base = la->base;
                c.b_base = lb->base;
                if (commutative && c1 == c2) { /* engine.py:241-257 */
                    int64_t i0 = 0;
                    c.n = na;
                    while (i0 < na && !r.stop) {
                        if (na - i0 > batch) {
                            for (int64_t j0 = i0; j0 < na && !r.stop; j0 += batch) {
                                c.kind = 4;
                                c.i0 = i0;
                                c.j0 = j0;
                                c.j1 = j0 + batch < na ? j0 + batch : na;
                                do_chunk(&r, &c);
                            }
                            i0++;
                            continue;
                        }
                        int64_t pairs = 0, i1 = i0;
                        while (i1 < na && pairs + (na - i1) <= batch) {
                            pairs += na - i1;
                            i1++;
                        }
                        c.kind = 3;
                        c.i0 = i0;
                        c.i1 = i1;
                        do_chunk(&r, &c);
                        i0 = i1;
                    }
                } else { /* engine.py:258-266 */
                    int64_t rows = batch / nb;
                    c.kind = 2;
                    if (rows >= 1) {
                        for (int64_t i0 = 0; i0 < na && !r.stop; i0 += rows) {
                            c.i0 = i0;
                            c.i1 = i0 + rows < na ? i0 + rows : na;
                            c.j0 = 0;
                            c.j1 = nb;
                            do_chunk(&r, &c);
                        }
                    } else {
                        for (int64_t i0 = 0; i0 < na && !r.stop; i0++)
                            for (int64_t j0 = 0; j0 < nb && !r.stop; j0 += batch) {
                                c.i0 = i0;
                                c.i1 = i0 + 1;
                                c.j0 = j0;
                                c.j1 = j0 + batch < nb ? j0 + batch : nb;
                                do_chunk(&r, &c);
                            }
                    }
                }
            }
        }
    }
    /* flush(), engine.py:399-412,447-449 */
    if (o->n_levels == o->levels_cap) {
        o->levels_cap = o->levels_cap ? o->levels_cap * 2 : 32;
        o->levels = (level_t *)realloc(o->levels, sizeof(level_t) * (size_t)o->levels_cap);
    }
    o->levels[o->n_levels++] = r.lv;
    *n_new = r.n_new;
    *sep_gid = r.sep_gid;
    *constructed_delta = r.constructed;
    return r.status;
}

double orc_now(void) { return now_s(); }
int64_t orc_total(const oracle_t *o) { return o->total; }
int64_t orc_approx_bytes(const oracle_t *o) { return o->approx_bytes; }
int orc_num_levels(const oracle_t *o) { return o->n_levels; }
/* analysis only (tools/dup_profile.py): duplicate histogram of the most recently expanded level */
void orc_dup_hist(const oracle_t *o, int64_t *out64) { memcpy(out64, o->dup_hist, sizeof(o->dup_hist)); }
int orc_row_bytes(const oracle_t *o) { return o->row_bytes; }

int orc_level_info(const oracle_t *o, int cost, int64_t *n, int64_t *base) {
    if (cost < 1 || cost > o->n_levels) return ST_BAD;
    *n = o->levels[cost - 1].n;
    *base = o->levels[cost - 1].base;
    return ST_OK;
}

/* copies the level arrays: cms = n x row_bytes (numpy tobytes image), op u8, left/right i64 */
int orc_level_copy(const oracle_t *o, int cost, uint8_t *cms, uint8_t *op, int64_t *left, int64_t *right) {
    if (cost < 1 || cost > o->n_levels) return ST_BAD;
    const level_t *lv = &o->levels[cost - 1];
    if (cms) memcpy(cms, o->rows + (size_t)lv->row0 * o->row_bytes, (size_t)lv->n * o->row_bytes);
    if (op) memcpy(op, lv->op, (size_t)lv->n);
    if (left) memcpy(left, lv->left, sizeof(int64_t) * (size_t)lv->n);
    if (right) memcpy(right, lv->right, sizeof(int64_t) * (size_t)lv->n);
    return ST_OK;
}
