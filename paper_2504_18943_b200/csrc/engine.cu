// engine.cu -- host side of the B200 enumeration engine and its C ABI (include/ltlsynth_b200.h).
//
// Owns the HBM-resident language cache (all finalised CMs by global id + the ordinal
// each entry won with), the dedup hash set and the per-level scratch, and drives one
// cost level per ltlb200_expand_level call:
//
//   plan      canonical block list of the level (reference _tasks_for_level,
//             engine.py:219-266, minus its batch chunking) -> ordinal offsets, tiles
//   enumerate persistent launches of the construction+dedup kernels (narrow.cuh / wide2.cuh), one per operator on
//             big levels, one for all on small ones, one for several tiny levels (narrow_tiny.cuh)
//   finalise  bitmap-rank compaction: winners ordered by ordinal, appended to the cache
//   account   `constructed` as the reference counts it, including its chunk rounding on
//             the level that holds the separator (engine.py:418,445-446)
//
// No CPU fallback exists: without a usable sm_100 device every entry point fails.
#include <cuda_runtime.h>

#include <algorithm>
#include <array>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <ctime>
#include <map>
#include <mutex>
#include <stdexcept>
#include <string>
#include <tuple>
#include <vector>

#include "../../include/ltlsynth_b200.h"
#include <deque>

#include "launch.h"
#include "narrow_fin.cuh"
#include "narrow_tiny.cuh"
#include "wide2_tiny.cuh"
#include "wide_fin.cuh"

namespace ltlb200 {

static thread_local std::string g_last_error;

struct CudaError : std::runtime_error {
    using std::runtime_error::runtime_error;
};
struct MemoryBudget : std::runtime_error {
    using std::runtime_error::runtime_error;
};

#define CUDA_CHECK(expr)                                                                              \
    do {                                                                                              \
        cudaError_t err__ = (expr);                                                                   \
        if (err__ != cudaSuccess)                                                                     \
            throw CudaError(std::string(#expr) + ": " + cudaGetErrorString(err__) + " (" __FILE__ ":" + \
                            std::to_string(__LINE__) + ")");                                          \
    } while (0)

static bool debug_on() {
    static const bool on = getenv("LTLB200_DEBUG") != nullptr;
    return on;
}
#define DBG(...)                                   \
    do {                                           \
        if (debug_on()) {                          \
            fprintf(stderr, "[ltlb200] " __VA_ARGS__); \
            fputc('\n', stderr);                   \
            fflush(stderr);                        \
        }                                          \
    } while (0)

static double monotonic_s() {
    timespec ts;
    clock_gettime(CLOCK_MONOTONIC, &ts);
    return (double)ts.tv_sec + 1e-9 * (double)ts.tv_nsec;
}

// LTLB200_TIMING=1: host-side phase timers of the level loop, printed when a handle is destroyed
struct PhaseTimers {
    static constexpr int N = 12;
    double acc[N] = {};
    const char *name[N] = {};
    bool on = getenv("LTLB200_TIMING") != nullptr;
    void add(int i, const char *n, double dt) {
        acc[i] += dt;
        name[i] = n;
    }
    void dump() const {
        if (!on) return;
        for (int i = 0; i < N; ++i)
            if (name[i]) fprintf(stderr, "[ltlb200 timing] %-28s %9.3f ms\n", name[i], 1e3 * acc[i]);
    }
};
static PhaseTimers g_phase;
#define PHASE(i, label, t0)                              \
    do {                                                 \
        if (g_phase.on) {                                \
            const double now__ = monotonic_s();          \
            g_phase.add(i, label, now__ - (t0));         \
            (t0) = now__;                                \
        }                                                \
    } while (0)

static u64 next_pow2(u64 x) {
    u64 p = 1;
    while (p < x) p <<= 1;
    return p;
}

// ---- process-wide device block cache ------------------------------------------------------
// A search regrows its hash set and its cache every level, and a caller typically runs many
// searches (one per specification, or one per benchmark step).  cudaMalloc/cudaFree cost
// milliseconds per GB and synchronise the device, so freed blocks are kept here, rounded to
// a few size classes per power of two, and handed to the next request of the same class.
// After the first search of a given size no allocation reaches the driver.
struct BlockCache {
    std::mutex mu;
    std::map<std::pair<int, u64>, std::vector<void *>> free_blocks;
    std::map<int, u64> cached_bytes;

    static u64 size_class(u64 bytes) {
        if (bytes <= 4096) return 4096;
        u64 p = next_pow2(bytes);           // 2^k >= bytes
        if (bytes <= (1u << 20)) return p;  // small: plain powers of two
        u64 q = p / 8;                      // large: eighths between 2^(k-1) and 2^k
        return ((bytes + q - 1) / q) * q;
    }
    void *get(int dev, u64 cls) {
        std::lock_guard<std::mutex> lock(mu);
        auto it = free_blocks.find({dev, cls});
        if (it == free_blocks.end() || it->second.empty()) return nullptr;
        void *p = it->second.back();
        it->second.pop_back();
        cached_bytes[dev] -= cls;
        return p;
    }
    void put(int dev, u64 cls, void *p) {
        std::lock_guard<std::mutex> lock(mu);
        free_blocks[{dev, cls}].push_back(p);
        cached_bytes[dev] += cls;
    }
    u64 cached(int dev) {
        std::lock_guard<std::mutex> lock(mu);
        return cached_bytes[dev];
    }
    void trim(int dev) {  // give everything cached for `dev` back to the driver
        std::lock_guard<std::mutex> lock(mu);
        for (auto &kv : free_blocks)
            if (kv.first.first == dev) {
                for (void *p : kv.second) cudaFree(p);
                kv.second.clear();
            }
        cached_bytes[dev] = 0;
    }
};
static BlockCache g_blocks;

struct DeviceInfo {
    int major = 0, sm_count = 0;
    bool known = false;
};
static DeviceInfo device_info(int dev) {
    static std::mutex mu;
    static std::map<int, DeviceInfo> cache;
    std::lock_guard<std::mutex> lock(mu);
    DeviceInfo &d = cache[dev];
    if (!d.known) {
        int major = 0, sms = 0;
        if (cudaDeviceGetAttribute(&major, cudaDevAttrComputeCapabilityMajor, dev) != cudaSuccess ||
            cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess) {
            cudaGetLastError();
            return DeviceInfo{};
        }
        d.major = major;
        d.sm_count = sms;
        d.known = true;
    }
    return d;
}

// pinned staging words for the per-level counter read-back, recycled across handles
static std::mutex g_pinned_mu;
static std::vector<u64 *> g_pinned_free;
static u64 *pinned_get() {
    {
        std::lock_guard<std::mutex> lock(g_pinned_mu);
        if (!g_pinned_free.empty()) {
            u64 *p = g_pinned_free.back();
            g_pinned_free.pop_back();
            return p;
        }
    }
    u64 *p = nullptr;
    if (cudaMallocHost(&p, 64 * sizeof(u64)) != cudaSuccess) {
        cudaGetLastError();
        throw std::runtime_error("cudaMallocHost failed");
    }
    return p;
}
static void pinned_put(u64 *p) {
    if (!p) return;
    std::lock_guard<std::mutex> lock(g_pinned_mu);
    g_pinned_free.push_back(p);
}

// Streams and events of a handle, recycled process-wide: a caller that runs one search per specification
// creates and destroys a handle per search, and creating five streams and ten events costs more than the
// small levels of the search (the end-to-end time of spec2 rose by 0.6 ms when the side streams were added).
struct StreamBundle {
    cudaStream_t own = nullptr;  // the handle's stream when the caller passed none
    cudaEvent_t ev[4] = {};      // timing: enumerate begin/end, finalise begin/end
    cudaStream_t side[4] = {};   // operator fan-out (Engine::fan_*)
    cudaEvent_t fork = nullptr, join[4] = {};
    cudaStream_t copy = nullptr;     // reads the level's counters while the last finalisation kernel still runs
    cudaEvent_t summary = nullptr;   // the counters are final
    cudaEvent_t fin[4] = {};         // finalisation begin / end, double-buffered (read one level late)
};
static std::mutex g_bundle_mu;
static std::map<int, std::vector<StreamBundle>> g_bundles;

static StreamBundle bundle_get(int dev) {
    {
        std::lock_guard<std::mutex> lock(g_bundle_mu);
        auto &pool = g_bundles[dev];
        if (!pool.empty()) {
            StreamBundle b = pool.back();
            pool.pop_back();
            return b;
        }
    }
    StreamBundle b;
    CUDA_CHECK(cudaStreamCreateWithFlags(&b.own, cudaStreamNonBlocking));
    for (auto &e : b.ev) CUDA_CHECK(cudaEventCreate(&e));
    for (auto &st : b.side) CUDA_CHECK(cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking));
    CUDA_CHECK(cudaEventCreateWithFlags(&b.fork, cudaEventDisableTiming));
    for (auto &e : b.join) CUDA_CHECK(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
    CUDA_CHECK(cudaStreamCreateWithFlags(&b.copy, cudaStreamNonBlocking));
    CUDA_CHECK(cudaEventCreateWithFlags(&b.summary, cudaEventDisableTiming));
    for (auto &e : b.fin) CUDA_CHECK(cudaEventCreate(&e));
    return b;
}

// (every stream of the bundle has drained: the handle synchronises before it lets go)
static void bundle_put(int dev, const StreamBundle &b) {
    std::lock_guard<std::mutex> lock(g_bundle_mu);
    g_bundles[dev].push_back(b);
}

// ---- small device kernels shared by both key widths --------------------------------

// exclusive scan of per-superblock popcounts, 1024 values per CTA; block totals go to `sums`
__global__ void __launch_bounds__(1024) sb_scan_kernel(const uint32_t *bitmap, u64 n_words, const uint32_t *in,
                                                      uint32_t *out, u64 n, uint32_t *sums) {
    __shared__ uint32_t warp_tot[32];
    const u64 i = (u64)blockIdx.x * 1024 + threadIdx.x;
    uint32_t v = 0;
    if (i < n) {
        if (bitmap) {  // first level: popcount of the 32 words of superblock i
            const u64 w0 = i << 5;
#pragma unroll 4
            for (int k = 0; k < 32; ++k)
                if (w0 + k < n_words) v += __popc(bitmap[w0 + k]);
        } else {
            v = in[i];
        }
    }
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    uint32_t incl = v;
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
        uint32_t t = __shfl_up_sync(0xFFFFFFFFu, incl, d);
        if (lane >= d) incl += t;
    }
    if (lane == 31) warp_tot[warp] = incl;
    __syncthreads();
    if (warp == 0) {
        uint32_t w = warp_tot[lane], wi = w;
#pragma unroll
        for (int d = 1; d < 32; d <<= 1) {
            uint32_t t = __shfl_up_sync(0xFFFFFFFFu, wi, d);
            if (lane >= d) wi += t;
        }
        warp_tot[lane] = wi - w;  // exclusive prefix of warp totals
        if (lane == 31 && sums) sums[blockIdx.x] = wi;
    }
    __syncthreads();
    if (i < n) out[i] = warp_tot[warp] + incl - v;
}

__global__ void __launch_bounds__(1024) sb_add_kernel(uint32_t *out, u64 n, const uint32_t *block_prefix) {
    const u64 i = (u64)blockIdx.x * 1024 + threadIdx.x;
    if (i < n) out[i] += block_prefix[blockIdx.x];
}

// counters of a level start at zero (CTR_SEP at "none"); the special-key register persists across levels;
// `time_left_ns` (all ones = no deadline) anchors the level's deadline on the device's own timer
__global__ void level_init_kernel(u64 *counters, u64 time_left_ns) {
    const int i = threadIdx.x;
    if (i < CTR_COUNT && i != CTR_SPECIAL) counters[i] = i == CTR_SEP ? VAL_EMPTY : 0ull;
    if (i == CTR_STOPAT) counters[i] = time_left_ns == VAL_EMPTY ? VAL_EMPTY : global_timer_ns() + time_left_ns;
}

// number of winners and rank of the separator's ordinal (the separator is counters[CTR_SEP])
__global__ void level_summary_kernel(const uint32_t *bitmap, const uint32_t *sb_rank, u64 n_bits, u64 *counters) {
    const u64 sep_ord = counters[CTR_SEP];
    counters[CTR_WINNERS] = n_bits ? ordinal_rank(bitmap, sb_rank, n_bits - 1) + ((bitmap[(n_bits - 1) >> 5] >> ((n_bits - 1) & 31)) & 1u) : 0;
    counters[CTR_SEPRANK] = sep_ord < n_bits ? ordinal_rank(bitmap, sb_rank, sep_ord) : ~0ull;
}

// counters[CTR_SEP] = smallest listed ordinal that is a winner (its bitmap bit is set)
__global__ void __launch_bounds__(256) first_fresh_kernel(const uint32_t *bitmap, const u64 *ords, u64 n, u64 *counters) {
    const u64 k = (u64)blockIdx.x * blockDim.x + threadIdx.x;
    if (k >= n) return;
    const u64 ord = ords[k];
    if (bitmap[ord >> 5] >> (ord & 31) & 1u) atomicMin(&counters[CTR_SEP], ord);
}

// ---- host-side level bookkeeping ------------------------------------------------------

struct LevelMeta {
    u64 n = 0, base = 0;
    std::vector<BlockDesc> blocks;
};

template <typename T>
struct DeviceArray {
    T *ptr = nullptr;
    u64 cap = 0;    // elements
    u64 bytes = 0;  // size class of the block
};

class Engine {
public:
    Engine(int T, int lane_bits, const uint64_t *masks, const uint64_t *target, const uint64_t *atoms, int n_atoms,
           int device, u64 budget, void *stream);
    ~Engine();

    int expand_level(int cost, uint32_t op_mask, bool exhaustive, int64_t batch, u64 mem_budget, double deadline,
                     int64_t *n_new, int64_t *sep_gid, int64_t *constructed_delta);
    int level_info(int cost, int64_t *n, int64_t *base) const;
    int64_t level_candidates(int cost, uint32_t op_mask);
    int level_copy(int cost, int64_t first, int64_t count, uint8_t *cms, uint8_t *op, int64_t *left, int64_t *right);
    int level_device(int cost, void **rows_dev, void **ords_dev);
    const uint4 *rows_in_id_order(u64 first, u64 count);
    void set_weights(const int32_t *weights, int count);
    // Tiny levels built ahead of the caller by ONE launch (narrow_tiny.cuh) and handed out one expand_level call
    // at a time: the rows, ordinals and set entries of these levels are on the device already; levels_ / total_
    // learn about a level when it is handed out.
    struct Lookahead {
        int cost;
        u64 n_new, sep_ord, sep_rank;
        u64 n_staged;  // wide: log entries the level takes
    };
    std::deque<Lookahead> lookahead_;
    uint32_t la_mask_ = 0;
    bool la_exhaustive_ = false;
    bool tiny_off_ = false;  // an exhaustive level held a separating candidate: so will the following ones (until reset)
    DeviceArray<u64> tiny_tab_, tiny_results_;
    bool tiny_eligible(int cost, uint32_t op_mask, bool exhaustive);
    void tiny_run(int cost, uint32_t op_mask, bool exhaustive);
    void tiny_run_wide(int cost, uint32_t op_mask, bool exhaustive);
    int tiny_reveal(int cost, uint32_t op_mask, bool exhaustive, int64_t batch, u64 mem_budget, double deadline, int64_t *n_new,
                    int64_t *sep_gid, int64_t *constructed_delta);
    void discard_lookahead();
    double deadline_ = -1.0;  // CLOCK_MONOTONIC deadline of the level being built (< 0: none)
    u64 time_left_ns() const {
        if (deadline_ < 0) return VAL_EMPTY;
        const double left = deadline_ - monotonic_s();
        return left <= 0 ? 1ull : (u64)(left * 1e9);
    }
    void set_regex(int n_bits, const uint32_t *offsets, const uint32_t *entries, u64 n_entries);
    int entry(int64_t gid, int32_t *op, int64_t *left, int64_t *right);
    void get_stats(ltlb200_stats *out);
    void reset();
    int level_begin(int cost, uint32_t op_mask, bool exhaustive, double deadline, u64 *n_claimed, u64 *sep_ord, u64 *n_seps,
                    bool defer = false);
    int level_end(u64 sep_ord, const u64 *seps, u64 n_seps, int64_t batch, u64 mem_budget, int64_t *n_new, int64_t *sep_gid,
                  int64_t *constructed_delta);
    int level_end_deferred(int64_t batch, u64 mem_budget, int64_t *n_new, int64_t *sep_gid, int64_t *constructed_delta);
    void launch_rank_scan(u64 n_words, u64 n_sb);
    static constexpr int kRetryLevel = 100;  // internal status: the deferred attempt overflowed, redo synchronously
    // one search sharded over several GPUs: owner-sharded set, candidates routed to their hash owners
    int route_begin(int cost, uint32_t op_mask, bool exhaustive, double deadline, int rank, int world, u64 *send_counts,
                    u64 *send_offsets, void **rows_dev, void **ords_dev, u64 *sep_ord, u64 *n_seps);
    void exchange_recv(u64 n_records, void **rows_dev, void **ords_dev);
    int owner_reduce(u64 n_records, u64 *n_claimed, void **bitmap_dev, u64 *bitmap_words);
    void level_abort();
    void winners_export(u64 sep_ord, u64 *n_winners, void **rows_dev, void **ords_dev);
    int level_commit(u64 sep_ord, const u64 *seps, u64 n_seps, const u64 *recv_counts, int n_sources, int64_t batch, u64 mem_budget,
                     int64_t *n_new, int64_t *sep_gid, int64_t *constructed_delta);
    RecordSources sources_{};  // layout of the winners received from the other owners (level_commit)
    u64 seps_copy(u64 *out, u64 cap);
    int key_bytes() const { return 16 * nvec_; }
    int num_levels() const { return (int)levels_.size(); }
    bool holds_separator() const { return store_has_separator_; }
    u64 approx_bytes() const { return approx_bytes_; }

private:
    // geometry
    int T_, lw_, row_bytes_, key_words_, n_atoms_;
    int device_;
    cudaStream_t stream_ = nullptr;
    bool own_stream_ = false;
    StreamBundle res_;  // recycled streams / events (ev_, side_, fork_ev_, join_ev_ below are copies of its handles)
    u64 budget_ = 0, held_ = 0;
    uint4 valid_{}, target_{};
    bool special_possible_ = false;
    bool wide_ = false;  // CMs of more than one uint4
    int nvec_ = 1, log2g_ = 0;
    uint4 *d_valid_ = nullptr, *d_target_ = nullptr;

    // device state
    uint4 *d_atoms_ = nullptr;
    DeviceArray<uint4> store_;
    DeviceArray<u64> ords_;
    DeviceArray<Slot16> slots_;
    u64 grown_size(u64 want_slots) const;
    DeviceArray<uint4> claim_key_;   // narrow path: this level's new CMs by claim index
    DeviceArray<u64> claim_ord_;
    DeviceArray<u64> wslots_;          // wide path: slot words
    // wide path: store_ is the ROW LOG (rows in the order they were staged, a level's new rows at its tail);
    // loc_[id] = log index of entry id; log_tail_ = log entries in use (finalised levels incl. their unused entries)
    DeviceArray<u64> loc_;
    DeviceArray<uint4> gather_;  // level_copy / level_device: rows of a level gathered into id order
    u64 log_tail_ = 0;
    DeviceArray<u64> stage_ord_;
    DeviceArray<uint32_t> bitmap_;
    DeviceArray<uint32_t> sb_rank_;
    DeviceArray<uint32_t> scan_tmp_;
    DeviceArray<u64> sep_list_;
    DeviceArray<uint8_t> misc_;
    DeviceArray<u64> xchg_;  // per-owner record counts of the route phase; winners cursor
    // sharded search: send side (route regions, then this owner's winners) and receive side (records from the
    // other ranks, then their winners) of the two exchanges of a level
    DeviceArray<uint4> xs_rows_, xr_rows_;
    DeviceArray<u64> xs_ords_, xr_ords_;
    int owner_world_ = 1, owner_rank_ = 0;  // the set holds the CMs whose hash owner is owner_rank_ (world 1: all)
    void set_sharding(int world, int rank);
    int finalize_level(u64 sep_ord, const u64 *seps, u64 n_seps, int64_t batch, u64 mem_budget, int64_t *n_new, int64_t *sep_gid,
                       int64_t *constructed_delta, bool global_bitmap, u64 n_received);
    bool store_has_separator_ = false;  // some stored CM separates: a separating candidate need not be fresh
    // Associativity pruning (narrow.cuh: run_binary_tile) is sound while every stored level is complete and
    // all levels were built with one operator set; the first cut level or change of operators ends it.
    bool prune_ok_ = true;
    uint32_t prune_mask_ = 0;  // operator set of the levels built so far (0 = none yet)
    // EXTENSION (not in the reference: "config-extensible", unimplemented): cost of one node per operator
    // tag, [0] = an atom.  All 1 = the reference's node count.
    int weights_[16] = {1, 1, 1, 1, 1, 1, 1, 1, 1, 1, 1, 1, 1, 1, 1, 1};
    bool unit_weights_ = true;
    // regex front-end (regex_ops.cuh): the infix-split guide table on the device; n_bits_ > 0 = regex grammar
    DeviceArray<uint32_t> guide_;
    int n_bits_ = 0;
    uint32_t guide_smem_words_ = 0;  // wide kernels: the tables are staged in the CTA's shared memory (LTLB200_GUIDE_SMEM=1)
    uint32_t guide_entries_ = 0, guide_rounds_ = 0;
    // Non-exhaustive level over a store that already holds a separating CM (narrow path, one GPU): the chunks
    // the reference truncates at a separating candidate are found by a scan pass and their tails excluded
    // from the enumeration (NarrowParams::dead).  batch_size is known to expand_level only.
    DeviceArray<u64> dead_;
    u64 dead_n_ = 0;
    int64_t mode_batch_ = 0;
    u64 sep_want_ = 0;  // separating candidates the last attempt counted beyond the list's capacity
    void collect_dead_ranges(const LevelMeta &lv, u64 constructed, u64 batch);
    static constexpr u64 kEntryCache = 1ull << 14;  // entries whose ordinals entry() keeps on the host (128 KB)
    std::vector<u64> entry_cache_;
    u64 entry_cache_total_ = 0;
    struct PendingLevel {
        LevelMeta lv;
        u64 constructed = 0, n_claimed = 0, sep_ord = ~0ull, n_seps = 0, claim_cap = 0;
        bool exhaustive = false, active = false, seps_overflow = false, deferred = false, routed = false, reduced = false;
        int cost = 0;
        u64 n_received = 0, n_winners = 0, region_cap = 0;
    } pending_;
    WideParams wide_params(bool exhaustive) const;
    NarrowParams narrow_params(bool exhaustive) const;
    static constexpr u64 kMinSlots = 1ull << 16;
    u64 *d_counters_ = nullptr;
    BlockDesc *d_blocks_ = nullptr;
    static constexpr int kMaxBlocks = 512;
    u64 *h_counters_ = nullptr;  // pinned
    cudaEvent_t ev_[4] = {};
    bool table_dirty_ = false;
    // The operator launches of one big level are independent of each other (they share the set, the claim
    // arrays and the counters, all updated atomically), so they go to different streams: the next operator's
    // CTAs move into the SMs as the previous launch's last tiles finish, instead of waiting for its tail.
    static constexpr int kSideStreams = 4;
    cudaStream_t side_[kSideStreams] = {};
    cudaEvent_t fork_ev_ = nullptr, join_ev_[kSideStreams] = {};
    uint32_t side_used_ = 0;  // side streams of the current fan-out
    void fan_begin();
    cudaStream_t fan_stream(int group);
    void fan_end();

    std::vector<LevelMeta> levels_;
    u64 total_ = 0, approx_bytes_ = 0, last_constructed_ = 0;
    int occupancy_ = 2;
    ltlb200_stats st_{};
    int sm_count_ = 148;

    template <typename T>
    void reserve(DeviceArray<T> &a, u64 want, bool keep, u64 keep_elems = 0);
    template <typename T>
    void release(DeviceArray<T> &a);
    void *pool_alloc(u64 bytes);
    void pool_free(void *p, u64 bytes);
    void recycle_retired(bool synchronise);
    std::vector<std::pair<void *, u64>> retired_;
    void plan_level(int cost, uint32_t op_mask, LevelMeta &lv, u64 &constructed, u64 &n_tiles);
    void rebuild_table(u64 slots);
    void read_counters();
    void read_counters_early();
    void collect_finalize_time(int slot, bool wait);
    int fin_slot_ = 0;
    bool fin_pending_[2] = {false, false};
    void decode(const LevelMeta &lv, u64 ord, int32_t *op, int64_t *left, int64_t *right) const;
    u64 constructed_through(const LevelMeta &lv, u64 sep_ord, u64 batch) const;
    void launch_enumerate(NarrowParams P, const LevelMeta &lv);
    void launch_narrow(int kind, int op, const NarrowParams &P, int grid, cudaStream_t st);
    void launch_wide(int kind, int op, const WideParams &P, int grid, cudaStream_t st);
    template <typename Params>
    void launch_level(Params P, const LevelMeta &lv);
    void launch_enumerate_wide(WideParams P, const LevelMeta &lv);
    u64 table_slots() const { return wide_ ? wslots_.cap : slots_.cap; }
    u64 chunk_exact_separator(const LevelMeta &lv, std::vector<u64> &seps, u64 batch);
};

// Blocks come from the process-wide cache (see BlockCache); `bytes` must be a size class.
void *Engine::pool_alloc(u64 bytes) {
    const double t0 = monotonic_s();
    void *p = g_blocks.get(device_, bytes);
    if (!p) {
        cudaError_t err = cudaMalloc(&p, bytes);
        if (err != cudaSuccess) {  // make room by dropping cached blocks of other classes, once
            cudaGetLastError();
            CUDA_CHECK(cudaStreamSynchronize(stream_));
            g_blocks.trim(device_);
            err = cudaMalloc(&p, bytes);
        }
        if (err != cudaSuccess) {
            cudaGetLastError();
            st_.alloc_ms += 1e3 * (monotonic_s() - t0);
            throw MemoryBudget(std::string("cudaMalloc failed: ") + cudaGetErrorString(err));
        }
    }
    st_.alloc_ms += 1e3 * (monotonic_s() - t0);
    return p;
}

// Stream-ordered reuse: a block released here may be handed out again to THIS handle while
// earlier work of its stream still reads it, which is safe because the next user runs on
// the same stream; blocks become visible to other handles only after the stream drained.
void Engine::pool_free(void *p, u64 bytes) {
    if (p) retired_.push_back({p, bytes});
}

void Engine::recycle_retired(bool synchronise) {
    if (retired_.empty()) return;
    if (synchronise) cudaStreamSynchronize(stream_);
    for (auto &r : retired_) g_blocks.put(device_, r.second, r.first);
    retired_.clear();
}

template <typename T>
void Engine::release(DeviceArray<T> &a) {
    if (a.ptr) {
        pool_free(a.ptr, a.bytes);
        held_ -= a.bytes;
    }
    a.ptr = nullptr;
    a.cap = 0;
    a.bytes = 0;
}

// grow `a` to at least `want` elements; with keep, the first keep_elems survive
template <typename T>
void Engine::reserve(DeviceArray<T> &a, u64 want, bool keep, u64 keep_elems) {
    if (want <= a.cap) return;
    u64 bytes = BlockCache::size_class(std::max<u64>(keep ? std::max(want, 2 * a.cap) : want, 1) * sizeof(T));
    u64 extra = bytes - (keep ? 0 : a.bytes);
    if (held_ + extra > budget_) {
        bytes = BlockCache::size_class(want * sizeof(T));  // retry without head-room
        extra = bytes - (keep ? 0 : a.bytes);
        if (held_ + extra > budget_) throw MemoryBudget("device memory budget exhausted");
    }
    if (!keep) release(a);
    T *p = static_cast<T *>(pool_alloc(bytes));
    held_ += bytes;
    if (keep && a.ptr) {
        if (keep_elems) CUDA_CHECK(cudaMemcpyAsync(p, a.ptr, keep_elems * sizeof(T), cudaMemcpyDeviceToDevice, stream_));
        pool_free(a.ptr, a.bytes);  // recycled once the stream has drained
        held_ -= a.bytes;
    }
    a.ptr = p;
    a.bytes = bytes;
    a.cap = bytes / sizeof(T);
}

// byte image of one CM row (T lanes, little endian), zero padded to nvec uint4 vectors
static void pack_row(const uint64_t *lanes, int T, int lane_bits, int nvec, uint4 *out) {
    std::vector<uint8_t> bytes((size_t)nvec * 16, 0);
    const int lb = lane_bits / 8;
    for (int t = 0; t < T; ++t) memcpy(bytes.data() + (size_t)t * lb, &lanes[t], lb);
    memcpy(out, bytes.data(), bytes.size());
}

Engine::Engine(int T, int lane_bits, const uint64_t *masks, const uint64_t *target, const uint64_t *atoms, int n_atoms,
               int device, u64 budget, void *stream)
    : T_(T), lw_(lane_bits), row_bytes_(T * lane_bits / 8), key_words_((T * lane_bits / 8 + 7) / 8), n_atoms_(n_atoms),
      device_(device) {
    const double t_create = monotonic_s();
    double tp = monotonic_s();
    CUDA_CHECK(cudaSetDevice(device_));
    PHASE(8, "create: set device", tp);
    const DeviceInfo info = device_info(device_);
    if (!info.known) throw CudaError("cannot query the CUDA device");
    if (info.major != 10) throw CudaError("device is not sm_100 (Blackwell B200); this library has no other code path");
    sm_count_ = info.sm_count;
    nvec_ = (row_bytes_ + 15) / 16;
    wide_ = nvec_ > 1;
    if (nvec_ > MAX_NVEC) throw std::invalid_argument("CMs wider than 512 bytes are not supported");
    for (log2g_ = wide_ ? 1 : 0; (1 << log2g_) < nvec_; ++log2g_) {}
    res_ = bundle_get(device_);
    if (stream) stream_ = (cudaStream_t)stream;
    else {
        stream_ = res_.own;
        own_stream_ = true;
    }
    PHASE(9, "create: stream", tp);
    if (budget) budget_ = budget;
    else {  // 90% of what was free when this process first asked (cudaMemGetInfo costs milliseconds once
            // gigabytes are mapped, and everything this library holds is either in use by a live
            // handle -- counted in held_ -- or parked in the process-wide block cache)
        static std::mutex mu;
        static std::map<int, u64> free_at_start;
        std::lock_guard<std::mutex> lock(mu);
        auto it = free_at_start.find(device_);
        if (it == free_at_start.end()) {
            size_t free_b = 0, total_b = 0;
            CUDA_CHECK(cudaMemGetInfo(&free_b, &total_b));
            it = free_at_start.emplace(device_, (u64)free_b + g_blocks.cached(device_)).first;
        }
        budget_ = (u64)(it->second * 0.9);
    }
    PHASE(10, "create: mem info", tp);
    std::vector<uint4> h_valid(nvec_), h_target(nvec_);
    pack_row(masks, T, lane_bits, nvec_, h_valid.data());
    pack_row(target, T, lane_bits, nvec_, h_target.data());
    valid_ = h_valid[0];
    target_ = h_target[0];
    // the all-ones vector doubles as the empty-slot marker; it is a legal CM only when
    // the row fills the vector and every lane is fully valid
    special_possible_ = (valid_.x & valid_.y & valid_.z & valid_.w) == 0xFFFFFFFFu;

    // one small block: counters | block descriptors | masks | target | atom rows
    const u64 off_blocks = 256, off_rows = off_blocks + kMaxBlocks * sizeof(BlockDesc);
    std::vector<uint4> h_rows((size_t)(2 + std::max(n_atoms, 1)) * nvec_);
    memcpy(h_rows.data(), h_valid.data(), (size_t)nvec_ * 16);
    memcpy(h_rows.data() + nvec_, h_target.data(), (size_t)nvec_ * 16);
    for (int p = 0; p < n_atoms; ++p) pack_row(atoms + (size_t)p * T, T, lane_bits, nvec_, h_rows.data() + (size_t)(2 + p) * nvec_);
    reserve(misc_, off_rows + h_rows.size() * sizeof(uint4), false);
    d_counters_ = reinterpret_cast<u64 *>(misc_.ptr);
    d_blocks_ = reinterpret_cast<BlockDesc *>(misc_.ptr + off_blocks);
    d_valid_ = reinterpret_cast<uint4 *>(misc_.ptr + off_rows);
    d_target_ = d_valid_ + nvec_;
    d_atoms_ = d_target_ + nvec_;
    CUDA_CHECK(cudaMemcpyAsync(d_valid_, h_rows.data(), h_rows.size() * sizeof(uint4), cudaMemcpyHostToDevice, stream_));
    st_.h2d_bytes += h_rows.size() * sizeof(uint4);
    h_counters_ = pinned_get();
    for (int k = 0; k < 4; ++k) ev_[k] = res_.ev[k];
    for (int k = 0; k < kSideStreams; ++k) side_[k] = res_.side[k];
    fork_ev_ = res_.fork;
    for (int k = 0; k < kSideStreams; ++k) join_ev_[k] = res_.join[k];
    u64 init[CTR_COUNT];
    for (auto &c : init) c = 0;
    init[CTR_SPECIAL] = VAL_EMPTY;
    CUDA_CHECK(cudaMemcpyAsync(d_counters_, init, sizeof(init), cudaMemcpyHostToDevice, stream_));
    CUDA_CHECK(cudaStreamSynchronize(stream_));  // h_rows / init leave scope
    PHASE(11, "create: copies + sync", tp);
    {   // occupancy queries once per process, device, lane width and (wide: shared memory depends on it) nvec
        static std::mutex mu;
        static std::map<std::tuple<int, int, int>, int> cache;
        std::lock_guard<std::mutex> lock(mu);
        auto it = cache.find({device_, lw_, nvec_});
        if (it == cache.end()) {
            int occ;
            if (wide_) occ = lw_ == 8 ? wide2_occupancy_8(nvec_, device_, 0) : lw_ == 16 ? wide2_occupancy_16(nvec_, device_, 0)
                             : lw_ == 32 ? wide2_occupancy_32(nvec_, device_, 0) : wide2_occupancy_64(nvec_, device_, 0);
            else occ = lw_ == 8 ? narrow_occupancy_8() : lw_ == 16 ? narrow_occupancy_16() : lw_ == 32 ? narrow_occupancy_32() : narrow_occupancy_64();
            it = cache.emplace(std::make_tuple(device_, lw_, nvec_), occ).first;
        }
        occupancy_ = it->second;
    }
    rebuild_table(kMinSlots);
    st_.row_bytes = row_bytes_;
    st_.key_bytes = 16 * nvec_;
    st_.create_ms = 1e3 * (monotonic_s() - t_create);
}

Engine::~Engine() {
    cudaSetDevice(device_);
    release(store_);
    release(ords_);
    release(slots_);
    release(dead_);
    release(claim_key_);
    release(claim_ord_);
    release(wslots_);
    release(loc_);
    release(gather_);
    release(stage_ord_);
    release(bitmap_);
    release(sb_rank_);
    release(scan_tmp_);
    release(sep_list_);
    release(misc_);
    release(tiny_tab_);
    release(tiny_results_);
    release(guide_);
    release(xchg_);
    release(xs_rows_);
    release(xr_rows_);
    release(xs_ords_);
    release(xr_ords_);
    recycle_retired(true);
    pinned_put(h_counters_);
    g_phase.dump();
    if (res_.own) {
        cudaStreamSynchronize(stream_);  // (side streams are joined into it at the end of every fan-out)
        bundle_put(device_, res_);
    }
}

// Regrowing re-inserts every stored CM and clears the new set, so it should be rare while it is
// cheap and tight once clearing costs real time (6 GB/ms): grow 8x (two to three levels of a search
// that widens ~2.5x per level) below 256 MiB, 4x below 1 GiB, 2x beyond, and exactly to what the
// level needs when even that is more than a quarter of the budget.
// (Clearing the next set ahead of time on a side stream was tried twice.  Launched at the level that needs it, the
// memset queues behind the persistent enumerate CTAs.  Launched two or three levels early -- the size of the next
// set is predictable: grown_size of twice the current one -- it does run in the background and the regrows of
// `spec2` drop from 0.68 to 0.31 ms, but the search does not get faster (6.06 -> 6.09 ms): the device is busy 92 % of
// the time, so the 2.5 GB of stores only move into the enumerate launches they overlap.  Cleared by copy-engine
// copies of a pattern instead of a memset kernel it overlaps too, and costs more than it hides: 5.91 -> 6.19 ms, the
// random probes and the scatter slow down beside 4 GB of streaming traffic.)
u64 Engine::grown_size(u64 want_slots) const {
    const u64 slot_bytes = wide_ ? sizeof(u64) : sizeof(Slot16);
    const u64 want_bytes = want_slots * slot_bytes;
    u64 grown = want_slots * (want_bytes >= (1ull << 30) ? 2 : want_bytes >= (256ull << 20) ? 4 : 8);
    while (grown > want_slots && (grown * slot_bytes > budget_ / 4 || grown > (1ull << 32) - 2)) grown /= 2;  // (slot indices are 32-bit)
    return grown;
}

// Fresh table of `slots` entries holding every finalised CM (val = global id).
void Engine::rebuild_table(u64 slots) {
    const double t0 = monotonic_s();
    cudaEvent_t tev[2] = {nullptr, nullptr};
    if (g_phase.on) {  // LTLB200_TIMING: device time of this rebuild (synchronises; measurement only)
        for (auto &e : tev) CUDA_CHECK(cudaEventCreate(&e));
        CUDA_CHECK(cudaStreamSynchronize(stream_));
        CUDA_CHECK(cudaEventRecord(tev[0], stream_));
    }
    slots = std::max<u64>(next_pow2(slots), kMinSlots);
    if (slots > (1ull << 32) - 2) throw MemoryBudget("hash set would exceed 2^32 slots");
    if (wide_) {
        if (slots != wslots_.cap) {
            release(wslots_);
            reserve(wslots_, slots, false);
            wslots_.cap = slots;  // capacity must stay a power of two
        }
        CUDA_CHECK(cudaMemsetAsync(wslots_.ptr, 0, wslots_.cap * sizeof(u64), stream_));
        if (total_) {
            int grid = (int)std::min<u64>((total_ + 255) / 256, (u64)sm_count_ * 16);
            wide_rebuild_kernel<<<grid, 256, 0, stream_>>>(wslots_.ptr, wslots_.cap - 1, store_.ptr, loc_.ptr, total_, nvec_, log2g_, (uint32_t)owner_world_, (uint32_t)owner_rank_);
            CUDA_CHECK(cudaGetLastError());
            st_.kernel_launches++;
        }
    } else {
        if (slots != slots_.cap) {
            release(slots_);
            reserve(slots_, slots, false);
            slots_.cap = slots;  // capacity must stay a power of two
        }
        CUDA_CHECK(cudaMemsetAsync(slots_.ptr, 0xFF, slots_.cap * sizeof(Slot16), stream_));
        u64 special = VAL_EMPTY;
        CUDA_CHECK(cudaMemcpyAsync(d_counters_ + CTR_SPECIAL, &special, sizeof(u64), cudaMemcpyHostToDevice, stream_));
        if (total_) {
            int grid = (int)std::min<u64>((total_ + 255) / 256, (u64)sm_count_ * 16);
            narrow_rebuild_kernel<<<grid, 256, 0, stream_>>>(slots_.ptr, slots_.cap - 1, store_.ptr, 0, total_, d_counters_, (uint32_t)owner_world_, (uint32_t)owner_rank_);
            CUDA_CHECK(cudaGetLastError());
            st_.kernel_launches++;
        }
    }
    if (g_phase.on) {
        CUDA_CHECK(cudaEventRecord(tev[1], stream_));
        CUDA_CHECK(cudaEventSynchronize(tev[1]));
        float ms = 0;
        CUDA_CHECK(cudaEventElapsedTime(&ms, tev[0], tev[1]));
        fprintf(stderr, "[ltlb200 timing] rebuild_table: %llu slots, %llu stored CMs: %.3f ms on the device, %.3f ms host\n",
                (unsigned long long)slots, (unsigned long long)total_, ms, 1e3 * (monotonic_s() - t0));
        for (auto &e : tev) cudaEventDestroy(e);
    }
    table_dirty_ = false;
    st_.table_rebuilds++;
    st_.rebuild_host_ms += 1e3 * (monotonic_s() - t0);
}

// Forget every level but keep the device buffers (and the hash set's capacity) for the next search.
void Engine::reset() {
    CUDA_CHECK(cudaSetDevice(device_));
    lookahead_.clear();
    tiny_off_ = false;
    levels_.clear();
    total_ = 0;
    log_tail_ = 0;
    approx_bytes_ = 0;
    last_constructed_ = 0;
    store_has_separator_ = false;
    prune_ok_ = unit_weights_;
    prune_mask_ = 0;
    entry_cache_total_ = 0;
    rebuild_table(kMinSlots);  // small levels probe an L2-resident set again; it regrows with the search
    st_.constructed = 0;
    st_.unique = 0;
}

void Engine::read_counters() {
    CUDA_CHECK(cudaMemcpyAsync(h_counters_, d_counters_, CTR_COUNT * sizeof(u64), cudaMemcpyDeviceToHost, stream_));
    CUDA_CHECK(cudaStreamSynchronize(stream_));
    st_.d2h_bytes += CTR_COUNT * sizeof(u64);
}

// The counters of a level are final once level_summary_kernel has run; the kernel behind it (the scatter of the
// winners' rows, or the row directory of the wide path) changes none of them.  Reading them from a second stream
// that waits for the summary only lets the host plan and launch the next level while that kernel runs: the device
// then goes from one level to the next without waiting for the host's turn-around (~30 us a level).  Everything the
// host does to the cache afterwards is queued on stream_ and so stays ordered behind the scatter.
void Engine::read_counters_early() {
    CUDA_CHECK(cudaStreamWaitEvent(res_.copy, res_.summary, 0));
    CUDA_CHECK(cudaMemcpyAsync(h_counters_, d_counters_, CTR_COUNT * sizeof(u64), cudaMemcpyDeviceToHost, res_.copy));
    CUDA_CHECK(cudaStreamSynchronize(res_.copy));
    st_.d2h_bytes += CTR_COUNT * sizeof(u64);
}

// finalisation time of a level whose last kernel was still running when the host moved on
void Engine::collect_finalize_time(int slot, bool wait) {
    if (!fin_pending_[slot]) return;
    if (wait) CUDA_CHECK(cudaEventSynchronize(res_.fin[2 * slot + 1]));
    float ms = 0;
    if (cudaEventElapsedTime(&ms, res_.fin[2 * slot], res_.fin[2 * slot + 1]) == cudaSuccess) {
        st_.finalize_ms += ms;
        fin_pending_[slot] = false;
    } else {
        cudaGetLastError();
    }
}

// Canonical block order of one level (reference engine.py:219-266 without the chunking).
void Engine::plan_level(int cost, uint32_t op_mask, LevelMeta &lv, u64 &constructed, u64 &n_tiles) {
    constructed = 0;
    n_tiles = 0;
    // tile geometry: narrow = one lane per vector row; wide = one group of G lanes per vector row
    const u64 tile_v = (u64)TILE_V;
    const u64 tile_s_max = wide_ ? (u64)wide2_tile_s(nvec_, lw_ == LW_REGEX) : (u64)TILE_S;
    const u64 tile_max = (u64)TILE_V * TILE_S;  // candidates of a full-size tile
    // A block is cut into at least ~4 tiles per resident warp so that small levels still
    // spread over the whole GPU instead of a few warps grinding through full-size tiles.
    const u64 want_tiles = (u64)sm_count_ * occupancy_ * WARPS_PER_CTA * 4;
    // ... but not below ~1024 candidates (8 probe batches) while that still leaves every warp a
    // tile: a ticket costs a global atomic, and the first ncu capture of mid-size levels had 28 %
    // of its stall samples waiting on one ticket per 256 candidates.
    const u64 resident_warps = (u64)sm_count_ * occupancy_ * WARPS_PER_CTA;
    auto tile_candidates = [&](u64 size) {
        const u64 floor_per = wide_ ? tile_v * 4 : std::max<u64>(tile_v * 4, std::min<u64>(1024, size / resident_warps));
        u64 per = std::max<u64>(size / want_tiles, floor_per);
        return std::min<u64>(next_pow2(per), tile_max);
    };
    auto ceil_div = [](u64 a, u64 b) { return (a + b - 1) / b; };
    auto push = [&](BlockDesc b) {
        if (b.size == 0) return;
        const u64 per = tile_candidates(b.size);
        if (b.kind == BK_UNARY) {
            b.tile_s = (uint32_t)std::min<u64>(std::max<u64>(per / tile_v, 4), UNARY_ITEMS);
            b.vg = 1;
            b.tiles_v = ceil_div(b.na, tile_v * b.tile_s);
            b.tiles_s = 1;
        } else {
            const u64 n_vec = b.vec_is_b ? b.nb : b.na, n_sc = b.vec_is_b ? b.na : b.nb;
            b.tile_s = (uint32_t)std::min<u64>(std::max<u64>(per / tile_v, 4), std::min(tile_s_max, n_sc));
            b.tiles_s = ceil_div(n_sc, b.tile_s);
            // few scalar rows per tile: widen the tile over several groups of vector rows
            b.vg = (uint32_t)std::min<u64>(256, std::max<u64>(1, per / (tile_v * b.tile_s)));
            b.tiles_v = ceil_div(n_vec, tile_v * b.vg);
        }
        b.ord0 = constructed;
        b.tile0 = n_tiles;
        constructed += b.size;
        n_tiles += b.tiles_v * b.tiles_s;
        lv.blocks.push_back(b);
    };
    // weights_[tag] = cost of one node of that operator ([0] = an atom); all 1 in the reference, where the lines
    // below read "atoms at cost 1, unary over level cost - 1, binary over c1 + c2 = cost - 1" (engine.py:219-266)
    const int *w = weights_;
    if (cost == w[OP_ATOM]) {
        BlockDesc b{};
        b.op = OP_ATOM;
        b.kind = BK_UNARY;
        b.from_atoms = 1;
        b.na = (u64)n_atoms_;
        b.size = b.na;
        push(b);
    }
    // (the regex operators -- question, star unary; concatenation, non-commutative, before union = OP_OR -- are only
    // ever enabled on a handle with the regex grammar, where none of the LTL tags is)
    static const int unary_tags[6] = {OP_NOT, OP_NEXT, OP_FUTURE, OP_GLOBALLY, OP_RE_QUESTION, OP_RE_STAR};
    static const int binary_tags[4] = {OP_AND, OP_UNTIL, OP_RE_CONCAT, OP_OR};
    for (int tag : unary_tags) {
        if (!(op_mask >> tag & 1u) || cost - w[tag] < 1) continue;
        const LevelMeta &prev = levels_[cost - w[tag] - 1];
        if (prev.n == 0) continue;
        BlockDesc b{};
        b.op = (uint32_t)tag;
        b.kind = BK_UNARY;
        b.a_off = prev.base;
        b.na = prev.n;
        b.size = prev.n;
        push(b);
    }
    for (int tag : binary_tags) {
        if (!(op_mask >> tag & 1u)) continue;
        const bool commutative = tag == OP_AND || tag == OP_OR;
        for (int c1 = 1; c1 < cost - w[tag]; ++c1) {
            const int c2 = cost - w[tag] - c1;
            if (commutative && c1 > c2) break;
            const LevelMeta &la = levels_[c1 - 1], &lb = levels_[c2 - 1];
            if (la.n == 0 || lb.n == 0) continue;
            BlockDesc b{};
            b.op = (uint32_t)tag;
            b.a_off = la.base;
            b.na = la.n;
            b.b_off = lb.base;
            b.nb = lb.n;
            if (commutative && c1 == c2) {
                b.kind = BK_TRI;
                b.vec_is_b = 1;
                b.size = la.n * (la.n + 1) / 2;
            } else {
                b.kind = BK_RECT;
                b.vec_is_b = lb.n >= la.n;
                b.size = la.n * lb.n;
            }
            b.c_left = (uint32_t)c1;
            if (tag == OP_AND && !wide_) {
                // left operand rows that are AND nodes; right operand rows that are AND nodes whose left child
                // costs less than c1 (AND blocks of a level are contiguous, in ascending order of their left cost)
                auto and_range = [](const LevelMeta &lv, uint32_t left_cost_below, u64 &lo, u64 &hi) {
                    lo = hi = 0;
                    bool any = false;
                    for (const BlockDesc &q : lv.blocks) {
                        if (q.op != (uint32_t)OP_AND || q.c_left >= left_cost_below) continue;
                        if (!any) lo = q.ord0;
                        hi = q.ord0 + q.size;
                        any = true;
                    }
                };
                and_range(la, ~0u, b.skip_a_lo, b.skip_a_hi);
                and_range(lb, (uint32_t)c1, b.skip_b_lo, b.skip_b_hi);
            }
            push(b);
        }
    }
    if ((int)lv.blocks.size() > kMaxBlocks) throw std::invalid_argument("too many operand blocks in one level");
}

// ordinal (within a triangle block over n rows) of the first pair of row i: sum of the row lengths n, n-1, ...
static u64 tri_row_start(u64 n, u64 i) { return i * n - (i ? (i * (i - 1)) / 2 : 0); }

// provenance of an entry from the ordinal it won with (engine.py:274-327)
void Engine::decode(const LevelMeta &lv, u64 ord, int32_t *op, int64_t *left, int64_t *right) const {
    size_t bi = 0;
    while (bi + 1 < lv.blocks.size() && ord >= lv.blocks[bi + 1].ord0) ++bi;
    const BlockDesc &b = lv.blocks[bi];
    const u64 k = ord - b.ord0;
    *op = (int32_t)b.op;
    if (b.kind == BK_UNARY) {
        *left = (int64_t)(b.from_atoms ? k : b.a_off + k);
        *right = -1;
    } else if (b.kind == BK_RECT) {
        *left = (int64_t)(b.a_off + k / b.nb);
        *right = (int64_t)(b.b_off + k % b.nb);
    } else {
        // row i of the triangle starts at i*n - i(i-1)/2; invert with a float guess + exact fix-up
        const u64 n = b.na;
        long double fn = (long double)(2 * n + 1);
        long double disc = fn * fn - 8.0L * (long double)k;
        u64 i = (u64)((fn - sqrtl(disc > 0 ? disc : 0)) / 2.0L);
        if (i >= n) i = n - 1;
        while (i > 0 && tri_row_start(n, i) > k) --i;
        while (i + 1 < n && tri_row_start(n, i + 1) <= k) ++i;
        const u64 j = i + (k - tri_row_start(n, i));
        *left = (int64_t)(b.a_off + i);
        *right = (int64_t)(b.a_off + j);
    }
}

// `stats.constructed` increment of a level cut short at the separator: the reference
// adds whole chunks (engine.py:418) and stops after the separator's chunk (:445-446),
// so the count is "everything up to the end of the chunk that holds sep_ord" under the
// chunk schedule of _tasks_for_level (:219-266) for this batch size.
u64 Engine::constructed_through(const LevelMeta &lv, u64 sep_ord, u64 batch) const {
    size_t bi = 0;
    while (bi + 1 < lv.blocks.size() && sep_ord >= lv.blocks[bi + 1].ord0) ++bi;
    const BlockDesc &b = lv.blocks[bi];
    const u64 k = sep_ord - b.ord0;
    u64 end;  // candidates of this block covered by chunks up to the separator's
    if (b.kind == BK_UNARY) {
        end = b.from_atoms ? b.size : std::min(b.size, (k / batch + 1) * batch);
    } else if (b.kind == BK_RECT) {
        const u64 rows = batch / b.nb, i = k / b.nb, j = k % b.nb;
        if (rows >= 1) end = std::min(b.na, (i / rows + 1) * rows) * b.nb;
        else end = i * b.nb + std::min(b.nb, (j / batch + 1) * batch);
    } else {
        const u64 n = b.na;
        int32_t op;
        int64_t l, r;
        decode(lv, sep_ord, &op, &l, &r);
        const u64 i = (u64)l - b.a_off, j = (u64)r - b.a_off;
        if (n - i > batch) {  // a long row is split over j on its own (trij chunks)
            end = tri_row_start(n, i) + std::min(n - i, ((j - i) / batch + 1) * batch);
        } else {  // greedy groups of whole rows with at most `batch` pairs
            u64 i0 = n > batch ? n - batch : 0;
            for (;;) {
                u64 pairs = 0, i1 = i0;
                while (i1 < n && pairs + (n - i1) <= batch) {
                    pairs += n - i1;
                    ++i1;
                }
                if (i < i1) {
                    end = i1 < n ? tri_row_start(n, i1) : b.size;
                    break;
                }
                i0 = i1;
            }
        }
    }
    return b.ord0 + end;
}

// Exhaustive mode: from the ordinals of ALL separating candidates of the level, pick what
// the reference's chunked merge loop reports -- walk the chunks in order, look only at each
// chunk's first separating candidate, and take the first of those that is fresh, i.e. that
// won its CM (bit set in the winners bitmap).  Leaves the result in counters[CTR_SEP].
u64 Engine::chunk_exact_separator(const LevelMeta &lv, std::vector<u64> &seps, u64 batch) {
    reserve(sep_list_, seps.size() + 1, false);
    std::sort(seps.begin(), seps.end());
    std::vector<u64> firsts;
    u64 chunk_end = 0;
    for (u64 o : seps) {
        if (o < chunk_end) continue;  // not the first separating candidate of its chunk
        firsts.push_back(o);
        chunk_end = constructed_through(lv, o, batch);
    }
    const u64 none = VAL_EMPTY;
    CUDA_CHECK(cudaMemcpyAsync(d_counters_ + CTR_SEP, &none, sizeof(u64), cudaMemcpyHostToDevice, stream_));
    CUDA_CHECK(cudaMemcpyAsync(sep_list_.ptr, firsts.data(), firsts.size() * sizeof(u64), cudaMemcpyHostToDevice, stream_));
    st_.h2d_bytes += firsts.size() * sizeof(u64);
    first_fresh_kernel<<<(unsigned)((firsts.size() + 255) / 256), 256, 0, stream_>>>(bitmap_.ptr, sep_list_.ptr, firsts.size(), d_counters_);
    CUDA_CHECK(cudaGetLastError());
    CUDA_CHECK(cudaStreamSynchronize(stream_));  // `firsts` must outlive the copy
    st_.kernel_launches++;
    return firsts.size();
}

// One launch per operator, in canonical operator order (blocks of a level are grouped by
// operator already); each launch covers all (c1, c2) blocks of its operator.
template <typename Params, typename Launch>
static void for_each_operator(Params P, const LevelMeta &lv, int sm_count, int occupancy, Launch launch) {
    size_t b0 = 0;
    int group = 0;
    while (b0 < lv.blocks.size()) {
        size_t b1 = b0;
        while (b1 < lv.blocks.size() && lv.blocks[b1].op == lv.blocks[b0].op) ++b1;
        const BlockDesc &last = lv.blocks[b1 - 1];
        P.block_begin = (int)b0;
        P.block_end = (int)b1;
        P.tile_begin = lv.blocks[b0].tile0;
        P.tile_end = last.tile0 + last.tiles_v * last.tiles_s;
        P.ticket = CTR_TICKET0 + group;
        const int grid = (int)std::min<u64>((P.tile_end - P.tile_begin + WARPS_PER_CTA - 1) / WARPS_PER_CTA, (u64)sm_count * occupancy);
        DBG("launch op=%d blocks=[%zu,%zu) tiles=[%llu,%llu) grid=%d", (int)lv.blocks[b0].op, b0, b1, (unsigned long long)P.tile_begin, (unsigned long long)P.tile_end, grid);
        launch((int)lv.blocks[b0].op, P, grid, group);
        if (debug_on()) {
            CUDA_CHECK(cudaDeviceSynchronize());
            DBG("  done");
        }
        b0 = b1;
        ++group;
    }
}

// levels up to this many candidates take the one-launch kernel (narrow_small_level_kernel)
static constexpr u64 kSmallLevel = 1ull << 19;

// LTLB200_OPSTREAMS=0: every operator launch of a level on the engine's own stream, one after the other
static bool fan_enabled() {
    static const bool on = [] {
        const char *e = getenv("LTLB200_OPSTREAMS");
        return !(e && e[0] == '0');
    }();
    return on;
}

void Engine::fan_begin() {
    side_used_ = 0;
    if (fan_enabled()) CUDA_CHECK(cudaEventRecord(fork_ev_, stream_));
}

// stream of the level's `group`-th operator launch: the first stays on the engine's stream, the others
// start on a side stream once everything queued before the fan-out (level init, memsets) is done
cudaStream_t Engine::fan_stream(int group) {
    if (group == 0 || !fan_enabled()) return stream_;
    const int k = (group - 1) % kSideStreams;
    if (!(side_used_ >> k & 1u)) {
        CUDA_CHECK(cudaStreamWaitEvent(side_[k], fork_ev_, 0));
        side_used_ |= 1u << k;
    }
    return side_[k];
}

// the engine's stream continues (finalisation, counters read-back) after every side stream has drained
void Engine::fan_end() {
    for (int k = 0; k < kSideStreams; ++k) {
        if (!(side_used_ >> k & 1u)) continue;
        CUDA_CHECK(cudaEventRecord(join_ev_[k], side_[k]));
        CUDA_CHECK(cudaStreamWaitEvent(stream_, join_ev_[k], 0));
    }
    side_used_ = 0;
}

void Engine::launch_narrow(int kind, int op, const NarrowParams &P, int grid, cudaStream_t st) {
    switch (lw_) {
        case 8: narrow_launch_8(kind, op, P, grid, st); break;
        case 16: narrow_launch_16(kind, op, P, grid, st); break;
        case 32: narrow_launch_32(kind, op, P, grid, st); break;
        default: narrow_launch_64(kind, op, P, grid, st); break;
    }
    CUDA_CHECK(cudaGetLastError());
    st_.kernel_launches++;
    st_.enumerate_launches++;
}

void Engine::launch_wide(int kind, int op, const WideParams &P, int grid, cudaStream_t st) {
    const size_t smem = wide2_warp_vecs(nvec_, lw_ == LW_REGEX) * sizeof(uint4) * WARPS_PER_CTA + (size_t)guide_smem_words_ * sizeof(uint32_t);
    switch (lw_) {
        case LW_REGEX: wide2_launch_1(kind, op, P, grid, smem, device_, st); break;
        case 8: wide2_launch_8(kind, op, P, grid, smem, device_, st); break;
        case 16: wide2_launch_16(kind, op, P, grid, smem, device_, st); break;
        case 32: wide2_launch_32(kind, op, P, grid, smem, device_, st); break;
        default: wide2_launch_64(kind, op, P, grid, smem, device_, st); break;
    }
    CUDA_CHECK(cudaGetLastError());
    st_.kernel_launches++;
    st_.enumerate_launches++;
}

// Small levels and the rare guarded mode (collect_dead_ranges) take ONE launch for every operator;
// big levels one launch per operator, fanned out over the side streams.
template <typename Params>
void Engine::launch_level(Params P, const LevelMeta &lv) {
    constexpr bool kWide = std::is_same<Params, WideParams>::value;
    const BlockDesc &last = lv.blocks.back();
    const u64 level_candidates = last.ord0 + last.size;
    const bool guarded = P.scan_only || P.dead_n;
    const bool route = P.route_rows != nullptr;  // sharded search: one launch per operator, whatever the size
    if (!route && (guarded || level_candidates <= kSmallLevel)) {
        P.block_begin = 0;
        P.block_end = (int)lv.blocks.size();
        P.tile_begin = 0;
        P.tile_end = last.tile0 + last.tiles_v * last.tiles_s;
        P.ticket = CTR_TICKET0;
        const int grid = (int)std::min<u64>((P.tile_end + WARPS_PER_CTA - 1) / WARPS_PER_CTA, (u64)sm_count_ * 2);
        if constexpr (kWide) launch_wide(guarded ? LK_GUARDED : LK_SMALL, 0, P, grid, stream_);
        else launch_narrow(guarded ? LK_GUARDED : LK_SMALL, 0, P, grid, stream_);
        return;
    }
    fan_begin();
    for_each_operator(P, lv, sm_count_, occupancy_, [&](int op, const Params &Q, int grid, int group) {
        cudaStream_t st = fan_stream(group);
        if constexpr (kWide) launch_wide(route ? LK_ROUTE : LK_OPERATOR, op, Q, grid, st);
        else launch_narrow(route ? LK_ROUTE : LK_OPERATOR, op, Q, grid, st);
    });
    fan_end();
}

void Engine::launch_enumerate(NarrowParams P, const LevelMeta &lv) { launch_level(P, lv); }
void Engine::launch_enumerate_wide(WideParams P, const LevelMeta &lv) { launch_level(P, lv); }

// ---- one level = begin (enumerate this rank's shard) [+ exchange] + end (finalise) ---------

// Enumerates the tiles of level `cost` that belong to shard `shard_index` of `shard_count`
// (tile-strided) into the local hash set.  Nothing is appended yet; level_end() does that.
// `defer` (single-GPU, non-exhaustive, narrow): do not wait for the enumeration -- level_end launches
// the finalisation right behind it with device-side bounds and synchronises once for both.
// Scan pass of a non-exhaustive level over a store that already holds a separating CM.  The reference cuts every
// chunk at its FIRST separating candidate, fresh or not (engine.py:330-335), and goes on with the next chunk
// until a fresh one ends the level (:425-446): whatever follows such a candidate inside its chunk does not
// exist for this level.  Here: every separating ordinal is recorded without touching the set, the host walks
// them chunk by chunk (constructed_through = end of the chunk that holds an ordinal) and the tails become
// the dead ranges of the enumeration that follows.
void Engine::collect_dead_ranges(const LevelMeta &lv, u64 constructed, u64 batch) {
    dead_n_ = 0;
    u64 want = std::max<u64>(1ull << 20, constructed / 16), n = 0;
    for (;;) {
        reserve(sep_list_, want, false);
        level_init_kernel<<<1, 32, 0, stream_>>>(d_counters_, time_left_ns());
        CUDA_CHECK(cudaGetLastError());
        if (wide_) {
            WideParams Q = wide_params(false);
            Q.scan_only = 1;
            Q.prune_after_sep = 0;
            Q.sep_list = sep_list_.ptr;
            Q.sep_list_cap = sep_list_.cap;
            launch_enumerate_wide(Q, lv);
        } else {
            NarrowParams Q = narrow_params(false);
            Q.scan_only = 1;
            Q.prune_after_sep = 0;
            Q.sep_list = sep_list_.ptr;
            Q.sep_list_cap = sep_list_.cap;
            Q.ords = nullptr;
            launch_enumerate(Q, lv);
        }
        read_counters();
        n = h_counters_[CTR_SEPCOUNT];
        if (n <= sep_list_.cap) break;
        want = n;
    }
    if (n == 0) return;
    std::vector<u64> seps((size_t)n);
    CUDA_CHECK(cudaMemcpyAsync(seps.data(), sep_list_.ptr, n * sizeof(u64), cudaMemcpyDeviceToHost, stream_));
    CUDA_CHECK(cudaStreamSynchronize(stream_));
    st_.d2h_bytes += n * sizeof(u64);
    std::sort(seps.begin(), seps.end());
    std::vector<u64> ranges;
    u64 chunk_end = 0;
    for (u64 o : seps) {
        if (o < chunk_end) continue;  // not the first separating candidate of its chunk
        chunk_end = constructed_through(lv, o, batch);
        if (o + 1 < chunk_end) {
            ranges.push_back(o + 1);
            ranges.push_back(chunk_end);
        }
    }
    if (ranges.empty()) return;
    reserve(dead_, ranges.size(), false);
    CUDA_CHECK(cudaMemcpyAsync(dead_.ptr, ranges.data(), ranges.size() * sizeof(u64), cudaMemcpyHostToDevice, stream_));
    CUDA_CHECK(cudaStreamSynchronize(stream_));  // `ranges` must outlive the copy
    st_.h2d_bytes += ranges.size() * sizeof(u64);
    dead_n_ = ranges.size() / 2;
}

int Engine::level_begin(int cost, uint32_t op_mask, bool exhaustive, double deadline, u64 *n_claimed_out, u64 *sep_ord_out,
                        u64 *n_seps_out, bool defer) {
    if (pending_.active) throw std::invalid_argument("level_begin: the previous level was not ended");
    if (cost != (int)levels_.size() + 1) throw std::invalid_argument("cost must be the next unbuilt level");
    CUDA_CHECK(cudaSetDevice(device_));
    set_sharding(1, 0);  // a level built by one handle needs the whole set
    deadline_ = deadline;
    pending_ = PendingLevel{};
    PendingLevel &pl = pending_;
    pl.lv.base = total_;
    pl.exhaustive = exhaustive;
    pl.cost = cost;
    *n_claimed_out = 0;
    *sep_ord_out = VAL_EMPTY;
    *n_seps_out = 0;
    if (deadline >= 0 && monotonic_s() > deadline) {  // engine.py:416-417, before the first chunk
        prune_ok_ = false;
        levels_.push_back(pl.lv);
        return LTLB200_TIME_BUDGET;
    }
    if (prune_mask_ == 0) prune_mask_ = op_mask;
    else if (prune_mask_ != op_mask) prune_ok_ = false;  // (see prune_ok_)
    u64 n_tiles = 0;
    double tp = monotonic_s();
    plan_level(cost, op_mask, pl.lv, pl.constructed, n_tiles);
    PHASE(0, "begin: plan", tp);
    pl.active = true;
    if (pl.constructed == 0) return LTLB200_OK;
    const LevelMeta &lv = pl.lv;
    const u64 constructed = pl.constructed;
    try {
        if (table_dirty_) rebuild_table(table_slots());
        CUDA_CHECK(cudaMemcpyAsync(d_blocks_, lv.blocks.data(), lv.blocks.size() * sizeof(BlockDesc), cudaMemcpyHostToDevice, stream_));
        st_.h2d_bytes += lv.blocks.size() * sizeof(BlockDesc);
        dead_n_ = 0;
        if (!exhaustive && store_has_separator_ && mode_batch_ > 0) {
            // The dead ranges delete candidates -- among them the smaller-ordinal witnesses x & (y & r) that the
            // associativity pruning of AND blocks relies on -- and leave this level incomplete: no pruning here
            // nor in any later level of this store.
            prune_ok_ = false;
            collect_dead_ranges(lv, constructed, (u64)mode_batch_);
            defer = false;  // (rare mode: the plain two-synchronisation path)
        }

        // expected number of new CMs: everything for small levels, else the previous level's
        // uniqueness with head-room; a wrong guess trips the overflow flag and the level is redone
        const u64 kExact = 1ull << 22, kSlack = 1ull << 21;
        u64 est = constructed;
        if (constructed > kExact) {
            double u = 1.0;
            // (head-room x1.5 over the previous level's uniqueness; x1.2 for levels of more than 2^28 candidates, whose
            // staging is tens of GB -- uniqueness moves by a few per cent from level to level, and a wrong guess is redone)
            const double head = constructed > (1ull << 28) ? 1.2 : 1.5;
            if (levels_.size() >= 2 && last_constructed_ > 0) u = std::min(1.0, head * (double)levels_.back().n / (double)last_constructed_ + 0.02);
            // LTLB200_EST_SCALE (tests): scales the guess so that the overflow -> regrow -> redo path runs
            static const double scale = [] {
                const char *e = getenv("LTLB200_EST_SCALE");
                return e ? atof(e) : 1.0;
            }();
            est = std::min(constructed, std::max(kExact, (u64)(scale * u * (double)constructed)));
        }
        for (int attempt = 0;; ++attempt) {
            const bool exact = est >= constructed;
            // staging / claim capacity: the estimate plus what warps may over-reserve in flight
            // (wide: every group of every operator launch may end with a partly used chunk of staging entries)
            const u64 wide_slack = (u64)sm_count_ * occupancy_ * WARPS_PER_CTA * std::max<u64>((u64)(32 >> log2g_) * WIDE_CHUNK, CLAIM_CHUNK) * 8 + 1024;
            // (narrow: every warp of every operator launch may end with a partly used chunk of claim indices)
            // (a small level is one launch of at most 2 CTAs per SM: narrow_small_level_kernel)
            const u64 narrow_slack = constructed <= kSmallLevel
                                         ? (u64)sm_count_ * 2 * WARPS_PER_CTA * CLAIM_CHUNK + 1024
                                         : (u64)sm_count_ * occupancy_ * WARPS_PER_CTA * CLAIM_CHUNK * 8 + 1024;
            const u64 claim_cap = est + (wide_ ? wide_slack : narrow_slack);
            // the set is sized for the CMs it can receive (est; exact for small levels, and beyond est the
            // claim arrays overflow first because est >= kExact > their slack), not for the claim slack:
            // small levels then probe a set that stays in the L2
            const u64 want_slots = next_pow2(2 * (total_ + est));
            DBG("level %d attempt %d: constructed=%llu est=%llu claim_cap=%llu slots=%llu want=%llu", cost, attempt, (unsigned long long)constructed, (unsigned long long)est, (unsigned long long)claim_cap, (unsigned long long)table_slots(), (unsigned long long)want_slots);
            if (want_slots > table_slots()) rebuild_table(grown_size(want_slots));
            if (exhaustive) reserve(sep_list_, std::max<u64>(std::max<u64>(1ull << 20, constructed / 16), sep_want_), false);
            // counters start at zero (CTR_SEP at "none"); the special-key register persists across levels
            level_init_kernel<<<1, 32, 0, stream_>>>(d_counters_, time_left_ns());
            CUDA_CHECK(cudaGetLastError());
            pl.claim_cap = claim_cap;
            if (wide_) {
                reserve(store_, (log_tail_ + claim_cap) * nvec_, true, log_tail_ * nvec_);  // new rows are staged at the log's tail
                reserve(stage_ord_, claim_cap, false);
                CUDA_CHECK(cudaMemsetAsync(stage_ord_.ptr, 0xFF, claim_cap * sizeof(u64), stream_));
                WideParams P = wide_params(exhaustive);
                CUDA_CHECK(cudaEventRecord(ev_[0], stream_));
                launch_enumerate_wide(P, lv);
            } else {
                reserve(claim_key_, claim_cap, false);
                reserve(claim_ord_, claim_cap, false);
                CUDA_CHECK(cudaMemsetAsync(claim_ord_.ptr, 0xFF, claim_cap * sizeof(u64), stream_));
                NarrowParams P = narrow_params(exhaustive);
                PHASE(1, "begin: setup (copies, memsets)", tp);
                CUDA_CHECK(cudaEventRecord(ev_[0], stream_));
                launch_enumerate(P, lv);
            }
            CUDA_CHECK(cudaEventRecord(ev_[1], stream_));
            PHASE(2, "begin: launches", tp);
            if (defer) {
                pl.deferred = true;
                st_.enumerate_candidates += constructed;
                return LTLB200_OK;
            }
            read_counters();
            PHASE(3, "begin: sync + read counters", tp);
            float ms = 0;
            CUDA_CHECK(cudaEventElapsedTime(&ms, ev_[0], ev_[1]));
            st_.enumerate_ms += ms;
            st_.enumerate_candidates += constructed;
            if (exhaustive && h_counters_[CTR_OVERFLOW] == 0 && h_counters_[CTR_SEPCOUNT] > sep_list_.cap) {
                // more separating candidates than the list holds: the chunk-exact separator needs all of them
                sep_want_ = h_counters_[CTR_SEPCOUNT] + 1024;
                if (attempt > 8) throw CudaError("separator list keeps overflowing");
                rebuild_table(table_slots());  // drops this attempt's claims
                continue;
            }
            if (h_counters_[CTR_OVERFLOW] == 0) break;
            if (attempt > 8 || (exact && !wide_)) throw CudaError("hash set overflow on an exactly sized table");
            est = std::min(constructed, est * 4);
            rebuild_table(next_pow2(2 * (total_ + est + kSlack)));  // drops this attempt's claims
        }
    } catch (const MemoryBudget &e) {
        g_last_error = e.what();
        table_dirty_ = true;
        pl.active = false;
        prune_ok_ = false;
        levels_.push_back(LevelMeta{0, total_, {}});
        return LTLB200_MEMORY_BUDGET;
    }
    DBG("level %d enumerated: claimed=%llu sep=%llx", cost, (unsigned long long)h_counters_[CTR_CLAIMED], (unsigned long long)h_counters_[CTR_SEP]);
    pl.n_claimed = h_counters_[CTR_CLAIMED];  // narrow: claimed slots; wide: reserved staging entries
    pl.sep_ord = h_counters_[CTR_SEP];
    if (pl.sep_ord != VAL_EMPTY || h_counters_[CTR_SEPCOUNT]) store_has_separator_ = true;
    pl.n_seps = std::min<u64>(h_counters_[CTR_SEPCOUNT], sep_list_.cap);
    pl.seps_overflow = h_counters_[CTR_SEPCOUNT] > sep_list_.cap;
    *n_claimed_out = pl.n_claimed;
    *sep_ord_out = pl.sep_ord;
    *n_seps_out = pl.n_seps;
    return LTLB200_OK;
}

NarrowParams Engine::narrow_params(bool exhaustive) const {
    NarrowParams P{};
    P.store = store_.ptr;
    P.atoms = d_atoms_;
    P.slots = slots_.ptr;
    P.slot_mask = slots_.cap - 1;
    P.claim_key = claim_key_.ptr;
    P.claim_ord = claim_ord_.ptr;
    P.claim_cap = pending_.claim_cap;
    P.epoch = (u64)pending_.cost << EPOCH_SHIFT;
    P.counters = d_counters_;
    P.blocks = d_blocks_;
    P.valid = valid_;
    P.target = target_;
    P.prune_after_sep = exhaustive ? 0 : 1;
    P.special_possible = special_possible_ ? 1 : 0;
    P.sep_list = exhaustive ? sep_list_.ptr : nullptr;
    P.sep_list_cap = exhaustive ? sep_list_.cap : 0;
    P.shard_stride = 1;
    P.shard_offset = 0;
    static const bool prune_on = [] {  // LTLB200_PRUNE=0: every AND candidate is probed
        const char *e = getenv("LTLB200_PRUNE");
        return !(e && e[0] == '0');
    }();
    P.ords = prune_on && prune_ok_ && total_ ? ords_.ptr : nullptr;
    P.dead = dead_n_ ? dead_.ptr : nullptr;
    P.dead_n = (uint32_t)dead_n_;
    P.scan_only = 0;
    return P;
}

WideParams Engine::wide_params(bool exhaustive) const {
    WideParams P{};
    P.store = store_.ptr;
    P.atoms = d_atoms_;
    P.slots = wslots_.ptr;
    P.slot_mask = wslots_.cap - 1;
    P.loc = loc_.ptr;
    P.stage_rows = store_.ptr + log_tail_ * nvec_;
    P.stage_ord = stage_ord_.ptr;
    P.stage_cap = pending_.claim_cap;
    P.total_before = log_tail_;
    P.counters = d_counters_;
    P.blocks = d_blocks_;
    P.valid = d_valid_;
    P.target = d_target_;
    P.nvec = nvec_;
    P.log2g = log2g_;
    P.prune_after_sep = exhaustive ? 0 : 1;
    P.sep_list = exhaustive ? sep_list_.ptr : nullptr;
    P.sep_list_cap = exhaustive ? sep_list_.cap : 0;
    P.shard_stride = 1;
    P.shard_offset = 0;
    P.dead = dead_n_ ? dead_.ptr : nullptr;
    P.dead_n = (uint32_t)dead_n_;
    P.scan_only = 0;
    P.guide = guide_.ptr;
    P.n_bits = n_bits_;
    P.guide_smem_words = guide_smem_words_;
    P.guide_entries = guide_entries_;
    P.guide_rounds = guide_rounds_;
    return P;
}

// Finalises the pending level.  `sep_ord` = smallest ordinal of a fresh separating candidate
// over ALL shards (all ones = none); `seps` = every separating ordinal of the level (exhaustive
// runs; NULL = use what this handle recorded itself).
int Engine::level_end(u64 sep_ord, const u64 *seps, u64 n_seps, int64_t batch, u64 mem_budget, int64_t *n_new,
                      int64_t *sep_gid, int64_t *constructed_delta) {
    if (pending_.routed) throw std::invalid_argument("level_end on a routed level (level_commit ends it)");
    return finalize_level(sep_ord, seps, n_seps, batch, mem_budget, n_new, sep_gid, constructed_delta, false, 0);
}

// `global_bitmap`: the winners bitmap already holds the marks of every owner (sharded search: owner_reduce marked,
// the ranks all-reduced); this owner's claims are placed as usual and `n_received` records published by the other
// owners (exchange_recv buffers) are placed by the rank of their ordinals.
int Engine::finalize_level(u64 sep_ord, const u64 *seps, u64 n_seps, int64_t batch, u64 mem_budget, int64_t *n_new,
                           int64_t *sep_gid, int64_t *constructed_delta, bool global_bitmap, u64 n_received) {
    if (!pending_.active) throw std::invalid_argument("level_end without level_begin");
    if (batch < 1) throw std::invalid_argument("batch_size must be >= 1");
    if (sep_ord != VAL_EMPTY || n_seps) store_has_separator_ = true;  // found by another shard
    CUDA_CHECK(cudaSetDevice(device_));
    PendingLevel &pl = pending_;
    LevelMeta &lv = pl.lv;
    const bool exhaustive = pl.exhaustive;
    const u64 constructed = pl.constructed;
    *n_new = 0;
    *sep_gid = -1;
    *constructed_delta = 0;
    pl.active = false;
    if (constructed == 0) {
        levels_.push_back(lv);
        return LTLB200_OK;
    }
    double tp = monotonic_s();
    if (pl.deferred) return level_end_deferred(batch, mem_budget, n_new, sep_gid, constructed_delta);
    try {
        const u64 n_claimed = std::min(h_counters_[CTR_CLAIMED], pl.claim_cap);
        const bool cut = !exhaustive && sep_ord != VAL_EMPTY;
        const u64 n_bits = cut ? sep_ord + 1 : constructed;
        const u64 n_words = (n_bits + 31) / 32, n_sb = (n_words + 31) / 32;
        reserve(bitmap_, n_words + 1, false);
        reserve(sb_rank_, n_sb + 1, false);
        if (wide_) {  // the staged rows stay where they are; received rows are appended behind them
            reserve(store_, (log_tail_ + n_claimed + n_received) * nvec_, true, (log_tail_ + n_claimed) * nvec_);
            reserve(loc_, total_ + n_claimed + n_received, true, total_);
        } else {
            reserve(store_, (total_ + n_claimed + n_received) * nvec_, true, total_ * nvec_);
        }
        reserve(ords_, total_ + n_claimed + n_received, true, total_);
        CUDA_CHECK(cudaEventRecord(ev_[2], stream_));
        if (!global_bitmap) CUDA_CHECK(cudaMemsetAsync(bitmap_.ptr, 0, (n_words + 1) * sizeof(uint32_t), stream_));
        CUDA_CHECK(cudaMemcpyAsync(d_counters_ + CTR_SEP, &sep_ord, sizeof(u64), cudaMemcpyHostToDevice, stream_));
        const u64 ord_limit = cut ? sep_ord : VAL_EMPTY - 1;
        FinalizeParams F{};
        WideFinalize W{};
        const int fgrid = (int)std::max<u64>(1, std::min<u64>((n_claimed + 255) / 256, (u64)sm_count_ * 16));
        if (wide_) {
            W.stage_ord = stage_ord_.ptr;
            W.n_staged = std::min(n_claimed, pl.claim_cap);
            W.bitmap = bitmap_.ptr;
            W.sb_rank = sb_rank_.ptr;
            W.ord_limit = ord_limit;
            W.loc = loc_.ptr;
            W.ords = ords_.ptr;
            W.base = total_;
            W.log_base = log_tail_;
            if (!global_bitmap) wide_mark_kernel<<<fgrid, 256, 0, stream_>>>(W);
        } else {
            F.claim_key = claim_key_.ptr;
            F.claim_ord = claim_ord_.ptr;
            F.n_claimed = std::min(n_claimed, pl.claim_cap);
            F.bitmap = bitmap_.ptr;
            F.sb_rank = sb_rank_.ptr;
            F.ord_limit = ord_limit;
            F.store = store_.ptr;
            F.ords = ords_.ptr;
            F.base = total_;
            if (!global_bitmap) narrow_mark_kernel<<<fgrid, 256, 0, stream_>>>(F);
        }
        CUDA_CHECK(cudaGetLastError());
        launch_rank_scan(n_words, n_sb);
        // exhaustive runs: the reference reports, per level, the first CHUNK whose first
        // separating candidate is fresh (engine.py:331,425-433); reproduce that exactly
        if (exhaustive) {
            std::vector<u64> all;
            if (seps) all.assign(seps, seps + n_seps);
            else if (pl.n_seps && !pl.seps_overflow) {
                all.resize((size_t)pl.n_seps);
                CUDA_CHECK(cudaMemcpyAsync(all.data(), sep_list_.ptr, pl.n_seps * sizeof(u64), cudaMemcpyDeviceToHost, stream_));
                CUDA_CHECK(cudaStreamSynchronize(stream_));
                st_.d2h_bytes += pl.n_seps * sizeof(u64);
            }
            if (!all.empty()) chunk_exact_separator(lv, all, (u64)batch);
        }
        level_summary_kernel<<<1, 1, 0, stream_>>>(bitmap_.ptr, sb_rank_.ptr, n_bits, d_counters_);
        if (wide_) {
            wide_rank_kernel<<<fgrid, 256, 0, stream_>>>(W);
        } else {
            narrow_scatter_kernel<<<fgrid, 256, 0, stream_>>>(F);
        }
        CUDA_CHECK(cudaGetLastError());
        if (n_received) {  // what the other owners published
            const u64 work = sources_.longest * (u64)sources_.n * (u64)(wide_ ? nvec_ : 1);
            const int rgrid = (int)std::max<u64>(1, std::min<u64>((work + 255) / 256, (u64)sm_count_ * 16));
            if (wide_) wide_append_records_kernel<<<rgrid, 256, 0, stream_>>>(xr_rows_.ptr, xr_ords_.ptr, sources_, nvec_, bitmap_.ptr, sb_rank_.ptr, store_.ptr, log_tail_ + n_claimed, loc_.ptr, ords_.ptr, total_);
            else narrow_scatter_records_kernel<<<rgrid, 256, 0, stream_>>>(xr_rows_.ptr, xr_ords_.ptr, sources_, bitmap_.ptr, sb_rank_.ptr, store_.ptr, ords_.ptr, total_);
            CUDA_CHECK(cudaGetLastError());
            st_.kernel_launches++;
        }
        CUDA_CHECK(cudaEventRecord(ev_[3], stream_));
        st_.kernel_launches += 3;
        PHASE(5, "end: reserve + launches", tp);
        read_counters();
        PHASE(6, "end: sync + read counters", tp);
        float fms = 0;
        CUDA_CHECK(cudaEventElapsedTime(&fms, ev_[2], ev_[3]));
        st_.finalize_ms += fms;
        recycle_retired(false);  // the stream has drained: blocks retired by regrows can be reused
        lv.n = h_counters_[CTR_WINNERS];
        if (global_bitmap && lv.n != pl.n_winners + n_received)
            throw CudaError("sharded level: the winners bitmap holds " + std::to_string(lv.n) + " entries, the owners published " +
                            std::to_string(pl.n_winners + n_received));
        if (wide_) log_tail_ += n_claimed + n_received;  // (unused and cut-off staging entries stay behind as dead log entries)
        sep_ord = h_counters_[CTR_SEP];
        if (sep_ord != VAL_EMPTY) *sep_gid = (int64_t)(total_ + h_counters_[CTR_SEPRANK]);
        if (cut) table_dirty_ = true;  // claims ordered after the separator stay flagged in the set
    } catch (const MemoryBudget &e) {
        g_last_error = e.what();
        table_dirty_ = true;
        prune_ok_ = false;
        levels_.push_back(LevelMeta{0, total_, {}});
        return LTLB200_MEMORY_BUDGET;
    }
    const bool found_cut = !exhaustive && sep_ord != VAL_EMPTY;
    if (found_cut) prune_ok_ = false;  // the level keeps only what precedes its separator: no longer complete
    *constructed_delta = (int64_t)(found_cut ? constructed_through(lv, sep_ord, (u64)batch) : constructed);
    last_constructed_ = constructed;
    *n_new = (int64_t)lv.n;
    total_ += lv.n;
    st_.constructed += (u64)*constructed_delta;
    st_.unique = total_;
    approx_bytes_ += lv.n * ((u64)row_bytes_ + (u64)key_words_ * 8 + 80);  // engine.py:442
    levels_.push_back(std::move(lv));
    PHASE(7, "end: bookkeeping", tp);
    if (h_counters_[CTR_TIMEOUT]) {  // the deadline passed while the level was being built: it holds what was built
        prune_ok_ = false;           // until then (the reference's partial level, engine.py:416-417 + 447-449)
        return LTLB200_TIME_BUDGET;
    }
    if (mem_budget && approx_bytes_ > mem_budget) return LTLB200_MEMORY_BUDGET;  // engine.py:443-444
    return LTLB200_OK;
}

// popcount prefix per 1024-bit superblock of the winners bitmap: up to three scan levels of 1024
void Engine::launch_rank_scan(u64 n_words, u64 n_sb) {
        {
    const u64 nb1 = (n_sb + 1023) / 1024;
    reserve(scan_tmp_, 2 * (nb1 + 1024) + 2048, false);
    uint32_t *sums1 = scan_tmp_.ptr, *pre1 = sums1 + nb1 + 8;
    sb_scan_kernel<<<(unsigned)nb1, 1024, 0, stream_>>>(bitmap_.ptr, n_words, nullptr, sb_rank_.ptr, n_sb, sums1);
    CUDA_CHECK(cudaGetLastError());
    st_.kernel_launches++;
    if (nb1 > 1) {
        const u64 nb2 = (nb1 + 1023) / 1024;
        uint32_t *sums2 = pre1 + nb1 + 8, *pre2 = sums2 + nb2 + 8;
        sb_scan_kernel<<<(unsigned)nb2, 1024, 0, stream_>>>(nullptr, 0, sums1, pre1, nb1, sums2);
        if (nb2 > 1) {
            if (nb2 > 1024) throw std::invalid_argument("level too large for the rank scan");
            sb_scan_kernel<<<1, 1024, 0, stream_>>>(nullptr, 0, sums2, pre2, nb2, nullptr);
            sb_add_kernel<<<(unsigned)nb2, 1024, 0, stream_>>>(pre1, nb1, pre2);
            st_.kernel_launches += 2;
        }
        sb_add_kernel<<<(unsigned)nb1, 1024, 0, stream_>>>(sb_rank_.ptr, n_sb, pre1);
        CUDA_CHECK(cudaGetLastError());
        st_.kernel_launches += 2;
    }
}
}

// Finalisation launched right behind the enumeration (see level_begin's `defer`): every bound the
// host would have read from the counters is resolved on the device, and the one synchronisation
// at the end serves both phases.  Returns kRetryLevel when the enumeration overflowed.
int Engine::level_end_deferred(int64_t batch, u64 mem_budget, int64_t *n_new, int64_t *sep_gid, int64_t *constructed_delta) {
    PendingLevel &pl = pending_;
    LevelMeta &lv = pl.lv;
    const u64 constructed = pl.constructed;
    const bool exhaustive = pl.exhaustive;
    double tp = monotonic_s();
    u64 sep_ord = VAL_EMPTY;
    try {
        const u64 n_bits = constructed;
        const u64 n_words = (n_bits + 31) / 32, n_sb = (n_words + 31) / 32;
        const bool small = n_bits <= SMALL_FIN_MAX_BITS;  // bitmap in shared memory, one launch
        if (!small || exhaustive) {
            reserve(bitmap_, n_sb * 32 + 1, false);
            reserve(sb_rank_, n_sb + 1, false);
        }
        if (wide_) reserve(loc_, total_ + pl.claim_cap, true, total_);  // (the rows are in the log already)
        else reserve(store_, (total_ + pl.claim_cap) * nvec_, true, total_ * nvec_);
        reserve(ords_, total_ + pl.claim_cap, true, total_);
        static const bool early_on = [] {  // LTLB200_EARLY_COUNTERS=0: one full synchronisation per level
            const char *e = getenv("LTLB200_EARLY_COUNTERS");
            return !(e && e[0] == '0');
        }();
        const bool early = early_on && !small;  // (a small level is one kernel: nothing to overlap)
        const int slot = fin_slot_;
        if (early) collect_finalize_time(slot, true);  // (two levels back: long finished)
        CUDA_CHECK(cudaEventRecord(early ? res_.fin[2 * slot] : ev_[2], stream_));
        // the grids are sized by what the level can have claimed at most (its candidates, or the claim arrays)
        const u64 claim_bound = std::min(constructed + (u64)sm_count_ * occupancy_ * WARPS_PER_CTA * CLAIM_CHUNK * 8, pl.claim_cap);
        const int fgrid = (int)std::max<u64>(1, std::min<u64>((claim_bound + 255) / 256, (u64)sm_count_ * 16));
        if (wide_) {
            WideFinalize W{};
            W.stage_ord = stage_ord_.ptr;
            W.bitmap = bitmap_.ptr;
            W.sb_rank = sb_rank_.ptr;
            W.loc = loc_.ptr;
            W.ords = ords_.ptr;
            W.base = total_;
            W.log_base = log_tail_;
            W.live = d_counters_;
            W.stage_cap = pl.claim_cap;
            W.cut_allowed = exhaustive ? 0 : 1;
            if (small) {
                const size_t smem = (size_t)n_sb * 32 * sizeof(uint32_t) + (size_t)n_sb * sizeof(uint32_t);
                small_finalize_kernel<WideFinalize><<<1, SMALL_FIN_THREADS, smem, stream_>>>(W, n_bits, d_counters_, exhaustive ? 1 : 0);
                CUDA_CHECK(cudaGetLastError());
                st_.kernel_launches++;
            } else {
                CUDA_CHECK(cudaMemsetAsync(bitmap_.ptr, 0, (n_words + 1) * sizeof(uint32_t), stream_));
                wide_mark_kernel<<<fgrid, 256, 0, stream_>>>(W);
                CUDA_CHECK(cudaGetLastError());
                launch_rank_scan(n_words, n_sb);
                level_summary_kernel<<<1, 1, 0, stream_>>>(bitmap_.ptr, sb_rank_.ptr, n_bits, d_counters_);
                if (early) CUDA_CHECK(cudaEventRecord(res_.summary, stream_));
                wide_rank_kernel<<<fgrid, 256, 0, stream_>>>(W);
                CUDA_CHECK(cudaGetLastError());
                st_.kernel_launches += 3;
            }
        } else {
            FinalizeParams F{};
            F.claim_key = claim_key_.ptr;
            F.claim_ord = claim_ord_.ptr;
            F.bitmap = bitmap_.ptr;
            F.sb_rank = sb_rank_.ptr;
            F.store = store_.ptr;
            F.ords = ords_.ptr;
            F.base = total_;
            F.live = d_counters_;
            F.claim_cap = pl.claim_cap;
            F.cut_allowed = exhaustive ? 0 : 1;
            if (small) {
                const size_t smem = (size_t)n_sb * 32 * sizeof(uint32_t) + (size_t)n_sb * sizeof(uint32_t);
                small_finalize_kernel<FinalizeParams><<<1, SMALL_FIN_THREADS, smem, stream_>>>(F, n_bits, d_counters_, exhaustive ? 1 : 0);
                CUDA_CHECK(cudaGetLastError());
                st_.kernel_launches++;
            } else {
                CUDA_CHECK(cudaMemsetAsync(bitmap_.ptr, 0, (n_words + 1) * sizeof(uint32_t), stream_));
                narrow_mark_kernel<<<fgrid, 256, 0, stream_>>>(F);
                CUDA_CHECK(cudaGetLastError());
                launch_rank_scan(n_words, n_sb);
                level_summary_kernel<<<1, 1, 0, stream_>>>(bitmap_.ptr, sb_rank_.ptr, n_bits, d_counters_);
                if (early) CUDA_CHECK(cudaEventRecord(res_.summary, stream_));
                narrow_scatter_kernel<<<fgrid, 256, 0, stream_>>>(F);
                CUDA_CHECK(cudaGetLastError());
                st_.kernel_launches += 3;
            }
        }
        CUDA_CHECK(cudaEventRecord(early ? res_.fin[2 * slot + 1] : ev_[3], stream_));
        PHASE(5, "end: reserve + launches", tp);
        if (early) read_counters_early();
        else read_counters();
        PHASE(6, "end: sync + read counters", tp);
        float ms = 0;
        CUDA_CHECK(cudaEventElapsedTime(&ms, ev_[0], ev_[1]));
        st_.enumerate_ms += ms;
        if (early) {
            fin_pending_[slot] = true;
            collect_finalize_time(slot ^ 1, false);  // the previous level's: its last kernel ran before this level's first
            fin_slot_ ^= 1;
        } else {
            CUDA_CHECK(cudaEventElapsedTime(&ms, ev_[2], ev_[3]));
            st_.finalize_ms += ms;
        }
        // (blocks retired during this level were last touched by work queued before the summary kernel)
        recycle_retired(false);
        pl.active = false;
        if (h_counters_[CTR_OVERFLOW]) {  // the guess of new CMs was too small: nothing was finalised
            table_dirty_ = true;
            return kRetryLevel;
        }
        if (exhaustive && h_counters_[CTR_SEPCOUNT] > sep_list_.cap) {  // redo with a list that holds them all
            sep_want_ = h_counters_[CTR_SEPCOUNT] + 1024;
            table_dirty_ = true;
            return kRetryLevel;
        }
        lv.n = h_counters_[CTR_WINNERS];
        if (wide_) log_tail_ += std::min(h_counters_[CTR_CLAIMED], pl.claim_cap);
        sep_ord = h_counters_[CTR_SEP];
        if (sep_ord != VAL_EMPTY || h_counters_[CTR_SEPCOUNT]) store_has_separator_ = true;
        if (exhaustive && h_counters_[CTR_SEPCOUNT]) {
            // the reference reports, per level, the first CHUNK whose first separating candidate is fresh
            // (engine.py:331,425-433): walk the recorded ordinals against the winners bitmap (one more round trip,
            // only on levels that contain a separating candidate at all)
            const u64 n_seps = std::min<u64>(h_counters_[CTR_SEPCOUNT], sep_list_.cap);
            std::vector<u64> all;
            if (h_counters_[CTR_SEPCOUNT] <= sep_list_.cap) {
                all.resize((size_t)n_seps);
                CUDA_CHECK(cudaMemcpyAsync(all.data(), sep_list_.ptr, n_seps * sizeof(u64), cudaMemcpyDeviceToHost, stream_));
                CUDA_CHECK(cudaStreamSynchronize(stream_));
                st_.d2h_bytes += n_seps * sizeof(u64);
            }
            if (!all.empty()) {
                chunk_exact_separator(lv, all, (u64)batch);
                level_summary_kernel<<<1, 1, 0, stream_>>>(bitmap_.ptr, sb_rank_.ptr, n_bits, d_counters_);
                CUDA_CHECK(cudaGetLastError());
                st_.kernel_launches++;
                read_counters();
                sep_ord = h_counters_[CTR_SEP];
            }
        }
        if (sep_ord != VAL_EMPTY) {
            *sep_gid = (int64_t)(total_ + h_counters_[CTR_SEPRANK]);
            if (!exhaustive) table_dirty_ = true;  // claims ordered after the separator stay flagged in the set
        }
    } catch (const MemoryBudget &e) {
        g_last_error = e.what();
        table_dirty_ = true;
        pl.active = false;
        prune_ok_ = false;
        levels_.push_back(LevelMeta{0, total_, {}});
        return LTLB200_MEMORY_BUDGET;
    }
    const bool found_cut = !exhaustive && sep_ord != VAL_EMPTY;
    if (found_cut) prune_ok_ = false;  // the level keeps only what precedes its separator: no longer complete
    *constructed_delta = (int64_t)(found_cut ? constructed_through(lv, sep_ord, (u64)batch) : constructed);
    last_constructed_ = constructed;
    *n_new = (int64_t)lv.n;
    total_ += lv.n;
    st_.constructed += (u64)*constructed_delta;
    st_.unique = total_;
    approx_bytes_ += lv.n * ((u64)row_bytes_ + (u64)key_words_ * 8 + 80);  // engine.py:442
    levels_.push_back(std::move(lv));
    PHASE(7, "end: bookkeeping", tp);
    if (h_counters_[CTR_TIMEOUT]) {  // the deadline passed while the level was being built: it holds what was built
        prune_ok_ = false;           // until then (the reference's partial level, engine.py:416-417 + 447-449)
        return LTLB200_TIME_BUDGET;
    }
    if (mem_budget && approx_bytes_ > mem_budget) return LTLB200_MEMORY_BUDGET;  // engine.py:443-444
    return LTLB200_OK;
}

int Engine::expand_level(int cost, uint32_t op_mask, bool exhaustive, int64_t batch, u64 mem_budget, double deadline,
                         int64_t *n_new, int64_t *sep_gid, int64_t *constructed_delta) {
    if (batch < 1) throw std::invalid_argument("batch_size must be >= 1");
    *n_new = 0;
    *sep_gid = -1;
    *constructed_delta = 0;
    // levels the tiny-levels kernel built ahead (same operators, same mode), or a new run of it
    if (!lookahead_.empty() && (lookahead_.front().cost != cost || la_mask_ != op_mask || la_exhaustive_ != exhaustive)) discard_lookahead();
    if (lookahead_.empty() && tiny_eligible(cost, op_mask, exhaustive)) tiny_run(cost, op_mask, exhaustive);
    if (!lookahead_.empty()) return tiny_reveal(cost, op_mask, exhaustive, batch, mem_budget, deadline, n_new, sep_gid, constructed_delta);
    u64 n_claimed = 0, sep_ord = VAL_EMPTY, n_seps = 0;
    static const bool defer = getenv("LTLB200_NO_DEFER") == nullptr;
    mode_batch_ = batch;  // (collect_dead_ranges needs the reference's chunk schedule)
    int rc = level_begin(cost, op_mask, exhaustive, deadline, &n_claimed, &sep_ord, &n_seps, defer);
    if (rc != LTLB200_OK) {
        mode_batch_ = 0;
        return rc;
    }
    mode_batch_ = 0;
    rc = level_end(sep_ord, nullptr, 0, batch, mem_budget, n_new, sep_gid, constructed_delta);
    if (rc != kRetryLevel) return rc;
    mode_batch_ = batch;
    rc = level_begin(cost, op_mask, exhaustive, deadline, &n_claimed, &sep_ord, &n_seps, false);
    mode_batch_ = 0;
    if (rc != LTLB200_OK) return rc;
    return level_end(sep_ord, nullptr, 0, batch, mem_budget, n_new, sep_gid, constructed_delta);
}

// ---- tiny levels: several levels per launch (narrow_tiny.cuh) --------------------------------------------------

// LTLB200_TINY=0: every level through its own expand_level launches
static bool tiny_enabled() {
    static const bool on = [] {
        const char *e = getenv("LTLB200_TINY");
        return !(e && e[0] == '0');
    }();
    return on;
}

// One CTA beats the per-level launches only while a level is a few thousand candidates.  One-vector CMs: measured on
// spec2 / c3 with 1024 / 2048 / 4096 / 8192 / 32768 candidates -- 6.03 / 6.03 / 6.03 / 6.03 / 6.12 ms and 2.33 / 2.28 /
// 2.26 / 2.26 / 2.39 ms.  (A thread-block cluster of eight CTAs sharing CTA 0's counters and bitmap through distributed
// shared memory was built for the levels in between, 4 K - 64 K candidates: parity green, level 8 of spec2 125 -> 58 us,
// and still slower than handing those levels to the whole device -- spec2 6.09 ms, c3 2.54 ms; removed.)
static u64 narrow_tiny_max_candidates() {
    static const u64 n = [] {
        const char *e = getenv("LTLB200_TINY_MAX");
        return e ? (u64)atoll(e) : 4096ull;
    }();
    return std::min<u64>(n, TINY_MAX_CANDIDATES);
}

// multi-vector CMs: eight warps (LTLB200_WIDE_TINY_MAX)
static u64 wide_tiny_max_candidates() {
    static const u64 n = [] {
        const char *e = getenv("LTLB200_WIDE_TINY_MAX");
        return e ? (u64)atoll(e) : 4096ull;
    }();
    return std::min<u64>(n, TINY_MAX_CANDIDATES);
}

bool Engine::tiny_eligible(int cost, uint32_t op_mask, bool exhaustive) {
    if (!tiny_enabled() || tiny_off_ || pending_.active || cost != (int)levels_.size() + 1 || cost > 60) return false;
    if (!exhaustive && store_has_separator_) return false;  // the chunk-truncation regime (collect_dead_ranges)
    LevelMeta lv;
    u64 constructed = 0, n_tiles = 0;
    plan_level(cost, op_mask, lv, constructed, n_tiles);
    const u64 slots = std::max<u64>(table_slots(), kMinSlots);
    return constructed <= (wide_ ? wide_tiny_max_candidates() : narrow_tiny_max_candidates()) && (int)lv.blocks.size() <= TINY_MAX_BLOCKS &&
           2 * (total_ + constructed) <= slots;
}

// Builds level `cost` and as many following levels as stay tiny, in one launch; queues their sizes.
void Engine::tiny_run(int cost, uint32_t op_mask, bool exhaustive) {
    CUDA_CHECK(cudaSetDevice(device_));
    set_sharding(1, 0);
    if (wide_) return tiny_run_wide(cost, op_mask, exhaustive);
    const u64 max_candidates = narrow_tiny_max_candidates();
    const u64 claim_cap = max_candidates + (u64)TINY_WARPS * CLAIM_CHUNK + 1024;
    const u64 growth = 4 * max_candidates;  // what one launch may add to the cache (the kernel stops before)
    try {
        if (table_dirty_) rebuild_table(table_slots());
        reserve(claim_key_, claim_cap, false);
        reserve(claim_ord_, claim_cap, false);
        reserve(store_, total_ + growth, true, total_);
        reserve(ords_, total_ + growth, true, total_);
        reserve(tiny_tab_, 2 * 128, false);
        reserve(tiny_results_, 5 * (TINY_MAX_LEVELS + 1), false);
    } catch (const MemoryBudget &) {
        return;  // (the usual path reports the memory budget)
    }
    std::vector<u64> tab(2 * 128, 0);
    for (size_t c = 1; c <= levels_.size(); ++c) {
        tab[2 * c] = levels_[c - 1].n;
        tab[2 * c + 1] = levels_[c - 1].base;
    }
    CUDA_CHECK(cudaMemcpyAsync(tiny_tab_.ptr, tab.data(), tab.size() * sizeof(u64), cudaMemcpyHostToDevice, stream_));
    CUDA_CHECK(cudaMemsetAsync(tiny_results_.ptr, 0, 5 * (TINY_MAX_LEVELS + 1) * sizeof(u64), stream_));
    CUDA_CHECK(cudaMemsetAsync(claim_ord_.ptr, 0xFF, claim_cap * sizeof(u64), stream_));
    st_.h2d_bytes += tab.size() * sizeof(u64);
    pending_ = PendingLevel{};
    pending_.claim_cap = claim_cap;
    pending_.cost = cost;
    TinyParams T{};
    T.P = narrow_params(exhaustive);
    T.P.ords = nullptr;  // (no associativity pruning here: it needs the block lists of the stored levels)
    T.P.sep_list = exhaustive ? d_counters_ : nullptr;  // capacity 0: separating candidates are only counted
    T.P.sep_list_cap = 0;
    T.store = store_.ptr;
    T.store_ords = ords_.ptr;
    T.level_tab = tiny_tab_.ptr;
    T.results = reinterpret_cast<TinyLevelResult *>(tiny_results_.ptr);
    T.total = total_;
    T.table_slots = table_slots();
    T.max_candidates = max_candidates;
    T.store_cap = total_ + growth;
    T.op_mask = op_mask;
    T.n_atoms = n_atoms_;
    T.cost_first = cost;
    T.cost_last = std::min(cost + TINY_MAX_LEVELS - 1, 62);
    T.exhaustive = exhaustive ? 1 : 0;
    for (int k = 0; k < 16; ++k) T.weights[k] = weights_[k];
    CUDA_CHECK(cudaEventRecord(ev_[0], stream_));
    switch (lw_) {
        case 8: narrow_tiny_8(T, device_, stream_); break;
        case 16: narrow_tiny_16(T, device_, stream_); break;
        case 32: narrow_tiny_32(T, device_, stream_); break;
        default: narrow_tiny_64(T, device_, stream_); break;
    }
    CUDA_CHECK(cudaGetLastError());
    CUDA_CHECK(cudaEventRecord(ev_[1], stream_));
    std::vector<u64> res(5 * (TINY_MAX_LEVELS + 1));
    CUDA_CHECK(cudaMemcpyAsync(res.data(), tiny_results_.ptr, res.size() * sizeof(u64), cudaMemcpyDeviceToHost, stream_));
    CUDA_CHECK(cudaStreamSynchronize(stream_));
    st_.d2h_bytes += res.size() * sizeof(u64);
    st_.kernel_launches++;
    float ms = 0;
    CUDA_CHECK(cudaEventElapsedTime(&ms, ev_[0], ev_[1]));
    st_.tiny_ms += ms;
    recycle_retired(false);
    const int asked = T.cost_last - T.cost_first + 1;
    int built = 0;
    while (built < asked && res[5 * built] == TINY_BUILT) {
        lookahead_.push_back(Lookahead{cost + built, res[5 * built + 1], res[5 * built + 2], res[5 * built + 3], 0});
        DBG("tiny level %d: %llu new, %.1f us", cost + built, (unsigned long long)res[5 * built + 1], 1e-3 * (double)res[5 * built + 4]);
        ++built;
    }
    la_mask_ = op_mask;
    la_exhaustive_ = exhaustive;
    // a level the kernel started but left to the host (set / claim arrays too small, an exhaustive level with a
    // separating candidate) has its claims in the set: rebuild it from the cache before the next level
    const u64 why = res[5 * TINY_MAX_LEVELS];
    if (built < asked && why != TINY_END_BIG) table_dirty_ = true;
    // once an exhaustive search holds a separating CM, (nearly) every later level contains a separating candidate,
    // and each of them would be built here only to be handed to the host: stop trying on this store
    if (why == TINY_END_SEPARATOR) tiny_off_ = true;
    DBG("tiny levels: asked %d from cost %d, built %d (end reason %llu)", asked, cost, built, (unsigned long long)why);
}

// The same for multi-vector CMs (wide2_tiny.cuh): the levels' rows are staged at the tail of the row log, which the
// kernel moves on level by level; the host learns how far when it hands a level out.
void Engine::tiny_run_wide(int cost, uint32_t op_mask, bool exhaustive) {
    const bool regex = lw_ == LW_REGEX;
    // as many warps as fit the CTA's shared memory beside the kernel's static part
    const size_t per_warp = wide2_warp_vecs(nvec_, regex) * sizeof(uint4);
    const int warps = (int)std::min<size_t>(W2_TINY_MAX_WARPS, (kMaxDynamicSmem - 16 * 1024) / per_warp);
    if (warps < 2) return;
    const u64 claim_cap = (u64)TINY_MAX_CANDIDATES + (u64)warps * CLAIM_CHUNK + 1024;
    const u64 growth = 1ull << 17;  // log entries (and cache entries) one launch may add; the kernel stops before
    try {
        if (table_dirty_) rebuild_table(table_slots());
        reserve(stage_ord_, claim_cap, false);
        reserve(store_, (log_tail_ + growth) * nvec_, true, log_tail_ * nvec_);
        reserve(loc_, total_ + growth, true, total_);
        reserve(ords_, total_ + growth, true, total_);
        reserve(tiny_tab_, 2 * 128, false);
        reserve(tiny_results_, 6 * (TINY_MAX_LEVELS + 1), false);
    } catch (const MemoryBudget &) {
        return;  // (the usual path reports the memory budget)
    }
    std::vector<u64> tab(2 * 128, 0);
    for (size_t c = 1; c <= levels_.size(); ++c) {
        tab[2 * c] = levels_[c - 1].n;
        tab[2 * c + 1] = levels_[c - 1].base;
    }
    CUDA_CHECK(cudaMemcpyAsync(tiny_tab_.ptr, tab.data(), tab.size() * sizeof(u64), cudaMemcpyHostToDevice, stream_));
    CUDA_CHECK(cudaMemsetAsync(tiny_results_.ptr, 0, 6 * (TINY_MAX_LEVELS + 1) * sizeof(u64), stream_));
    CUDA_CHECK(cudaMemsetAsync(stage_ord_.ptr, 0xFF, claim_cap * sizeof(u64), stream_));
    st_.h2d_bytes += tab.size() * sizeof(u64);
    pending_ = PendingLevel{};
    pending_.claim_cap = claim_cap;
    pending_.cost = cost;
    WideTinyParams T{};
    T.P = wide_params(exhaustive);
    T.P.stage_cap = claim_cap;
    T.P.sep_list = exhaustive ? d_counters_ : nullptr;  // capacity 0: separating candidates are only counted
    T.P.sep_list_cap = 0;
    T.P.dead = nullptr;
    T.P.dead_n = 0;
    T.store = store_.ptr;
    T.loc = loc_.ptr;
    T.ords = ords_.ptr;
    T.level_tab = tiny_tab_.ptr;
    T.results = reinterpret_cast<WideTinyLevelResult *>(tiny_results_.ptr);
    T.total = total_;
    T.log_tail = log_tail_;
    T.log_cap = log_tail_ + growth;
    T.table_slots = table_slots();
    T.max_candidates = wide_tiny_max_candidates();
    T.op_mask = op_mask;
    T.n_atoms = n_atoms_;
    T.cost_first = cost;
    T.cost_last = std::min(cost + TINY_MAX_LEVELS - 1, 62);
    T.exhaustive = exhaustive ? 1 : 0;
    for (int k = 0; k < 16; ++k) T.weights[k] = weights_[k];
    const size_t smem = per_warp * (size_t)warps;
    CUDA_CHECK(cudaEventRecord(ev_[0], stream_));
    switch (lw_) {
        case LW_REGEX: wide2_tiny_1(T, warps, smem, device_, stream_); break;
        case 8: wide2_tiny_8(T, warps, smem, device_, stream_); break;
        case 16: wide2_tiny_16(T, warps, smem, device_, stream_); break;
        case 32: wide2_tiny_32(T, warps, smem, device_, stream_); break;
        default: wide2_tiny_64(T, warps, smem, device_, stream_); break;
    }
    CUDA_CHECK(cudaGetLastError());
    CUDA_CHECK(cudaEventRecord(ev_[1], stream_));
    std::vector<u64> res(6 * (TINY_MAX_LEVELS + 1));
    CUDA_CHECK(cudaMemcpyAsync(res.data(), tiny_results_.ptr, res.size() * sizeof(u64), cudaMemcpyDeviceToHost, stream_));
    CUDA_CHECK(cudaStreamSynchronize(stream_));
    st_.d2h_bytes += res.size() * sizeof(u64);
    st_.kernel_launches++;
    float ms = 0;
    CUDA_CHECK(cudaEventElapsedTime(&ms, ev_[0], ev_[1]));
    st_.tiny_ms += ms;
    recycle_retired(false);
    const int asked = T.cost_last - T.cost_first + 1;
    int built = 0;
    while (built < asked && res[6 * built] == TINY_BUILT) {
        lookahead_.push_back(Lookahead{cost + built, res[6 * built + 1], res[6 * built + 2], res[6 * built + 3], res[6 * built + 5]});
        DBG("tiny level %d: %llu new, %llu staged, %.1f us", cost + built, (unsigned long long)res[6 * built + 1],
            (unsigned long long)res[6 * built + 5], 1e-3 * (double)res[6 * built + 4]);
        ++built;
    }
    la_mask_ = op_mask;
    la_exhaustive_ = exhaustive;
    const u64 why = res[6 * TINY_MAX_LEVELS];
    if (built < asked && why != TINY_END_BIG) table_dirty_ = true;  // (see tiny_run)
    if (why == TINY_END_SEPARATOR) tiny_off_ = true;
    DBG("tiny levels (wide): asked %d from cost %d, built %d (end reason %llu)", asked, cost, built, (unsigned long long)why);
}

// Hands out the first queued level: the bookkeeping of level_end, with the block list replayed on the host.
int Engine::tiny_reveal(int cost, uint32_t op_mask, bool exhaustive, int64_t batch, u64 mem_budget, double deadline, int64_t *n_new,
                        int64_t *sep_gid, int64_t *constructed_delta) {
    if (deadline >= 0 && monotonic_s() > deadline) {  // engine.py:416-417, before the first chunk
        discard_lookahead();
        prune_ok_ = false;
        levels_.push_back(LevelMeta{0, total_, {}});
        return LTLB200_TIME_BUDGET;
    }
    const Lookahead la = lookahead_.front();
    lookahead_.pop_front();
    if (prune_mask_ == 0) prune_mask_ = op_mask;
    else if (prune_mask_ != op_mask) prune_ok_ = false;
    LevelMeta lv;
    lv.base = total_;
    u64 constructed = 0, n_tiles = 0;
    plan_level(cost, op_mask, lv, constructed, n_tiles);
    lv.n = la.n_new;
    const bool found_cut = !exhaustive && la.sep_ord != VAL_EMPTY;
    if (la.sep_ord != VAL_EMPTY) {
        store_has_separator_ = true;
        *sep_gid = (int64_t)(total_ + la.sep_rank);
    }
    if (found_cut) {
        prune_ok_ = false;    // the level keeps only what precedes its separator: no longer complete
        table_dirty_ = true;  // claims ordered after the separator stay flagged in the set
    }
    *constructed_delta = (int64_t)(found_cut ? constructed_through(lv, la.sep_ord, (u64)batch) : constructed);
    st_.enumerate_candidates += constructed;
    last_constructed_ = constructed;
    *n_new = (int64_t)lv.n;
    total_ += lv.n;
    log_tail_ += la.n_staged;  // (wide: unused and cut-off staging entries stay behind as dead log entries)
    st_.constructed += (u64)*constructed_delta;
    st_.unique = total_;
    approx_bytes_ += lv.n * ((u64)row_bytes_ + (u64)key_words_ * 8 + 80);  // engine.py:442
    levels_.push_back(std::move(lv));
    if (mem_budget && approx_bytes_ > mem_budget) return LTLB200_MEMORY_BUDGET;  // engine.py:443-444
    return LTLB200_OK;
}

// Levels built ahead that the caller does not want after all (other operators, another mode, a sharded level):
// their rows lie beyond total_ and are simply overwritten; their set entries go with a rebuild.
void Engine::discard_lookahead() {
    if (lookahead_.empty()) return;
    lookahead_.clear();
    table_dirty_ = true;
}

// ---- one search sharded over several GPUs ----------------------------------------------------------------------
//
// The language cache (rows + winning ordinals of every finished level) is replicated: any rank reads any operand.
// The dedup set is OWNER-SHARDED: rank r holds the CMs with hash owner r, of every level, so the set of an N-GPU
// search has N times the capacity and every rank probes 1/N of the candidates.  One level =
//
//   route_begin    build this rank's tile-strided share of the pair space; every candidate that is not a duplicate
//                  by construction goes, as a record {CM, ordinal}, to the send region of its owner (phase A)
//   [all-to-all]   the caller moves the regions (exchange_recv hands out the receive buffers)
//   owner_reduce   insert-or-min of the received records into the owned part of the set (phase B); marks the
//                  ordinals of this owner's winners in the level's bitmap
//   [all-reduce]   the caller sums the bitmaps (disjoint bits: a sum is the union); min of the separator
//   winners_export this owner's winners up to the separator as dense records, in ordinal order (so that what the
//                  other ranks receive goes to ascending ids)
//   [all-gather]   every rank receives the winners of the others (exchange_recv again)
//   level_commit   ranks of the global bitmap -> ids; own winners and received records appended to the cache
//
// Per rank: C/N candidates built, (K+8)C/N bytes out and in, C/N random probes, and the u*C new rows every replica
// of the cache has to store anyway.

void Engine::set_sharding(int world, int rank) {
    if (world == owner_world_ && rank == owner_rank_) return;
    owner_world_ = world;
    owner_rank_ = rank;
    table_dirty_ = true;  // the set is rebuilt with the CMs this rank owns now
}

int Engine::route_begin(int cost, uint32_t op_mask, bool exhaustive, double deadline, int rank, int world, u64 *send_counts,
                        u64 *send_offsets, void **rows_dev, void **ords_dev, u64 *sep_ord_out, u64 *n_seps_out) {
    if (pending_.active) throw std::invalid_argument("route_begin: the previous level was not ended");
    if (cost != (int)levels_.size() + 1) throw std::invalid_argument("cost must be the next unbuilt level");
    if (world < 1 || world > ROUTE_MAX_WORLD || rank < 0 || rank >= world) throw std::invalid_argument("bad shard (at most 8 ranks)");
    CUDA_CHECK(cudaSetDevice(device_));
    discard_lookahead();
    set_sharding(world, rank);
    deadline_ = deadline;
    pending_ = PendingLevel{};
    PendingLevel &pl = pending_;
    pl.lv.base = total_;
    pl.exhaustive = exhaustive;
    pl.cost = cost;
    pl.routed = true;
    for (int o = 0; o < world; ++o) send_counts[o] = send_offsets[o] = 0;
    *rows_dev = *ords_dev = nullptr;
    *sep_ord_out = VAL_EMPTY;
    *n_seps_out = 0;
    if (deadline >= 0 && monotonic_s() > deadline) {  // engine.py:416-417, before the first chunk
        prune_ok_ = false;
        levels_.push_back(pl.lv);
        return LTLB200_TIME_BUDGET;
    }
    if (!exhaustive && store_has_separator_)
        throw std::invalid_argument("a non-exhaustive level over a store that holds a separating CM follows the reference's chunk "
                                    "truncation: build it with ltlb200_expand_level on every rank");
    if (prune_mask_ == 0) prune_mask_ = op_mask;
    else if (prune_mask_ != op_mask) prune_ok_ = false;
    u64 n_tiles = 0;
    plan_level(cost, op_mask, pl.lv, pl.constructed, n_tiles);
    pl.active = true;
    if (pl.constructed == 0) return LTLB200_OK;
    const LevelMeta &lv = pl.lv;
    const u64 constructed = pl.constructed;
    std::vector<u64> counts((size_t)world, 0);
    try {
        if (table_dirty_) rebuild_table(table_slots());
        CUDA_CHECK(cudaMemcpyAsync(d_blocks_, lv.blocks.data(), lv.blocks.size() * sizeof(BlockDesc), cudaMemcpyHostToDevice, stream_));
        st_.h2d_bytes += lv.blocks.size() * sizeof(BlockDesc);
        dead_n_ = 0;
        reserve(xchg_, 16, false);
        // a rank builds ~1/world of the candidates and a uniform hash sends ~1/world of those to each owner; a
        // region that overflows is only counted, and the level is routed again with the exact sizes
        u64 cap = (u64)((double)(constructed / (u64)world + 1) / (double)world * 1.25) + (1ull << 16);
        cap = std::min(cap, constructed + 64);
        for (int attempt = 0;; ++attempt) {
            if (exhaustive) reserve(sep_list_, std::max<u64>(std::max<u64>(1ull << 20, constructed / 16), sep_want_), false);
            reserve(xs_rows_, (u64)world * cap * nvec_, false);
            reserve(xs_ords_, (u64)world * cap, false);
            level_init_kernel<<<1, 32, 0, stream_>>>(d_counters_, time_left_ns());
            CUDA_CHECK(cudaGetLastError());
            CUDA_CHECK(cudaMemsetAsync(xchg_.ptr, 0, 16 * sizeof(u64), stream_));
            pl.claim_cap = 0;
            CUDA_CHECK(cudaEventRecord(ev_[0], stream_));
            if (wide_) {
                WideParams P = wide_params(exhaustive);
                P.shard_stride = (u64)world;
                P.shard_offset = (u64)rank;
                P.route_rows = xs_rows_.ptr;
                P.route_ords = xs_ords_.ptr;
                P.route_cap = cap;
                P.route_counts = xchg_.ptr;
                P.route_world = (uint32_t)world;
                P.route_sep_any = store_has_separator_ ? 0 : 1;
                launch_enumerate_wide(P, lv);
            } else {
                NarrowParams P = narrow_params(exhaustive);
                P.shard_stride = (u64)world;
                P.shard_offset = (u64)rank;
                P.route_rows = xs_rows_.ptr;
                P.route_ords = xs_ords_.ptr;
                P.route_cap = cap;
                P.route_counts = xchg_.ptr;
                P.route_world = (uint32_t)world;
                P.route_sep_any = store_has_separator_ ? 0 : 1;
                launch_enumerate(P, lv);
            }
            CUDA_CHECK(cudaEventRecord(ev_[1], stream_));
            CUDA_CHECK(cudaMemcpyAsync(h_counters_ + CTR_COUNT, xchg_.ptr, (u64)world * sizeof(u64), cudaMemcpyDeviceToHost, stream_));
            read_counters();
            st_.d2h_bytes += (u64)world * sizeof(u64);
            float ms = 0;
            CUDA_CHECK(cudaEventElapsedTime(&ms, ev_[0], ev_[1]));
            st_.enumerate_ms += ms;
            st_.route_ms += ms;
            st_.enumerate_candidates += constructed / (u64)world;
            u64 need = 0;
            for (int o = 0; o < world; ++o) {
                counts[o] = h_counters_[CTR_COUNT + o];
                need = std::max(need, counts[o]);
            }
            if (attempt > 4) throw CudaError("route regions keep overflowing");
            if (need > cap) {
                cap = need + 1024;
                continue;
            }
            if (exhaustive && h_counters_[CTR_SEPCOUNT] > sep_list_.cap) {
                sep_want_ = h_counters_[CTR_SEPCOUNT] + 1024;
                continue;
            }
            break;
        }
        pl.region_cap = cap;
        if (h_counters_[CTR_TIMEOUT]) {  // the deadline passed while this rank was building its share: the level ends
            level_abort();               // empty here, and the caller tells the other ranks
            return LTLB200_TIME_BUDGET;
        }
    } catch (const MemoryBudget &e) {
        g_last_error = e.what();
        pl.active = false;
        prune_ok_ = false;
        levels_.push_back(LevelMeta{0, total_, {}});
        return LTLB200_MEMORY_BUDGET;
    }
    pl.sep_ord = h_counters_[CTR_SEP];
    pl.n_seps = h_counters_[CTR_SEPCOUNT];
    for (int o = 0; o < world; ++o) {
        st_.routed_records += counts[o];
        send_counts[o] = counts[o];
        send_offsets[o] = (u64)o * pl.region_cap;
    }
    *rows_dev = xs_rows_.ptr;
    *ords_dev = xs_ords_.ptr;
    *sep_ord_out = pl.sep_ord;
    *n_seps_out = pl.n_seps;
    return LTLB200_OK;
}

// receive buffers of the next exchange (records of the route phase, then the winners of the other owners)
void Engine::exchange_recv(u64 n_records, void **rows_dev, void **ords_dev) {
    if (!pending_.active || !pending_.routed) throw std::invalid_argument("exchange_recv outside a routed level");
    CUDA_CHECK(cudaSetDevice(device_));
    reserve(xr_rows_, std::max<u64>(n_records, 1) * nvec_, false);
    reserve(xr_ords_, std::max<u64>(n_records, 1), false);
    *rows_dev = xr_rows_.ptr;
    *ords_dev = xr_ords_.ptr;
}

// Phase B: the first `n_records` records of the receive buffers are folded into the owned part of the set; then
// the ordinals of this owner's winners are marked in the level's bitmap (one bit per candidate of the WHOLE level,
// so that the bitmaps of all owners add up to the level's winners).
int Engine::owner_reduce(u64 n_records, u64 *n_claimed_out, void **bitmap_dev, u64 *bitmap_words) {
    PendingLevel &pl = pending_;
    if (!pl.active || !pl.routed) throw std::invalid_argument("owner_reduce outside a routed level");
    CUDA_CHECK(cudaSetDevice(device_));
    *n_claimed_out = 0;
    *bitmap_dev = nullptr;
    *bitmap_words = 0;
    try {
    const u64 constructed = pl.constructed;
    const u64 n_words = (constructed + 31) / 32, n_sb = (n_words + 31) / 32;
    pl.n_received = n_records;
    st_.received_records += n_records;
    const u64 kExact = 1ull << 22, kSlack = 1ull << 21;
    u64 est = n_records;
    if (n_records > kExact) {
        double u = 1.0;
        if (levels_.size() >= 2 && last_constructed_ > 0) u = std::min(1.0, 1.5 * (double)levels_.back().n / (double)last_constructed_ + 0.02);
        est = std::min(n_records, std::max(kExact, (u64)(u * (double)n_records)));
    }
    const u64 owned = total_ / (u64)owner_world_ + total_ / (u64)(8 * owner_world_) + 1024;  // this rank's share of the stored CMs
    for (int attempt = 0;; ++attempt) {
        const u64 slack = wide_ ? (u64)sm_count_ * 8 * (u64)(CTA_THREADS >> log2g_) * WIDE_CHUNK + 1024
                                : (u64)sm_count_ * occupancy_ * WARPS_PER_CTA * CLAIM_CHUNK * 2 + 1024;
        const u64 claim_cap = est + slack;
        const u64 want_slots = next_pow2(2 * (owned + est));
        if (want_slots > table_slots()) rebuild_table(grown_size(want_slots));
        else if (table_dirty_) rebuild_table(table_slots());
        level_init_kernel<<<1, 32, 0, stream_>>>(d_counters_, time_left_ns());
        CUDA_CHECK(cudaGetLastError());
        pl.claim_cap = claim_cap;
        if (wide_) {
            reserve(store_, (log_tail_ + claim_cap) * nvec_, true, log_tail_ * nvec_);
            reserve(stage_ord_, claim_cap, false);
            CUDA_CHECK(cudaMemsetAsync(stage_ord_.ptr, 0xFF, claim_cap * sizeof(u64), stream_));
            CUDA_CHECK(cudaEventRecord(ev_[0], stream_));
            if (n_records) {
                WideParams P = wide_params(pl.exhaustive);
                P.sep_list = nullptr;
                P.sep_list_cap = 0;
                const u64 groups = (u64)(CTA_THREADS >> log2g_);
                const int grid = (int)std::max<u64>(1, std::min<u64>((n_records + groups - 1) / groups, (u64)sm_count_ * 8));
                wide_import_kernel<<<grid, CTA_THREADS, 0, stream_>>>(P, xr_rows_.ptr, xr_ords_.ptr, n_records);
                CUDA_CHECK(cudaGetLastError());
                st_.kernel_launches++;
            }
        } else {
            reserve(claim_key_, claim_cap, false);
            reserve(claim_ord_, claim_cap, false);
            CUDA_CHECK(cudaMemsetAsync(claim_ord_.ptr, 0xFF, claim_cap * sizeof(u64), stream_));
            CUDA_CHECK(cudaEventRecord(ev_[0], stream_));
            if (n_records) {
                NarrowParams P = narrow_params(pl.exhaustive);
                P.sep_list = nullptr;  // separating candidates were recorded where they were built
                P.sep_list_cap = 0;
                P.prune_after_sep = 0;
                const u64 steps = (n_records + 32 * PROBE_BATCH - 1) / (32 * PROBE_BATCH);
                const int grid = (int)std::max<u64>(1, std::min<u64>((steps + WARPS_PER_CTA - 1) / WARPS_PER_CTA, (u64)sm_count_ * LTLB200_PROBE_CTAS));
                switch (lw_) {
                    case 8: narrow_probe_8(P, xr_rows_.ptr, xr_ords_.ptr, n_records, grid, stream_); break;
                    case 16: narrow_probe_16(P, xr_rows_.ptr, xr_ords_.ptr, n_records, grid, stream_); break;
                    case 32: narrow_probe_32(P, xr_rows_.ptr, xr_ords_.ptr, n_records, grid, stream_); break;
                    default: narrow_probe_64(P, xr_rows_.ptr, xr_ords_.ptr, n_records, grid, stream_); break;
                }
                CUDA_CHECK(cudaGetLastError());
                st_.kernel_launches++;
            }
        }
        CUDA_CHECK(cudaEventRecord(ev_[1], stream_));
        read_counters();
        float ms = 0;
        CUDA_CHECK(cudaEventElapsedTime(&ms, ev_[0], ev_[1]));
        st_.enumerate_ms += ms;
        st_.probe_ms += ms;
        if (h_counters_[CTR_OVERFLOW] == 0) break;
        // the records are still in the receive buffers: regrow locally and fold them in again, no new exchange
        if (attempt > 8 || est >= n_records) throw CudaError("hash set overflow while folding in received records");
        est = std::min(n_records, est * 4);
        rebuild_table(next_pow2(2 * (owned + est + kSlack)));
    }
    const u64 n_claimed = std::min(h_counters_[CTR_CLAIMED], pl.claim_cap);
    pl.n_claimed = n_claimed;
    pl.reduced = true;
    reserve(bitmap_, n_words + 1, false);
    reserve(sb_rank_, n_sb + 1, false);
    CUDA_CHECK(cudaMemsetAsync(bitmap_.ptr, 0, (n_words + 1) * sizeof(uint32_t), stream_));
    if (n_claimed) {
        const int fgrid = (int)std::max<u64>(1, std::min<u64>((n_claimed + 255) / 256, (u64)sm_count_ * 16));
        if (wide_) {
            WideFinalize W{};
            W.stage_ord = stage_ord_.ptr;
            W.n_staged = n_claimed;
            W.bitmap = bitmap_.ptr;
            W.ord_limit = VAL_EMPTY - 1;
            wide_mark_kernel<<<fgrid, 256, 0, stream_>>>(W);
        } else {
            FinalizeParams F{};
            F.claim_ord = claim_ord_.ptr;
            F.n_claimed = n_claimed;
            F.bitmap = bitmap_.ptr;
            F.ord_limit = VAL_EMPTY - 1;
            narrow_mark_kernel<<<fgrid, 256, 0, stream_>>>(F);
        }
        CUDA_CHECK(cudaGetLastError());
        st_.kernel_launches++;
    }
    CUDA_CHECK(cudaStreamSynchronize(stream_));  // the caller's collective may run on another stream
    *n_claimed_out = n_claimed;
    *bitmap_dev = bitmap_.ptr;
    *bitmap_words = n_words + 1;
    } catch (const MemoryBudget &e) {  // the device is full: the level ends empty here; the caller tells the other ranks
        g_last_error = e.what();
        level_abort();
        return LTLB200_MEMORY_BUDGET;
    }
    return LTLB200_OK;
}

// Ends the pending level empty (another rank ran out of budget; every rank stops or none does).
void Engine::level_abort() {
    if (!pending_.active) return;
    pending_.active = false;
    table_dirty_ = true;
    prune_ok_ = false;
    levels_.push_back(LevelMeta{0, total_, {}});
}

// this owner's winners with an ordinal <= the level's separator (all of them in an exhaustive run), dense, in ordinal order
void Engine::winners_export(u64 sep_ord, u64 *n_winners, void **rows_dev, void **ords_dev) {
    PendingLevel &pl = pending_;
    if (!pl.active || !pl.reduced) throw std::invalid_argument("winners_export needs owner_reduce first");
    CUDA_CHECK(cudaSetDevice(device_));
    const bool cut = !pl.exhaustive && sep_ord != VAL_EMPTY;
    const u64 limit = cut ? sep_ord : VAL_EMPTY - 1;
    const u64 n = pl.n_claimed;
    reserve(xs_rows_, std::max<u64>(n, 1) * nvec_, false);
    reserve(xs_ords_, std::max<u64>(n, 1), false);
    CUDA_CHECK(cudaMemsetAsync(xchg_.ptr, 0, sizeof(u64), stream_));
    CUDA_CHECK(cudaEventRecord(ev_[2], stream_));
    if (n) {
        // the winners leave in ordinal order: their places are the ranks of their ordinals among this owner's own marks
        // (the bitmap is still the owner's: the ranks all-reduce it after this call, and level_commit ranks it again)
        const u64 n_words = (pl.constructed + 31) / 32, n_sb = (n_words + 31) / 32;
        launch_rank_scan(n_words, n_sb);
        const int grid = (int)std::max<u64>(1, std::min<u64>((n + 255) / 256, (u64)sm_count_ * 8));
        if (wide_) wide_winners_kernel<<<grid, 256, 0, stream_>>>(store_.ptr + log_tail_ * nvec_, stage_ord_.ptr, n, nvec_, limit, bitmap_.ptr, sb_rank_.ptr, xchg_.ptr, xs_rows_.ptr, xs_ords_.ptr);
        else narrow_winners_kernel<<<grid, 256, 0, stream_>>>(claim_key_.ptr, claim_ord_.ptr, n, limit, bitmap_.ptr, sb_rank_.ptr, xchg_.ptr, xs_rows_.ptr, xs_ords_.ptr);
        CUDA_CHECK(cudaGetLastError());
        st_.kernel_launches++;
    }
    CUDA_CHECK(cudaEventRecord(ev_[3], stream_));
    u64 count = 0;
    CUDA_CHECK(cudaMemcpyAsync(&count, xchg_.ptr, sizeof(u64), cudaMemcpyDeviceToHost, stream_));
    CUDA_CHECK(cudaStreamSynchronize(stream_));
    st_.d2h_bytes += sizeof(u64);
    float ms = 0;
    CUDA_CHECK(cudaEventElapsedTime(&ms, ev_[2], ev_[3]));
    st_.finalize_ms += ms;  // (publishing the winners is part of finalising a sharded level)
    pl.n_winners = count;
    *n_winners = count;
    *rows_dev = xs_rows_.ptr;
    *ords_dev = xs_ords_.ptr;
}

int Engine::level_commit(u64 sep_ord, const u64 *seps, u64 n_seps, const u64 *recv_counts, int n_sources, int64_t batch,
                         u64 mem_budget, int64_t *n_new, int64_t *sep_gid, int64_t *constructed_delta) {
    PendingLevel &pl = pending_;
    if (!pl.active || !pl.routed) throw std::invalid_argument("level_commit outside a routed level");
    if (pl.constructed && !pl.reduced) throw std::invalid_argument("level_commit needs owner_reduce and winners_export first");
    if (n_sources < 0 || n_sources > 8 || (n_sources && !recv_counts)) throw std::invalid_argument("level_commit: at most 8 sources");
    // the receive buffers hold the winners of the other owners source by source (dense)
    sources_ = RecordSources{};
    u64 n_received = 0;
    for (int k = 0; k < n_sources; ++k) {
        if (recv_counts[k] == 0) continue;
        sources_.offsets[sources_.n] = n_received;
        sources_.counts[sources_.n] = recv_counts[k];
        sources_.longest = std::max<u64>(sources_.longest, recv_counts[k]);
        sources_.n++;
        n_received += recv_counts[k];
    }
    // (counters as owner_reduce left them: CTR_CLAIMED = this owner's claims)
    return finalize_level(sep_ord, seps, n_seps, batch, mem_budget, n_new, sep_gid, constructed_delta, true, n_received);
}

// every separating ordinal this handle recorded in the pending level (exhaustive runs)
u64 Engine::seps_copy(u64 *out, u64 cap) {
    const u64 n = std::min(pending_.n_seps, cap);
    if (n) {
        CUDA_CHECK(cudaMemcpyAsync(out, sep_list_.ptr, n * sizeof(u64), cudaMemcpyDeviceToHost, stream_));
        CUDA_CHECK(cudaStreamSynchronize(stream_));
    }
    return n;
}

// candidates the next level would construct in full (the closed form of engine.py:219-266: sum of the block sizes)
int64_t Engine::level_candidates(int cost, uint32_t op_mask) {
    if (cost != (int)levels_.size() + 1) throw std::invalid_argument("cost must be the next unbuilt level");
    LevelMeta lv;
    u64 constructed = 0, n_tiles = 0;
    plan_level(cost, op_mask, lv, constructed, n_tiles);
    return (int64_t)constructed;
}

int Engine::level_info(int cost, int64_t *n, int64_t *base) const {
    if (cost < 1 || cost > (int)levels_.size()) return LTLB200_ERR_ARGUMENT;
    *n = (int64_t)levels_[cost - 1].n;
    *base = (int64_t)levels_[cost - 1].base;
    return LTLB200_OK;
}

int Engine::level_copy(int cost, int64_t first, int64_t count, uint8_t *cms, uint8_t *op, int64_t *left, int64_t *right) {
    if (cost < 1 || cost > (int)levels_.size()) return LTLB200_ERR_ARGUMENT;
    const LevelMeta &lv = levels_[cost - 1];
    if (first < 0 || count < 0 || (u64)(first + count) > lv.n) return LTLB200_ERR_ARGUMENT;
    if (count == 0) return LTLB200_OK;
    CUDA_CHECK(cudaSetDevice(device_));
    const u64 g0 = lv.base + (u64)first;
    if (cms) {
        std::vector<uint4> rows((size_t)count * nvec_);
        CUDA_CHECK(cudaMemcpyAsync(rows.data(), rows_in_id_order(g0, (u64)count), rows.size() * sizeof(uint4), cudaMemcpyDeviceToHost, stream_));
        CUDA_CHECK(cudaStreamSynchronize(stream_));
        st_.d2h_bytes += rows.size() * sizeof(uint4);
        for (int64_t k = 0; k < count; ++k) memcpy(cms + (size_t)k * row_bytes_, &rows[(size_t)k * nvec_], (size_t)row_bytes_);
    }
    if (op || left || right) {
        std::vector<u64> ords((size_t)count);
        CUDA_CHECK(cudaMemcpyAsync(ords.data(), ords_.ptr + g0, (size_t)count * sizeof(u64), cudaMemcpyDeviceToHost, stream_));
        CUDA_CHECK(cudaStreamSynchronize(stream_));
        st_.d2h_bytes += (u64)count * sizeof(u64);
        for (int64_t k = 0; k < count; ++k) {
            int32_t o;
            int64_t l, r;
            decode(lv, ords[(size_t)k], &o, &l, &r);
            if (op) op[k] = (uint8_t)o;
            if (left) left[k] = l;
            if (right) right[k] = r;
        }
    }
    return LTLB200_OK;
}

// The regex front-end (first slice): the handle was created with the CS bitsets as byte rows
// (masks = the bits of all example strings, target = the bits of the positives, atoms = the CSs of the empty word
// and of the letters); this switches its kernels to the regex operators and uploads the infix-split guide table.
void Engine::set_regex(int n_bits, const uint32_t *offsets, const uint32_t *entries, u64 n_entries) {
    if (!levels_.empty()) throw std::invalid_argument("the grammar must be set before the first level");
    // The regex operators live in the multi-vector kernels only (wide2_regex.cuh: two row areas of 32 rows per warp in
    // shared memory, 32 vectors = 4096 bits), so the rows must be wider than one uint4: short sequences are created
    // with zero lanes up to 17 bytes.  (A one-vector instantiation that walked the table per candidate existed; the
    // bit-sliced tiles are faster at every width: 111-bit sequences to cost 10, 3.8 -> 1.1 ms.)
    if (n_bits < 1 || n_bits > 4096 || lw_ != 8 || (n_bits + 7) / 8 > row_bytes_ || !wide_)
        throw std::invalid_argument("regex front-end: characteristic sequences of up to 4096 bits, created as max(17, ceil(bits / 8)) "
                                    "lanes of 8 bits");
    CUDA_CHECK(cudaSetDevice(device_));
    // device layout (wide2_regex.cuh: RegexGuide): the table as given (offsets | entries u | v << 16, sorted by the
    // result infix w) | w of every entry | the entries grouped by their LEFT part u (offsets | v | w << 16) | grouped
    // by their RIGHT part v (offsets | u | w << 16) | the entry offsets of the star's rounds.  A round holds the
    // infixes of one split depth: depth(w) = 1 + max depth(v) over the splits w = u v with u non-empty, which is the
    // length of w; the star of 32 rows at a time settles one round after the other.
    if (n_entries > 0xFFFFFFFFull / 8) throw std::invalid_argument("regex guide table: too many entries");
    const size_t nb1 = (size_t)n_bits + 1, E = (size_t)n_entries;
    if (offsets[0] != 0 || offsets[n_bits] != n_entries) throw std::invalid_argument("regex guide table: offsets do not span the entries");
    std::vector<uint32_t> w_of(E), depth(n_bits, 0), left_n(nb1, 0), right_n(nb1, 0);
    for (int w = 0; w < n_bits; ++w) {
        if (offsets[w] > offsets[w + 1]) throw std::invalid_argument("regex guide table: offsets are not ascending");
        for (uint32_t e = offsets[w]; e < offsets[w + 1]; ++e) {
            const uint32_t u = entries[e] & 0xFFFFu, v = entries[e] >> 16;
            if (u >= (uint32_t)n_bits || v >= (uint32_t)n_bits) throw std::invalid_argument("regex guide table: infix index out of range");
            w_of[e] = (uint32_t)w;
            left_n[u + 1]++;
            right_n[v + 1]++;
            if (u != 0u) {
                if (v >= (uint32_t)w) throw std::invalid_argument("regex guide table: infixes must be sorted by length (a split's right part after the whole)");
                depth[w] = std::max(depth[w], depth[v] + 1);
            }
        }
        if (w > 0 && depth[w] < depth[w - 1]) throw std::invalid_argument("regex guide table: infixes must be sorted by length");
    }
    std::vector<uint32_t> rounds;  // rounds[d] = first entry of the infixes of depth d
    for (int w = 0; w < n_bits; ++w)
        while (rounds.size() <= depth[w]) rounds.push_back(offsets[w]);
    const uint32_t n_rounds = (uint32_t)rounds.size();
    rounds.push_back((uint32_t)E);
    std::vector<uint32_t> h;
    h.reserve(3 * nb1 + 4 * E + rounds.size());
    h.insert(h.end(), offsets, offsets + nb1);
    h.insert(h.end(), entries, entries + E);
    h.insert(h.end(), w_of.begin(), w_of.end());
    for (int side = 0; side < 2; ++side) {
        std::vector<uint32_t> &cnt = side == 0 ? left_n : right_n;
        for (size_t k = 1; k < nb1; ++k) cnt[k] += cnt[k - 1];  // exclusive offsets
        std::vector<uint32_t> ent(E), at(cnt.begin(), cnt.end() - 1);
        for (size_t e = 0; e < E; ++e) {
            const uint32_t u = entries[e] & 0xFFFFu, v = entries[e] >> 16;
            ent[at[side == 0 ? u : v]++] = (side == 0 ? v : u) | (w_of[e] << 16);
        }
        h.insert(h.end(), cnt.begin(), cnt.end());
        h.insert(h.end(), ent.begin(), ent.end());
    }
    h.insert(h.end(), rounds.begin(), rounds.end());
    guide_entries_ = (uint32_t)E;
    guide_rounds_ = n_rounds;
    reserve(guide_, h.size(), false);
    CUDA_CHECK(cudaMemcpyAsync(guide_.ptr, h.data(), h.size() * sizeof(uint32_t), cudaMemcpyHostToDevice, stream_));
    CUDA_CHECK(cudaStreamSynchronize(stream_));
    st_.h2d_bytes += h.size() * sizeof(uint32_t);
    n_bits_ = n_bits;
    lw_ = LW_REGEX;
    prune_ok_ = false;  // (the associativity pruning is an argument about LTL's AND)
    {
        // LTLB200_GUIDE_SMEM=1: stage the tables in shared memory behind the warps' areas.  Off by default: measured on
        // the e-mail example (57 KB of tables) the staged copy costs two of the four resident CTAs per SM and the
        // search to cost 12 gets slower, while the tables read through L1 hit at 95 %
        const size_t warps = wide2_warp_vecs(nvec_, true) * sizeof(uint4) * WARPS_PER_CTA, table = h.size() * sizeof(uint32_t);
        const char *env = getenv("LTLB200_GUIDE_SMEM");
        const bool want = env && atoi(env) != 0;
        guide_smem_words_ = want && warps + table <= kMaxDynamicSmem ? (uint32_t)h.size() : 0u;
        if (warps > kMaxDynamicSmem) throw std::invalid_argument("regex front-end: sequences too wide for the shared-memory areas of the wide kernels");
        occupancy_ = wide2_occupancy_1(nvec_, device_, (int)guide_smem_words_);
    }
}

void Engine::set_weights(const int32_t *weights, int count) {
    if (!levels_.empty()) throw std::invalid_argument("operator weights must be set before the first level");
    if (count < 1 || count > 16) throw std::invalid_argument("operator weights: 1..16 entries");
    unit_weights_ = true;
    for (int k = 0; k < count; ++k) {
        if (weights[k] < 1 || weights[k] > 64) throw std::invalid_argument("operator weights must be in 1..64");
        weights_[k] = weights[k];
        unit_weights_ = unit_weights_ && weights[k] == 1;
    }
    // the argument behind the associativity pruning of AND blocks was made for the reference's node-count cost
    if (!unit_weights_) prune_ok_ = false;
}

// device pointer to `count` rows from id `first` on, in id order: the cache itself on the narrow path; on the wide
// path, where rows live in claim order, their place in a gathered image of the whole cache (filled on demand, range
// by range; valid until the next level is built)
const uint4 *Engine::rows_in_id_order(u64 first, u64 count) {
    if (!wide_) return store_.ptr + first;
    reserve(gather_, std::max<u64>(total_, 1) * nvec_, false);
    const u64 work = count * (u64)nvec_;
    const int grid = (int)std::max<u64>(1, std::min<u64>((work + 255) / 256, (u64)sm_count_ * 16));
    wide_gather_kernel<<<grid, 256, 0, stream_>>>(store_.ptr, loc_.ptr, first, count, nvec_, gather_.ptr + first * nvec_);
    CUDA_CHECK(cudaGetLastError());
    st_.kernel_launches++;
    return gather_.ptr + first * nvec_;
}

// the level where it lives: rows of key_bytes() bytes and winning ordinals, valid until the next level is built
int Engine::level_device(int cost, void **rows_dev, void **ords_dev) {
    if (cost < 1 || cost > (int)levels_.size()) return LTLB200_ERR_ARGUMENT;
    CUDA_CHECK(cudaSetDevice(device_));
    CUDA_CHECK(cudaStreamSynchronize(stream_));
    const LevelMeta &lv = levels_[cost - 1];
    *rows_dev = lv.n ? (void *)rows_in_id_order(lv.base, lv.n) : nullptr;
    CUDA_CHECK(cudaStreamSynchronize(stream_));
    *ords_dev = lv.n ? (void *)(ords_.ptr + lv.base) : nullptr;
    return LTLB200_OK;
}

int Engine::entry(int64_t gid, int32_t *op, int64_t *left, int64_t *right) {
    if (gid < 0 || (u64)gid >= total_) return LTLB200_ERR_ARGUMENT;
    size_t li = 0;
    while (li + 1 < levels_.size() && (u64)gid >= levels_[li + 1].base) ++li;
    while (levels_[li].n == 0 || (u64)gid < levels_[li].base) --li;
    CUDA_CHECK(cudaSetDevice(device_));
    // Witness reconstruction walks a tree whose nodes are almost all in the low levels: the ordinals of the first
    // kEntryCache entries come over in ONE copy on the first call and serve every later one (finalised entries
    // never change; reset() and new levels below the prefix size drop the copy), instead of a copy + synchronise
    // per node.
    if (entry_cache_total_ != std::min<u64>(total_, kEntryCache)) {
        entry_cache_total_ = std::min<u64>(total_, kEntryCache);
        entry_cache_.resize((size_t)entry_cache_total_);
        CUDA_CHECK(cudaMemcpyAsync(entry_cache_.data(), ords_.ptr, entry_cache_total_ * sizeof(u64), cudaMemcpyDeviceToHost, stream_));
        CUDA_CHECK(cudaStreamSynchronize(stream_));
        st_.d2h_bytes += entry_cache_total_ * sizeof(u64);
    }
    u64 ord = 0;
    if ((u64)gid < entry_cache_total_) {
        ord = entry_cache_[(size_t)gid];
    } else {
        CUDA_CHECK(cudaMemcpyAsync(&ord, ords_.ptr + gid, sizeof(u64), cudaMemcpyDeviceToHost, stream_));
        CUDA_CHECK(cudaStreamSynchronize(stream_));
        st_.d2h_bytes += sizeof(u64);
    }
    decode(levels_[li], ord, op, left, right);
    return LTLB200_OK;
}

void Engine::get_stats(ltlb200_stats *out) {
    if (fin_pending_[0] || fin_pending_[1]) {
        CUDA_CHECK(cudaSetDevice(device_));
        collect_finalize_time(0, true);
        collect_finalize_time(1, true);
    }
    st_.table_slots = table_slots();
    st_.device_bytes = held_;
    *out = st_;
}

}  // namespace ltlb200

// ---- C ABI -----------------------------------------------------------------------------
using ltlb200::Engine;
using ltlb200::g_last_error;

struct ltlb200_engine {
    Engine *impl;
};

template <typename Fn>
static int guarded(Fn &&fn) {
    try {
        g_last_error.clear();
        return fn();
    } catch (const ltlb200::CudaError &e) {
        g_last_error = e.what();
        return LTLB200_ERR_CUDA;
    } catch (const std::invalid_argument &e) {
        g_last_error = e.what();
        return LTLB200_ERR_ARGUMENT;
    } catch (const std::exception &e) {
        g_last_error = e.what();
        return LTLB200_ERR_CUDA;
    }
}

extern "C" {

int ltlb200_abi_version(void) { return LTLB200_ABI_VERSION; }

const char *ltlb200_last_error(void) { return g_last_error.c_str(); }

int ltlb200_device_count(void) {
    int n = 0;
    cudaError_t err = cudaGetDeviceCount(&n);
    if (err != cudaSuccess) {
        g_last_error = std::string("cudaGetDeviceCount: ") + cudaGetErrorString(err);
        cudaGetLastError();
        return 0;
    }
    int usable = 0;
    for (int d = 0; d < n; ++d) {
        if (ltlb200::device_info(d).major == 10) ++usable;
    }
    if (!usable) g_last_error = "no sm_100 (B200) device visible";
    return usable;
}

ltlb200_engine *ltlb200_create(int32_t trace_count, int32_t lane_bits, const uint64_t *masks, const uint64_t *target,
                               const uint64_t *atoms, int32_t n_atoms, int32_t device, uint64_t hbm_budget_bytes,
                               void *cuda_stream) {
    ltlb200_engine *h = nullptr;
    int rc = guarded([&] {
        if (trace_count < 1 || n_atoms < 1 || !masks || !target || !atoms ||
            (lane_bits != 8 && lane_bits != 16 && lane_bits != 32 && lane_bits != 64))
            throw std::invalid_argument("bad specification geometry");
        Engine *impl = new Engine(trace_count, lane_bits, masks, target, atoms, n_atoms, device, hbm_budget_bytes, cuda_stream);
        h = new ltlb200_engine{impl};
        return 0;
    });
    return rc == 0 ? h : nullptr;
}

void ltlb200_destroy(ltlb200_engine *e) {
    if (!e) return;
    delete e->impl;
    delete e;
}

int ltlb200_expand_level(ltlb200_engine *e, int32_t cost, uint32_t op_mask, int32_t exhaustive, int64_t batch_size,
                         uint64_t memory_budget_bytes, double deadline_s, int64_t *n_new, int64_t *sep_gid,
                         int64_t *constructed_delta) {
    if (!e || !n_new || !sep_gid || !constructed_delta) return LTLB200_ERR_ARGUMENT;
    return guarded([&] {
        return e->impl->expand_level(cost, op_mask, exhaustive != 0, batch_size, memory_budget_bytes, deadline_s, n_new,
                                     sep_gid, constructed_delta);
    });
}

int ltlb200_route_begin(ltlb200_engine *e, int32_t cost, uint32_t op_mask, int32_t exhaustive, double deadline_s, int32_t rank,
                        int32_t world, uint64_t *send_counts, uint64_t *send_offsets, void **rows_dev, void **ords_dev,
                        uint64_t *sep_ord, uint64_t *n_seps) {
    if (!e || !send_counts || !send_offsets || !rows_dev || !ords_dev || !sep_ord || !n_seps) return LTLB200_ERR_ARGUMENT;
    return guarded([&] {
        ltlb200::u64 sep = 0, ns = 0;
        int rc = e->impl->route_begin(cost, op_mask, exhaustive != 0, deadline_s, rank, world, (ltlb200::u64 *)send_counts,
                                      (ltlb200::u64 *)send_offsets, rows_dev, ords_dev, &sep, &ns);
        *sep_ord = sep;
        *n_seps = ns;
        return rc;
    });
}

int ltlb200_exchange_recv(ltlb200_engine *e, uint64_t n_records, void **rows_dev, void **ords_dev) {
    if (!e || !rows_dev || !ords_dev) return LTLB200_ERR_ARGUMENT;
    return guarded([&] {
        e->impl->exchange_recv(n_records, rows_dev, ords_dev);
        return LTLB200_OK;
    });
}

int ltlb200_owner_reduce(ltlb200_engine *e, uint64_t n_records, uint64_t *n_claimed, void **bitmap_dev, uint64_t *bitmap_words) {
    if (!e || !n_claimed || !bitmap_dev || !bitmap_words) return LTLB200_ERR_ARGUMENT;
    return guarded([&] {
        ltlb200::u64 nc = 0, words = 0;
        const int rc = e->impl->owner_reduce(n_records, &nc, bitmap_dev, &words);
        *n_claimed = nc;
        *bitmap_words = words;
        return rc;
    });
}

int ltlb200_level_abort(ltlb200_engine *e) {
    if (!e) return LTLB200_ERR_ARGUMENT;
    return guarded([&] {
        e->impl->level_abort();
        return LTLB200_OK;
    });
}

int ltlb200_winners_export(ltlb200_engine *e, uint64_t sep_ord, uint64_t *n_winners, void **rows_dev, void **ords_dev) {
    if (!e || !n_winners || !rows_dev || !ords_dev) return LTLB200_ERR_ARGUMENT;
    return guarded([&] {
        ltlb200::u64 n = 0;
        e->impl->winners_export(sep_ord, &n, rows_dev, ords_dev);
        *n_winners = n;
        return LTLB200_OK;
    });
}

int ltlb200_level_commit(ltlb200_engine *e, uint64_t sep_ord, const uint64_t *seps, uint64_t n_seps, const uint64_t *recv_counts,
                         int32_t n_sources, int64_t batch_size, uint64_t memory_budget_bytes, int64_t *n_new, int64_t *sep_gid,
                         int64_t *constructed_delta) {
    if (!e || !n_new || !sep_gid || !constructed_delta) return LTLB200_ERR_ARGUMENT;
    return guarded([&] {
        return e->impl->level_commit(sep_ord, (const ltlb200::u64 *)seps, n_seps, (const ltlb200::u64 *)recv_counts, n_sources,
                                     batch_size, memory_budget_bytes, n_new, sep_gid, constructed_delta);
    });
}

int64_t ltlb200_seps_copy(ltlb200_engine *e, uint64_t *out, uint64_t cap) {
    if (!e || (!out && cap)) return LTLB200_ERR_ARGUMENT;
    int64_t n = 0;
    int rc = guarded([&] {
        n = (int64_t)e->impl->seps_copy((ltlb200::u64 *)out, cap);
        return LTLB200_OK;
    });
    return rc < 0 ? rc : n;
}

int32_t ltlb200_key_bytes(const ltlb200_engine *e) { return e ? e->impl->key_bytes() : 0; }

double ltlb200_now(void) { return ltlb200::monotonic_s(); }

int ltlb200_level_info(const ltlb200_engine *e, int32_t cost, int64_t *n, int64_t *base) {
    if (!e || !n || !base) return LTLB200_ERR_ARGUMENT;
    return e->impl->level_info(cost, n, base);
}

int ltlb200_level_candidates(ltlb200_engine *e, int32_t cost, uint32_t op_mask, int64_t *n) {
    if (!e || !n) return LTLB200_ERR_ARGUMENT;
    return guarded([&] {
        *n = e->impl->level_candidates(cost, op_mask);
        return LTLB200_OK;
    });
}

int32_t ltlb200_holds_separator(const ltlb200_engine *e) { return e && e->impl->holds_separator() ? 1 : 0; }

int32_t ltlb200_num_levels(const ltlb200_engine *e) { return e ? e->impl->num_levels() : 0; }

int ltlb200_level_copy(ltlb200_engine *e, int32_t cost, int64_t first, int64_t count, uint8_t *cms, uint8_t *op,
                       int64_t *left, int64_t *right) {
    if (!e) return LTLB200_ERR_ARGUMENT;
    return guarded([&] { return e->impl->level_copy(cost, first, count, cms, op, left, right); });
}

int ltlb200_set_weights(ltlb200_engine *e, const int32_t *weights) {
    if (!e || !weights) return LTLB200_ERR_ARGUMENT;
    return guarded([&] {
        e->impl->set_weights(weights, 16);
        return LTLB200_OK;
    });
}

int ltlb200_set_regex(ltlb200_engine *e, int32_t n_bits, const uint32_t *offsets, const uint32_t *entries, uint64_t n_entries) {
    if (!e || !offsets || (!entries && n_entries)) return LTLB200_ERR_ARGUMENT;
    return guarded([&] {
        e->impl->set_regex(n_bits, offsets, entries, n_entries);
        return LTLB200_OK;
    });
}

int ltlb200_level_device(ltlb200_engine *e, int32_t cost, void **rows_dev, void **ords_dev) {
    if (!e || !rows_dev || !ords_dev) return LTLB200_ERR_ARGUMENT;
    return guarded([&] { return e->impl->level_device(cost, rows_dev, ords_dev); });
}

int ltlb200_entry(ltlb200_engine *e, int64_t gid, int32_t *op, int64_t *left, int64_t *right) {
    if (!e || !op || !left || !right) return LTLB200_ERR_ARGUMENT;
    return guarded([&] { return e->impl->entry(gid, op, left, right); });
}

int ltlb200_reset(ltlb200_engine *e) {
    if (!e) return LTLB200_ERR_ARGUMENT;
    return guarded([&] {
        e->impl->reset();
        return LTLB200_OK;
    });
}

void ltlb200_trim(int32_t device) {
    cudaSetDevice(device);
    cudaDeviceSynchronize();
    ltlb200::g_blocks.trim(device);
}

uint64_t ltlb200_approx_bytes(const ltlb200_engine *e) { return e ? e->impl->approx_bytes() : 0; }

int ltlb200_get_stats(ltlb200_engine *e, ltlb200_stats *out) {
    if (!e || !out) return LTLB200_ERR_ARGUMENT;
    e->impl->get_stats(out);
    return LTLB200_OK;
}

}  // extern "C"
