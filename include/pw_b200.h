/* pw_b200.h -- C ABI of the B200-native batched graph-ANNS search path.
 *
 * Drop-in boundary for the reference package shardann 0.1.0 (PathWeaver,
 * arXiv 2507.17094).  The reference has no FFI of its own (pure Python +
 * numpy); each entry point below replaces one reference interface, cited as
 * /root/reference/pkg/src/shardann/<file>:<line>.  Plain pointers and sizes
 * only; no torch or C++ types cross this boundary; no C++ exceptions escape.
 *
 * Status codes: 0 ok; PW_EINVAL (-1) -> ValueError, PW_ENOMEM (-2) ->
 * MemoryError, PW_ECUDA (-3) -> RuntimeError.  pw_last_error() returns the
 * thread-local message of the last failure (text matches the reference's
 * ValueError messages where one exists).
 */
#ifndef PW_B200_H
#define PW_B200_H
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define PW_OK 0
#define PW_EINVAL (-1)
#define PW_ENOMEM (-2)
#define PW_ECUDA (-3)

#define PW_METRIC_L2 0 /* squared L2, reported as sqrt (data.py:70-79, search.py:325) */
#define PW_METRIC_IP 1 /* inner product: distance = -(q . x), pairwise-ordered; parity unpinned */
#define PW_DTYPE_F32 0
#define PW_DTYPE_U8 1

#define PW_SEL_FULL 0
#define PW_SEL_DIRECTION 1
#define PW_SEL_RANDOM 2

#define PW_SEED_NEIGHBORS 0
#define PW_SEED_MIXED 1

#define PW_MODE_BASELINE 0
#define PW_MODE_PIPELINED 1

/* search.py:39-73 SearchParams (field for field). */
typedef struct {
    int32_t k, l, m, r, max_iter;
    uint64_t seed;
    int32_t selection;       /* PW_SEL_* */
    double discard_ratio;
    double cooldown_ratio;
    int32_t ghost_enabled;
    int32_t ghost_max_iter;
    int32_t seed_mode;       /* PW_SEED_* */
    int32_t buffer_cap;      /* 0 = None */
    int32_t log_visits;
    int32_t metric;          /* PW_METRIC_*: L2 (the reference's only metric) or IP (extension) */
} pw_params;

/* Device-side knobs outside SearchParams (SURVEY.md §5 "Config"). 0 = default. */
typedef struct {
    int32_t visited_slots;   /* shared-memory visited-hash slots per query (power of 2) */
    int32_t stage_rows;      /* rows in flight per warp (gather staging) */
    int32_t warps_per_sm;    /* cap on resident query-warps per SM */
    int32_t row_copy;        /* reserved (vector rows always use cp.async; TMA measured slower) */
    int32_t flags;           /* bit 0: L2-prefetch predicted parent rows (off by default: measured slower);
                                bit 1: lossy visited cache (ids exact, distance_computations may grow);
                                bit 2: TMA bulk copies for expansion rows (bits 0 and 2 are measured slower;
                                kept for A/B) */
    /* Opt-in path-extension knobs beyond the reference (its run_pipelined
     * forwards exactly one entry per query and uses one budget for every
     * stage; SPEC.md "DESIGN DECISIONS" names both as configurable).  0 =
     * the reference's behaviour; results then differ from the reference. */
    int32_t forward_count;   /* entries forwarded per query to the next shard (top-F of the
                                stage's queue through inter_map); 1..8.  Entry
                                buffers / inboxes then hold F words per query. */
    int32_t late_l;          /* queue length l of stages >= 1 (k <= late_l); 0 = params->l */
    int32_t late_max_iter;   /* max_iter of stages >= 1; 0 = params->max_iter */
} pw_tuning;

/* One shard (pipeline.py:121-155 build_contexts output for one ShardPack):
 * host arrays, copied to the current device by pw_shard_create. */
typedef struct {
    int64_t n;                    /* n_local */
    int32_t d;
    int32_t j;                    /* graph degree (adj.shape[1]); may be 0 */
    int32_t dtype;                /* PW_DTYPE_* of vectors */
    const void* vectors;          /* (n, d) row-major */
    const int32_t* adj;           /* (n, j) shard-local ids */
    const int32_t* global_ids;    /* (n,) */
    const uint32_t* direction;    /* (n, j, ceil(d/32)) packed sign bits or NULL */
    const int32_t* inter_map;     /* (n,) local ids in the next shard, or NULL */
    int64_t ghost_n;              /* 0 = no ghost index */
    int32_t ghost_j;
    const int32_t* ghost_ids;     /* (ghost_n,) parent-local ids, sorted */
    const int32_t* ghost_adj;     /* (ghost_n, ghost_j) ghost-local ids */
    int32_t on_device;            /* 1: every pointer above is a device pointer (copied D2D) */
} pw_shard_desc;

typedef struct pw_shard pw_shard;

/* numpy PCG64 state as exposed by Generator.bit_generator.state. */
typedef struct {
    uint64_t state_hi, state_lo, inc_hi, inc_lo;
    int32_t has_uint32;
    uint32_t uinteger;
} pw_rng;

/* search.py:76-100 SearchCounters + SearchResult scalars. */
typedef struct {
    int64_t iterations, distance_computations, total_visits, nodes_expanded,
        dgs_skipped, inserted_total;
    int32_t converged, retained, n_out, pad_;
    int64_t n_visited;
} pw_search_out;

const char* pw_last_error(void);
const char* pw_version(void);

/* Replaces pipeline.py:121-155 build_contexts (one shard; uploads to the
 * current CUDA device).  Ghost vectors are gathered on the device from
 * vectors[ghost_ids] (pipeline.py:139-144). */
int pw_shard_create(const pw_shard_desc* desc, pw_shard** out);
int pw_shard_destroy(pw_shard* shard);
/* device memory footprint of a shard in bytes */
int64_t pw_shard_bytes(const pw_shard* shard);

/* Replaces search.py:269-335 search(query, ctx, params, seeds, rng=...) and,
 * with use_ghost=1, the inner search of pipeline.py:158-184
 * run_ghost_stage (params must already be the ghost params).
 * Host buffers; rng is advanced exactly as numpy would advance it.
 * out_ids/out_dists/out_local: k entries; visit_log: visit_cap entries. */
int pw_search_one(pw_shard* shard, int32_t use_ghost, const pw_params* params,
                  const float* query, const int64_t* seeds, int32_t n_seeds,
                  pw_rng* rng, int32_t* out_ids, float* out_dists, int32_t* out_local,
                  pw_search_out* out, int32_t* visit_log, int64_t visit_cap);

/* One pipeline stage for a contiguous query range on one shard -- the
 * per-(GPU, stage) launch of pipeline.py:329-342 `process` (pipelined) and
 * :294-297 `do` (baseline).  ALL pointers are DEVICE pointers.
 *   queries      (q_total, d) float32; rows [q0, q0+n) are searched
 *   entries_in   (q_total,) int32 entry ids in this shard, or NULL (stage 0 / baseline)
 *   forward_out  (q_total,) int32 <- inter_map[top1], or NULL (last stage)
 *   shard_ids/shard_dists (q_total, n_cols, k) written at column `col`
 *   stats_i32 (4, q_total): iterations, ghost_iterations, retained, converged
 *   stats_i64 (6, q_total): distance_computations, total_visits, inserted, dgs_skipped,
 *                           nodes_expanded, ghost_nodes_expanded (the last two are not
 *                           StageStats fields; they feed the gather-roofline byte count)
 * Counters accumulate (+=) like pipeline.py:224-243; converged is assigned.
 * stream: cudaStream_t (NULL = legacy default stream). */
int pw_search_stage(pw_shard* shard, const pw_params* params, const pw_tuning* tuning,
                    const float* queries, int64_t q0, int64_t n, int32_t stage,
                    const int32_t* entries_in, int32_t* forward_out,
                    int32_t* shard_ids, float* shard_dists, int32_t n_cols, int32_t col,
                    int32_t* stats_i32, int64_t* stats_i64, int64_t q_total, void* stream);

/* pipeline.py:187-196 reduce_topk + :249-267 finish over device arrays:
 * (q, n_cand) candidate lists (n_cand = N*k for (q, N, k) shard lists) ->
 * (q, k) by (sqrt'd float32 distance, global id); ids < 0 are padding.
 * err_dev: device int32 flag set to 1 when some query has no valid candidate;
 * NULL = synchronise and return PW_EINVAL "cannot reduce empty candidate lists". */
int pw_reduce_topk(const int32_t* shard_ids, const float* shard_dists, int64_t q,
                   int32_t n_cand, int32_t k, int32_t* final_ids, float* final_dists,
                   int32_t* err_dev, void* stream);

/* Output initialisation of a device-resident run (no reference counterpart:
 * the reference allocates fresh arrays per call, pipeline.py:288-305): ids[n]
 * = -1 and dists[n] = +inf (the shard-column padding), s32[n32] = 0 and
 * s64[n64] = 0 (StageStats), in one launch on `stream`. */
int pw_init_outputs(int32_t* ids, float* dists, int64_t n, int32_t* s32, int64_t n32,
                    int64_t* s64, int64_t n64, void* stream);

/* Replaces pipeline.py:270-305 run_sharded_baseline (mode 0) and
 * :308-350 run_pipelined (mode 1) for n_shards shards resident on the
 * current device (logical shards; the multi-GPU ring lives in the host
 * layer).  HOST buffers in and out: queries (q, d); shard_ids/dists (q, N, k);
 * final_ids/dists (q, k); stats_i32 (N, 4, q) / stats_i64 (N, 6, q) as in
 * pw_search_stage;
 * comm (N, N) int64 bytes per (stage, sending shard).
 * Result block: when the six output buffers are one allocation laid out as
 * shard_ids | shard_dists | final_ids | final_dists | stats_i32 | stats_i64,
 * each starting at the previous one's start + its size rounded up to 256
 * bytes, the results arrive in one copy instead of six (any other layout
 * works too). */
int pw_run(pw_shard* const* shards, int32_t n_shards, const pw_params* params,
           const pw_tuning* tuning, const float* queries, int64_t q, int32_t mode,
           int32_t* shard_ids, float* shard_dists, int32_t* final_ids, float* final_dists,
           int32_t* stats_i32, int64_t* stats_i64, int64_t* comm);

/* Device-resident variant of pw_run (all pointers device; stats_i64 is
 * (N, 6, q); no host copies, no synchronisation): the kernel-only timing
 * path of bench.py. */
int pw_run_device(pw_shard* const* shards, int32_t n_shards, const pw_params* params,
                  const pw_tuning* tuning, const float* queries, int64_t q, int32_t mode,
                  int32_t* shard_ids, float* shard_dists, int32_t* final_ids,
                  float* final_dists, int32_t* stats_i32, int64_t* stats_i64,
                  int32_t* entries_a, int32_t* entries_b, void* stream);

/* Dataflow ring: the pipelined path extension of pipeline.py:308-347 as ONE
 * persistent K1 launch per shard.  Shard g runs every (stage s, query q) task
 * with chunk(q) = (g - s) mod N in stage-major order; a stage s > 0 task
 * waits on inbox[q] (epoch << 32 | entry) and a finished stage s < N-1 task
 * stores epoch << 32 | inter_map[top1] into next_inbox[q] -- shard g+1's
 * inbox, a peer (NVLink) mapping when the shards live on different GPUs
 * (pw_ipc_*), so stage boundaries never stop a GPU.  Outputs may also be
 * peer mappings (the reducing rank's buffers): shard_ids/dists (q, N, k)
 * column g; stats_i32 (N, 4, q) / stats_i64 (N, 6, q) row `stage`.
 * epoch: a run tag equal on every shard, new for every run (inboxes are
 * never reset).  sm_limit > 0 caps the CTAs (several shards sharing one GPU
 * must all be resident).  Device pointers; asynchronous on `stream`. */
int pw_search_dataflow(pw_shard* shard, const pw_params* params, const pw_tuning* tuning,
                       const float* queries, int64_t q, int32_t g, int32_t n_shards,
                       uint32_t epoch, const uint64_t* inbox, uint64_t* next_inbox,
                       int32_t* shard_ids, float* shard_dists, int32_t* stats_i32,
                       int64_t* stats_i64, int32_t sm_limit, void* stream);

/* Exact squared L2 of row pairs for the GPU index builder (graphs.py:90-101
 * rescoring): out[t] = squared_l2(b[ib[t]], a[ia[t]]), numpy pairwise float32
 * order, bit-identical to data.py:70-79.  a (.., d), b (.., d) float32; ia,
 * ib (n,) int64; out (n,) float32; device pointers, asynchronous. */
int pw_l2_pairs(const float* a, const float* b, int32_t d, const int64_t* ia, const int64_t* ib,
                int64_t n, float* out, void* stream);

/* Measurement probe (not a reference interface): gather n_ids rows of
 * row_bytes (a 16-byte multiple) from table at random ids with as many rows
 * in flight as the SMs hold -- the achievable HBM bandwidth of K1's access
 * pattern, reported beside K1's roofline (tools/gather_probe.py).  Device
 * pointers; sink: one device u32; asynchronous. */
int pw_gather_probe(const void* table, int64_t row_bytes, const int32_t* ids, int64_t n_ids,
                    uint32_t* sink, int32_t blocks, void* stream);

/* K4 tensor-core kNN screen (replaces the distance screen of
 * graphs.py:65-78 `_knn_block`, which keeps k + 8 candidates per row by a
 * GEMM-style distance before the exact rescore): for each of the nq query
 * rows q (device, (nq, d) f32), the kc base rows x (device, (n, d) f32) with
 * the smallest approximate |x_c|^2 - 2 q.x_c (TF32 tensor cores, FP32
 * accumulation; xn = |x_c|^2, (n,) f32), query row r excluding base row
 * r + self_off when self_off >= 0.  Outputs (nq, kc) int32 ids / f32 values,
 * unsorted, -1 / +inf when n - 1 < kc.  d % 4 == 0, kc <= 64.  The values only
 * select candidates: exact.py rescores them bit-exactly and certifies each
 * row against the TF32 error bound. */
int pw_knn_screen(const float* q, int64_t nq, const float* x, int64_t n, int32_t d, const float* xn,
                  int64_t self_off, int32_t kc, int32_t* out_ids, float* out_vals, void* stream);

/* Validate a shard's inter_map (pipeline.py:339 forwards inter_map[top1]
 * as the next shard's entry) against the next shard's size n_next: every
 * value must be in [0, n_next).  Synchronous once per (shard, n_next);
 * pw_run / pw_run_device call it for every pipelined ring.  0 or PW_EINVAL. */
int pw_shard_validate_inter(pw_shard* shard, int64_t n_next);

/* Stream-ordered cross-GPU flags for the pipelined dataflow ring (batches
 * in flight without host synchronisation):
 *   pw_signal  after all earlier work on `stream` (a persistent K1's peer
 *              stores included) is visible system-wide, store `value` into
 *              *flag (a device word, possibly a peer / IPC mapping);
 *   pw_wait    hold `stream` until every *flags[i] >= value (flags: DEVICE
 *              array of n <= 32 device pointers); after ~1 minute without it
 *              sets bit 32 in *err (device int32) and releases the stream. */
int pw_signal(uint64_t* flag, uint64_t value, void* stream);
int pw_wait(const uint64_t* const* flags, int32_t n, uint64_t value, int32_t* err, void* stream);

/* Synchronous check of a shard's device error flag (table overflow, a
 * dataflow inbox that never filled); clears it.  0 or PW_ECUDA + message. */
int pw_shard_check(pw_shard* shard);

/* Device buffers shareable across processes (cudaMalloc'd, so an IPC handle
 * maps exactly this allocation) and their CUDA IPC handles (64 bytes). */
int pw_dev_alloc(int64_t bytes, void** out);
int pw_dev_free(void* ptr);
int pw_ipc_get(const void* ptr, void* handle64);
int pw_ipc_open(const void* handle64, void** out);
int pw_ipc_close(void* ptr);

/* Bit-exact data.py:70-79 squared_l2 of rows[ids] against one query, on the
 * device (test hook for the distance primitive).  Device pointers. */
int pw_squared_l2_rows(pw_shard* shard, const int32_t* ids, int64_t n_ids,
                       const float* query, float* out, void* stream);

/* Launch configuration K1 would use for (shard, params, tuning) without
 * launching: out[0] warps per CTA (= resident query-warps per SM), out[1]
 * shared-memory bytes per warp, out[2] visited-table slots, out[3] staging
 * rows, out[4] specialised dimension (0 = generic), out[5] blocks. */
int pw_launch_config(pw_shard* shard, const pw_params* params, const pw_tuning* tuning,
                     int32_t* out6);

/* Per-phase cycle totals of K1 summed over warps (init, score, merge,
 * select, expand, dedup, visited, other) -- non-zero only in the
 * PW_PHASE_TIMERS build (libpwb200_timers.so, tools/phase_timers.py). */
int pw_phase_cycles(pw_shard* shard, int64_t* out8, int32_t reset);

/* CRC-32C (Castagnoli, reflected 0x82F63B78; init ~0, final ~) for the
 * `.pwix` index container.
 * pw_crc32c          replaces shardann/_crc32c.py:98-130 crc32c on a HOST
 *                    buffer: SSE4.2 crc32 instruction, split over `threads`
 *                    host threads (<= 0: all cores) and combined.
 * pw_crc32c_combine  replaces shardann/_crc32c.py:85-89 crc32c_combine.
 * pw_crc32c_device   the section checks of shardann/container.py:117-124
 *                    (_read_array) on DEVICE buffers already in HBM: n
 *                    buffers, one K3 launch on `stream`, synchronous, CRCs
 *                    written to out_host[n]. */
int pw_crc32c(const void* buf, int64_t n, int32_t threads, uint32_t* out);
int pw_crc32c_combine(uint32_t crc1, uint32_t crc2, int64_t len2, uint32_t* out);
int pw_crc32c_device(const void* const* ptrs, const int64_t* lens, int32_t n, uint32_t* out_host,
                     void* stream);

/* Number of kernel launches issued by this library since load (evidence for
 * bench.py's gpu_launches). */
int64_t pw_launch_count(void);

#ifdef __cplusplus
}
#endif
#endif
