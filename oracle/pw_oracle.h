/* pw_oracle.h -- CPU restatement of the reference's batched graph-ANNS search
 * path (shardann 0.1.0).  TEST INFRASTRUCTURE ONLY: this is the parity
 * checker; only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
 * --impl reference legs may load it.  The product path never links it.
 *
 * Every function cites the reference file:line it restates
 * (paths relative to /root/reference/pkg/src/shardann/).  numpy's own
 * algorithms used by the reference (pairwise float32 sum, SeedSequence,
 * PCG64, Generator.choice / permutation) are restated from numpy 2.3.5's
 * published sources (numpy/_core/src/umath/loops_utils.h.src pairwise_sum,
 * numpy/random/bit_generator.pyx SeedSequence, numpy/random/_generator.pyx
 * choice/shuffle, numpy/random/src/distributions/distributions.c bounded
 * integers, numpy/random/src/pcg64/pcg64.h).
 */
#ifndef PW_ORACLE_H
#define PW_ORACLE_H
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* One searchable graph: search.py:130-151 ShardContext (vectors/adj/global_ids/direction). */
typedef struct {
    const float* vectors;      /* (n, d) float32 row-major */
    int64_t n;
    int32_t d;
    const int32_t* adj;        /* (n, j) int32 */
    int32_t j;
    const int32_t* global_ids; /* (n,) int32 */
    const uint32_t* direction; /* (n, j, W) uint32 or NULL */
} orc_graph;

/* ShardContext + ghost (search.py:117-151). */
typedef struct {
    orc_graph main;
    const int32_t* inter_map;  /* (n,) int32 or NULL */
    int32_t has_ghost;
    orc_graph ghost;           /* ghost.global_ids = parent-shard local ids */
} orc_shard;

/* search.py:39-73 SearchParams. */
typedef struct {
    int32_t k, l, m, r, max_iter;
    uint64_t seed;
    int32_t selection;        /* 0 full, 1 direction, 2 random */
    double discard_ratio;
    double cooldown_ratio;
    int32_t ghost_enabled;
    int32_t ghost_max_iter;
    int32_t seed_mode;        /* 0 neighbors, 1 mixed */
    int32_t buffer_cap;       /* 0 = None */
    int32_t log_visits;
    int32_t metric;           /* 0 L2 (the reference); 1 inner product (extension, parity unpinned) */
    /* opt-in path-extension knobs (the GPU's pw_tuning fields of the same
     * names; 0 = the reference's run_pipelined) */
    int32_t forward_count;    /* top-F entries forwarded per query (F <= k) */
    int32_t late_l;           /* l of stages >= 1 */
    int32_t late_max_iter;    /* max_iter of stages >= 1 */
} orc_params;

/* numpy PCG64 bit generator state (128-bit state/inc + buffered uint32). */
typedef struct {
    uint64_t state_hi, state_lo, inc_hi, inc_lo;
    int32_t has_uint32;
    uint32_t uinteger;
} orc_pcg64;

/* search.py:76-100 SearchCounters. */
typedef struct {
    int64_t iterations, distance_computations, total_visits, nodes_expanded,
        dgs_skipped, inserted_total;
} orc_counters;

typedef struct {
    int32_t n_out;       /* <= k */
    int32_t converged;
    int32_t retained;
    orc_counters c;
    int64_t n_visited;   /* entries written to visit_log (log_visits) */
} orc_result;

const char* orc_last_error(void);

/* rng.py:26-44 */
uint64_t orc_splitmix64(uint64_t x);
uint64_t orc_derive_seed(uint64_t seed, const uint64_t* parts, int n_parts);
void orc_pcg64_seed(uint64_t seed64, orc_pcg64* g);     /* np.random.PCG64(seed64) */
uint64_t orc_pcg64_next64(orc_pcg64* g);
uint32_t orc_pcg64_next32(orc_pcg64* g);
/* Generator.choice(pop, size, replace=False) -> out[size] */
int orc_choice(orc_pcg64* g, int64_t pop, int64_t size, int64_t* out);
/* Generator.permutation(n) -> out[n] */
void orc_permutation(orc_pcg64* g, int64_t n, int64_t* out);

/* data.py:70-79 squared_l2 (numpy pairwise float32 order). */
void orc_squared_l2(const float* points, int64_t rows, int32_t d, const float* q, float* out);

/* direction.py helpers */
void orc_pack_sign_bits(const uint8_t* bits, int64_t rows, int32_t d, uint32_t* out);
int32_t orc_keep_count(int32_t j, double discard_ratio);
int32_t orc_in_cooldown(int32_t iteration, int32_t max_iter, double cooldown_ratio);

/* search.py:269-335; returns 0 or -1 (ValueError, see orc_last_error). */
int orc_search(const orc_graph* ctx, const float* query, const orc_params* p,
               const int64_t* seeds, int32_t n_seeds, orc_pcg64* rng,
               int32_t* out_ids, float* out_dists, int32_t* out_local,
               orc_result* res, int32_t* visit_log, int64_t visit_cap);

/* pipeline.py:158-184 run_ghost_stage -> parent-local entry id. */
int orc_ghost_stage(const orc_shard* sh, const float* query, const orc_params* p,
                    orc_pcg64* rng, int32_t* entry, orc_counters* c);

/* pipeline.py:270-305 (mode 0) / 308-350 (mode 1) + finish 249-267.
 * stats_i32: (N_stages, 4, Q) iterations, ghost_iterations, retained, converged
 * stats_i64: (N_stages, 4, Q) distance_computations, total_visits, inserted, dgs_skipped
 * comm: (N_stages, N).  threads <= 0 -> all cores (OpenMP).  */
int orc_run(const orc_shard* shards, int32_t n_shards, const float* queries, int64_t q,
            const orc_params* p, int32_t mode, int32_t threads,
            int32_t* shard_ids, float* shard_dists, int32_t* final_ids, float* final_dists,
            int32_t* stats_i32, int64_t* stats_i64, int64_t* comm);

/* One stage launch, mirroring pw_search_stage: queries [q0, q0+n) of the
 * (q_total, d) array searched on one shard at `stage` (pipeline.py:329-342 /
 * :294-297).  entries_in/forward_out: (q_total,) or NULL; shard_ids/dists:
 * (q_total, n_cols, k) written at column col; stats_i32 (4, q_total) /
 * stats_i64 (4, q_total) accumulate as in orc_run. */
int orc_run_stage(const orc_shard* shard, const float* queries, int64_t q_total, int64_t q0,
                  int64_t n, const orc_params* p, int32_t stage, const int32_t* entries_in,
                  int32_t* forward_out, int32_t* shard_ids, float* shard_dists, int32_t n_cols,
                  int32_t col, int32_t* stats_i32, int64_t* stats_i64, int32_t threads);

/* pipeline.py:187-196 reduce_topk over one query's n candidates. returns count or -1. */
int orc_reduce_topk(const int32_t* ids, const float* dists, int64_t n, int32_t k,
                    int32_t* out_ids, float* out_dists);

/* _crc32c.py:17-39: CRC-32C, byte-table serial path (_make_tables table 0 +
 * _update_serial), starting from raw register `state`; crc32c(buf) =
 * ~orc_crc32c_update(0xFFFFFFFF, buf, n). */
uint32_t orc_crc32c_update(uint32_t state, const uint8_t* buf, int64_t n);

#ifdef __cplusplus
}
#endif
#endif
