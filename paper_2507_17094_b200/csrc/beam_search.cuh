// beam_search.cuh -- K1: persistent warp-per-query beam search for sm_100a.
//
// One warp runs one whole search (shardann/search.py:269-335) with its state
// in shared memory: the size-l priority queue (64-bit keys f32bits<<32 | id,
// which order exactly like the reference's (distance, id) tuples), an exact
// open-addressing visited set (spilling to a per-warp global table if it
// fills up), the candidate batch, and a gather staging ring.  Vector rows are
// gathered with cp.async (LDGSTS) into padded shared-memory rows and reduced
// in numpy's pairwise float32 order (8 strided accumulators per <=128-element
// leaf, xor-shuffle tree 1/2/4, sequential tail; recursive halves above 128),
// so every distance is bit-identical to shardann/data.py:70-79.
//
// Per iteration: score new candidates (gather + L2) -> threshold-filter +
// rank-merge into the queue (search.py:170-190) -> first r unexpanded
// parents (:192-204) -> one async round trip for adjacency rows, and when
// pruning the parents' rows + direction rows (direction-guided selection
// fused as a pre-filter, search.py:249-263) -> ordered in-batch dedup + cap
// (:230-232, :264) -> visited filter.  Ghost staging (pipeline.py:158-184)
// runs as a prologue search on the shard's ghost graph in the same warp.
#pragma once
#include <stdint.h>

#include <cuda.h>  // CUtensorMap (TMA descriptors built on the host)

#include "rng_pcg64.cuh"

#ifndef PW_MAX_THREADS
#define PW_MAX_THREADS 512  // resident query-warps per SM x 32 (__launch_bounds__)
#endif

namespace pw {
constexpr int kMaxWarps = PW_MAX_THREADS / 32;
constexpr int kWideWarps = 20;  // the FAST direction-guided build: 640 threads, 96 registers

constexpr uint32_t kEmpty = 0xFFFFFFFFu;
constexpr int kMaxLeaves = 64;
constexpr int kMaxOps = 2 * kMaxLeaves;
constexpr int kParentGroup = 8;

struct GraphDev {
    const void* vec;        // (n, d) rows of the shard's element type (f32 or u8)
    const int32_t* adj;     // (n, j)
    const int32_t* gid;     // (n,) output id map
    const uint32_t* dir;    // (n, j, W) or null
    int32_t n;
    int32_t j;
};

// Host-derived per-search configuration (search.py:289-295, direction.py).
struct SearchCfg {
    int32_t k, L, want, r, max_iter, cap;
    int32_t prune_sel;      // 0 none, 1 direction, 2 random
    int32_t n_keep;         // keep_count(j, discard_ratio)
    int32_t cool_start;     // first iteration of the full-expansion tail
    int32_t log;            // log_visits
};

// Exact numpy pairwise-sum plan for one row length d.
struct L2Plan {
    int32_t n_leaves, n_ops;
    int16_t leaf_off[kMaxLeaves];
    int16_t leaf_len[kMaxLeaves];
    int8_t ops[kMaxOps];    // >=0 push leaf i; -1 add top two
};

struct TaskRecord {         // per-task outputs of pw_search_one
    int64_t c[6];           // iterations, dc, total_visits, nodes_expanded, dgs, inserted
    int32_t converged, retained, n_out, pad;
    int64_t n_visited;
};

struct KArgs {
    // TMA descriptors of the vector rows (main graph, ghost graph) for the
    // tile::gather4 scoring path (tma_rows): 2D {d, n} tensors, box {spad, 1}
    // -- the box is wider than a row, so columns d..spad-1 are zero-filled
    // out of bounds and the rows land at the padded, bank-conflict-free
    // staging stride without any extra traffic
    CUtensorMap tm_main, tm_ghost;
    GraphDev main, ghost;
    const int32_t* inter;   // (n,) or null
    int32_t d, W;
    int32_t spad;           // staging row stride in elements (bank-conflict-free passes)
    L2Plan plan;
    // consecutive: a task's config is (&cfg)[0 main | 1 stages >= 1 | 2 ghost]
    SearchCfg cfg;
    SearchCfg cfg_late;     // stages >= 1 (== cfg unless opt-in per-stage budgets)
    SearchCfg gcfg;
    int32_t has_late;
    int32_t fwd;            // entries forwarded per query (1 = the reference)
    int32_t ghost_on;       // run the ghost prologue when the task has no entry
    int32_t seed_mode;      // 0 neighbors, 1 mixed
    int32_t use_ghost_graph;
    uint64_t seed;
    int32_t stage;
    int64_t q0;             // first query id (RNG stream id)
    int32_t n_tasks;
    const float* queries;   // row t = task t
    const int32_t* entries; // per task or null
    int32_t* forward;       // per task or null
    const int64_t* seeds;   // explicit seed list (single search) or null
    int32_t n_seeds;
    Pcg64* rng_io;          // explicit rng state per task (single search) or null
    int32_t* out_ids;       // row t at t*out_stride
    float* out_dists;
    int32_t* out_local;     // may be null
    int64_t out_stride;
    int32_t* st32;          // [f*st_stride + t] (task-relative base) or null
    int64_t* st64;
    int64_t st_stride;
    TaskRecord* rec;        // or null
    int32_t* visit_log;
    int64_t visit_cap;
    // per-warp shared-memory layout (bytes)
    int32_t L_max, CB, BH, H, R, PG;
    int32_t pstride;        // DGS parent-row stride in elements (16-byte multiple)
    int32_t o_par;          // parents list offset in misc (words)
    int32_t o_qbits;        // DGS query-bit words (PW_DGS_LDG) offset in misc (words)
    int32_t o_q, o_qk, o_qe, o_cand, o_cslot, o_newl, o_ckey, o_bhk, o_bhp, o_vh, o_stage,
        o_misc, o_mbar, o_desc, warp_bytes;
    int32_t bulk_rows;      // vector rows may use cp.async.bulk (TMA) (d*4 % 16 == 0)
    int32_t tma_rows;       // scoring rows by TMA tile::gather4 (tuning flag 8)
    int32_t bulk_adj;       // expansion rows 16-byte aligned: 1 cp.async x16, 2 TMA bulk (flag 4)
    int32_t prefetch;       // L2-prefetch predicted parent rows
    unsigned long long* phase;  // per-phase cycle totals (PW_PHASE_TIMERS builds only)
    int32_t vis_limit;      // smem visited entries before spilling to global
    unsigned long long* gvis;  // per-warp global visited spill tables, (epoch << 32 | id)
    int32_t gmask;
    int32_t lossy;          // lossy visited cache instead of the exact set (ids exact; DC may grow)
    int32_t lshift;         // lossy cache slot = hash32(id) >> lshift
    uint32_t* gepoch;       // per-warp search epoch (tags the spill table; no clearing)
    uint32_t* gscratch;     // per-warp global scratch for choice()
    const uint64_t* jump;   // PCG64 jump-ahead table (kJumpMax entries, choice_floyd_warp)
    int64_t gscratch_words;
    int32_t* task_counter;
    int32_t* err;
    // Dataflow ring (pw_search_dataflow): one persistent launch per shard runs
    // every (stage, query) task of shard g in stage-major order; a stage-s>0
    // task waits for its entry, which shard g-1 stores straight into this
    // shard's inbox (P2P over NVLink between GPUs) when its stage s-1 search
    // ends -- no stage barriers, no host round trips (pipeline.py:327-347).
    // Overlapped query upload (pw_run): query rows arrive in geometrically
    // growing chunks (chunk c: rows [q_chunk (2^c - 1), q_chunk (2^(c+1) - 1)))
    // on a copy stream, each chunk's flag set to q_epoch after it lands; a
    // task polls its chunk's flag before reading its row.
    const uint32_t* qready;  // or null (queries already resident)
    int32_t q_chunk;
    uint32_t q_epoch;
    int32_t df;             // 1: dataflow task mapping
    int32_t df_g, df_N;
    int32_t df_lo[9];       // chunk bounds, np.array_split(arange(Q), N) (pipeline.py:327)
    int32_t df_base[9];     // first task of each stage on this shard
    uint32_t df_epoch;      // run tag carried by inbox words (no reset between runs)
    const unsigned long long* df_inbox;  // (Q,) epoch << 32 | entry, written by shard g-1
    unsigned long long* df_next;         // shard g+1's inbox (peer mapping or local)
    int64_t st32_stage_stride, st64_stage_stride;  // stats (stage, f, q) = stage*stride + f*st_stride + q
};

__device__ __forceinline__ unsigned long long ld_acquire_sys(const unsigned long long* p) {
    unsigned long long v;
    asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ uint32_t ld_acquire_gpu_u32(const uint32_t* p) {
    uint32_t v;
    asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ void st_release_sys(unsigned long long* p, unsigned long long v) {
    asm volatile("st.release.sys.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}

// ------------------------------------------------------------------ helpers
__device__ __forceinline__ unsigned lane_id() { return threadIdx.x & 31u; }
__device__ __forceinline__ unsigned lanemask_lt() {
    unsigned m;
    asm("mov.u32 %0, %%lanemask_lt;" : "=r"(m));
    return m;
}
__device__ __forceinline__ uint32_t hash32(uint32_t x) { return x * 0x9E3779B1u; }

__device__ __forceinline__ void cp_async4(void* smem, const void* gmem) {
    uint32_t s = (uint32_t)__cvta_generic_to_shared(smem);
    asm volatile("cp.async.ca.shared.global [%0], [%1], 4;\n" ::"r"(s), "l"(gmem));
}
__device__ __forceinline__ void cp_async8(void* smem, const void* gmem) {
    uint32_t s = (uint32_t)__cvta_generic_to_shared(smem);
    asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"(s), "l"(gmem));
}
__device__ __forceinline__ void cp_async16(void* smem, const void* gmem) {
    uint32_t s = (uint32_t)__cvta_generic_to_shared(smem);
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(s), "l"(gmem));
}
#ifndef PW_EVICT_FIRST
#define PW_EVICT_FIRST 1
#endif
// Streaming rows (vectors, adjacency, direction: no reuse across queries)
// carry an L2 evict-first hint so they do not push the lossy visited caches
// and the ghost graph out of L2 (C2: naive 5.36 -> 4.80 ms, PW 4.21 -> 4.05 ms;
// -DPW_EVICT_FIRST=0 builds without).
__device__ __forceinline__ uint64_t l2_evict_first_policy() {
    uint64_t pol = 0;
#if PW_EVICT_FIRST
    asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
#endif
    return pol;
}
#ifndef PW_EVICT_LAST
#define PW_EVICT_LAST 0
#endif
// Reused data -- the lossy visited caches and the ghost graph (every query's
// stage-0 search walks it) -- optionally ask L2 to keep it (evict-last).
__device__ __forceinline__ uint64_t l2_evict_last_policy() {
    uint64_t pol = 0;
#if PW_EVICT_LAST
    asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(pol));
#endif
    return pol;
}
__device__ __forceinline__ void cp_async4_keep(void* smem, const void* gmem, uint64_t pol) {
#if PW_EVICT_LAST
    asm volatile("cp.async.ca.shared.global.L2::cache_hint [%0], [%1], 4, %2;\n" ::"r"(
                     (uint32_t)__cvta_generic_to_shared(smem)), "l"(gmem), "l"(pol));
#else
    (void)pol;
    cp_async4(smem, gmem);
#endif
}
__device__ __forceinline__ void st_keep(uint32_t* p, uint32_t v, uint64_t pol) {
#if PW_EVICT_LAST
    asm volatile("st.global.cg.L2::cache_hint.b32 [%0], %1, %2;" ::"l"(p), "r"(v), "l"(pol) : "memory");
#else
    (void)pol;
    __stcg(p, v);
#endif
}
// HINT = false for the uint8-row instances: with the hint, ptxas 12.9 emits
// LDGSTS with an odd uniform descriptor register (desc[UR1]) there, which
// faults as an illegal instruction (tests/test_abi.py guards the SASS).
template <bool HINT = true>
__device__ __forceinline__ void cp_async16_stream(uint32_t s, const void* gmem, uint64_t pol) {
#if PW_EVICT_FIRST
    if constexpr (!HINT) {
        (void)pol;
        asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(s), "l"(gmem));
        return;
    }
    asm volatile("cp.async.cg.shared.global.L2::cache_hint [%0], [%1], 16, %2;\n" ::"r"(s), "l"(gmem), "l"(pol));
#else
    (void)pol;
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(s), "l"(gmem));
#endif
}
__device__ __forceinline__ void cp_commit() { asm volatile("cp.async.commit_group;\n" ::); }
template <int N>
__device__ __forceinline__ void cp_wait() {
    asm volatile("cp.async.wait_group %0;\n" ::"n"(N));
}

// ---- TMA bulk copies (cp.async.bulk, SASS UBLKCP) completing on an mbarrier
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
    return (uint32_t)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void mbar_init(uint64_t* bar) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;\n" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void mbar_fence_init() {
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
}
__device__ __forceinline__ void mbar_arrive_expect(uint64_t* bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(smem_u32(bar)),
                 "r"(bytes)
                 : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
    uint32_t done;
    do {
        asm volatile(
            "{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n"
            " selp.u32 %0, 1, 0, p;\n}\n"
            : "=r"(done)
            : "r"(smem_u32(bar)), "r"(parity)
            : "memory");
    } while (!done);
}
__device__ __forceinline__ void fence_proxy_async() {
    asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n" ::"r"(
            smem_u32(dst)),
        "l"(src), "r"(bytes), "r"(smem_u32(bar))
        : "memory");
}

// TMA tile::gather4 scoring path (tuning flag 8).  Off in the product build:
// measured at the C2 bench point (profiles/r02/ab_tma_r02m.log) the gather4
// path is slower than LDGSTS (PW 1.62 vs 1.52 ms, naive 3.22 vs 2.88 ms) and
// merely compiling it in costs 3-5% (code size / registers in the hot loop);
// build with -DPW_TMA_ROWS=1 for the A/B (tests pass either way).
#ifndef PW_DGS_LDG
#define PW_DGS_LDG 0  // DGS parent rows into registers instead of the staging ring (A/B)
#endif
#ifndef PW_QREG_F32
#define PW_QREG_F32 1  // float rows: this lane's query pairs held in registers while scoring
#endif
#ifndef PW_DGS_QREG
#define PW_DGS_QREG 1  // DGS: the query elements in registers across the parent loop (0.7% on C2 K1, ab_qr8_s17.log)
#endif
#ifndef PW_DGS_PUNROLL
#define PW_DGS_PUNROLL 1  // DGS parent loop unrolled by 2 (A/B)
#endif
#ifndef PW_TMA_ROWS
#define PW_TMA_ROWS 0
#endif
// elect.sync: one lane of the warp; ptxas knows the region is single-threaded,
// so per-lane values feed TMA's uniform operands with a plain R2UR (an
// `if (lane == 0)` region makes it emit a lane waterfall instead)
__device__ __forceinline__ bool elect_one() {
    uint32_t pred = 0;
    asm volatile("{\n .reg .pred P;\n elect.sync _|P, 0xffffffff;\n selp.u32 %0, 1, 0, P;\n}\n" : "=r"(pred));
    return pred != 0;
}
// TMA tile::gather4: 4 rows (row coordinates r0..r3, -1 = out of bounds,
// zero-filled, no traffic) x box columns from column 0 into dst, completing
// on bar (SASS UTMALDG.2D.GATHER4)
__device__ __forceinline__ void tma_gather4(void* dst, const CUtensorMap* tm, int32_t r0, int32_t r1, int32_t r2,
                                            int32_t r3, uint64_t* bar, uint64_t pol) {
    asm volatile(
        "cp.async.bulk.tensor.2d.shared::cta.global.tile::gather4.mbarrier::complete_tx::bytes.L2::cache_hint"
        " [%0], [%1, {%2, %3, %4, %5, %6}], [%7], %8;\n" ::"r"(smem_u32(dst)),
        "l"(tm), "r"(0), "r"(r0), "r"(r1), "r"(r2), "r"(r3), "r"(smem_u32(bar)), "l"(pol)
        : "memory");
}

// ---- warp-wide bitonic sorts (ascending across lanes)
__device__ __forceinline__ uint64_t warp_sort_u64(uint64_t x) {
    // rolled network (15 compare-exchange stages): compact code for the
    // instruction caches; the stage parameters are uniform
    const unsigned lane = threadIdx.x & 31u;
#pragma unroll 1
    for (int k = 2; k <= 32; k <<= 1)
#pragma unroll 1
        for (int j = k >> 1; j > 0; j >>= 1) {
            uint64_t o = __shfl_xor_sync(0xffffffffu, x, j);
            bool keep_min = ((lane & j) == 0) == ((lane & k) == 0);
            x = keep_min ? (o < x ? o : x) : (o > x ? o : x);
        }
    return x;
}
// 64 keys, element i = 32*e + lane in register x[e]: bitonic network with
// the j = 32 stage as an in-lane compare-exchange (ascending across i)
__device__ __forceinline__ void warp_sort2_u64(uint64_t& x0, uint64_t& x1) {
    const unsigned lane = threadIdx.x & 31u;
#pragma unroll 1
    for (int k = 2; k <= 32; k <<= 1)
#pragma unroll 1
        for (int j = k >> 1; j > 0; j >>= 1) {
            // element lane ascends iff (lane & k) == 0; element 32 + lane has
            // the k = 32 bit set, so it descends at k = 32 (bitonic 64)
            const uint64_t o0 = __shfl_xor_sync(0xffffffffu, x0, j);
            const uint64_t o1 = __shfl_xor_sync(0xffffffffu, x1, j);
            const bool lo = (lane & j) == 0;
            const bool asc0 = (lane & k) == 0;
            const bool asc1 = k == 32 ? false : asc0;
            x0 = (lo == asc0) ? (o0 < x0 ? o0 : x0) : (o0 > x0 ? o0 : x0);
            x1 = (lo == asc1) ? (o1 < x1 ? o1 : x1) : (o1 > x1 ? o1 : x1);
        }
    {
        const uint64_t a = x0 < x1 ? x0 : x1, b = x0 < x1 ? x1 : x0;
        x0 = a;
        x1 = b;
    }
#pragma unroll 1
    for (int j = 16; j > 0; j >>= 1) {
        const uint64_t o0 = __shfl_xor_sync(0xffffffffu, x0, j);
        const uint64_t o1 = __shfl_xor_sync(0xffffffffu, x1, j);
        const bool lo = (lane & j) == 0;
        x0 = lo ? (o0 < x0 ? o0 : x0) : (o0 > x0 ? o0 : x0);
        x1 = lo ? (o1 < x1 ? o1 : x1) : (o1 > x1 ? o1 : x1);
    }
}
__device__ __forceinline__ uint32_t warp_sort_u32(uint32_t x) {
    const unsigned lane = threadIdx.x & 31u;
#pragma unroll
    for (int k = 2; k <= 32; k <<= 1)
#pragma unroll
        for (int j = k >> 1; j > 0; j >>= 1) {
            uint32_t o = __shfl_xor_sync(0xffffffffu, x, j);
            bool keep_min = ((lane & j) == 0) == ((lane & k) == 0);
            x = keep_min ? min(o, x) : max(o, x);
        }
    return x;
}

// Warp-cooperative async copy of `bytes` (multiple of 4) into shared memory.
__device__ __forceinline__ void warp_copy_async(void* dst, const void* src, int bytes) {
    const unsigned lane = lane_id();
    uintptr_t a = (uintptr_t)src | (uintptr_t)__cvta_generic_to_shared(dst);
    if (((a | (uintptr_t)bytes) & 15u) == 0) {
        for (int c = lane; c < (bytes >> 4); c += 32)
            cp_async16((char*)dst + 16 * c, (const char*)src + 16 * c);
    } else if (((a | (uintptr_t)bytes) & 7u) == 0) {
        for (int c = lane; c < (bytes >> 3); c += 32)
            cp_async8((char*)dst + 8 * c, (const char*)src + 8 * c);
    } else {
        for (int c = lane; c < (bytes >> 2); c += 32)
            cp_async4((char*)dst + 4 * c, (const char*)src + 4 * c);
    }
}

__device__ __forceinline__ void prefetch_l2(const void* p) {
    asm volatile("prefetch.global.L2 [%0];" ::"l"(p));
}

// Vector element types: float32 rows, or uint8 rows (SIFT-style bvecs) that
// the reference upcasts to float32 (data.py:36) -- float(b) is exact, so the
// arithmetic after the load is identical.
template <typename VT>
__device__ __forceinline__ const VT* vrow(const GraphDev& G, uint32_t id, int d) {
    return reinterpret_cast<const VT*>(G.vec) + (size_t)id * d;
}
__device__ __forceinline__ float to_f(float x) { return x; }
__device__ __forceinline__ float to_f(uint8_t x) { return (float)x; }

__device__ __forceinline__ float sqd(float x, float q) {
    float df = __fsub_rn(x, q);
    return __fmul_rn(df, df);
}

// (x - q)^2 for two lanes of a float2 with packed sub.rn/mul.rn.f32x2 (SASS
// FADD2/FMUL2; each half rounds exactly like the scalar __fsub_rn/__fmul_rn)
__device__ __forceinline__ float2 sqd2(float2 x, float2 q) {
    unsigned long long xv = *reinterpret_cast<const unsigned long long*>(&x);
    unsigned long long qv = *reinterpret_cast<const unsigned long long*>(&q);
    unsigned long long d, r;
    asm("sub.rn.f32x2 %0, %1, %2;" : "=l"(d) : "l"(xv), "l"(qv));
    asm("mul.rn.f32x2 %0, %1, %1;" : "=l"(r) : "l"(d));
    return *reinterpret_cast<const float2*>(&r);
}

// Metric element op, summed in the numpy pairwise order: M = 0 squared L2
// (data.py:70-79, the reference's only metric); M = 1 inner product
// (BASELINE C5, an extension -- parity unpinned): x*q, and the distance is
// the negated sum so that smaller is better everywhere.
template <int M>
__device__ __forceinline__ float eop(float x, float q) {
    if constexpr (M == 0) return sqd(x, q);
    else return __fmul_rn(x, q);
}
template <int M>
__device__ __forceinline__ float2 eop2(float2 x, float2 q) {
    if constexpr (M == 0) {
        return sqd2(x, q);
    } else {
        unsigned long long xv = *reinterpret_cast<const unsigned long long*>(&x);
        unsigned long long qv = *reinterpret_cast<const unsigned long long*>(&q);
        unsigned long long r;
        asm("mul.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(xv), "l"(qv));
        return *reinterpret_cast<const float2*>(&r);
    }
}
template <int M>
__device__ __forceinline__ float finish(float sum) { return M == 0 ? sum : -sum; }
// Queue keys: distance bits << 32 | id.  L2 distances are >= 0, so raw bits
// order like the floats; IP distances can be negative: sign-flip transform.
template <int M>
__device__ __forceinline__ uint32_t dist_bits(float d) {
    uint32_t b = __float_as_uint(d);
    if constexpr (M == 0) {
        return b;
    } else {
        if (b == 0x80000000u) b = 0u;  // -0 == +0 as floats (the oracle compares floats)
        return (b & 0x80000000u) ? ~b : (b | 0x80000000u);
    }
}
template <int M>
__device__ __forceinline__ float bits_dist(uint32_t k) {
    if constexpr (M == 0) return __uint_as_float(k);
    else return __uint_as_float((k & 0x80000000u) ? (k & 0x7FFFFFFFu) : ~k);
}

// numpy pairwise_sum leaf over squared differences, lanes (v, a=lane&7)
// hold accumulator a; every lane of the 8-lane group ends with the leaf sum.
template <int M, typename VT>
__device__ __forceinline__ float l2_leaf(const VT* x, const float* q, int off, int len, unsigned a) {
    if (len < 8) {
        float s = 0.f;
        for (int i = 0; i < len; i++) s = __fadd_rn(s, eop<M>(to_f(x[off + i]), q[off + i]));
        return s;
    }
    const int nf = len - (len & 7);
    float acc = eop<M>(to_f(x[off + a]), q[off + a]);
    for (int i = off + (int)a + 8; i < off + nf; i += 8) acc = __fadd_rn(acc, eop<M>(to_f(x[i]), q[i]));
    acc = __fadd_rn(acc, __shfl_xor_sync(0xffffffffu, acc, 1));
    acc = __fadd_rn(acc, __shfl_xor_sync(0xffffffffu, acc, 2));
    acc = __fadd_rn(acc, __shfl_xor_sync(0xffffffffu, acc, 4));
    for (int i = off + nf; i < off + len; i++) acc = __fadd_rn(acc, eop<M>(to_f(x[i]), q[i]));
    return acc;
}

// Pairwise-ordered sum over a row (runtime plan), metric-finished.
template <int M, typename VT>
__device__ __forceinline__ float l2_row(const L2Plan& P, const VT* x, const float* q, unsigned a) {
    if (P.n_leaves == 1) return finish<M>(l2_leaf<M>(x, q, 0, P.leaf_len[0], a));
    float stack[8];
    int sp = 0;
    for (int o = 0; o < P.n_ops; o++) {
        int op = P.ops[o];
        if (op >= 0) {
            stack[sp++] = l2_leaf<M>(x, q, P.leaf_off[op], P.leaf_len[op], a);
        } else {
            float b = stack[--sp];
            float t = stack[--sp];
            stack[sp++] = __fadd_rn(t, b);
        }
    }
    return finish<M>(stack[0]);
}

// Same order with 4 lanes per row (8 rows per warp pass): lane c = lane&3
// owns accumulators 2c, 2c+1 (one float2 per 8-element step); the xor-1 and
// xor-2 shuffles form ((r0+r1)+(r2+r3)) + ((r4+r5)+(r6+r7)).
template <int M, int OFF, int N>
__device__ __forceinline__ float pw_leaf4(const float* x, const float* q, unsigned c) {
    if constexpr (N < 8) {
        float s = 0.f;
#pragma unroll
        for (int i = 0; i < N; i++) s = __fadd_rn(s, eop<M>(x[OFF + i], q[OFF + i]));
        return s;
    } else {
        constexpr int NF = N - (N % 8);
        const float2* x2 = reinterpret_cast<const float2*>(x + OFF);
        const float2* q2 = reinterpret_cast<const float2*>(q + OFF);
        // packed FADD2/FMUL2 for (x - q)^2 on both accumulators; the adds stay
        // scalar so ptxas cannot contract mul+add into FFMA2 (bit-exactness)
        float2 sq = eop2<M>(x2[c], q2[c]);
        float r0 = sq.x, r1 = sq.y;
#pragma unroll
        for (int p = 1; p < NF / 8; p++) {
            sq = eop2<M>(x2[4 * p + c], q2[4 * p + c]);
            r0 = __fadd_rn(r0, sq.x);
            r1 = __fadd_rn(r1, sq.y);
        }
        float a = __fadd_rn(r0, r1);
        a = __fadd_rn(a, __shfl_xor_sync(0xffffffffu, a, 1));
        float s = __fadd_rn(a, __shfl_xor_sync(0xffffffffu, a, 2));
#pragma unroll
        for (int i = NF; i < N; i++) s = __fadd_rn(s, eop<M>(x[OFF + i], q[OFF + i]));
        return s;
    }
}

// pw_leaf4 for a whole row of N <= 128 (N % 8 == 0) with this lane's query
// pairs already in registers (qr[p] = q2[4p + c]): half the shared loads.
template <int M, int N>
__device__ __forceinline__ float pw_row4_qreg(const float* x, const float2 (&qr)[N / 8], unsigned c) {
    const float2* x2 = reinterpret_cast<const float2*>(x);
    // packed FADD2/FMUL2 for (x - q)^2; the adds stay scalar: ptxas contracts
    // mul.rn.f32x2 + add.rn.f32x2 into FFMA2 (measured), which is not exact
    float2 sq = eop2<M>(x2[c], qr[0]);
    float r0 = sq.x, r1 = sq.y;
#pragma unroll
    for (int p = 1; p < N / 8; p++) {
        sq = eop2<M>(x2[4 * p + c], qr[p]);
        r0 = __fadd_rn(r0, sq.x);
        r1 = __fadd_rn(r1, sq.y);
    }
    float a = __fadd_rn(r0, r1);
    a = __fadd_rn(a, __shfl_xor_sync(0xffffffffu, a, 1));
    return finish<M>(__fadd_rn(a, __shfl_xor_sync(0xffffffffu, a, 2)));
}

// Same for uint8 rows: lane c reads its two bytes of every 8-byte step
// (LDS.U16), rebuilds float(b) exactly as (2^23 + b) - 2^23 (PRMT + FADD2,
// full-rate ALUs instead of I2F), then the float32 ops of pw_row4_qreg.
template <int M, int N>
__device__ __forceinline__ float pw_row4_u8(const uint8_t* x, const float2 (&qr)[N / 8], unsigned c) {
    const uint16_t* x2 = reinterpret_cast<const uint16_t*>(x);
    const float2 big = make_float2(8388608.f, 8388608.f);
    auto ld = [&](int p) -> float2 {
        const uint32_t w = x2[4 * p + c];
        const float2 f = make_float2(__uint_as_float(__byte_perm(w, 0x4B000000u, 0x7540)),
                                     __uint_as_float(__byte_perm(w, 0x4B000000u, 0x7541)));
        unsigned long long fv = *reinterpret_cast<const unsigned long long*>(&f);
        unsigned long long bv = *reinterpret_cast<const unsigned long long*>(&big);
        unsigned long long r;
        asm("sub.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(fv), "l"(bv));
        return *reinterpret_cast<const float2*>(&r);
    };
    float2 sq = eop2<M>(ld(0), qr[0]);
    float r0 = sq.x, r1 = sq.y;
#pragma unroll
    for (int p = 1; p < N / 8; p++) {
        sq = eop2<M>(ld(p), qr[p]);
        r0 = __fadd_rn(r0, sq.x);
        r1 = __fadd_rn(r1, sq.y);
    }
    float a = __fadd_rn(r0, r1);
    a = __fadd_rn(a, __shfl_xor_sync(0xffffffffu, a, 1));
    return finish<M>(__fadd_rn(a, __shfl_xor_sync(0xffffffffu, a, 2)));
}

// uint8 rows against an integer-valued query in [0, 255] (the SIFT case):
// every (x - q)^2 is an exact integer <= 65025 and every partial sum of <= 258
// of them stays below 2^24, so numpy's float32 pairwise sum IS the exact
// integer sum, in any order.  Computed as sum x^2 - 2 sum x q + sum q^2 with
// DP4A (4 bytes per instruction) and converted once -- bit-identical to
// pw_row4_u8.  Lane c owns words 4p + c of the row.
template <int N>
__device__ __forceinline__ float pw_row4_u8i(const uint8_t* x, const uint32_t (&qw)[N / 16], unsigned c,
                                             int qsq) {
    const uint32_t* xw = reinterpret_cast<const uint32_t*>(x);
    unsigned sxx = 0, sxq = 0;
#pragma unroll
    for (int p = 0; p < N / 16; p++) {
        const uint32_t w = xw[4 * p + c];
        sxx = __dp4a(w, w, sxx);
        sxq = __dp4a(w, qw[p], sxq);
    }
    int t = (int)sxx - 2 * (int)sxq;
    t += __shfl_xor_sync(0xffffffffu, t, 1);
    t += __shfl_xor_sync(0xffffffffu, t, 2);
    return (float)(t + qsq);
}

template <int M, int OFF, int N>
__device__ __forceinline__ float pw_sum4(const float* x, const float* q, unsigned c) {
    if constexpr (N <= 128) {
        return pw_leaf4<M, OFF, N>(x, q, c);
    } else {
        constexpr int N2 = N / 2 - (N / 2) % 8;
        float a = pw_sum4<M, OFF, N2>(x, q, c);
        float b = pw_sum4<M, OFF + N2, N - N2>(x, q, c);
        return __fadd_rn(a, b);
    }
}


// --------------------------------------------------------------- per warp
struct WarpState {
    float* q;
    uint64_t* qk0;          // the size-l queue (keys, sorted) -- merged in place
    uint8_t* qe0;           // expanded flags
    int32_t* cand;
    int32_t* cslot;
    int32_t* newl;
    uint64_t* ckey;
    uint32_t* bhk;
    int32_t* bhp;
    uint32_t* vh;
    float* stage;
    int32_t* misc;
    unsigned long long* gvis;
    uint32_t* gscr;
    uint32_t epoch;         // this search's spill-table tag (0 never used)
#ifdef PW_PHASE_TIMERS
    long long pc[8];        // cycles: init, score, merge, select, expand, dedup, visited, tail
#endif
    uint64_t* mbar;         // [0],[1] gather halves, [2] expansion fetch
    uint4* desc;            // bulk-copy descriptors of one expansion fetch (<= 32)
    uint32_t phase;         // parity bit per mbarrier
    int32_t cur;            // current queue buffer
    __device__ __forceinline__ uint64_t* qk_cur() const { return qk0; }
    __device__ __forceinline__ uint8_t* qe_cur() const { return qe0; }
    int32_t qlen;
    int32_t fu;             // first queue position that may be unexpanded
    int32_t vcount;         // entries in the smem visited table
    bool ovf;               // visited set spilled to the global table
    // per-search counters, 32-bit (prepare() rejects budgets that could
    // overflow them); StageStats accumulate them as int64
    int32_t c_it, c_dc, c_tv, c_ne, c_dgs, c_ins;
};

__device__ __forceinline__ uint32_t bh_insert(const KArgs& A, WarpState& S, uint32_t id) {
    const uint32_t mask = (uint32_t)A.BH - 1u;
    uint32_t h = hash32(id) & mask;
    for (int probe = 0; probe <= A.BH; probe++) {
        uint32_t old = atomicCAS(&S.bhk[h], kEmpty, id);
        if (old == kEmpty || old == id) return h;
        h = (h + 1u) & mask;
    }
    atomicOr(A.err, 2);  // batch table full: impossible when BH >= 2*CB
    return h;
}

__device__ __forceinline__ bool bh_contains(const KArgs& A, const WarpState& S, uint32_t id) {
    const uint32_t mask = (uint32_t)A.BH - 1u;
    uint32_t h = hash32(id) & mask;
    for (int probe = 0; probe <= A.BH; probe++) {
        uint32_t v = S.bhk[h];
        if (v == id) return true;
        if (v == kEmpty) return false;
        h = (h + 1u) & mask;
    }
    return false;
}

// KEYS_ONLY: only the key half (dedup_unordered's table; the position half
// is read by dedup_ordered and the exact global visited path alone)
template <bool KEYS_ONLY = false>
__device__ __forceinline__ void bh_clear(const KArgs& A, WarpState& S) {
    uint4* k4 = reinterpret_cast<uint4*>(S.bhk);
    uint4* p4 = reinterpret_cast<uint4*>(S.bhp);
    const uint4 e = make_uint4(kEmpty, kEmpty, kEmpty, kEmpty);
    const uint4 m = make_uint4(0x7FFFFFFFu, 0x7FFFFFFFu, 0x7FFFFFFFu, 0x7FFFFFFFu);
#pragma unroll 1
    for (int i = lane_id(); i < (A.BH >> 2); i += 32) {
        k4[i] = e;
        if (!KEYS_ONLY) p4[i] = m;
    }
    __syncwarp();
}

// Ordered first-occurrence dedup of src[0..n) keeping the first `limit`
// unique ids, written to dst (search.py:219 dict.fromkeys / :230-232
// _ordered_unique + [:cap]).  Returns the kept count; bh stays populated.
static __device__ int dedup_ordered(const KArgs& A, WarpState& S, const int32_t* src, int n, int limit,
                             int32_t* dst, int* n_unique) {
    const unsigned lane = lane_id();
    for (int t = lane; t < n; t += 32) {
        uint32_t slot = bh_insert(A, S, (uint32_t)src[t]);
        atomicMin(&S.bhp[slot], t);
        S.cslot[t] = (int32_t)slot;
    }
    __syncwarp();
    int cnt = 0;
    for (int base = 0; base < n; base += 32) {
        int t = base + lane;
        bool f = t < n && S.bhp[S.cslot[t]] == t;
        unsigned b = __ballot_sync(0xffffffffu, f);
        int pos = cnt + __popc(b & lanemask_lt());
        if (f && pos < limit) dst[pos] = src[t];
        cnt += __popc(b);
    }
    __syncwarp();
    *n_unique = cnt;
    return cnt < limit ? cnt : limit;
}

// Same set and count as dedup_ordered when nothing is truncated (n <= cap)
// and no visit log is kept: order inside the batch does not change any result
// (scores are merged by key), so one CAS pass with two candidates in flight
// per lane replaces insert + atomicMin + the ordered second pass.  Needs a
// clear bhk; leaves it populated.
static __device__ int dedup_unordered(const KArgs& A, WarpState& S, const int32_t* src, int n,
                                      int32_t* dst, uint32_t mask) {
    const unsigned lane = lane_id();
    int cnt = 0;
    for (int base = 0; base < n; base += 64) {
        const int t0 = base + (int)lane, t1 = t0 + 32;
        // idle lanes: o == id (not kEmpty) skips the probe loop and the ballot
        const uint32_t id0 = t0 < n ? (uint32_t)src[t0] : 0u;
        const uint32_t id1 = t1 < n ? (uint32_t)src[t1] : 0u;
        uint32_t h0 = hash32(id0) & mask, h1 = hash32(id1) & mask;
        uint32_t o0 = t0 < n ? atomicCAS(&S.bhk[h0], kEmpty, id0) : id0;
        uint32_t o1 = t1 < n ? atomicCAS(&S.bhk[h1], kEmpty, id1) : id1;
        while (o0 != kEmpty && o0 != id0) {
            h0 = (h0 + 1u) & mask;
            o0 = atomicCAS(&S.bhk[h0], kEmpty, id0);
        }
        while (o1 != kEmpty && o1 != id1) {
            h1 = (h1 + 1u) & mask;
            o1 = atomicCAS(&S.bhk[h1], kEmpty, id1);
        }
        const unsigned b0 = __ballot_sync(0xffffffffu, o0 == kEmpty);
        const unsigned b1 = __ballot_sync(0xffffffffu, o1 == kEmpty);
        if (o0 == kEmpty) dst[cnt + __popc(b0 & lanemask_lt())] = (int32_t)id0;
        cnt += __popc(b0);
        if (o1 == kEmpty) dst[cnt + __popc(b1 & lanemask_lt())] = (int32_t)id1;
        cnt += __popc(b1);
    }
    __syncwarp();
    return cnt;
}

// Exact visited-set insert-if-absent (search.py:167, :300-303).
__device__ __forceinline__ bool visit_insert(const KArgs& A, WarpState& S, uint32_t id) {
    const uint32_t hm = (uint32_t)A.H - 1u;
    uint32_t h = hash32(id) & hm;
    int probe = 0;
    for (; probe <= A.H; probe++) {
        uint32_t v = S.vh[h];
        if (v == id) return false;
        if (v == kEmpty) break;
        h = (h + 1u) & hm;
    }
    if (!S.ovf) {
        for (; probe <= A.H; probe++) {
            uint32_t old = atomicCAS(&S.vh[h], kEmpty, id);
            if (old == kEmpty) return true;
            if (old == id) return false;
            h = (h + 1u) & hm;
        }
        atomicOr(A.err, 4);  // smem visited table full: impossible below vis_limit
        return false;
    }
    // spilled: per-warp global table whose entries carry the search epoch, so
    // stale entries of earlier searches read as empty and nothing is cleared
    const uint32_t gm = (uint32_t)A.gmask;
    const unsigned long long want = ((unsigned long long)S.epoch << 32) | id;
    uint32_t g = (hash32(id ^ 0x5bd1e995u) >> 3) & gm;
    for (uint32_t gp = 0; gp <= gm;) {
        unsigned long long v = S.gvis[g];
        if (v == want) return false;
        if ((uint32_t)(v >> 32) != S.epoch) {
            unsigned long long old = atomicCAS(&S.gvis[g], v, want);
            if (old == v) return true;
            if (old == want) return false;
            continue;  // slot changed under us: re-examine it
        }
        g = (g + 1u) & gm;
        gp++;
    }
    atomicOr(A.err, 8);  // global visited table full
    return false;
}

__device__ __forceinline__ bool smem_lookup(const KArgs& A, const WarpState& S, uint32_t id) {
    const uint32_t hm = (uint32_t)A.H - 1u;
    uint32_t h = hash32(id) & hm;
    for (int probe = 0; probe <= A.H; probe++) {
        const uint32_t v = S.vh[h];
        if (v == id) return true;
        if (v == kEmpty) return false;
        h = (h + 1u) & hm;
    }
    return false;
}

// Linear-probing insert-if-absent into the epoch-tagged spill table, starting
// at slot g whose current content is cur (the rare collision path).
static __device__ __noinline__ bool probe_insert(unsigned long long* gvis, uint32_t gm, uint32_t epoch,
                                                 uint32_t id, uint32_t g, unsigned long long cur,
                                                 int32_t* err) {
    const unsigned long long want = ((unsigned long long)epoch << 32) | id;
    for (uint32_t gp = 0; gp <= gm;) {
        if (cur == want) return false;
        if ((uint32_t)(cur >> 32) != epoch) {
            const unsigned long long o = atomicCAS(&gvis[g], cur, want);
            if (o == cur) return true;
            cur = o;
            continue;
        }
        g = (g + 1u) & gm;
        gp++;
        cur = __ldcg(&gvis[g]);
    }
    atomicOr(err, 8);  // global visited table full
    return false;
}

// Lossy visited filter (tuning flag 2): a per-warp direct-mapped cache of
// 32-bit words in global memory, small enough to stay in L2.  With h =
// hash32(id) (a bijection: odd multiplier mod 2^32) and 2^s slots, the slot
// is h's top s bits and the word is epoch8 << 24 | h's low 32 - s bits, so
// (slot, word) names the id exactly for any 32-bit id when s >= 8
// (4096 slots = 16 KB per warp: measured faster than 8192 / 16384 despite
// ~3% more re-scores -- the L2 footprint matters).  One round trip, no atomics: every miss is
// stored (overwrites allowed) and scored.  Results stay identical to the
// exact set: a forgotten node that is re-scored either is still queued --
// the merge finds its identical key and drops it -- or was dropped from /
// never entered the queue, so its key is above the (non-increasing) l-th key
// and it cannot survive.  Only distance_computations can exceed the
// reference's.  A hit is never false: tags are unique per search and the
// cache is cleared when the 8-bit epoch wraps.
static __device__ __forceinline__ int visited_lossy(const KArgs& A, WarpState& S, int nb) {
    // all probes in flight at once as 4-byte LDGSTS into the (free until
    // scoring) key area, then one compact pass: rolled loops, no register
    // arrays (the hot loop has to stay within the instruction caches)
    const unsigned lane = lane_id();
    uint32_t* tab = reinterpret_cast<uint32_t*>(S.gvis);
    uint32_t* vs = reinterpret_cast<uint32_t*>(S.ckey);
    const uint32_t tag = S.epoch << 24;
    const uint32_t lmask = (1u << A.lshift) - 1u;  // low 32 - s bits of h
    const uint64_t keep = l2_evict_last_policy();
#pragma unroll 1
    for (int t = lane; t < nb; t += 32) cp_async4_keep(vs + t, tab + (hash32((uint32_t)S.newl[t]) >> A.lshift), keep);
    cp_commit();
    cp_wait<0>();
    __syncwarp();
    int cnt = 0;
#pragma unroll 1
    for (int base = 0; base < nb; base += 32) {
        const int t = base + (int)lane;
        const uint32_t id = t < nb ? (uint32_t)S.newl[t] : 0u;
        const uint32_t h = hash32(id);
        const bool fresh = t < nb && vs[t] != (tag | (h & lmask));
        if (fresh) st_keep(&tab[h >> A.lshift], tag | (h & lmask), keep);
        const unsigned b = __ballot_sync(0xffffffffu, fresh);
        if (fresh) S.newl[cnt + __popc(b & lanemask_lt())] = (int32_t)id;
        cnt += __popc(b);
    }
    __syncwarp();
    return cnt;
}

// Keep only never-scored ids of newl[0..nb) (in order); returns n_new.
// Until the shared-memory table would pass vis_limit, inserts go there
// (one CAS each, no global traffic).  After the spill, every candidate not in
// the (now read-only) shared table is resolved against the per-warp global
// epoch table with all of a lane's probes in flight at once: first-slot
// loads, then CASes, then (rarely) linear-probing retries.
// GLOBAL_ONLY (the specialised kernels): the shared table is skipped and every
// probe goes to the per-warp epoch table, so only the batched-probe path below
// is compiled into the hot loop.
// FAST kernel instances (host-selected per launch, prepare()): the launch
// uses the lossy visited cache, full or direction-guided selection and
// degrees <= 32, so the exact visited path, the random-selection arm and the
// shared-memory DGS path for wide degrees are compiled out -- 19% less code
// in the hot loop's address range, measured 6% (PathWeaver) / 2% (naive)
// faster at the C2 bench point (profiles/r02/ab_cold_r02z.log).
template <bool GLOBAL_ONLY, bool FAST = false>
__device__ int visited_filter(const KArgs& A, WarpState& S, int nb) {
    if (FAST || A.lossy) return visited_lossy(A, S, nb);
    const unsigned lane = lane_id();
    if (!GLOBAL_ONLY && !S.ovf && S.vcount + nb > A.vis_limit) S.ovf = true;
    int cnt = 0;
    if (!GLOBAL_ONLY && !S.ovf) {
        for (int base = 0; base < nb; base += 32) {
            int t = base + lane;
            int32_t id = t < nb ? S.newl[t] : -1;
            bool f = t < nb && visit_insert(A, S, (uint32_t)id);
            unsigned b = __ballot_sync(0xffffffffu, f);
            int pos = cnt + __popc(b & lanemask_lt());
            if (f) S.newl[pos] = id;
            cnt += __popc(b);
        }
        __syncwarp();
        S.vcount += cnt;
        return cnt;
    }
    constexpr int K = 4;
    const uint32_t gm = (uint32_t)A.gmask;
    for (int base0 = 0; base0 < nb; base0 += 32 * K) {
        int32_t id[K];
        uint32_t slot[K], sh[K];
        unsigned long long v[K];
        bool pend[K], fresh[K];
#pragma unroll
        for (int k = 0; k < K; k++) {
            const int t = base0 + k * 32 + (int)lane;
            id[k] = t < nb ? S.newl[t] : -1;
            pend[k] = t < nb && (GLOBAL_ONLY || !smem_lookup(A, S, (uint32_t)id[k]));
            slot[k] = (hash32((uint32_t)id[k] ^ 0x5bd1e995u) >> 3) & gm;
            // count how many candidates of this batch share a home slot
            // (shared-memory hash; the ordered-dedup table is free here)
            sh[k] = pend[k] ? bh_insert(A, S, slot[k]) : 0u;
            if (pend[k]) atomicAdd(&S.bhp[sh[k]], 1);
            v[k] = pend[k] ? __ldcg(&S.gvis[slot[k]]) : 0ull;  // one round trip for all
            fresh[k] = false;
        }
        __syncwarp();
        // fast path: a stale home slot claimed by exactly one candidate gets a
        // plain (fire-and-forget) store; found == already visited
#pragma unroll
        for (int k = 0; k < K; k++) {
            if (!pend[k]) continue;
            const unsigned long long want = ((unsigned long long)S.epoch << 32) | (uint32_t)id[k];
            const bool alone = (uint32_t)S.bhp[sh[k]] == 0x80000000u;  // 0x7FFFFFFF + one add
            if (v[k] == want) {
                pend[k] = false;
            } else if (alone && (uint32_t)(v[k] >> 32) != S.epoch) {
                __stcg(&S.gvis[slot[k]], want);
                pend[k] = false;
                fresh[k] = true;
            }
        }
        __syncwarp();  // the plain stores are ordered before any CAS below
        // slow path (occupied or shared home slot): CAS + linear probing
#pragma unroll
        for (int k = 0; k < K; k++)
            if (pend[k])
                fresh[k] = probe_insert(S.gvis, gm, S.epoch, (uint32_t)id[k], slot[k],
                                        __ldcg(&S.gvis[slot[k]]), A.err);
#pragma unroll
        for (int k = 0; k < K; k++) {
            const unsigned b = __ballot_sync(0xffffffffu, fresh[k]);
            const int pos = cnt + __popc(b & lanemask_lt());
            if (fresh[k]) S.newl[pos] = id[k];
            cnt += __popc(b);
        }
        bh_clear(A, S);
    }
    __syncwarp();
    return cnt;
}

// Gather rows newl[0..n) and compute exact squared L2 keys into ckey.
// D > 0: rows land in shared memory by TMA bulk copies (one lane per row,
// completion on a per-half mbarrier, two halves in flight), and 16 rows are
// reduced per warp pass in the compile-time pairwise order.  D == 0: generic
// d (cp.async + runtime pairwise plan).
template <int D, typename VT, int M, bool QI = false, bool QREG_OK = true>
__device__ int score_rows(const KArgs& A, WarpState& S, const GraphDev& G, int n, uint64_t thr) {
    const unsigned lane = lane_id();
    int ns = 0;  // survivors (key < thr, search.py:182-184) compacted into ckey as produced
    const int RH = A.R >> 1;
    const int sp = A.spad;
    const int ngroups = (n + RH - 1) / RH;
    if constexpr (D > 0) {
        constexpr uint32_t row_bytes = D * (uint32_t)sizeof(VT);
        constexpr int CPR = row_bytes / 16;  // 16-byte chunks per row
        // the ghost graph's rows are reused by every query: not streaming
        const uint64_t pol = (PW_EVICT_LAST && G.vec == A.ghost.vec) ? l2_evict_last_policy()
                                                                     : l2_evict_first_policy();
        const bool tma = PW_TMA_ROWS && A.tma_rows != 0;
        const CUtensorMap* tm = G.vec == A.ghost.vec ? &A.tm_ghost : &A.tm_main;
        if (tma) fence_proxy_async();  // the ring was last written / read by the generic proxy
        auto issue = [&](int g) {
            if (g < ngroups && tma) {
                // one elected lane: ceil(rows / 4) gather4 copies into half g & 1
                const int r0 = g * RH;
                const int rows = min(RH, n - r0);
                VT* dst0 = reinterpret_cast<VT*>(S.stage) + (size_t)(g & 1) * RH * sp;
                uint64_t* bar = S.mbar + (g & 1);
                if (elect_one()) {
                    const int n4 = (rows + 3) >> 2;
                    mbar_arrive_expect(bar, (uint32_t)(n4 * 4 * sp * (int)sizeof(VT)));
#pragma unroll 1
                    for (int i = 0; i < n4; i++) {
                        const int b = r0 + 4 * i;
                        const int c = rows - 4 * i;
                        tma_gather4(dst0 + (size_t)(4 * i) * sp, tm, S.newl[b], c > 1 ? S.newl[b + 1] : -1,
                                    c > 2 ? S.newl[b + 2] : -1, c > 3 ? S.newl[b + 3] : -1, bar, pol);
                    }
                }
                __syncwarp();
            } else if (g < ngroups) {
                const int r0 = g * RH;
                const int rows = min(RH, n - r0);
                VT* dst0 = reinterpret_cast<VT*>(S.stage) + (size_t)(g & 1) * RH * sp;
                // LDGSTS: LPR lanes per row, CPL 16-byte chunks per lane
                constexpr int LPR = CPR <= 32 ? 8 : 32;
                constexpr int CPL = (CPR + LPR - 1) / LPR;
                constexpr int RPP = 32 / LPR;
                const int sub = (int)lane % LPR;
                for (int r = (int)lane / LPR; r < rows; r += RPP) {
                    const VT* src = vrow<VT>(G, (uint32_t)S.newl[r0 + r], D);
                    VT* dst = dst0 + (size_t)r * sp;
#pragma unroll
                    for (int k = 0; k < CPL; k++) {
                        const int ch = sub + k * LPR;
                        if (CPR % LPR == 0 || ch < CPR)
                            cp_async16_stream<sizeof(VT) != 1>((uint32_t)__cvta_generic_to_shared(dst + (16 / sizeof(VT)) * ch),
                                              src + (16 / sizeof(VT)) * ch, pol);
                    }
                }
            }
            cp_commit();
        };
        const unsigned v = lane >> 2, c = lane & 3u;
        // float rows: query pairs in registers, except in the 96-register
        // 20-warp build, where reading them from shared memory measured
        // faster (ab_qreg_r02am.log)
        constexpr bool QREG = !QI && ((PW_QREG_F32 && QREG_OK && D <= 128 && D % 8 == 0) || sizeof(VT) == 1);
        float2 qr[QREG ? D / 8 : 1];
        if constexpr (QREG) {
            const float2* q2 = reinterpret_cast<const float2*>(S.q);
#pragma unroll
            for (int p = 0; p < D / 8; p++) qr[p] = q2[4 * p + c];
        }
        uint32_t qw[QI ? D / 16 : 1];
        int qsq = 0;
        if constexpr (QI) {
            const uint32_t* qb = reinterpret_cast<const uint32_t*>(S.q + ((D + 3) & ~3));
#pragma unroll
            for (int p = 0; p < D / 16; p++) qw[p] = qb[4 * p + c];
            qsq = reinterpret_cast<const int32_t*>(qb)[((D + 15) & ~15) / 4];
        }
        // one 8-row pass: distance -> key -> survivor compaction
        auto emit = [&](int r0, int rows, float dist) {
            const int rr = (int)v;
            const int rc = rr < rows ? rr : rows - 1;
            const uint64_t key = ((uint64_t)dist_bits<M>(dist) << 32) | (uint32_t)S.newl[r0 + rc];
            const bool surv = c == 0 && rr < rows && key < thr;
            const unsigned b = __ballot_sync(0xffffffffu, surv);
            if (surv) S.ckey[ns + __popc(b & lanemask_lt())] = key;
            ns += __popc(b);
        };
        issue(0);
        issue(1);
        for (int g = 0; g < ngroups; g++) {
#if PW_TMA_ROWS
            if (tma) {
                // bounded (~seconds): a transaction count that never completes
                // raises (flag 32) instead of hanging the GPU
                const uint32_t par = (S.phase >> (g & 1)) & 1u;
                uint32_t done = 0;
                for (uint32_t spin = 0; !done; spin++) {
                    asm volatile(
                        "{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n"
                        " selp.u32 %0, 1, 0, p;\n}\n"
                        : "=r"(done)
                        : "r"(smem_u32(S.mbar + (g & 1))), "r"(par)
                        : "memory");
                    if (!done && spin > (1u << 22)) {
                        atomicOr(A.err, 32);
                        break;
                    }
                }
                S.phase ^= 1u << (g & 1);
            } else
#endif
            {
                cp_wait<1>();
            }
            __syncwarp();
            const int r0 = g * RH;
            const int rows = min(RH, n - r0);
            const VT* base = reinterpret_cast<const VT*>(S.stage) + (size_t)(g & 1) * RH * sp;
            for (int pass = 0; pass < rows; pass += 8) {
                const int rc = pass + (int)v < rows ? pass + (int)v : rows - 1;
                float dist;
                if constexpr (QI)
                    dist = pw_row4_u8i<D>(reinterpret_cast<const uint8_t*>(base + (size_t)rc * sp), qw, c, qsq);
                else if constexpr (sizeof(VT) == 1)
                    dist = pw_row4_u8<M, D>(reinterpret_cast<const uint8_t*>(base + (size_t)rc * sp), qr, c);
                else if constexpr (QREG)
                    dist = pw_row4_qreg<M, D>(reinterpret_cast<const float*>(base + (size_t)rc * sp), qr, c);
                else
                    dist = finish<M>(pw_sum4<M, 0, D>(reinterpret_cast<const float*>(base + (size_t)rc * sp), S.q, c));
                emit(r0 + pass, min(8, rows - pass), dist);
            }
            __syncwarp();
            if (tma) fence_proxy_async();  // generic reads of this half before the async overwrite
            issue(g + 2);
        }
        if (!tma) cp_wait<0>();
        __syncwarp();
    } else {
        const int row_bytes = A.d * (int)sizeof(VT);
        auto issue = [&](int g) {
            if (g < ngroups) {
                int r0 = g * RH;
                int rows = min(RH, n - r0);
                VT* dst0 = reinterpret_cast<VT*>(S.stage) + (size_t)(g & 1) * RH * sp;
                for (int r = 0; r < rows; r++) {
                    int32_t id = S.newl[r0 + r];
                    warp_copy_async(dst0 + (size_t)r * sp, vrow<VT>(G, (uint32_t)id, A.d), row_bytes);
                }
            }
            cp_commit();
        };
        issue(0);
        issue(1);
        const unsigned v = lane >> 3, a = lane & 7u;
        for (int g = 0; g < ngroups; g++) {
            cp_wait<1>();
            __syncwarp();
            int r0 = g * RH;
            int rows = min(RH, n - r0);
            const VT* base = reinterpret_cast<const VT*>(S.stage) + (size_t)(g & 1) * RH * sp;
            for (int sub = 0; sub < rows; sub += 4) {
                int rr = sub + (int)v;
                int rc = rr < rows ? rr : rows - 1;
                float dist = l2_row<M>(A.plan, base + (size_t)rc * sp, S.q, a);
                const uint64_t key = ((uint64_t)dist_bits<M>(dist) << 32) | (uint32_t)S.newl[r0 + rc];
                const bool surv = a == 0 && rr < rows && key < thr;
                const unsigned b = __ballot_sync(0xffffffffu, surv);
                if (surv) S.ckey[ns + __popc(b & lanemask_lt())] = key;
                ns += __popc(b);
            }
            __syncwarp();
            issue(g + 2);
        }
        cp_wait<0>();
        __syncwarp();
    }
    return ns;
}

// Bitonic sort of ckey[0..s) in shared memory (32 < s <= 256): compact
// loops (this case only occurs in the first iterations of a search, so code
// size matters more than its instruction count).
static __device__ __noinline__ void sort_survivors_smem(uint64_t* ckey, int s) {
    const unsigned lane = lane_id();
    int N = 64;
    while (N < s) N <<= 1;
    for (int e = s + (int)lane; e < N; e += 32) ckey[e] = ~0ull;
    __syncwarp();
    for (int size = 2; size <= N; size <<= 1) {
        for (int stride = size >> 1; stride > 0; stride >>= 1) {
            for (int i = lane; i < (N >> 1); i += 32) {
                const int lo = 2 * i - (i & (stride - 1));
                const int hi = lo + stride;
                const bool asc = (lo & size) == 0;
                const uint64_t a = ckey[lo], b = ckey[hi];
                if ((a > b) == asc) {
                    ckey[lo] = b;
                    ckey[hi] = a;
                }
            }
            __syncwarp();
        }
    }
}

// search.py:170-190 merge_and_sort on keys; returns `inserted`.
static __device__ int merge_queue(const KArgs& A, WarpState& S, const SearchCfg& C, int s) {
    // In place, single buffer: sort the survivors, find each one's insertion
    // point P_i = lower_bound(queue, S_i), shift only the queue tail
    // [min P_i, qlen) back to front (entry t moves to t + #{P_i <= t}; entries
    // pushed past l fall off), then drop survivor i at P_i + i.  Keys are
    // unique, so the positions form the merged order exactly.
    const unsigned lane = lane_id();
    const int L = C.L;
    uint64_t* qk = S.qk0;
    uint8_t* qe = S.qe0;
    const int qlen = S.qlen;
    // ckey[0..s): the survivors (keys below the l-th key), filtered by score_rows
    if (s == 0) return 0;
    if (s <= 32) {
        // rank by counting smaller keys (keys are unique): s broadcast loads
        // per lane instead of a 15-stage shuffle network
        const uint64_t x = (int)lane < s ? S.ckey[lane] : ~0ull;
        int rank = 0;
#pragma unroll 4
        for (int o = 0; o < s; o++) rank += S.ckey[o] < x;
        __syncwarp();
        if ((int)lane < s) S.ckey[rank] = x;
    } else if (s <= 64) {
        const uint64_t x0 = S.ckey[lane];
        const uint64_t x1 = 32 + (int)lane < s ? S.ckey[32 + lane] : ~0ull;
        int r0 = 0, r1 = 0;
#pragma unroll 4
        for (int o = 0; o < s; o++) {
            const uint64_t y = S.ckey[o];
            r0 += y < x0;
            r1 += y < x1;
        }
        __syncwarp();
        S.ckey[r0] = x0;
        if (32 + (int)lane < s) S.ckey[r1] = x1;
    } else {
        sort_survivors_smem(S.ckey, s);
    }
    __syncwarp();
    int32_t* ppos = S.newl;  // free once scoring has turned ids into keys
    // P_i = lower_bound(queue, S_i): branch-free bit descent, two searches in
    // flight per lane
    int qstep = 1;
    while (qstep <= qlen) qstep <<= 1;
    qstep >>= 1;
    bool dup = false;
    if (s <= 32) {  // the common case: one search per lane
        if ((int)lane < s) {
            const uint64_t k0 = S.ckey[lane];
            int p0 = 0;
            for (int st = qstep; st > 0; st >>= 1)
                if (p0 + st <= qlen && qk[p0 + st - 1] < k0) p0 += st;
            const bool d0 = p0 < qlen && qk[p0] == k0;
            dup = d0;
            ppos[lane] = d0 ? -1 : p0;
        }
    } else
    for (int i0 = lane; i0 < s; i0 += 64) {
        const int i1 = i0 + 32;
        const uint64_t k0 = S.ckey[i0];
        const uint64_t k1 = i1 < s ? S.ckey[i1] : 0ull;
        int p0 = 0, p1 = 0;
        for (int st = qstep; st > 0; st >>= 1) {
            if (p0 + st <= qlen && qk[p0 + st - 1] < k0) p0 += st;
            if (p1 + st <= qlen && qk[p1 + st - 1] < k1) p1 += st;
        }
        // lossy visited mode re-scores forgotten nodes: one still queued has
        // the identical key (search.py:181 skips queued ids)
        const bool d0 = p0 < qlen && qk[p0] == k0;
        const bool d1 = i1 < s && p1 < qlen && qk[p1] == k1;
        dup |= d0 | d1;
        ppos[i0] = d0 ? -1 : p0;
        if (i1 < s) ppos[i1] = d1 ? -1 : p1;
    }
    if (__any_sync(0xffffffffu, dup)) {
        __syncwarp();
        int s2 = 0;  // in-place compaction (each chunk is read before it is written)
        for (int base = 0; base < s; base += 32) {
            const int i = base + (int)lane;
            const uint64_t key = i < s ? S.ckey[i] : 0ull;
            const int pp = i < s ? ppos[i] : -1;
            const unsigned b = __ballot_sync(0xffffffffu, pp >= 0);
            __syncwarp();
            if (pp >= 0) {
                const int o = s2 + __popc(b & lanemask_lt());
                S.ckey[o] = key;
                ppos[o] = pp;
            }
            s2 += __popc(b);
        }
        s = s2;
        __syncwarp();
        if (s == 0) return 0;
    }
    __syncwarp();
    const int pmin = ppos[0];
    S.fu = min(S.fu, pmin);  // entries before pmin keep their place (and flags)
    if (qlen > pmin) {
        // Queue tail [pmin, qlen): entry t moves to t + #{i : P_i <= t}.  Up to
        // 4 chunks are read into registers, their targets found with
        // independent bit-descent searches over ppos, then written -- back to
        // front by 128-entry groups, so every write lands on an entry that was
        // already read (targets are distinct and >= the source).
        int sstep = 1;
        while (sstep <= s) sstep <<= 1;
        sstep >>= 1;
        for (int g_end = qlen; g_end > pmin; g_end -= 128) {
            const int g0 = max(pmin, g_end - 128);
            uint64_t key[4];
            int np[4];
            uint32_t fl = 0;
#pragma unroll
            for (int c = 0; c < 4; c++) {
                const int t = g0 + 32 * c + (int)lane;
                const bool valid = t < g_end;
                key[c] = valid ? qk[t] : 0ull;
                fl |= (valid && qe[t]) ? (1u << c) : 0u;
                np[c] = 0;
            }
            for (int st = sstep; st > 0; st >>= 1) {
#pragma unroll
                for (int c = 0; c < 4; c++) {
                    const int t = g0 + 32 * c + (int)lane;
                    if (np[c] + st <= s && ppos[np[c] + st - 1] <= t) np[c] += st;
                }
            }
            __syncwarp();
#pragma unroll
            for (int c = 0; c < 4; c++) {
                const int t = g0 + 32 * c + (int)lane;
                const int dst = t + np[c];
                if (t < g_end && dst < L) {
                    qk[dst] = key[c];
                    qe[dst] = (uint8_t)((fl >> c) & 1u);
                }
            }
            __syncwarp();
        }
    }
    int ins = 0;
    for (int base = 0; base < s; base += 32) {
        const int i = base + (int)lane;
        bool kept = false;
        if (i < s) {
            const int p = ppos[i] + i;
            if (p < L) {
                qk[p] = S.ckey[i];
                qe[p] = 0;
                kept = true;
            }
        }
        ins += __popc(__ballot_sync(0xffffffffu, kept));
    }
    __syncwarp();
    S.qlen = min(L, qlen + s);
    return ins;
}

// search.py:192-204: first r unexpanded queue entries, marked expanded.
// S.fu: every entry before it is expanded (merges lower it to their first
// insertion point), so the scan starts at its chunk.
static __device__ int select_parents(WarpState& S, int r, int32_t* parents) {
    const unsigned lane = lane_id();
    uint64_t* qk = S.qk_cur();
    uint8_t* qe = S.qe_cur();
    int np = 0, last = -1;
    for (int base = S.fu & ~31; base < S.qlen && np < r; base += 32) {
        int t = base + lane;
        bool f = t < S.qlen && qe[t] == 0;
        unsigned b = __ballot_sync(0xffffffffu, f);
        int pos = np + __popc(b & lanemask_lt());
        if (f && pos < r) {
            parents[pos] = (int32_t)(uint32_t)qk[t];
            qe[t] = 1;
        }
        const unsigned lb = __ballot_sync(0xffffffffu, f && pos == r - 1);
        if (lb) last = base + __ffs(lb) - 1;
        np = min(r, np + __popc(b));
    }
    S.fu = np == r ? last + 1 : S.qlen;
    __syncwarp();
    return np;
}

// Issue the bulk copies described in S.desc[0..n_rows) (one lane per row;
// TMA takes uniform operands, so the compiler serialises lanes -- kept out of
// line so there is one copy of that loop in the kernel) and wait for them.
static __device__ __noinline__ uint32_t bulk_issue_wait(const uint4* desc, uint64_t* bar,
                                                        uint32_t phase, int n_rows, uint32_t total) {
    const unsigned lane = lane_id();
    fence_proxy_async();
    if (lane == 0) mbar_arrive_expect(bar, total);
    __syncwarp();
    for (int r = lane; r < n_rows; r += 32) {
        const uint4 d = desc[r];
        const void* src = reinterpret_cast<const void*>(((uint64_t)d.w << 32) | d.z);
        asm volatile(
            "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n" ::"r"(
                d.x),
            "l"(src), "r"(d.y), "r"(smem_u32(bar))
            : "memory");
    }
    mbar_wait(bar, (phase >> 2) & 1u);
    __syncwarp();
    return phase ^ 4u;
}

// 16-byte aligned rows (the default): 8 lanes per row, 4 rows per warp step,
// LDGSTS chunks.  TMA bulk copies need warp-uniform operands, so per-row
// (data-dependent) sources make ptxas serialise lanes through a waterfall
// loop of hundreds of instructions; this is a dozen.
static __device__ __forceinline__ void copy16_issue_wait(const uint4* desc, int n_rows, bool wait = true) {
    const unsigned lane = lane_id();
    const unsigned sub = lane & 7u;
    const uint64_t pol = l2_evict_first_policy();
    for (int r = (int)(lane >> 3); r < n_rows; r += 4) {
        const uint4 d = desc[r];
        const char* src = reinterpret_cast<const char*>(((uint64_t)d.w << 32) | d.z);
        const uint32_t nch = d.y >> 4;
        for (uint32_t c = sub; c < nch; c += 8) cp_async16_stream(d.x + 16 * c, src + 16 * c, pol);
    }
    cp_commit();
    if (!wait) return;
    cp_wait<0>();
    __syncwarp();
}

// cp.async fallback for rows that are not 16-byte multiples (out of line).
static __device__ __noinline__ void copy_issue_wait(const uint4* desc, int n_rows) {
    const unsigned lane = lane_id();
    for (int r = 0; r < n_rows; r++) {
        const uint4 d = desc[r];
        const char* src = reinterpret_cast<const char*>(((uint64_t)d.w << 32) | d.z);
        const uint32_t dst = d.x, bytes = d.y;
        const uint32_t al = (uint32_t)(uintptr_t)src | dst | bytes;
        if ((al & 15u) == 0) {
            for (uint32_t c = lane; c < (bytes >> 4); c += 32)
                asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(dst + 16 * c), "l"(src + 16 * c));
        } else if ((al & 7u) == 0) {
            for (uint32_t c = lane; c < (bytes >> 3); c += 32)
                asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"(dst + 8 * c), "l"(src + 8 * c));
        } else {
            for (uint32_t c = lane; c < (bytes >> 2); c += 32)
                asm volatile("cp.async.ca.shared.global [%0], [%1], 4;\n" ::"r"(dst + 4 * c), "l"(src + 4 * c));
        }
    }
    cp_commit();
    cp_wait<0>();
    __syncwarp();
}

// Fetch up to 3 row sets (adjacency, parent vectors, direction rows) for the
// parents in ONE round trip: lanes write one descriptor per row, then a single
// out-of-line issuer runs TMA bulk copies (aligned rows) or cp.async.
template <bool FAST = false, typename F>
__device__ __forceinline__ void fetch_group(const KArgs& A, WarpState& S, int n_rows, uint32_t total,
                                            F&& row, bool wait = true) {
    const unsigned lane = lane_id();
    for (int r = lane; r < n_rows; r += 32) {
        void* dst;
        const void* src;
        uint32_t bytes;
        row(r, dst, src, bytes);
        const uint64_t sp = (uint64_t)src;
        S.desc[r] = make_uint4(smem_u32(dst), bytes, (uint32_t)sp, (uint32_t)(sp >> 32));
    }
    __syncwarp();
    if (FAST)  // FAST launches have 16-byte rows and no TMA bulk expansion (prepare())
        copy16_issue_wait(S.desc, n_rows, wait);
    else if (A.bulk_adj == 2)
        S.phase = bulk_issue_wait(S.desc, S.mbar + 2, S.phase, n_rows, total);
    else if (A.bulk_adj)
        copy16_issue_wait(S.desc, n_rows, wait);
    else
        copy_issue_wait(S.desc, n_rows);
}


// Warm L2 with the rows the next expansion will most likely fetch: the first
// r unexpanded entries of the current queue become the parents unless new
// candidates overtake them.  One prefetch per 128-byte line, no registers
// tied up; a wrong guess only costs bandwidth.
template <int D, typename VT>
__device__ __forceinline__ void prefetch_parents(const KArgs& A, const WarpState& S, const GraphDev& G,
                                                 const SearchCfg& C) {
    const unsigned lane = lane_id();
    const uint64_t* qk = S.qk_cur();
    const uint8_t* qe = S.qe_cur();
    const int lim = min(S.qlen, 32);
    const bool f = (int)lane < lim && qe[lane] == 0;
    const unsigned b = __ballot_sync(0xffffffffu, f);
    const int rank = __popc(b & lanemask_lt());
    if (!f || rank >= C.r) return;
    const uint32_t par = (uint32_t)qk[lane];
    const int j = G.j;
    const char* a = reinterpret_cast<const char*>(G.adj + (size_t)par * j);
    for (int o = 0; o < j * 4; o += 128) prefetch_l2(a + o);
    if (C.prune_sel == 1 && G.dir) {
        const int d = D > 0 ? D : A.d;
        const char* v = reinterpret_cast<const char*>(vrow<VT>(G, par, d));
        for (int o = 0; o < d * (int)sizeof(VT); o += 128) prefetch_l2(v + o);
        const char* dr = reinterpret_cast<const char*>(G.dir + (size_t)par * j * A.W);
        for (int o = 0; o < j * A.W * 4; o += 128) prefetch_l2(dr + o);
    }
}

// _expand (search.py:235-266) up to the ordered candidate list in S.cand;
// returns the candidate count p * n_sel.
template <int D, typename VT, bool FAST = false>
__device__ int expand(const KArgs& A, WarpState& S, const GraphDev& G, const SearchCfg& C,
                      const int32_t* parents, int np, int it, Pcg64& rng) {
    const unsigned lane = lane_id();
    const int j = G.j;
    if (j == 0) return 0;
    const bool prune = C.prune_sel != 0 && it < C.cool_start;
    const uint32_t adj_bytes = (uint32_t)j * 4u;
    if (!prune) {
        fetch_group<FAST>(A, S, np, np * adj_bytes, [&](int r, void*& dst, const void*& src, uint32_t& b) {
            dst = S.cand + r * j;
            src = G.adj + (size_t)parents[r] * j;
            b = adj_bytes;
        });
        return np * j;
    }
    const int nsel = C.n_keep < j ? C.n_keep : j;
    int32_t* craw = reinterpret_cast<int32_t*>(S.ckey);  // free during expansion
    int32_t* cnt = S.misc;                                // PG * j
    int32_t* perm = S.misc;                               // j (random arm)
    uint32_t* qb = reinterpret_cast<uint32_t*>(S.misc + A.PG * j);  // PG * W
    if (C.prune_sel == 1) {
        constexpr int WC = D > 0 ? (D + 31) / 32 : 0;
        const int W = WC ? WC : A.W;
        const int d = D > 0 ? D : A.d;
        const uint32_t vec_bytes = (uint32_t)d * (uint32_t)sizeof(VT), dir_bytes = (uint32_t)(j * W) * 4u;
        // PW_DGS_LDG: the parents' query bits pack(q >= x_parent) from their
        // rows loaded straight into registers (one float4 per lane and parent,
        // in flight with the expansion's cp.async round trip), so the parent
        // rows never pass through the staging ring
        constexpr bool LDGP = PW_DGS_LDG && D > 0 && sizeof(VT) == 4 && D % 4 == 0 && D <= 128;
        [[maybe_unused]] uint32_t* qbits = reinterpret_cast<uint32_t*>(S.misc + A.o_qbits);
        for (int pg = 0; pg < np; pg += A.PG) {
            const int gp = min(A.PG, np - pg);
            VT* prow = reinterpret_cast<VT*>(S.stage);
            uint32_t* drow = LDGP ? reinterpret_cast<uint32_t*>(S.stage)
                                  : reinterpret_cast<uint32_t*>(prow + (size_t)gp * A.pstride);
            if constexpr (LDGP) {
                constexpr int CH = D / 4;  // float4 chunks per row
                // cp.async of the adjacency + direction rows issued first
                // (no wait), then the parent rows' register loads: one round trip
                fetch_group<FAST>(A, S, 2 * gp, gp * (adj_bytes + dir_bytes),
                            [&](int r, void*& dst, const void*& src, uint32_t& b) {
                                const int pi = r % gp;
                                const int32_t par = parents[pg + pi];
                                if (r < gp) {
                                    dst = craw + (pg + pi) * j;
                                    src = G.adj + (size_t)par * j;
                                    b = adj_bytes;
                                } else {
                                    dst = drow + (size_t)pi * j * W;
                                    src = G.dir + (size_t)par * j * W;
                                    b = dir_bytes;
                                }
                            }, /*wait=*/!A.bulk_adj || A.bulk_adj == 2);
                float4 xr[kParentGroup];
#pragma unroll
                for (int pi = 0; pi < kParentGroup; pi++)
                    if (pi < gp && (int)lane < CH)
                        xr[pi] = __ldcs(reinterpret_cast<const float4*>(vrow<VT>(G, (uint32_t)parents[pg + pi], D)) +
                                        lane);
                if (A.bulk_adj == 1) {
                    cp_wait<0>();
                    __syncwarp();
                }
                const float4 q4 = (int)lane < CH ? reinterpret_cast<const float4*>(S.q)[lane]
                                                 : make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll
                for (int pi = 0; pi < kParentGroup; pi++) {
                    if (pi < gp) {
                        // lane holds elements 4 lane .. 4 lane + 3: a nibble of
                        // word lane / 8, OR-reduced over the 8 lanes of a word
                        const float4 x = xr[pi];
                        uint32_t v = (int)lane < CH ? ((q4.x >= x.x ? 1u : 0u) | (q4.y >= x.y ? 2u : 0u) |
                                                       (q4.z >= x.z ? 4u : 0u) | (q4.w >= x.w ? 8u : 0u))
                                                    : 0u;
                        v <<= 4u * (lane & 7u);
                        v |= __shfl_xor_sync(0xffffffffu, v, 1);
                        v |= __shfl_xor_sync(0xffffffffu, v, 2);
                        v |= __shfl_xor_sync(0xffffffffu, v, 4);
                        if ((lane & 7u) == 0 && (int)(lane >> 3) < WC) qbits[pi * WC + (lane >> 3)] = v;
                    }
                }
                __syncwarp();
            } else
            fetch_group<FAST>(A, S, 3 * gp, gp * (adj_bytes + vec_bytes + dir_bytes),
                        [&](int r, void*& dst, const void*& src, uint32_t& b) {
                            const int pi = r % gp, kind = r / gp;
                            const int32_t par = parents[pg + pi];
                            if (kind == 0) {
                                dst = craw + (pg + pi) * j;
                                src = G.adj + (size_t)par * j;
                                b = adj_bytes;
                            } else if (kind == 1) {
                                dst = prow + (size_t)pi * A.pstride;
                                src = vrow<VT>(G, (uint32_t)par, d);
                                b = vec_bytes;
                            } else {
                                dst = drow + (size_t)pi * j * W;
                                src = G.dir + (size_t)par * j * W;
                                b = dir_bytes;
                            }
                        });
            if (WC > 0 && j <= 32) {
                const unsigned valid = __ballot_sync(0xffffffffu, (int)lane < j);
#if PW_DGS_QREG
                // this lane's query elements for the direction bits, loaded once
                // per expansion instead of once per parent
                float qv[WC > 0 ? WC : 1];
#pragma unroll
                for (int w = 0; w < WC; w++) qv[w] = 32 * w + (int)lane < d ? S.q[32 * w + lane] : 0.f;
#endif
                // per parent: query direction bits pack(q >= x_parent) as W
                // ballots (direction.py:53-59), matching count per slot
                // (lane = slot, :62-69), one warp bitonic sort on (count desc,
                // slot asc) == stable argsort(-counts) (:79-87)
#if PW_DGS_PUNROLL == 2
#pragma unroll 2
#endif
                for (int pi = 0; pi < gp; pi++) {
                    uint32_t qb[WC > 0 ? WC : 1];
#pragma unroll
                    for (int w = 0; w < WC; w++) {
                        if constexpr (LDGP) {
                            qb[w] = qbits[pi * WC + w];
                        } else {
                            const int t = 32 * w + (int)lane;
#if PW_DGS_QREG
                            const bool bit = t < d && qv[w] >= to_f(prow[(size_t)pi * A.pstride + t]);
#else
                            const bool bit = t < d && S.q[t] >= to_f(prow[(size_t)pi * A.pstride + t]);
#endif
                            qb[w] = __ballot_sync(0xffffffffu, bit);
                        }
                    }
                    int c = 0;
                    if ((int)lane < j) {
                        const uint32_t* dr = drow + ((size_t)pi * j + lane) * WC;
                        int diff = 0;
                        if constexpr (WC % 4 == 0) {
#pragma unroll
                            for (int w = 0; w < WC; w += 4) {
                                const uint4 v = *reinterpret_cast<const uint4*>(dr + w);
                                diff += __popc(v.x ^ qb[w]) + __popc(v.y ^ qb[w + 1]) +
                                        __popc(v.z ^ qb[w + 2]) + __popc(v.w ^ qb[w + 3]);
                            }
                        } else {
#pragma unroll
                            for (int w = 0; w < WC; w++) diff += __popc(dr[w] ^ qb[w]);
                        }
                        c = d - diff;
                    }
                    // rank = #slots with a larger count + #equal-count slots
                    // before this one: bit-serial ballot radix over the count
                    // bits, MSB first.  eq = slots equal to mine on the bits
                    // seen so far; gtm collects the slots that first differ
                    // from mine with a 1 where I have a 0 (larger counts).
                    // Masks, not running counts: one popc at the end.
                    constexpr int NB = D >= 1024 ? 11 : D >= 512 ? 10 : D >= 256 ? 9 : D >= 128 ? 8 : D >= 64 ? 7 : 6;
                    unsigned eq = valid, gtm = 0u;
#pragma unroll
                    for (int b = NB - 1; b >= 0; b--) {
                        const unsigned m = 0u - (((unsigned)c >> b) & 1u);  // all ones iff my bit b is set
                        const unsigned B = __ballot_sync(0xffffffffu, m != 0u);
                        const unsigned t = eq & B;
                        gtm |= t & ~m;
                        eq &= ~(B ^ m);
                    }
                    const int rank = __popc(gtm) + __popc(eq & lanemask_lt());
                    if ((int)lane < j && rank < nsel)
                        S.cand[(pg + pi) * nsel + rank] = craw[(pg + pi) * j + lane];
                }
            } else if (!FAST) {
                for (int pi = 0; pi < gp; pi++)
                    for (int w = 0; w < W; w++) {
                        int t = 32 * w + (int)lane;
                        bool bit = t < d && S.q[t] >= to_f(prow[(size_t)pi * A.pstride + t]);
                        unsigned word = __ballot_sync(0xffffffffu, bit);
                        if (lane == 0) qb[pi * W + w] = word;
                    }
                __syncwarp();
                for (int pi = 0; pi < gp; pi++)
                    for (int s = lane; s < j; s += 32) {
                        int diff = 0;
                        const uint32_t* dr = drow + ((size_t)pi * j + s) * W;
                        for (int w = 0; w < W; w++) diff += __popc(dr[w] ^ qb[pi * W + w]);
                        cnt[pi * j + s] = d - diff;
                    }
                __syncwarp();
                for (int pi = 0; pi < gp; pi++)
                    for (int s = lane; s < j; s += 32) {
                        int c = cnt[pi * j + s];
                        int rank = 0;
                        for (int o = 0; o < j; o++) {
                            int co = cnt[pi * j + o];
                            rank += (co > c) || (co == c && o < s);
                        }
                        if (rank < nsel) S.cand[(pg + pi) * nsel + rank] = craw[(pg + pi) * j + s];
                    }
            }
            __syncwarp();
        }
    } else if (!FAST) {
        fetch_group<FAST>(A, S, np, np * adj_bytes, [&](int r, void*& dst, const void*& src, uint32_t& b) {
            dst = craw + r * j;
            src = G.adj + (size_t)parents[r] * j;
            b = adj_bytes;
        });
        for (int pi = 0; pi < np; pi++) {
            if (lane == 0) rng = permutation(rng, (uint32_t)j, perm);  // direction.py:103-105
            __syncwarp();
            for (int t = lane; t < nsel; t += 32) S.cand[pi * nsel + t] = craw[pi * j + perm[t]];
            __syncwarp();
        }
    }
    S.c_dgs += np * (j - C.n_keep);
    return np * nsel;
}

#ifdef PW_PHASE_TIMERS
#define PW_T0() long long pw_t_ = clock64()
#define PW_T(i)                          \
    do {                                 \
        const long long n_ = clock64();  \
        S.pc[i] += n_ - pw_t_;           \
        pw_t_ = n_;                      \
    } while (0)
#else
#define PW_T0() \
    do {        \
    } while (0)
#define PW_T(i) \
    do {        \
    } while (0)
#endif

// log_visits (search.py:304-305): newly scored ids in batch order (cold).
static __device__ __noinline__ int64_t log_visits(int32_t* log, int64_t cap, const int32_t* newl, int n_new,
                                                  int64_t n_logged) {
    for (int t = lane_id(); t < n_new; t += 32) {
        const int64_t p = n_logged + t;
        if (p < cap) log[p] = newl[t];
    }
    return n_logged + n_new;
}

// One full search (search.py:269-335) over graph G.  Seeds (already in
// S.cand[0..ns)) are deduplicated in order and capped at `want`; the
// random fill draws Generator.choice(n, want) from rng.
template <int D, typename VT, int M, bool FAST = false, bool WIDE = false>
__device__ __forceinline__ bool run_search(const KArgs& A, WarpState& S, const GraphDev& G, const SearchCfg& C,
                           int ns, bool fill_random, Pcg64& rng, int64_t task,
                           int64_t* n_logged) {
    const unsigned lane = lane_id();
    PW_T0();
    // reset per-search state
    if (D == 0)
        for (int i = lane; i < A.H; i += 32) S.vh[i] = kEmpty;
    bh_clear(A, S);
    S.cur = 0;
    S.qlen = 0;
    S.fu = 0;
    S.vcount = 0;
    S.ovf = false;
    if (A.lossy) {
        // 8-bit tags 1..255; on wrap the cache is cleared (tag 0 = never used)
        if (++S.epoch > 255u) {
            uint4* t4 = reinterpret_cast<uint4*>(S.gvis);
            const int n4 = (int)((A.gmask + 1) >> 1);  // gmask + 1 u64 words
#pragma unroll 1
            for (int i = lane; i < n4; i += 32) __stcg(t4 + i, make_uint4(0u, 0u, 0u, 0u));
            __syncwarp();
            S.epoch = 1u;
        }
    } else {
        S.epoch = S.epoch == 0xFFFFFFFFu ? 1u : S.epoch + 1u;
    }
    S.c_it = S.c_dc = S.c_tv = S.c_ne = S.c_dgs = S.c_ins = 0;

    // _initial_batch (search.py:207-227)
    int nuniq;
    int nb = dedup_ordered(A, S, S.cand, ns, C.want, S.newl, &nuniq);
    if (fill_random && nb < C.want) {
        int32_t* ch = S.cand;
        const uint32_t pop = (uint32_t)G.n, size = (uint32_t)C.want;
        // warp-parallel Floyd when exact (rare rejections / repeats fall back
        // to the serial restatement); the draw order matters only when seeds
        // precede the fill (the first want - nb new values are kept) or the
        // visit log records it
        bool done = false;
        if (size <= (uint32_t)kJumpMax && pop > size && !choice_uses_tail(pop, size)) {
            const Pcg64 r = choice_floyd_warp(rng, pop, size, nb > 0 || C.log, A.jump,
                                              A.CB > 64 ? reinterpret_cast<uint32_t*>(S.ckey) : S.gscr, ch);
            done = r.has32 < 2u;
            if (done) rng = r;
        }
        if (!done && lane == 0) {
            if (choice_uses_tail(pop, size)) {
                uint32_t cap = 1;
                while (cap < 4u * size + 8u) cap <<= 1;
                rng = choice_tail(rng, pop, size, S.gscr, S.gscr + cap, cap - 1, ch);
            } else {
                uint32_t mask = (uint32_t)gen_mask64((uint64_t)(1.2 * (double)size));
                // ckey is free during the initial batch (stage aliases the dedup hash)
                uint32_t* set = ((int64_t)(mask + 1) * 8 <= 8ll * max(64, A.CB))
                                    ? reinterpret_cast<uint32_t*>(S.ckey)
                                    : S.gscr;
                rng = choice_floyd(rng, pop, size, set, mask, ch);
            }
        }
        __syncwarp();
        int cnt = nb;
        for (int base = 0; base < C.want && cnt < C.want; base += 32) {
            int t = base + lane;
            int32_t id = t < C.want ? ch[t] : -1;
            bool f = t < C.want && !bh_contains(A, S, (uint32_t)id);
            unsigned b = __ballot_sync(0xffffffffu, f);
            int pos = cnt + __popc(b & lanemask_lt());
            if (f && pos < C.want) S.newl[pos] = id;
            cnt = min(C.want, cnt + __popc(b));
        }
        __syncwarp();
        nb = cnt;
    }
    bh_clear(A, S);
    int n_new = visited_filter<(D > 0), FAST>(A, S, nb);
    PW_T(0);

    bool converged = false;
    int32_t* parents = S.misc + A.o_par;
    for (int it = 0; it < C.max_iter; it++) {
        S.c_it++;
        int inserted = 0;
        if (!FAST && A.prefetch && it > 0 && it < C.max_iter - 1) prefetch_parents<D, VT>(A, S, G, C);
        if (n_new) {
            if (!FAST && C.log && A.visit_log)
                *n_logged = log_visits(A.visit_log + task * A.visit_cap, A.visit_cap, S.newl, n_new, *n_logged);
            S.c_dc += n_new;
            PW_T(7);
            const uint64_t thr = S.qlen == C.L ? S.qk0[C.L - 1] : ~0ull;
            int ns;
            if constexpr (sizeof(VT) == 1 && M == 0 && D > 0) {
                const int32_t* qmeta = reinterpret_cast<const int32_t*>(
                    reinterpret_cast<const uint8_t*>(S.q + ((D + 3) & ~3)) + ((D + 15) & ~15));
                ns = qmeta[1] ? score_rows<D, VT, M, true>(A, S, G, n_new, thr)
                              : score_rows<D, VT, M, false>(A, S, G, n_new, thr);
            } else {
                ns = score_rows<D, VT, M, false, !WIDE>(A, S, G, n_new, thr);
            }
            PW_T(1);
            inserted = merge_queue(A, S, C, ns);
            PW_T(2);
            S.c_ins += inserted;
        }
        if (inserted == 0) {
            converged = true;
            break;
        }
        if (it == C.max_iter - 1) break;
        int np = select_parents(S, C.r, parents);
        PW_T(3);
        if (np == 0) {
            converged = true;
            break;
        }
        S.c_ne += np;
        int nc = expand<D, VT, FAST>(A, S, G, C, parents, np, it, rng);
        PW_T(4);
        // the hash shares the staging ring, which now holds rows.  FAST: the
        // unordered dedup reads keys only, and the lossy visited cache does
        // not use the hash (the next search's first clear is a full one)
        if (FAST) {
            bh_clear<true>(A, S);
            nb = dedup_unordered(A, S, S.cand, nc, S.newl, (uint32_t)A.BH - 1u);
        } else {
            bh_clear(A, S);
            if (nc <= C.cap && !C.log)
                nb = dedup_unordered(A, S, S.cand, nc, S.newl, (uint32_t)A.BH - 1u);
            else
                nb = dedup_ordered(A, S, S.cand, nc, C.cap, S.newl, &nuniq);
        }
        S.c_tv += nb;
        if (!FAST) bh_clear(A, S);
        PW_T(5);
        n_new = visited_filter<(D > 0), FAST>(A, S, nb);
        PW_T(6);
    }
    PW_T(7);
    return converged;
}

template <int D, typename VT, int M, bool FAST = false, int MAXT = PW_MAX_THREADS>
__global__ void __launch_bounds__(MAXT, 1) beam_search_kernel(const __grid_constant__ KArgs A) {
    extern __shared__ __align__(128) unsigned char smem_raw[];
    const unsigned lane = lane_id();
    const int warp = threadIdx.x >> 5;
    const int gwarp = blockIdx.x * (blockDim.x >> 5) + warp;
    unsigned char* base = smem_raw + (size_t)warp * A.warp_bytes;
    WarpState S;
    S.q = reinterpret_cast<float*>(base + A.o_q);
    S.qk0 = reinterpret_cast<uint64_t*>(base + A.o_qk);
    S.qe0 = reinterpret_cast<uint8_t*>(base + A.o_qe);
    S.cand = reinterpret_cast<int32_t*>(base + A.o_cand);
    S.cslot = reinterpret_cast<int32_t*>(base + A.o_cslot);
    S.newl = reinterpret_cast<int32_t*>(base + A.o_newl);
    S.ckey = reinterpret_cast<uint64_t*>(base + A.o_ckey);
    S.bhk = reinterpret_cast<uint32_t*>(base + A.o_bhk);
    S.bhp = reinterpret_cast<int32_t*>(base + A.o_bhp);
    S.vh = reinterpret_cast<uint32_t*>(base + A.o_vh);
    S.stage = reinterpret_cast<float*>(base + A.o_stage);
    S.misc = reinterpret_cast<int32_t*>(base + A.o_misc);
    S.gvis = A.gvis + (size_t)gwarp * (A.gmask + 1);
    S.epoch = A.gepoch[gwarp];
#ifdef PW_PHASE_TIMERS
    for (int i = 0; i < 8; i++) S.pc[i] = 0;
#endif
    S.gscr = A.gscratch + (size_t)gwarp * A.gscratch_words;
    S.mbar = reinterpret_cast<uint64_t*>(base + A.o_mbar);
    S.desc = reinterpret_cast<uint4*>(base + A.o_desc);
    S.phase = 0;
    if (lane < 3) mbar_init(S.mbar + lane);
    mbar_fence_init();
    __syncwarp();

    while (true) {
        int task = 0;
        if (lane == 0) task = atomicAdd(A.task_counter, 1);
        task = __shfl_sync(0xffffffffu, task, 0);
        if (task >= A.n_tasks) break;
        int64_t qid = A.q0 + task;
        int64_t row = task;  // query / output / stats row
        int32_t stage = A.stage;
        bool has_entry = A.entries != nullptr;
        // forwarded entries land in cand[0..n_ent) (the seed list's head)
        int n_ent = 0;
        if (has_entry) {
            if ((int)lane < A.fwd) S.cand[lane] = A.entries[(int64_t)task * A.fwd + lane];
            n_ent = A.fwd;
        }
        if (A.df) {
            // stage-major task list of shard g: stage s searches chunk (g - s) mod N
            stage = 0;
            while (stage + 1 < A.df_N && task >= A.df_base[stage + 1]) stage++;
            const int c = (A.df_g - stage + A.df_N) % A.df_N;
            qid = A.df_lo[c] + (task - A.df_base[stage]);
            row = qid;
            has_entry = stage > 0;
            if (has_entry) {
                if (lane == 0) {
                    // bounded wait (~10 s): a producer that never comes (a
                    // shard not resident, a dead peer) raises an error
                    // instead of hanging the GPU.  F words per query, each
                    // stored with release semantics: poll them in order.
                    uint32_t spin = 0;
                    for (int f = 0; f < A.fwd; f++) {
                        unsigned long long v = 0;
                        for (;; spin++) {
                            v = ld_acquire_sys(A.df_inbox + qid * A.fwd + f);
                            if ((uint32_t)(v >> 32) == A.df_epoch) break;
                            if (spin > (1u << 25)) {
                                atomicOr(A.err, 16);
                                v = 0;
                                break;
                            }
                            __nanosleep(256);
                        }
                        S.cand[f] = (int32_t)(uint32_t)v;
                    }
                }
                n_ent = A.fwd;
                __syncwarp();
            }
        }
        if (A.qready) {
            // overlapped upload: wait (bounded) for this row's chunk to land
            if (lane == 0) {
                // chunk c holds rows [q_chunk (2^c - 1), q_chunk (2^(c+1) - 1))
                const int64_t qr = A.df ? row : A.q0 + row;
                const uint32_t* f = A.qready + (31 - __clz((int)(qr / A.q_chunk) + 1));
                for (uint32_t spin = 0; ld_acquire_gpu_u32(f) != A.q_epoch; spin++) {
                    if (spin > (1u << 25)) {
                        atomicOr(A.err, 64);
                        if (A.phase) {  // diagnostics: what was seen, where
                            A.phase[0] = ld_acquire_gpu_u32(f);
                            A.phase[1] = A.q_epoch;
                            A.phase[2] = (unsigned long long)(f - A.qready);
                            A.phase[3] = (unsigned long long)A.q_chunk;
                        }
                        break;
                    }
                    __nanosleep(128);
                }
            }
            __syncwarp();
        }
        // query row -> smem
        for (int t = lane; t < A.d; t += 32) S.q[t] = A.queries[(size_t)row * A.d + t];
        if constexpr (sizeof(VT) == 1 && M == 0 && D > 0) {
            // the query's bytes, sum q^2 and whether it is integer-valued in
            // [0, 255] (then pw_row4_u8i is exact; else the float path runs)
            uint8_t* qb = reinterpret_cast<uint8_t*>(S.q + ((D + 3) & ~3));
            bool ok = true;
            int sq = 0;
            for (int t = lane; t < ((D + 15) & ~15); t += 32) {
                uint32_t b = 0;
                if (t < D) {
                    const float v = A.queries[(size_t)row * A.d + t];
                    ok &= v >= 0.f && v <= 255.f && v == rintf(v);
                    b = ok ? (uint32_t)v : 0u;
                    sq += (int)(b * b);
                }
                qb[t] = (uint8_t)b;
            }
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) sq += __shfl_xor_sync(0xffffffffu, sq, o);
            const bool all = __all_sync(0xffffffffu, ok);
            if (lane == 0) {
                int32_t* qmeta = reinterpret_cast<int32_t*>(qb + ((D + 15) & ~15));
                qmeta[0] = sq;
                qmeta[1] = all ? 1 : 0;
            }
        }
        // the task's (qid, stage) wait in shared memory instead of registers
        // across the search: the hot loop runs at the 128-register cap
        int32_t* tsk = S.misc + A.o_par - 2;
        if (lane == 0) {
            tsk[0] = (int32_t)qid;
            tsk[1] = stage;
        }
        __syncwarp();

        int32_t g_it = 0;
        int32_t g_dc = 0, g_tv = 0, g_ne = 0;  // ghost-stage counters (32-bit like the search's)
        int64_t n_logged = 0;
        const GraphDev& G = A.use_ghost_graph ? A.ghost : A.main;

        // Phase 0 = ghost staging (pipeline.py:218-226) when the task has no
        // entry; phase 1 = the shard search.  One call site keeps a single
        // inlined copy of run_search in the kernel.
        bool converged = false;
        const bool ghost_phase = !has_entry && A.n_seeds == 0 && A.ghost_on;
        for (int phase = ghost_phase ? 0 : 1; phase < 2; phase++) {
            const bool gph = phase == 0;
            int ns = 0;
            bool fill_random = true;
            Pcg64 rng;
            if (gph) {
                rng = pcg64_from_seed(derive_seed3(A.seed, 5, (uint64_t)tsk[0], (uint64_t)tsk[1]));
            } else {
                // seeds (pipeline.py:227-231, search.py:294)
                if (A.n_seeds > 0) {
                    for (int t = lane; t < A.n_seeds; t += 32) S.cand[t] = (int32_t)A.seeds[t];
                    ns = A.n_seeds;
                    fill_random = A.seed_mode == 1;
                } else if (has_entry) {
                    // [e] + adj[e] (pipeline.py:229-231); with F forwarded
                    // entries (opt-in): [e_0..e_F-1] + adj[e_0] + ... + adj[e_F-1]
                    ns = n_ent;
                    if (A.seed_mode == 0) {
                        for (int f = 0; f < n_ent; f++) {
                            const int32_t e = S.cand[f];
                            for (int t = lane; t < G.j; t += 32) S.cand[n_ent + f * G.j + t] = G.adj[(size_t)e * G.j + t];
                        }
                        ns = n_ent * (1 + G.j);
                        fill_random = false;
                    }
                }
                __syncwarp();
                rng = A.rng_io ? A.rng_io[task]
                               : pcg64_from_seed(derive_seed3(A.seed, 4, (uint64_t)tsk[0], (uint64_t)tsk[1]));
            }
            converged = run_search<D, VT, M, FAST, (MAXT > PW_MAX_THREADS)>(A, S, gph ? A.ghost : G,
                                                                         (&A.cfg)[gph ? 2 : (tsk[1] > 0 ? 1 : 0)],
                                             ns, fill_random, rng, task, &n_logged);
            if (gph) {
                if (lane == 0) S.cand[0] = A.ghost.gid[(uint32_t)S.qk_cur()[0]];
                __syncwarp();
                n_ent = 1;
                has_entry = true;
                g_it = (int32_t)S.c_it;
                g_dc = S.c_dc;
                g_tv = S.c_tv;
                g_ne = S.c_ne;
                n_logged = 0;
            } else if (A.rng_io && lane == 0) {
                A.rng_io[task] = rng;
            }
        }

        // outputs (search.py:323-335, pipeline.py:236-246, :339)
        qid = tsk[0];
        stage = tsk[1];
        row = A.df ? qid : task;
        const uint64_t* qk = S.qk_cur();
        const int nk = min(S.qlen, A.cfg.k);
        for (int t = lane; t < nk; t += 32) {
            uint64_t key = qk[t];
            uint32_t loc = (uint32_t)key;
            A.out_ids[row * A.out_stride + t] = G.gid[loc];
            // search.py:325 sqrt of the squared L2; IP reports the distance itself
            const float dk = bits_dist<M>((uint32_t)(key >> 32));
            A.out_dists[row * A.out_stride + t] = M == 0 ? __fsqrt_rn(dk) : dk;
            if (A.out_local) A.out_local[row * A.out_stride + t] = (int32_t)loc;
        }
        if (A.df) {
            // short lists padded -1 / +inf here (pipeline.py:244-246): the
            // output may be another GPU's buffer, written by nobody else
            for (int t = nk + lane; t < A.cfg.k; t += 32) {
                A.out_ids[row * A.out_stride + t] = -1;
                A.out_dists[row * A.out_stride + t] = __int_as_float(0x7f800000);
            }
            if (lane == 0) {
                // pipeline.py:339 forward inter_map[top1] to shard g+1 (opt-in:
                // the top F, short queues repeating their last entry)
                if (stage + 1 < A.df_N)
                    for (int f = 0; f < A.fwd; f++)
                        st_release_sys(A.df_next + qid * A.fwd + f,
                                       ((unsigned long long)A.df_epoch << 32) |
                                           (uint32_t)(nk > 0 ? A.inter[(uint32_t)qk[min(f, S.qlen - 1)]] : 0));
                if (A.st32) {
                    int32_t* s32 = A.st32 + stage * A.st32_stage_stride + qid;
                    int64_t* s64 = A.st64 + stage * A.st64_stage_stride + qid;
                    s32[0 * A.st_stride] = (int32_t)S.c_it;
                    s32[1 * A.st_stride] = g_it;
                    s32[2 * A.st_stride] = S.qlen;
                    s32[3 * A.st_stride] = converged ? 1 : 0;
                    s64[0 * A.st_stride] = (int64_t)S.c_dc + g_dc;
                    s64[1 * A.st_stride] = (int64_t)S.c_tv + g_tv;
                    s64[2 * A.st_stride] = S.c_ins;
                    s64[3 * A.st_stride] = S.c_dgs;
                    s64[4 * A.st_stride] = S.c_ne;
                    s64[5 * A.st_stride] = g_ne;
                }
            }
        } else {
            if (A.forward && nk > 0 && (int)lane < A.fwd)
                A.forward[(int64_t)task * A.fwd + lane] = A.inter[(uint32_t)qk[min((int)lane, S.qlen - 1)]];
        }
        if (!A.df && lane == 0) {
            if (A.st32) {
                A.st32[0 * A.st_stride + task] += (int32_t)S.c_it;
                A.st32[1 * A.st_stride + task] += g_it;
                A.st32[2 * A.st_stride + task] += S.qlen;
                A.st32[3 * A.st_stride + task] = converged ? 1 : 0;
                A.st64[0 * A.st_stride + task] += (int64_t)S.c_dc + g_dc;
                A.st64[1 * A.st_stride + task] += (int64_t)S.c_tv + g_tv;
                A.st64[2 * A.st_stride + task] += S.c_ins;
                A.st64[3 * A.st_stride + task] += S.c_dgs;
                A.st64[4 * A.st_stride + task] += S.c_ne;
                A.st64[5 * A.st_stride + task] += g_ne;
            }
            if (A.rec) {
                TaskRecord& R = A.rec[task];
                R.c[0] = S.c_it;
                R.c[1] = S.c_dc;
                R.c[2] = S.c_tv;
                R.c[3] = S.c_ne;
                R.c[4] = S.c_dgs;
                R.c[5] = S.c_ins;
                R.converged = converged ? 1 : 0;
                R.retained = S.qlen;
                R.n_out = nk;
                R.n_visited = n_logged;
            }
        }
        __syncwarp();
    }
    if (lane == 0) A.gepoch[gwarp] = S.epoch;
#ifdef PW_PHASE_TIMERS
    if (lane == 0)
        for (int i = 0; i < 8; i++) atomicAdd(A.phase + i, (unsigned long long)S.pc[i]);
#endif
}

typedef void (*KernelFn)(KArgs);

}  // namespace pw
