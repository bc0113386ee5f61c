// knn_screen.cu -- K4: fused tensor-core kNN screen for the exact index build
// (shardann/graphs.py:65-78 `_knn_block`: a GEMM-style distance screen keeping
// k + pad candidates per row, which the builder then rescores exactly).
//
// One CTA owns 128 query rows and streams every column tile of the base rows:
//   warp 0      TMA producer: the query block once, then base tiles (BN rows x
//               d, K-major, 128-byte swizzle) into a STAGES-deep ring
//   warp 1      MMA issuer: tcgen05.mma kind::tf32 (M=128, N=BN, K=8 per
//               instruction) into one of two TMEM accumulators (BN columns
//               each), tcgen05.commit to free ring slots / hand a tile over
//   warps 2..5  epilogue: tcgen05.ld of the row's BN accumulators, approximate
//               squared distance |x_c|^2 - 2 q.x_c, and a per-row list of the
//               KC smallest (self excluded) in shared memory; a value only
//               enters when it beats the row's current worst (a compare per
//               value once the list is warm)
// Nothing of the n x n distance matrix is ever written to memory.  The
// approximate values (TF32 operands, FP32 accumulation) only SELECT
// candidates: the builder rescores them with the bit-exact numpy-pairwise L2
// and certifies each row (exact.py: a row whose margin between its KC-th
// screened value and its j-th exact distance exceeds the TF32 error bound is
// provably exact; the rest are redone by the FP32 screen).
#include <cuda.h>
#include <cuda_runtime.h>
#include <stdint.h>
#include <cstdio>
#include <cstdlib>

namespace knn {

constexpr int BM = 128;        // query rows per CTA (MMA M, TMEM lanes)
constexpr int NTHREADS = 192;  // warp 0 TMA, warp 1 MMA, warps 2..5 epilogue
constexpr int ATOM = 128;      // bytes per 128B-swizzle row (32 fp32 of K)

struct Args {
    int64_t nq, n;             // query rows, base rows
    int32_t d, ka;             // dimension, K atoms (ceil(d / 32))
    int32_t bn, stages, kc;    // column tile, ring depth, candidates per row
    int64_t self_off;          // query row r is base row r + self_off (excluded); < 0: none
    const float* xn;           // (n,) |x_c|^2
    int32_t* out_ids;          // (nq, kc)
    float* out_vals;           // (nq, kc)
    uint32_t o_b, o_bar, o_lv, o_li, o_tmem, o_nb, o_scr;  // shared-memory offsets
    int32_t debug;             // A/B probes: 1 skip the compare loop, 2 no norm loads
    int32_t stream_a;          // 1: the query block does not fit beside the ring (d > 128 with
                               // 64-candidate lists): ring stages hold one K atom of the query
                               // block AND of the column tile, the query atoms re-read (L2) per tile
};

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

__device__ __forceinline__ bool elect_one() {
    uint32_t pred = 0;
    asm volatile("{\n .reg .pred P;\n elect.sync _|P, 0xffffffff;\n selp.u32 %0, 1, 0, P;\n}\n" : "=r"(pred));
    return pred != 0;
}

__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(smem_u32(bar)), "r"(bytes)
                 : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];\n" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
    uint32_t done = 0;
    while (!done) {
        asm volatile(
            "{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2, 1000000;\n selp.u32 %0, 1, 0, p;\n}\n"
            : "=r"(done)
            : "r"(smem_u32(bar)), "r"(parity)
            : "memory");
    }
}

// 2D TMA tile load {x (K elements), y (rows)} completing on bar
__device__ __forceinline__ void tma_load_2d(void* dst, const CUtensorMap* tm, int32_t x, int32_t y, uint64_t* bar) {
    asm volatile(
        "cp.async.bulk.tensor.2d.shared::cta.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];\n" ::"r"(
            smem_u32(dst)),
        "l"(tm), "r"(x), "r"(y), "r"(smem_u32(bar))
        : "memory");
}

// UMMA shared-memory descriptor, K-major, 128-byte swizzle: 8-row groups
// 1024 bytes apart (SBO), version 1 (sm_100), layout SWIZZLE_128B
__device__ __forceinline__ uint64_t sw128_desc(uint32_t saddr) {
    uint64_t desc = 0;
    desc |= (uint64_t)((saddr & 0x3FFFFu) >> 4);          // start address [0,14)
    desc |= (uint64_t)(16u >> 4) << 16;                   // LBO (unused for swizzled K-major)
    desc |= (uint64_t)(1024u >> 4) << 32;                 // SBO [32,46)
    desc |= (uint64_t)1 << 46;                            // version [46,48)
    desc |= (uint64_t)2 << 61;                            // SWIZZLE_128B [61,64)
    return desc;
}

// instruction descriptor kind::tf32: D f32, A/B tf32, both K-major, M x N
__host__ __device__ constexpr uint32_t idesc_tf32(int m, int n) {
    return (1u << 4) | (2u << 7) | (2u << 10) | ((uint32_t)(n >> 3) << 17) | ((uint32_t)(m >> 4) << 24);
}

__device__ __forceinline__ void mma_tf32(uint32_t d_tmem, uint64_t a, uint64_t b, uint32_t idesc, uint32_t acc) {
    asm volatile(
        "{\n .reg .pred p;\n setp.ne.b32 p, %4, 0;\n"
        " tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n}\n" ::"r"(d_tmem),
        "l"(a), "l"(b), "r"(idesc), "r"(acc));
}
__device__ __forceinline__ void mma_commit(uint64_t* bar) {
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n" ::"r"(smem_u32(bar))
                 : "memory");
}
__device__ __forceinline__ void tc_fence_before() { asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory"); }
__device__ __forceinline__ void tc_fence_after() { asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory"); }

// 32 consecutive fp32 columns of this thread's TMEM lane; the caller waits
// (tcgen05.wait::ld) before touching v, so a load can overlap other work
__device__ __forceinline__ void tmem_ld32_issue(uint32_t addr, float (&v)[32]) {
    uint32_t* r = reinterpret_cast<uint32_t*>(v);
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0, %1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, %14, "
        "%15, %16, %17, %18, %19, %20, %21, %22, %23, %24, %25, %26, %27, %28, %29, %30, %31}, [%32];\n"
        : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
          "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15]),
          "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]),
          "=r"(r[24]), "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
        : "r"(addr));
}
__device__ __forceinline__ void tmem_ld_wait() { asm volatile("tcgen05.wait::ld.sync.aligned;\n" ::: "memory"); }

__global__ void __launch_bounds__(NTHREADS, 1)
    knn_screen_kernel(const __grid_constant__ CUtensorMap tm_q, const __grid_constant__ CUtensorMap tm_x,
                      const __grid_constant__ Args A) {
    extern __shared__ __align__(1024) unsigned char sm[];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int64_t row0 = (int64_t)blockIdx.x * BM;
    const int BN = A.bn, ST = A.stages, KA = A.ka;
    unsigned char* sa = sm;                    // query block: KA atoms x (BM x 128 B)
    unsigned char* sb = sm + A.o_b;            // ring: ST x KA atoms x (BN x 128 B)
    uint64_t* bar = reinterpret_cast<uint64_t*>(sm + A.o_bar);
    uint64_t* a_full = bar;                    // [0]
    uint64_t* full = bar + 1;                  // [1, 1 + ST)
    uint64_t* empty = bar + 1 + ST;            // [1 + ST, 1 + 2 ST)
    uint64_t* acc_full = bar + 1 + 2 * ST;     // [2]
    uint64_t* acc_empty = bar + 3 + 2 * ST;    // [2]
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(sm + A.o_tmem);
    const int64_t ntiles = (A.n + BN - 1) / BN;
    const uint32_t b_stage_bytes = (uint32_t)(BN * KA * ATOM);

    if (warp == 0 && lane == 0) {
        mbar_init(a_full, 1);
        for (int s = 0; s < ST; s++) {
            mbar_init(full + s, 1);
            mbar_init(empty + s, 1);
        }
        for (int b = 0; b < 2; b++) {
            mbar_init(acc_full + b, 1);
            mbar_init(acc_empty + b, 4);  // one arrive per epilogue warp
        }
        asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
    }
    if (warp == 1) {  // TMEM: two accumulators of BN fp32 columns
        const uint32_t cols = 2u * (uint32_t)BN;
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;\n" ::"r"(smem_u32(tmem_slot)),
                     "r"(cols));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;\n");
    }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = *tmem_slot;

    if (warp == 0) {
        // ---------------- TMA producer
        if (elect_one()) {
            asm volatile("prefetch.tensormap [%0];\n" ::"l"(&tm_q) : "memory");
            asm volatile("prefetch.tensormap [%0];\n" ::"l"(&tm_x) : "memory");
            if (!A.stream_a) {
                mbar_expect_tx(a_full, (uint32_t)(BM * KA * ATOM));
                for (int a = 0; a < KA; a++)
                    tma_load_2d(sa + (size_t)a * BM * ATOM, &tm_q, 32 * a, (int32_t)row0, a_full);
                for (int64_t t = 0; t < ntiles; t++) {
                    const int s = (int)(t % ST);
                    const uint32_t ph = (uint32_t)((t / ST) & 1);
                    mbar_wait(empty + s, ph ^ 1u);
                    mbar_expect_tx(full + s, b_stage_bytes);
                    unsigned char* dst = sb + (size_t)s * b_stage_bytes;
                    for (int a = 0; a < KA; a++)
                        tma_load_2d(dst + (size_t)a * BN * ATOM, &tm_x, 32 * a, (int32_t)(t * BN), full + s);
                }
            } else {
                // one stage per (tile, K atom): the query atom, then the column atom
                const uint32_t st_bytes = (uint32_t)((BM + BN) * ATOM);
                int64_t i = 0;
                for (int64_t t = 0; t < ntiles; t++)
                    for (int a = 0; a < KA; a++, i++) {
                        const int s = (int)(i % ST);
                        const uint32_t ph = (uint32_t)((i / ST) & 1);
                        mbar_wait(empty + s, ph ^ 1u);
                        mbar_expect_tx(full + s, st_bytes);
                        unsigned char* dst = sb + (size_t)s * st_bytes;
                        tma_load_2d(dst, &tm_q, 32 * a, (int32_t)row0, full + s);
                        tma_load_2d(dst + (size_t)BM * ATOM, &tm_x, 32 * a, (int32_t)(t * BN), full + s);
                    }
            }
        }
    } else if (warp == 1) {
        // ---------------- MMA issuer (one thread)
        const uint32_t idesc = idesc_tf32(BM, BN);
        const uint32_t sa_u = smem_u32(sa), sb_u = smem_u32(sb);
        if (!A.stream_a) {
            mbar_wait(a_full, 0);
            for (int64_t t = 0; t < ntiles; t++) {
                const int s = (int)(t % ST);
                const uint32_t ph = (uint32_t)((t / ST) & 1);
                const int buf = (int)(t & 1);
                const uint32_t aph = (uint32_t)((t >> 1) & 1);
                mbar_wait(acc_empty + buf, aph ^ 1u);  // epilogue drained this accumulator
                mbar_wait(full + s, ph);               // tile landed
                tc_fence_after();
                if (elect_one()) {
                    const uint32_t d_tmem = tmem + (uint32_t)(buf * BN);
                    const uint32_t b0 = sb_u + (uint32_t)s * b_stage_bytes;
                    for (int a = 0; a < KA; a++)
                        for (int kk = 0; kk < 4; kk++) {  // K = 8 tf32 = 32 bytes per instruction
                            const uint64_t da = sw128_desc(sa_u + (uint32_t)(a * BM * ATOM + kk * 32));
                            const uint64_t db = sw128_desc(b0 + (uint32_t)(a * BN * ATOM + kk * 32));
                            mma_tf32(d_tmem, da, db, idesc, (a | kk) ? 1u : 0u);
                        }
                    mma_commit(empty + s);        // ring slot free once these MMAs have read it
                    mma_commit(acc_full + buf);   // accumulator ready for the epilogue
                }
                __syncwarp();
            }
        } else {
            const uint32_t st_bytes = (uint32_t)((BM + BN) * ATOM);
            int64_t i = 0;
            for (int64_t t = 0; t < ntiles; t++) {
                const int buf = (int)(t & 1);
                const uint32_t aph = (uint32_t)((t >> 1) & 1);
                const uint32_t d_tmem = tmem + (uint32_t)(buf * BN);
                mbar_wait(acc_empty + buf, aph ^ 1u);
                for (int a = 0; a < KA; a++, i++) {
                    const int s = (int)(i % ST);
                    const uint32_t ph = (uint32_t)((i / ST) & 1);
                    mbar_wait(full + s, ph);
                    tc_fence_after();
                    if (elect_one()) {
                        const uint32_t a0 = sb_u + (uint32_t)s * st_bytes, b0 = a0 + (uint32_t)(BM * ATOM);
                        for (int kk = 0; kk < 4; kk++)
                            mma_tf32(d_tmem, sw128_desc(a0 + (uint32_t)(kk * 32)), sw128_desc(b0 + (uint32_t)(kk * 32)),
                                     idesc, (a | kk) ? 1u : 0u);
                        mma_commit(empty + s);
                        if (a == KA - 1) mma_commit(acc_full + buf);
                    }
                    __syncwarp();
                }
            }
        }
    } else {
        // ---------------- epilogue: warp w reads TMEM lanes 32 * (w % 4) ..
        const int quad = warp & 3;
        const int r_local = quad * 32 + lane;
        const int64_t row = row0 + r_local;
        const bool live = row < A.nq;
        const int64_t self_col = (A.self_off >= 0 && live) ? row + A.self_off : -1;
        float* lv = reinterpret_cast<float*>(sm + A.o_lv);    // [kc][BM], column per thread
        int32_t* li = reinterpret_cast<int32_t*>(sm + A.o_li);
        float* nb = reinterpret_cast<float*>(sm + A.o_nb);    // [2][BN] column norms per accumulator
        float* scr = reinterpret_cast<float*>(sm + A.o_scr);  // [32][BM] slow-path values
        const int KC = A.kc;
        for (int k = 0; k < KC; k++) {
            lv[k * BM + r_local] = __int_as_float(0x7f800000);
            li[k * BM + r_local] = -1;
        }
        const float inf = __int_as_float(0x7f800000);
        float tau = inf;  // the list's current worst
        int tpos = 0;
        // column norms one tile ahead (thread i < BN loads norm i, coalesced);
        // columns past n get +inf, so zero-filled rows never qualify
        auto norm_of = [&](int64_t t) -> float {
            const int64_t c = t * BN + r_local;
            return (r_local < BN && c < A.n && !(A.debug & 2)) ? __ldg(A.xn + c) : (c < A.n ? 0.f : inf);
        };
        float nnext = norm_of(0);
        for (int64_t t = 0; t < ntiles; t++) {
            const int buf = (int)(t & 1);
            const uint32_t aph = (uint32_t)((t >> 1) & 1);
            if (r_local < BN) nb[buf * BN + r_local] = nnext;
            asm volatile("bar.sync 1, 128;\n" ::: "memory");  // the 4 epilogue warps
            nnext = t + 1 < ntiles ? norm_of(t + 1) : 0.f;
            mbar_wait(acc_full + buf, aph);
            tc_fence_after();
            const int64_t c_base = t * BN;
            const float4* nb4 = reinterpret_cast<const float4*>(nb + buf * BN);
            const uint32_t taddr = tmem + ((uint32_t)(quad * 32) << 16) + (uint32_t)(buf * BN);
            float accb[2][32];
            tmem_ld32_issue(taddr, accb[0]);
            tmem_ld_wait();
#pragma unroll
            for (int c0 = 0; c0 < 128; c0 += 32) {
                if (c0 >= BN || (A.debug & 1)) break;
                float (&acc)[32] = accb[(c0 >> 5) & 1];
                // the next chunk's TMEM load overlaps this chunk's compare
                if (c0 + 32 < BN) tmem_ld32_issue(taddr + (uint32_t)(c0 + 32), accb[((c0 >> 5) + 1) & 1]);
                // fast path: 32 values, four independent running minima
                float m0 = inf, m1 = inf, m2 = inf, m3 = inf;
#pragma unroll
                for (int i = 0; i < 32; i += 4) {
                    const float4 xn4 = nb4[(c0 + i) >> 2];
                    acc[i] = __fmaf_rn(-2.f, acc[i], xn4.x);
                    acc[i + 1] = __fmaf_rn(-2.f, acc[i + 1], xn4.y);
                    acc[i + 2] = __fmaf_rn(-2.f, acc[i + 2], xn4.z);
                    acc[i + 3] = __fmaf_rn(-2.f, acc[i + 3], xn4.w);
                    m0 = fminf(m0, acc[i]);
                    m1 = fminf(m1, acc[i + 1]);
                    m2 = fminf(m2, acc[i + 2]);
                    m3 = fminf(m3, acc[i + 3]);
                }
                if (fminf(fminf(m0, m1), fminf(m2, m3)) < tau) {
                    // slow path (rare once the list is warm): park the 32
                    // values in this thread's scratch column (registers stay
                    // statically indexed), then insert
                    const int64_t cb = c_base + c0;
#pragma unroll
                    for (int i = 0; i < 32; i++) scr[i * BM + r_local] = acc[i];
#pragma unroll 1
                    for (int i = 0; i < 32; i++) {
                        const float v = scr[i * BM + r_local];
                        if (v < tau && cb + i != self_col) {
                            lv[tpos * BM + r_local] = v;
                            li[tpos * BM + r_local] = (int32_t)(cb + i);
                            float w = lv[r_local];
                            int wp = 0;
                            for (int k = 1; k < KC; k++) {
                                const float x = lv[k * BM + r_local];
                                if (x > w) {
                                    w = x;
                                    wp = k;
                                }
                            }
                            tau = w;
                            tpos = wp;
                        }
                    }
                }
                tmem_ld_wait();
            }
            tc_fence_before();
            __syncwarp();
            if (lane == 0) mbar_arrive(acc_empty + buf);
        }
        if (live) {
            for (int k = 0; k < KC; k++) {
                A.out_ids[row * KC + k] = li[k * BM + r_local];
                A.out_vals[row * KC + k] = lv[k * BM + r_local];
            }
        }
    }
    tc_fence_before();
    __syncthreads();
    if (warp == 1) {
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;\n" ::"r"(tmem), "r"(2u * (uint32_t)BN));
    }
}

}  // namespace knn

// ------------------------------------------------------------------ host
namespace {

typedef CUresult (*EncodeTiledFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                  const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                  CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

EncodeTiledFn knn_encode() {
    static EncodeTiledFn fn = nullptr;
    static bool tried = false;
    if (!tried) {
        tried = true;
        void* p = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
            q == cudaDriverEntryPointSuccess)
            fn = reinterpret_cast<EncodeTiledFn>(p);
    }
    return fn;
}

// {d, rows} fp32 rows, box {32, box_rows}, 128-byte swizzle, OOB zero fill
bool knn_map(CUtensorMap* tm, const float* base, int64_t rows, int32_t d, int32_t box_rows) {
    EncodeTiledFn fn = knn_encode();
    if (!fn) return false;
    const cuuint64_t dims[2] = {(cuuint64_t)d, (cuuint64_t)rows};
    const cuuint64_t strides[1] = {(cuuint64_t)d * 4u};
    const cuuint32_t box[2] = {32u, (cuuint32_t)box_rows};
    const cuuint32_t estr[2] = {1u, 1u};
    return fn(tm, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, const_cast<float*>(base), dims, strides, box, estr,
              CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
              CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

}  // namespace

// status: 0 ok, -1 bad argument / unsupported shape, -3 CUDA error; msg (>= 256 bytes) on failure
extern "C" int pw_knn_screen_impl(const float* q, int64_t nq, const float* x, int64_t n, int32_t d,
                                  const float* xn, int64_t self_off, int32_t kc, int32_t* out_ids,
                                  float* out_vals, void* stream, char* msg) {
    using namespace knn;
    static const int debug = getenv("PW_KNN_DEBUG") ? atoi(getenv("PW_KNN_DEBUG")) : 0;
    if (nq <= 0) return 0;
    if (!q || !x || !xn || !out_ids || !out_vals || n <= 0 || d < 1 || kc < 1 || kc > 64 || n >= (1ll << 31) ||
        nq >= (1ll << 31) || (d * 4) % 16 != 0) {
        snprintf(msg, 256, "knn screen: unsupported arguments (d %% 4 == 0, 1 <= kc <= 64, n < 2^31)");
        return -1;
    }
    const int ka = (d + 31) / 32;
    // shared memory: query block + ring + barriers + lists; pick the widest
    // column tile and deepest ring that fit
    int dev = 0;
    cudaGetDevice(&dev);
    int optin = 0;
    cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev);
    const size_t a_bytes = (size_t)BM * ka * ATOM;
    const size_t lists = (size_t)kc * BM * 8;
    const size_t fixed = 1024 + lists + 2048 + 32 * BM * 4;
    int bn = 0, st = 0, stream_a = 0;
    for (int cand_bn : {128, 64, 32})
        for (int cand_st : {4, 3, 2}) {
            const size_t need = a_bytes + (size_t)cand_st * cand_bn * ka * ATOM + fixed;
            if (!bn && need <= (size_t)optin) {
                bn = cand_bn;
                st = cand_st;
            }
        }
    if (!bn || (bn < 128 && ka > 4)) {
        // large d: stream the query block per K atom beside the column atoms
        // (1-atom stages, so the ring is deep enough to cover the TMA latency)
        bn = 0;
        for (int cand_st : {8, 6, 5, 4, 3})
            if (!bn && (size_t)cand_st * (BM + 128) * ATOM + fixed <= (size_t)optin) {
                bn = 128;
                st = cand_st;
                stream_a = 1;
            }
    }
    if (!bn) {
        snprintf(msg, 256, "knn screen: d=%d needs more shared memory than the device has", d);
        return -1;
    }
    Args A{};
    A.nq = nq;
    A.n = n;
    A.d = d;
    A.ka = ka;
    A.bn = bn;
    A.stages = st;
    A.kc = kc;
    A.self_off = self_off;
    A.xn = xn;
    A.out_ids = out_ids;
    A.out_vals = out_vals;
    A.debug = debug;
    A.stream_a = stream_a;
    size_t off = stream_a ? 0 : a_bytes;
    A.o_b = (uint32_t)off;
    off += stream_a ? (size_t)st * (BM + bn) * ATOM : (size_t)st * bn * ka * ATOM;
    A.o_bar = (uint32_t)off;
    off += 8 * (1 + 2 * st + 4);
    A.o_tmem = (uint32_t)off;
    off += 16;
    off = (off + 15) / 16 * 16;
    A.o_lv = (uint32_t)off;
    off += (size_t)kc * BM * 4;
    A.o_li = (uint32_t)off;
    off += (size_t)kc * BM * 4;
    A.o_nb = (uint32_t)off;
    off += (size_t)2 * bn * 4;
    A.o_scr = (uint32_t)off;
    off += (size_t)32 * BM * 4;
    CUtensorMap tq, tx;
    if (!knn_map(&tq, q, nq, d, BM) || !knn_map(&tx, x, n, d, bn)) {
        snprintf(msg, 256, "knn screen: cuTensorMapEncodeTiled failed");
        return -3;
    }
    cudaError_t e = cudaFuncSetAttribute(knn_screen_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)off);
    if (e == cudaSuccess) {
        const int64_t blocks = (nq + BM - 1) / BM;
        knn_screen_kernel<<<(unsigned)blocks, NTHREADS, off, (cudaStream_t)stream>>>(tq, tx, A);
        e = cudaGetLastError();
    }
    if (e != cudaSuccess) {
        snprintf(msg, 256, "knn screen: %s", cudaGetErrorString(e));
        return -3;
    }
    return 0;
}
