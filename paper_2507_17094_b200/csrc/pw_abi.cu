// pw_abi.cu -- host side of the C ABI (include/pw_b200.h) + K2 reduce_topk.
//
// Owns device copies of shards (pipeline.py:121-155 build_contexts), derives
// per-search configuration from SearchParams exactly as search.py:289-295
// and direction.py:72-100 do, sizes the per-warp shared-memory layout of the
// beam-search kernel, and drives stages (pipeline.py:270-350).
#include <cuda_runtime.h>

#include <algorithm>
#include <atomic>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <mutex>
#include <string>
#include <type_traits>
#include <vector>

#include "../../include/pw_b200.h"
#include "beam_search.cuh"

using namespace pw;

namespace {

thread_local std::string g_err;
std::atomic<int64_t> g_launches{0};

int set_err(int code, const std::string& msg) {
    g_err = msg;
    return code;
}

#define PW_CUDA(call)                                                                  \
    do {                                                                               \
        cudaError_t e_ = (call);                                                       \
        if (e_ != cudaSuccess)                                                         \
            return set_err(e_ == cudaErrorMemoryAllocation ? PW_ENOMEM : PW_ECUDA,     \
                           std::string(#call) + ": " + cudaGetErrorString(e_));       \
    } while (0)

int words_per_vector(int d) { return (d + 31) / 32; }
int pw_fill_inf(float* p, int64_t n, cudaStream_t st);
int pw_init_run(int32_t* ids, float* dists, int64_t n, int32_t* s32, int64_t n32, int64_t* s64, int64_t n64,
                cudaStream_t st);

int32_t keep_count(int32_t j, double discard) {  // direction.py:72-76
    int32_t v = (int32_t)((1.0 - discard) * (double)j + 0.5);
    return v > 1 ? v : 1;
}
int32_t cooldown_start(int32_t max_iter, double ratio) {  // direction.py:90-100
    return max_iter - (int32_t)std::floor(ratio * (double)max_iter + 1e-9);
}
int64_t next_pow2(int64_t v) {
    int64_t p = 1;
    while (p < v) p <<= 1;
    return p;
}

// numpy pairwise_sum structure (loops_utils.h.src): leaves of <= 128
// elements, split at n2 = n/2 - (n/2)%8; postfix ops for the device stack.
void plan_rec(L2Plan& P, int off, int n) {
    if (n <= 128) {
        int i = P.n_leaves++;
        P.leaf_off[i] = (int16_t)off;
        P.leaf_len[i] = (int16_t)n;
        P.ops[P.n_ops++] = (int8_t)i;
        return;
    }
    int n2 = n / 2;
    n2 -= n2 % 8;
    plan_rec(P, off, n2);
    plan_rec(P, off + n2, n - n2);
    P.ops[P.n_ops++] = -1;
}

bool make_plan(int d, L2Plan& P) {
    std::memset(&P, 0, sizeof P);
    if (d > 128 * kMaxLeaves / 2 || d > 32767) return false;
    plan_rec(P, 0, d);
    return P.n_leaves <= kMaxLeaves && P.n_ops <= kMaxOps;
}

// Dimensions with a compile-time specialisation of K1 (TMA row gathers +
// compile-time pairwise order); any other d runs the generic instance.
// (PW_DIMS must match paper_2507_17094_b200/build_ext.py DIMS)
#define PW_DIMS(X) X(16) X(32) X(64) X(96) X(100) X(128) X(200) X(256) X(384) X(512) X(768) X(960) X(1024)
// uint8 rows: single-leaf specialisations with 16-byte rows (d <= 128, d % 16 == 0)
#define PW_DIMS_U8(X) X(96) X(128)
// inner product (float32 rows)
#define PW_DIMS_IP(X) X(96) X(128) X(200)
typedef KernelFn kernel_fn;
}  // namespace
#define PW_DECL(v) KernelFn pw_kernel_##v(); KernelFn pw_kernel_f_##v(); KernelFn pw_kernel_fw_##v();
#define PW_DECL_U8(v) KernelFn pw_kernel_u8_##v(); KernelFn pw_kernel_u8_f_##v(); KernelFn pw_kernel_u8_fw_##v();
#define PW_DECL_IP(v) KernelFn pw_kernel_ip_##v(); KernelFn pw_kernel_ip_f_##v(); KernelFn pw_kernel_ip_fw_##v();
PW_DIMS(PW_DECL)
PW_DIMS_U8(PW_DECL_U8)
PW_DIMS_IP(PW_DECL_IP)
KernelFn pw_kernel_0();
KernelFn pw_kernel_u8_0();
KernelFn pw_kernel_ip_0();
#undef PW_DECL
#undef PW_DECL_U8
#undef PW_DECL_IP
namespace {
// fast: the FAST instance of a specialised d (beam_search.cuh); the generic
// instance has none
kernel_fn pick_kernel(int d, int dtype, int metric, bool fast = false, bool wide = false) {
    if (metric == PW_METRIC_IP) {
        switch (d) {
#define PW_CASE(v) \
    case v:        \
        return fast ? (wide ? pw_kernel_ip_fw_##v() : pw_kernel_ip_f_##v()) : pw_kernel_ip_##v();
            PW_DIMS_IP(PW_CASE)
#undef PW_CASE
            default:
                return pw_kernel_ip_0();
        }
    }
    if (dtype == PW_DTYPE_U8) {
        switch (d) {
#define PW_CASE(v) \
    case v:        \
        return fast ? (wide ? pw_kernel_u8_fw_##v() : pw_kernel_u8_f_##v()) : pw_kernel_u8_##v();
            PW_DIMS_U8(PW_CASE)
#undef PW_CASE
            default:
                return pw_kernel_u8_0();
        }
    }
    switch (d) {
#define PW_CASE(v) \
    case v:        \
        return fast ? (wide ? pw_kernel_fw_##v() : pw_kernel_f_##v()) : pw_kernel_##v();
        PW_DIMS(PW_CASE)
#undef PW_CASE
        default:
            return pw_kernel_0();
    }
}
bool is_generic(kernel_fn f) { return f == pw_kernel_0() || f == pw_kernel_u8_0() || f == pw_kernel_ip_0(); }

struct DevInfo {
    int sms = 0;
    int smem_optin = 0;
    bool attr_set = false;
    uint64_t* jump = nullptr;  // PCG64 jump-ahead table on this device
};

// {A^k, A^(k-1) + ... + A + 1} mod 2^128 for k = 1..kJumpMax (numpy PCG64's
// 128-bit LCG multiplier A), as {M_hi, M_lo, S_hi, S_lo} per k.
std::vector<uint64_t> pcg_jump_table() {
    typedef unsigned __int128 u128;
    const u128 A = ((u128)2549297995355413924ULL << 64) | 4865540595714422341ULL;
    std::vector<uint64_t> t(4 * kJumpMax);
    u128 M = 1, S = 0;
    for (int k = 1; k <= kJumpMax; k++) {
        S = S + M;  // S_k = S_(k-1) + A^(k-1)
        M = M * A;  // A^k
        uint64_t* e = &t[4 * (k - 1)];
        e[0] = (uint64_t)(M >> 64);
        e[1] = (uint64_t)M;
        e[2] = (uint64_t)(S >> 64);
        e[3] = (uint64_t)S;
    }
    return t;
}
std::mutex g_dev_mu;
DevInfo g_dev[64];

int dev_info(int dev, DevInfo** out) {
    std::lock_guard<std::mutex> lk(g_dev_mu);
    DevInfo& I = g_dev[dev];
    if (I.sms == 0) {
        PW_CUDA(cudaDeviceGetAttribute(&I.sms, cudaDevAttrMultiProcessorCount, dev));
        PW_CUDA(cudaDeviceGetAttribute(&I.smem_optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev));
    }
    // per-device state below is created on `dev` (the caller's current
    // device is restored on return)
    int cur = dev;
    PW_CUDA(cudaGetDevice(&cur));
    struct Restore {
        int d;
        ~Restore() { cudaSetDevice(d); }
    } restore{cur};
    if (cur != dev) PW_CUDA(cudaSetDevice(dev));
    if (!I.jump) {
        const std::vector<uint64_t> t = pcg_jump_table();
        PW_CUDA(cudaMalloc(&I.jump, t.size() * sizeof(uint64_t)));
        PW_CUDA(cudaMemcpy(I.jump, t.data(), t.size() * sizeof(uint64_t), cudaMemcpyHostToDevice));
    }
    if (!I.attr_set) {
        PW_CUDA(cudaFuncSetAttribute((const void*)pw_kernel_0(),
                                     cudaFuncAttributeMaxDynamicSharedMemorySize, I.smem_optin));
        PW_CUDA(cudaFuncSetAttribute((const void*)pw_kernel_u8_0(),
                                     cudaFuncAttributeMaxDynamicSharedMemorySize, I.smem_optin));
        PW_CUDA(cudaFuncSetAttribute((const void*)pw_kernel_ip_0(),
                                     cudaFuncAttributeMaxDynamicSharedMemorySize, I.smem_optin));
#define PW_ATTR(v)                                                                             \
    PW_CUDA(cudaFuncSetAttribute((const void*)pw_kernel_##v(),                                 \
                                 cudaFuncAttributeMaxDynamicSharedMemorySize, I.smem_optin)); \
    PW_CUDA(cudaFuncSetAttribute((const void*)pw_kernel_f_##v(),                               \
                                 cudaFuncAttributeMaxDynamicSharedMemorySize, I.smem_optin)); \
    PW_CUDA(cudaFuncSetAttribute((const void*)pw_kernel_fw_##v(), cudaFuncAttributeMaxDynamicSharedMemorySize, I.smem_optin));
        PW_DIMS(PW_ATTR)
#undef PW_ATTR
#define PW_ATTR(v)                                                                             \
    PW_CUDA(cudaFuncSetAttribute((const void*)pw_kernel_u8_##v(),                              \
                                 cudaFuncAttributeMaxDynamicSharedMemorySize, I.smem_optin)); \
    PW_CUDA(cudaFuncSetAttribute((const void*)pw_kernel_u8_f_##v(),                            \
                                 cudaFuncAttributeMaxDynamicSharedMemorySize, I.smem_optin)); \
    PW_CUDA(cudaFuncSetAttribute((const void*)pw_kernel_u8_fw_##v(), cudaFuncAttributeMaxDynamicSharedMemorySize, I.smem_optin));
        PW_DIMS_U8(PW_ATTR)
#undef PW_ATTR
#define PW_ATTR(v)                                                                             \
    PW_CUDA(cudaFuncSetAttribute((const void*)pw_kernel_ip_##v(),                              \
                                 cudaFuncAttributeMaxDynamicSharedMemorySize, I.smem_optin)); \
    PW_CUDA(cudaFuncSetAttribute((const void*)pw_kernel_ip_f_##v(),                            \
                                 cudaFuncAttributeMaxDynamicSharedMemorySize, I.smem_optin)); \
    PW_CUDA(cudaFuncSetAttribute((const void*)pw_kernel_ip_fw_##v(), cudaFuncAttributeMaxDynamicSharedMemorySize, I.smem_optin));
        PW_DIMS_IP(PW_ATTR)
#undef PW_ATTR
        I.attr_set = true;
    }
    *out = &I;
    return 0;
}

}  // namespace

struct pw_shard {
    int device = 0;
    int64_t n = 0;
    int32_t d = 0, j = 0, W = 0, dtype = 0;
    void* vec = nullptr;          // (n, d) f32 or u8 rows (dtype)
    int32_t* adj = nullptr;
    int32_t* gid = nullptr;
    uint32_t* dir = nullptr;
    int32_t* inter = nullptr;
    int64_t gn = 0;
    int32_t gj = 0;
    void* gvec = nullptr;
    int32_t* gadj = nullptr;
    int32_t* gids = nullptr;
    int64_t bytes = 0;
    int64_t inter_ok_n = -1;  // inter_map validated against a next shard of this size
    // launch workspace (grow-only)
    int32_t* counter = nullptr;
    unsigned long long* phase = nullptr;  // 8 cycle counters (timer builds)
    unsigned long long* gvis = nullptr;
    size_t gvis_words = 0;
    uint32_t* gepoch = nullptr;
    size_t gepoch_n = 0;
    int64_t gvis_stride = 0;  // per-warp table size the epochs are valid for
    int gvis_lossy = 0;       // table holds lossy-cache words (else exact epoch entries)
    uint32_t* gscr = nullptr;
    size_t gscr_words = 0;
    std::mutex mu;
};

namespace {

template <typename T>
int upload(T** dst, const void* src, size_t count, int64_t* bytes, bool on_device = false) {
    size_t c = count == 0 ? 1 : count;
    PW_CUDA(cudaMalloc((void**)dst, c * sizeof(T)));
    if (src && count)
        PW_CUDA(cudaMemcpy(*dst, src, count * sizeof(T),
                           on_device ? cudaMemcpyDeviceToDevice : cudaMemcpyHostToDevice));
    *bytes += (int64_t)(c * sizeof(T));
    return 0;
}

__global__ void gather_rows_kernel(const uint8_t* __restrict__ vec, const int32_t* __restrict__ ids,
                                   int64_t n_ids, int64_t row_bytes, uint8_t* __restrict__ out) {
    int64_t total = n_ids * row_bytes;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total;
         i += (int64_t)gridDim.x * blockDim.x) {
        int64_t r = i / row_bytes, c = i % row_bytes;
        out[i] = vec[(int64_t)ids[r] * row_bytes + c];
    }
}

// Index validation: count entries of p[0..n) outside [0, hi) and record the
// first such position (ids become gather indices inside K1, so a bad id in a
// CRC-valid but inconsistent container must be rejected before any search).
__global__ void range_check_kernel(const int32_t* __restrict__ p, int64_t n, int64_t hi,
                                   unsigned long long* __restrict__ out) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        const int32_t v = p[i];
        if (v < 0 || (int64_t)v >= hi) {
            atomicAdd(&out[0], 1ull);
            atomicMin(&out[1], (unsigned long long)i);
        }
    }
}

// Returns PW_EINVAL with "<what> id <v> at <pos> outside [0, hi)" when some
// entry is out of range (synchronous; shard creation / first pipelined use).
int check_ids(const int32_t* p, int64_t n, int64_t hi, const char* what) {
    if (!p || n <= 0) return 0;
    unsigned long long* d = nullptr;
    PW_CUDA(cudaMalloc(&d, 2 * sizeof(unsigned long long)));
    unsigned long long h[2] = {0ull, ~0ull};
    cudaError_t e = cudaMemcpy(d, h, sizeof h, cudaMemcpyHostToDevice);
    if (e == cudaSuccess) {
        range_check_kernel<<<(int)std::min<int64_t>(4096, (n + 255) / 256), 256>>>(p, n, hi, d);
        e = cudaGetLastError();
    }
    if (e == cudaSuccess) e = cudaMemcpy(h, d, sizeof h, cudaMemcpyDeviceToHost);
    int32_t v = 0;
    if (e == cudaSuccess && h[0]) e = cudaMemcpy(&v, p + h[1], sizeof v, cudaMemcpyDeviceToHost);
    cudaFree(d);
    g_launches++;
    if (e != cudaSuccess) return set_err(PW_ECUDA, std::string("index validation: ") + cudaGetErrorString(e));
    if (h[0])
        return set_err(PW_EINVAL, std::string(what) + " id " + std::to_string(v) + " at position " +
                                      std::to_string(h[1]) + " outside shard of " + std::to_string(hi) +
                                      " nodes (" + std::to_string(h[0]) + " such entries)");
    return 0;
}

// K2: per-query best k of n_cols*k candidates by (distance, id)
// (pipeline.py:187-196).  One warp per query; rank selection in shared memory.
__global__ void reduce_topk_kernel(const int32_t* __restrict__ ids, const float* __restrict__ dists,
                                   int64_t q, int32_t n, int32_t k, int32_t* __restrict__ out_ids,
                                   float* __restrict__ out_dists, int32_t* err) {
    extern __shared__ uint64_t rk_keys[];
    const int warps = blockDim.x >> 5;
    const int w = threadIdx.x >> 5;
    const unsigned lane = threadIdx.x & 31u;
    uint64_t* keys = rk_keys + (size_t)w * n;
    for (int64_t qi = (int64_t)blockIdx.x * warps + w; qi < q; qi += (int64_t)gridDim.x * warps) {
        int cnt = 0;
        for (int base = 0; base < n; base += 32) {
            int t = base + lane;
            int32_t id = t < n ? ids[qi * n + t] : -1;
            bool f = id >= 0;
            unsigned b = __ballot_sync(0xffffffffu, f);
            int pos = cnt + __popc(b & lanemask_lt());
            // order-preserving bits (IP distances can be negative; for L2's
            // non-negative values this is the plain float order too)
            if (f) keys[pos] = ((uint64_t)dist_bits<1>(dists[qi * n + t]) << 32) | (uint32_t)id;
            cnt += __popc(b);
        }
        __syncwarp();
        if (cnt == 0 && lane == 0) atomicExch(err, 1);
        for (int t = lane; t < k; t += 32) {
            out_ids[qi * k + t] = -1;
            out_dists[qi * k + t] = __int_as_float(0x7f800000);
        }
        __syncwarp();
        for (int t = lane; t < cnt; t += 32) {
            uint64_t key = keys[t];
            int rank = 0;
            // ties on (distance, id) keep candidate order, like the stable
            // np.lexsort (pipeline.py:195): equal keys get distinct ranks
            for (int o = 0; o < cnt; o++) rank += keys[o] < key || (keys[o] == key && o < t);
            if (rank < k) {
                out_ids[qi * k + rank] = (int32_t)(uint32_t)key;
                out_dists[qi * k + rank] = bits_dist<1>((uint32_t)(key >> 32));
            }
        }
        __syncwarp();
    }
}

// Cross-GPU ordering for the pipelined dataflow ring (ring.DataflowRing):
// signal_kernel publishes `value` into a (peer-mapped) flag after everything
// earlier on its stream -- the persistent K1's stores into other GPUs'
// buffers included -- is visible system-wide; wait_kernel holds its stream
// until every flag reaches `value` (bounded: a peer that never signals sets
// err instead of hanging the GPU).
__global__ void signal_kernel(unsigned long long* flag, unsigned long long value) {
    asm volatile("fence.acq_rel.sys;" ::: "memory");
    st_release_sys(flag, value);
}
__global__ void wait_kernel(const unsigned long long* const* flags, int32_t n, unsigned long long value,
                            int32_t* err) {
    const int i = threadIdx.x;
    if (i < n) {
        for (uint32_t spin = 0;; spin++) {
            if (ld_acquire_sys(flags[i]) >= value) break;
            if (spin > (1u << 26)) {
                atomicOr(err, 32);
                break;
            }
            __nanosleep(512);
        }
    }
    __syncthreads();
    asm volatile("fence.acq_rel.sys;" ::: "memory");
}

// Test hook: exact squared L2 of rows[ids] vs query (data.py:70-79).
template <typename VT>
__global__ void l2_rows_kernel(const VT* __restrict__ vec, int32_t d, int32_t spad, L2Plan plan,
                               const int32_t* __restrict__ ids, int64_t n_ids,
                               const float* __restrict__ query, float* __restrict__ out) {
    extern __shared__ float l2s[];
    float* q = l2s;
    float* rows = l2s + ((d + 3) & ~3);
    const unsigned lane = threadIdx.x & 31u;
    for (int t = lane; t < d; t += 32) q[t] = query[t];
    for (int64_t r0 = (int64_t)blockIdx.x * 4; r0 < n_ids; r0 += (int64_t)gridDim.x * 4) {
        __syncwarp();
        for (int v = 0; v < 4; v++) {
            int64_t r = r0 + v < n_ids ? r0 + v : n_ids - 1;
            for (int t = lane; t < d; t += 32) rows[v * spad + t] = to_f(vec[(int64_t)ids[r] * d + t]);
        }
        __syncwarp();
        const unsigned v = lane >> 3, a = lane & 7u;
        float dist = l2_row<0, float>(plan, rows + v * spad, q, a);
        if (a == 0 && r0 + v < n_ids) out[r0 + v] = dist;
    }
}

// Exact squared L2 of row pairs (index builder rescoring, graphs.py:90-101,
// :124-126): out[t] = squared_l2(b[ib[t]], a[ia[t]]) in numpy's pairwise
// float32 order.  8 lanes per pair (the runtime pairwise plan), 4 pairs per
// warp, rows read straight from HBM.
__global__ void l2_pairs_kernel(const float* __restrict__ a, const float* __restrict__ b, int32_t d,
                                L2Plan plan, const int64_t* __restrict__ ia, const int64_t* __restrict__ ib,
                                int64_t n, float* __restrict__ out) {
    const unsigned lane = threadIdx.x & 31u;
    const int64_t warps = (int64_t)gridDim.x * (blockDim.x >> 5);
    for (int64_t w = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5); w * 4 < n; w += warps) {
        const int64_t t = w * 4 + (lane >> 3);
        const int64_t tc = t < n ? t : n - 1;
        const float* x = b + ib[tc] * (int64_t)d;
        const float* q = a + ia[tc] * (int64_t)d;
        const float dist = l2_row<0, float>(plan, x, q, lane & 7u);
        if ((lane & 7u) == 0 && t < n) out[t] = dist;
    }
}

// cuTensorMapEncodeTiled through the runtime's driver entry point (no -lcuda)
typedef CUresult (*EncodeTiledFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                  const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                  CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
EncodeTiledFn encode_tiled() {
    static EncodeTiledFn fn = nullptr;
    static std::once_flag once;
    std::call_once(once, [] {
        void* p = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
            q == cudaDriverEntryPointSuccess)
            fn = reinterpret_cast<EncodeTiledFn>(p);
    });
    return fn;
}

// 2D {d, n} row tensor with a {box_w, 1} box (box_w >= d: the extra columns
// are out of bounds, zero-filled, so rows land at stride box_w) for gather4
int make_row_tensor_map(CUtensorMap* tm, const void* base, int64_t n, int32_t d, int32_t elem, int32_t box_w) {
    EncodeTiledFn fn = encode_tiled();
    if (!fn) return set_err(PW_ECUDA, "cuTensorMapEncodeTiled unavailable");
    const cuuint64_t dims[2] = {(cuuint64_t)d, (cuuint64_t)std::max<int64_t>(n, 1)};
    const cuuint64_t strides[1] = {(cuuint64_t)d * (cuuint64_t)elem};
    const cuuint32_t box[2] = {(cuuint32_t)box_w, 1u};
    const cuuint32_t estr[2] = {1u, 1u};
    CUresult r = fn(tm, elem == 4 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT32 : CU_TENSOR_MAP_DATA_TYPE_UINT8, 2,
                    const_cast<void*>(base), dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                    CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_128B,
                    CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) return set_err(PW_ECUDA, "cuTensorMapEncodeTiled failed (" + std::to_string((int)r) + ")");
    return 0;
}

// cuStreamWriteValue32 through the runtime's driver entry point: a 32-bit
// store executed by the stream itself after its preceding copies (no kernel,
// so it cannot wait behind a persistent K1 that holds every SM)
typedef CUresult (*WriteValue32Fn)(CUstream, CUdeviceptr, cuuint32_t, unsigned int);
WriteValue32Fn write_value32() {
    static WriteValue32Fn fn = nullptr;
    static std::once_flag once;
    std::call_once(once, [] {
        void* p = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuStreamWriteValue32", &p, cudaEnableDefault, &q) == cudaSuccess &&
            q == cudaDriverEntryPointSuccess)
            fn = reinterpret_cast<WriteValue32Fn>(p);
    });
    return fn;
}

SearchCfg make_cfg(const pw_params& p, int64_t n, int32_t j) {
    SearchCfg c;
    c.k = p.k;
    c.L = p.l;
    c.want = (int32_t)std::min<int64_t>(p.m, n);
    c.r = p.r;
    c.max_iter = p.max_iter;
    c.cap = p.buffer_cap ? p.buffer_cap : std::max(p.m, p.r * j);  // search.py:289
    c.prune_sel = (p.selection != PW_SEL_FULL && p.discard_ratio > 0.0) ? p.selection : 0;
    c.n_keep = keep_count(j, p.discard_ratio);
    c.cool_start = cooldown_start(p.max_iter, p.cooldown_ratio);
    c.log = p.log_visits;
    return c;
}

int validate_params(const pw_params& p) {  // search.py:58-70
    if (!(1 <= p.k && p.k <= p.l && 1 <= p.r && p.r <= p.l))
        return set_err(PW_EINVAL, "need k <= l and r <= l, got k=" + std::to_string(p.k) +
                                      " l=" + std::to_string(p.l) + " r=" + std::to_string(p.r));
    if (p.m < 1 || p.max_iter < 1 || p.ghost_max_iter < 1)
        return set_err(PW_EINVAL, "m, max_iter and ghost_max_iter must be >= 1");
    if (!(0.0 <= p.discard_ratio && p.discard_ratio < 1.0))
        return set_err(PW_EINVAL, "discard_ratio must be in [0, 1)");
    if (!(0.0 <= p.cooldown_ratio && p.cooldown_ratio <= 1.0))
        return set_err(PW_EINVAL, "cooldown_ratio must be in [0, 1]");
    if (p.selection < 0 || p.selection > 2) return set_err(PW_EINVAL, "selection must be one of ('full', 'direction', 'random')");
    if (p.seed_mode < 0 || p.seed_mode > 1) return set_err(PW_EINVAL, "seed_mode must be one of ('neighbors', 'mixed')");
    if (p.buffer_cap < 0) return set_err(PW_EINVAL, "buffer_cap must be positive");
    if (p.metric != PW_METRIC_L2 && p.metric != PW_METRIC_IP) return set_err(PW_EINVAL, "metric must be one of ('l2', 'ip')");
    return 0;
}

// Build the launch description (shared-memory layout, configs) for one shard.
struct Launch {
    KArgs A;
    int warps_per_block = 0;
    int blocks = 0;
    size_t smem = 0;
    kernel_fn fn = nullptr;
};

int64_t visit_bound(const SearchCfg& c, int32_t j, int64_t n) {
    int64_t per = std::min<int64_t>(c.cap, (int64_t)c.r * j);
    int64_t b = c.want + (int64_t)(c.max_iter - 1) * per;
    return std::min<int64_t>(b, n);
}

// st: the stream the launch will use.  Workspace (re)initialisation is
// stream-ordered on it -- never a device-wide synchronisation, which would
// deadlock against another shard's persistent dataflow kernel waiting for
// this shard's entries.  A shard's searches share one stream (or are ordered
// by the caller).
int prepare(pw_shard* sh, const pw_params& p, const pw_tuning* tun, bool use_ghost_graph,
            int32_t n_seeds, bool ghost_on, Launch& Lc, cudaStream_t st = 0, int64_t n_tasks_hint = 0) {
    int rc = validate_params(p);
    if (rc) return rc;
    KArgs& A = Lc.A;
    std::memset(&A, 0, sizeof A);
    A.main = GraphDev{sh->vec, sh->adj, sh->gid, sh->dir, (int32_t)sh->n, sh->j};
    A.ghost = GraphDev{sh->gvec, sh->gadj, sh->gids, nullptr, (int32_t)sh->gn, sh->gj};
    A.inter = sh->inter;
    A.d = sh->d;
    A.W = sh->W;
    if (!make_plan(sh->d, A.plan)) return set_err(PW_EINVAL, "dimension too large");
    const GraphDev& G = use_ghost_graph ? A.ghost : A.main;
    if (use_ghost_graph && sh->gn == 0) return set_err(PW_EINVAL, "ghost index absent for this shard");
    A.cfg = make_cfg(p, G.n, G.j);
    pw_params gp = p;  // pipeline.py:174-182
    gp.k = 1;
    gp.max_iter = p.ghost_max_iter;
    gp.selection = PW_SEL_FULL;
    gp.discard_ratio = 0.0;
    gp.log_visits = 0;
    gp.buffer_cap = 0;
    A.gcfg = make_cfg(gp, std::max<int64_t>(sh->gn, 1), sh->gj);
    // opt-in path-extension knobs (pw_tuning: forward_count, late_l, late_max_iter)
    A.fwd = (tun && tun->forward_count > 0) ? tun->forward_count : 1;
    if (A.fwd > 8 || A.fwd > p.k) return set_err(PW_EINVAL, "forward_count must be in [1, min(8, k)]");
    pw_params lp = p;
    if (tun && tun->late_l > 0) lp.l = tun->late_l;
    if (tun && tun->late_max_iter > 0) lp.max_iter = tun->late_max_iter;
    A.has_late = (lp.l != p.l || lp.max_iter != p.max_iter) ? 1 : 0;
    A.cfg_late = A.cfg;
    if (A.has_late) {
        if ((rc = validate_params(lp))) return rc;
        A.cfg_late = make_cfg(lp, G.n, G.j);
    }
    static_assert(offsetof(KArgs, cfg_late) == offsetof(KArgs, cfg) + sizeof(SearchCfg) &&
                      offsetof(KArgs, gcfg) == offsetof(KArgs, cfg) + 2 * sizeof(SearchCfg),
                  "K1 indexes (&cfg)[0..2]");
    const int32_t Lq = std::max(p.l, lp.l);  // queue capacity (smem layout)
    // K1 keeps per-search counters in 32 bits: every counter is bounded by
    // want + max_iter * max(cap, r * j) (visits, scored rows, DGS skips)
    for (const SearchCfg* c : {&A.cfg, &A.cfg_late})
        if ((int64_t)c->want + (int64_t)c->max_iter * std::max<int64_t>(c->cap, (int64_t)c->r * G.j) >= (1ll << 31))
            return set_err(PW_EINVAL, "max_iter too large for the device's per-search counters");
    A.ghost_on = ghost_on ? 1 : 0;
    A.seed_mode = p.seed_mode;
    A.use_ghost_graph = use_ghost_graph ? 1 : 0;
    A.seed = p.seed;
    if (A.cfg.prune_sel == PW_SEL_DIRECTION && !sh->dir)
        return set_err(PW_EINVAL, "direction table required for direction-guided selection");

    // ---- shared-memory layout per warp
    const bool want_tma = PW_TMA_ROWS && tun && (tun->flags & 8);
    const int jm = std::max(G.j, ghost_on ? sh->gj : 0);
    const int d = sh->d;
    const int elem = sh->dtype == PW_DTYPE_U8 ? 1 : 4;  // bytes per vector element
    int spad;
    if (elem == 4) {
        spad = (d + 31) / 32 * 32 + 8;  // == 8 mod 32 floats: conflict-free (v, a) access
        if (spad - 32 >= d) spad -= 32;
    } else {
        // u8: 16-byte rows; the 8 rows of a pass read 8 bytes each (4 lanes x
        // LDS.U16) -- pick a stride whose 8 row offsets hit distinct bank pairs
        auto ok = [](int sp) {
            uint32_t used = 0;
            for (int v = 0; v < 8; v++) {
                const int b = (v * sp / 4) % 32;
                const uint32_t m = (1u << b) | (1u << ((b + 1) % 32));
                if (used & m) return false;
                used |= m;
            }
            return true;
        };
        spad = (d + 15) / 16 * 16;
        while (!ok(spad)) spad += 16;
    }
    A.spad = spad;
    int64_t cb = std::max<int64_t>({(int64_t)p.r * jm, (int64_t)A.cfg.want, (int64_t)A.fwd * (1 + jm),
                                    (int64_t)n_seeds, (int64_t)A.gcfg.want, 32});
    cb = (cb + 31) / 32 * 32;
    A.CB = (int32_t)cb;
    A.BH = (int32_t)next_pow2(2 * cb);
    A.L_max = Lq;
    int64_t bound = visit_bound(A.cfg, G.j, G.n);
    if (A.has_late) bound = std::max(bound, visit_bound(A.cfg_late, G.j, G.n));
    if (ghost_on) bound = std::max(bound, visit_bound(A.gcfg, sh->gj, sh->gn));
    // Default: a small shared-memory visited table (first iterations) backed
    // by the per-warp epoch-tagged global table (batched probes): measured on
    // C2 (10M x 96, l=256) this fits ~10 query-warps per SM instead of 5 and
    // is faster for both the naive and the PathWeaver arm (profiles/r01).
    if (p.metric == PW_METRIC_IP && sh->dtype != PW_DTYPE_F32)
        return set_err(PW_EINVAL, "inner-product search needs float32 vectors");
    Lc.fn = pick_kernel(d, sh->dtype, p.metric);
    const bool specialised = !is_generic(Lc.fn);
    // Specialised kernels keep the exact visited set only in the per-warp
    // epoch-tagged global table (batched probes; no shared table, which buys
    // resident warps).  The generic-d kernel uses a shared table spilling to
    // the same global table.
    int64_t H = specialised ? 0
                            : (tun && tun->visited_slots > 0 ? next_pow2(tun->visited_slots)
                                                             : std::min<int64_t>(256, next_pow2(bound * 4 / 3 + 2)));
    if (!specialised) H = std::max<int64_t>(H, 64);
    A.H = (int32_t)H;
    A.vis_limit = (int32_t)(H * 3 / 4);
    int R;
    if (tun && tun->stage_rows > 0) {
        R = tun->stage_rows;
    } else if (specialised && elem == 1) {
        // u8 rows are small: fill the region the dedup hash needs anyway
        // (8*BH + 4*CB bytes) with rows in flight, in 8-row compute passes
        R = (int)std::max<int64_t>(16, (8 * (int64_t)A.BH + 4 * cb) / spad / 16 * 16);
        R = std::min(R, 64);
    } else if (specialised) {
        // rows in flight per warp: two halves of 8 rows (one 8-row compute
        // pass each); large rows shrink to keep staging <= ~10 KB
        R = 16;
        while (R > 4 && (int64_t)R * spad * 4 > 10240) R >>= 1;
    } else {
        R = std::max(2, std::min(16, (16384 / (spad * elem)) & ~1));
    }
    R &= ~1;
    if (R < 2) R = 2;
    int W = sh->W;
    int PG = 1;
    // DGS parent rows are packed at a 16-byte stride (bit tests only, no
    // bank-conflict concern) so that kParentGroup parents fit the staging
    // ring and one expansion is ONE fetch round trip (C2: 8 x (96 + 96) words)
    const int pstride = elem == 4 ? (d + 3) & ~3 : (d + 15) & ~15;  // elements, 16-byte rows
    // PW_DGS_LDG (specialised f32 kernels, d <= 128): parent rows go to
    // registers, only adjacency + direction rows to the staging ring
    const bool dgs_ldg = PW_DGS_LDG && specialised && elem == 4 && d % 4 == 0 && d <= 128 && G.j <= 32;
    const int64_t per_vec = dgs_ldg ? 0 : (int64_t)pstride * elem;
    if (A.cfg.prune_sel == PW_SEL_DIRECTION) {
        const int64_t per = per_vec + 4ll * G.j * W;  // bytes per parent
        while ((int64_t)R * spad * elem < per) R += 2;
        PG = (int)std::min<int64_t>(kParentGroup, ((int64_t)R * spad * elem) / per);
        PG = std::max(PG, 1);
    }
    A.pstride = pstride;
    // specialised kernels with j <= 32 keep the DGS counts/bits in registers
    const bool dgs_regs = specialised && G.j <= 32;
    const int64_t n_desc = std::max<int64_t>({32, (int64_t)p.r, 3ll * kParentGroup});
    // Per-warp shared-memory layout for R staging rows; returns bytes per warp.
    auto layout = [&](int Rr) -> int64_t {
        A.R = Rr;
        // The in-batch dedup hash (bhk/bhp) and its slot list (cslot) are live
        // only between expansion and the visited filter, the staging ring only
        // in scoring and DGS expansion (before the dedup): they share one region.
        const int64_t hash_bytes = 8 * (int64_t)A.BH + 4 * cb;
        const int64_t stage_bytes = std::max<int64_t>((int64_t)elem * Rr * spad, hash_bytes);
        if (A.cfg.prune_sel == PW_SEL_DIRECTION) {  // DGS parents per fetch round trip
            const int64_t per = per_vec + 4ll * G.j * W;
            PG = (int)std::max<int64_t>(1, std::min<int64_t>(kParentGroup, stage_bytes / per));
        }
        A.PG = PG;
        auto al = [](int64_t x) { return (x + 15) / 16 * 16; };
        int64_t off = 0;
        // query (f32); uint8-row shards also keep the query's bytes and
        // (sum q^2, integral flag) for the exact integer distance path
        A.o_q = (int32_t)off;
        off = al(off + 4 * (int64_t)((d + 3) & ~3) + (elem == 1 ? ((d + 15) & ~15) + 16 : 0));
        A.o_qk = (int32_t)off; off = al(off + 8 * (int64_t)Lq);  // one queue buffer (in-place merge)
        A.o_qe = (int32_t)off; off = al(off + (int64_t)Lq);
        A.o_newl = (int32_t)off; off = al(off + 4 * cb);
        // keys (pow2 for the survivor sort); the candidate list lives in their
        // upper half: candidates are live from expansion to the dedup, while the
        // key area then holds at most the DGS raw adjacency (r*j ints, lower
        // half) and the visited probes (lower half); keys return only in scoring
        const int64_t ckey_n = std::max<int64_t>(64, next_pow2(cb));
        A.o_ckey = (int32_t)off;
        A.o_cand = (int32_t)(off + 4 * ckey_n);
        off = al(off + 8 * ckey_n);
        A.o_vh = (int32_t)off; off = al(off + 4 * H);
        if (want_tma) off = (off + 127) / 128 * 128;  // TMA destinations: 128-byte aligned
        A.o_stage = (int32_t)off;
        A.o_bhk = (int32_t)off;
        A.o_bhp = (int32_t)(off + 4 * (int64_t)A.BH);
        A.o_cslot = (int32_t)(off + 8 * (int64_t)A.BH);
        off = al(off + stage_bytes);
        A.o_misc = (int32_t)off;
        // misc words: [DGS counts PG*j | perm j] [DGS bits PG*W] 8 pad (task
        // scalars) | parents r | 8 pad
        const int64_t misc_cnt = dgs_regs ? (int64_t)jm : (int64_t)std::max(jm, PG * jm);
        const int64_t misc_bits = (dgs_regs && !dgs_ldg) ? 0 : (int64_t)PG * W;
        A.o_qbits = (int32_t)misc_cnt;
        A.o_par = (int32_t)(misc_cnt + misc_bits + 8);
        const int64_t misc = misc_cnt + misc_bits + 8 + p.r + 8;
        off = al(off + 4 * misc);
        A.o_mbar = (int32_t)off;
        off = al(off + 3 * 8);
        // expansion row descriptors live only inside one fetch, while the new-id
        // list is dead (consumed by scoring, rewritten by the dedup)
        if (16 * n_desc <= 4 * cb) {
            A.o_desc = A.o_newl;
        } else {
            A.o_desc = (int32_t)off;
            off = al(off + 16 * n_desc);
        }
        if (want_tma) off = (off + 127) / 128 * 128;
        A.warp_bytes = (int32_t)off;
        return off;
    };
    DevInfo* I;
    if ((rc = dev_info(sh->device, &I))) return rc;
    int64_t off = layout(R);
    // kernels built for more than 16 resident warps (PW_MAX_THREADS): shrink
    // the staging ring (down to 12 rows) until they fit
    while (specialised && elem == 4 && !(tun && tun->stage_rows > 0) && R > 12 &&
           I->smem_optin / off < kMaxWarps) {
        R -= 2;
        off = layout(R);
    }
    // Small batches need fewer resident query-warps per SM (launch() spreads
    // them over every SM), so the staging ring may take the shared memory the
    // absent warps would have used: more rows per compute pass.  This is what
    // large rows need most (d=960: 2 rows at full occupancy, one row per
    // 8-row pass).
    if (n_tasks_hint > 0 && specialised && elem == 4 && !(tun && tun->stage_rows > 0)) {
        const int64_t need = std::min<int64_t>(kMaxWarps, (n_tasks_hint + I->sms - 1) / I->sms);
        int Rb = R;
        while (Rb + 2 <= 16 && layout(Rb + 2) * need <= I->smem_optin) Rb += 2;
        R = Rb;
        off = layout(R);
    }
    // TMA bulk copies need 16-byte sizes/alignment for every expansion row kind
    auto b16 = [](int64_t bytes) { return bytes % 16 == 0; };
    A.bulk_rows = 0;
    // TMA tile::gather4 scoring rows (tuning flag 8): specialised kernels whose
    // padded staging row fits one box (<= 256 elements) and whose global row
    // stride is a 16-byte multiple
    A.tma_rows = 0;
    // every gather4 destination (half base + 4-row groups) 128-byte aligned
    const int64_t row_b = (int64_t)A.spad * elem;
    if (want_tma && specialised && A.spad <= 256 && ((int64_t)d * elem) % 16 == 0 && (4 * row_b) % 128 == 0 &&
        ((int64_t)(A.R / 2) * row_b) % 128 == 0 && A.o_stage % 128 == 0 && A.warp_bytes % 128 == 0) {
        if ((rc = make_row_tensor_map(&A.tm_main, sh->vec, sh->n, d, elem, A.spad))) return rc;
        if (sh->gn > 0 && (rc = make_row_tensor_map(&A.tm_ghost, sh->gvec, sh->gn, d, elem, A.spad))) return rc;
        A.tma_rows = 1;
    }
    A.prefetch = (tun && (tun->flags & 1)) ? 1 : 0;
    A.bulk_adj = (b16(4ll * G.j) && (!ghost_on || b16(4ll * sh->gj)) &&
                  (A.cfg.prune_sel != PW_SEL_DIRECTION || (b16((int64_t)elem * d) && b16(4ll * G.j * W))))
                     ? ((tun && (tun->flags & 4)) ? 2 : 1)
                     : 0;

    // the FAST K1 instance when this launch never needs the cold paths it
    // drops: lossy visited cache, no random selection, degrees <= 32; for
    // direction-guided launches its 20-warp build (96 registers; measured 3%
    // faster for PathWeaver, 3% slower for full selection, ab_warps_r02ad.log)
    const bool lossy_req = tun && (tun->flags & 2) && !p.log_visits;
    const bool fast = specialised && lossy_req && A.cfg.prune_sel != PW_SEL_RANDOM &&
                      A.cfg_late.prune_sel != PW_SEL_RANDOM && G.j <= 32 && (!ghost_on || sh->gj <= 32) &&
                      !(PW_TMA_ROWS && A.tma_rows) && !p.buffer_cap && !A.prefetch && A.bulk_adj == 1;
    const bool wide = fast && A.cfg.prune_sel == PW_SEL_DIRECTION && !(tun && tun->warps_per_sm > 0 &&
                                                                       tun->warps_per_sm <= kMaxWarps);
    if (fast) Lc.fn = pick_kernel(d, sh->dtype, p.metric, true, wide);
    const int max_w = wide ? kWideWarps : kMaxWarps;
    int wpb = (int)std::min<int64_t>(max_w, I->smem_optin / off);
    if (tun && tun->warps_per_sm > 0) wpb = std::min(wpb, tun->warps_per_sm);
    if (wpb < 1) return set_err(PW_EINVAL, "search configuration needs " + std::to_string(off) +
                                              " bytes of shared memory per query (l or degree too large)");
    Lc.warps_per_block = wpb;
    Lc.blocks = I->sms;
    Lc.smem = (size_t)wpb * off;

    // ---- global workspace: visited spill tables + choice scratch
    const int total_warps = Lc.blocks * wpb;
    // the spill triggers when (smem entries + batch) > vis_limit, so a table is
    // needed whenever bound + CB can exceed it; it holds <= bound entries
    int64_t gsz = (specialised || bound + cb > A.vis_limit) ? next_pow2(2 * bound + 2) : 1;
    // lossy visited cache (tuning flag 2): u32 slots holding epoch8 << 24 |
    // the low 32 - s bits of hash32(id) (any shard size: >= 2^8 slots make
    // slot + word name the id exactly); never with log_visits (the log lists
    // exact visits)
    const bool lossy = tun && (tun->flags & 2) && !p.log_visits;
    A.lossy = lossy ? 1 : 0;
    if (lossy) {
        const int64_t slots = std::min<int64_t>(
            1ll << 24, std::max<int64_t>(256, next_pow2(tun->visited_slots > 0 ? tun->visited_slots : 4096)));
        int lg = 0;
        while ((1ll << lg) < slots) lg++;
        A.lshift = 32 - lg;
        gsz = slots / 2;  // u64 words of the per-warp region
    }
    A.gmask = (int32_t)(gsz - 1);
    int64_t want_max = std::max(A.cfg.want, A.gcfg.want);
    int64_t scr = std::max<int64_t>(next_pow2(4 * want_max + 8) * 2, next_pow2((int64_t)(1.2 * want_max) + 1));
    std::lock_guard<std::mutex> lk(sh->mu);
    if (!sh->counter) {
        PW_CUDA(cudaMalloc(&sh->counter, sizeof(int32_t) * 2));
        PW_CUDA(cudaMemsetAsync(sh->counter, 0, sizeof(int32_t) * 2, st));
        PW_CUDA(cudaMalloc(&sh->phase, sizeof(unsigned long long) * 8));
        PW_CUDA(cudaMemsetAsync(sh->phase, 0, sizeof(unsigned long long) * 8, st));
    }
    A.phase = sh->phase;
    const bool grow = sh->gvis_words < (size_t)total_warps * gsz || sh->gepoch_n < (size_t)total_warps;
    const bool rezero = !grow && (sh->gvis_stride != gsz || sh->gvis_lossy != (int)lossy);
    if (grow) {
        // epoch-tagged tables: zero once (epoch 0 is never used by a search);
        // stream-ordered free / alloc / zero
        if (sh->gvis) PW_CUDA(cudaFreeAsync(sh->gvis, st));
        if (sh->gepoch) PW_CUDA(cudaFreeAsync(sh->gepoch, st));
        sh->gvis = nullptr;
        sh->gepoch = nullptr;
        const size_t words = std::max(sh->gvis_words, (size_t)total_warps * gsz);
        PW_CUDA(cudaMallocAsync((void**)&sh->gvis, sizeof(unsigned long long) * words, st));
        PW_CUDA(cudaMemsetAsync(sh->gvis, 0, sizeof(unsigned long long) * words, st));
        PW_CUDA(cudaMallocAsync((void**)&sh->gepoch, sizeof(uint32_t) * (size_t)total_warps, st));
        PW_CUDA(cudaMemsetAsync(sh->gepoch, 0, sizeof(uint32_t) * (size_t)total_warps, st));
        sh->gvis_words = words;
        sh->gepoch_n = (size_t)total_warps;
        sh->gvis_stride = gsz;
    } else if (rezero) {
        // a different per-warp stride maps regions to other warps: re-zero so no
        // stale (epoch, id) of another warp can match
        PW_CUDA(cudaMemsetAsync(sh->gvis, 0, sizeof(unsigned long long) * sh->gvis_words, st));
        PW_CUDA(cudaMemsetAsync(sh->gepoch, 0, sizeof(uint32_t) * sh->gepoch_n, st));
        sh->gvis_stride = gsz;
    }
    sh->gvis_lossy = (int)lossy;
    if (sh->gscr_words < (size_t)total_warps * scr) {
        if (sh->gscr) PW_CUDA(cudaFreeAsync(sh->gscr, st));
        sh->gscr = nullptr;
        PW_CUDA(cudaMallocAsync((void**)&sh->gscr, sizeof(uint32_t) * (size_t)total_warps * scr, st));
        sh->gscr_words = (size_t)total_warps * scr;
    }
    A.gvis = sh->gvis;
    A.gepoch = sh->gepoch;
    A.gscratch = sh->gscr;
    A.jump = I->jump;
    A.gscratch_words = scr;
    A.task_counter = sh->counter;
    A.err = sh->counter + 1;
    return 0;
}

// Device-side consistency flag (bounded probes in K1); read after a sync.
int check_err(pw_shard* sh) {
    int32_t e = 0;
    PW_CUDA(cudaMemcpy(&e, sh->counter + 1, sizeof e, cudaMemcpyDeviceToHost));
    if (e) {
        cudaMemset(sh->counter + 1, 0, sizeof(int32_t));
        return set_err(PW_ECUDA, (e & 64)   ? std::string("query upload wait timed out (flag ") + std::to_string(e) + ")"
                                 : (e & 16) ? std::string("dataflow inbox wait timed out (flag ") + std::to_string(e) + ")"
                                 : (e & 32) ? std::string("TMA gather never completed (flag ") + std::to_string(e) + ")"
                                            : "beam_search_kernel internal table overflow (flag " + std::to_string(e) + ")");
    }
    return 0;
}

int launch(pw_shard* sh, Launch& Lc, cudaStream_t st) {
    if (Lc.A.n_tasks <= 0) return 0;
    PW_CUDA(cudaSetDevice(sh->device));
    PW_CUDA(cudaMemsetAsync(sh->counter, 0, sizeof(int32_t), st));  // task counter only; err sticks
    // Small batches (fewer tasks than resident query-warps, e.g. 1K GIST
    // queries or one ring chunk) are spread over every SM with fewer warps per
    // CTA instead of packing 16 warps into the first SMs: each query then
    // shares its SM's issue slots and L1 with fewer others.  K1 indexes its
    // per-warp workspace by blockIdx * (blockDim / 32) + warp, a subset of
    // the prepared blocks x warps_per_block.
    int wpb = Lc.warps_per_block;
    int64_t blocks = Lc.blocks;
    if (blocks * wpb > (int64_t)Lc.A.n_tasks) {
        wpb = (int)std::min<int64_t>(wpb, std::max<int64_t>(1, (Lc.A.n_tasks + blocks - 1) / blocks));
        blocks = std::min<int64_t>(blocks, ((int64_t)Lc.A.n_tasks + wpb - 1) / wpb);
    }
    const size_t smem = Lc.smem / (size_t)Lc.warps_per_block * (size_t)wpb;
    void* args[] = {(void*)&Lc.A};
    PW_CUDA(cudaLaunchKernel((const void*)Lc.fn, dim3((unsigned)blocks), dim3(32 * wpb), args, smem, st));
    g_launches++;
    PW_CUDA(cudaGetLastError());
    return 0;
}

}  // namespace

// shared with the other translation units of libpwb200.so (pw_crc32c.cu)
int pw_internal_set_err(int code, const char* msg) { return set_err(code, msg); }
void pw_internal_count_launch() { g_launches++; }

extern "C" {

const char* pw_last_error(void) { return g_err.c_str(); }
const char* pw_version(void) { return "pwb200 0.1.0 (sm_100a)"; }
int64_t pw_launch_count(void) { return g_launches.load(); }

int pw_shard_create(const pw_shard_desc* D, pw_shard** out) {
    if (!D || !out) return set_err(PW_EINVAL, "null argument");
    if (D->n <= 0) return set_err(PW_EINVAL, "empty graph");
    if (D->n >= (1ll << 31)) return set_err(PW_EINVAL, "shard too large (n_local >= 2^31)");
    if (D->d < 1 || D->j < 0) return set_err(PW_EINVAL, "bad dimensions");
    if (D->dtype != PW_DTYPE_F32 && D->dtype != PW_DTYPE_U8)
        return set_err(PW_EINVAL, "vectors must be float32 or uint8");
    if (D->dtype == PW_DTYPE_U8 && D->d % 4 != 0)
        return set_err(PW_EINVAL, "uint8 vectors need d % 4 == 0 (4-byte row copies)");
    pw_shard* sh = new pw_shard();
    int dev = 0;
    cudaGetDevice(&dev);
    sh->device = dev;
    sh->n = D->n;
    sh->d = D->d;
    sh->j = D->j;
    sh->W = words_per_vector(D->d);
    sh->dtype = D->dtype;
    int rc = 0;
    auto fail = [&](int code) {
        pw_shard_destroy(sh);
        return code;
    };
    const bool od = D->on_device != 0;
    const size_t elem = D->dtype == PW_DTYPE_U8 ? 1 : 4;
    if ((rc = upload((uint8_t**)&sh->vec, D->vectors, (size_t)D->n * D->d * elem, &sh->bytes, od)))
        return fail(rc);
    if ((rc = upload(&sh->adj, D->adj, (size_t)D->n * D->j, &sh->bytes, od))) return fail(rc);
    if ((rc = upload(&sh->gid, D->global_ids, (size_t)D->n, &sh->bytes, od))) return fail(rc);
    if ((rc = check_ids(sh->adj, (int64_t)D->n * D->j, D->n, "adjacency"))) return fail(rc);
    if (D->direction &&
        (rc = upload(&sh->dir, D->direction, (size_t)D->n * D->j * sh->W, &sh->bytes, od)))
        return fail(rc);
    if (D->inter_map && (rc = upload(&sh->inter, D->inter_map, (size_t)D->n, &sh->bytes, od)))
        return fail(rc);
    if (D->ghost_n > 0) {
        sh->gn = D->ghost_n;
        sh->gj = D->ghost_j;
        if ((rc = upload(&sh->gids, D->ghost_ids, (size_t)D->ghost_n, &sh->bytes, od))) return fail(rc);
        if ((rc = upload(&sh->gadj, D->ghost_adj, (size_t)D->ghost_n * D->ghost_j, &sh->bytes, od)))
            return fail(rc);
        if ((rc = upload((uint8_t**)&sh->gvec, nullptr, (size_t)D->ghost_n * D->d * elem, &sh->bytes)))
            return fail(rc);
        if ((rc = check_ids(sh->gids, sh->gn, sh->n, "ghost parent"))) return fail(rc);
        if ((rc = check_ids(sh->gadj, sh->gn * sh->gj, sh->gn, "ghost adjacency"))) return fail(rc);
        gather_rows_kernel<<<256, 256>>>((const uint8_t*)sh->vec, sh->gids, sh->gn, (int64_t)sh->d * elem,
                                         (uint8_t*)sh->gvec);
        g_launches++;
        cudaError_t e = cudaDeviceSynchronize();
        if (e != cudaSuccess) return fail(set_err(PW_ECUDA, cudaGetErrorString(e)));
    }
    *out = sh;
    return 0;
}

int pw_shard_destroy(pw_shard* sh) {
    if (!sh) return 0;
    int cur = 0;
    cudaGetDevice(&cur);
    cudaSetDevice(sh->device);
    void* ptrs[] = {sh->vec, sh->adj, sh->gid, sh->dir, sh->inter, sh->gvec, sh->gadj, sh->gids,
                    sh->counter, sh->gvis, sh->gscr, sh->gepoch, sh->phase};
    for (void* p : ptrs)
        if (p) cudaFree(p);
    cudaSetDevice(cur);
    delete sh;
    return 0;
}

int64_t pw_shard_bytes(const pw_shard* sh) { return sh ? sh->bytes : 0; }

// Overlapped query upload of the current pw_run call (this thread), read by
// the launch builders below; null outside pw_run.
struct QUpload {
    const uint32_t* flags;
    int32_t chunk;
    uint32_t epoch;
};
thread_local const QUpload* tl_upload = nullptr;

int pw_search_stage(pw_shard* sh, const pw_params* params, const pw_tuning* tuning,
                    const float* queries, int64_t q0, int64_t n, int32_t stage,
                    const int32_t* entries_in, int32_t* forward_out, int32_t* shard_ids,
                    float* shard_dists, int32_t n_cols, int32_t col, int32_t* stats_i32,
                    int64_t* stats_i64, int64_t q_total, void* stream) {
    if (!sh || !params) return set_err(PW_EINVAL, "null argument");
    if (forward_out && !sh->inter)
        return set_err(PW_EINVAL, "pipelined mode requires inter-shard tables for every shard");
    Launch Lc;
    bool ghost_on = params->ghost_enabled && !entries_in && sh->gn > 0;
    int rc = prepare(sh, *params, tuning, false, 0, ghost_on, Lc, (cudaStream_t)stream, n);
    if (rc) return rc;
    KArgs& A = Lc.A;
    A.stage = stage;
    A.q0 = q0;
    A.n_tasks = (int32_t)n;
    A.queries = queries + q0 * sh->d;
    if (tl_upload) {
        A.qready = tl_upload->flags;
        A.q_chunk = tl_upload->chunk;
        A.q_epoch = tl_upload->epoch;
    }
    A.entries = entries_in ? entries_in + q0 * A.fwd : nullptr;
    A.forward = forward_out ? forward_out + q0 * A.fwd : nullptr;
    const int64_t k = params->k;
    A.out_ids = shard_ids + (q0 * n_cols + col) * k;
    A.out_dists = shard_dists + (q0 * n_cols + col) * k;
    A.out_local = nullptr;
    A.out_stride = (int64_t)n_cols * k;
    A.st32 = stats_i32 ? stats_i32 + q0 : nullptr;
    A.st64 = stats_i64 ? stats_i64 + q0 : nullptr;
    A.st_stride = q_total;
    return launch(sh, Lc, (cudaStream_t)stream);
}

int pw_search_dataflow(pw_shard* sh, const pw_params* params, const pw_tuning* tuning,
                       const float* queries, int64_t q, int32_t g, int32_t N, uint32_t epoch,
                       const uint64_t* inbox, uint64_t* next_inbox, int32_t* shard_ids,
                       float* shard_dists, int32_t* stats_i32, int64_t* stats_i64, int32_t sm_limit,
                       void* stream) {
    if (!sh || !params) return set_err(PW_EINVAL, "null argument");
    if (N < 1 || N > 8 || g < 0 || g >= N) return set_err(PW_EINVAL, "dataflow ring needs 1 <= N <= 8, 0 <= g < N");
    if (q < 1 || q >= (1ll << 31)) return set_err(PW_EINVAL, "bad query count");
    if (N > 1 && !sh->inter)
        return set_err(PW_EINVAL, "pipelined mode requires inter-shard tables for every shard");
    if (N > 1 && (!inbox || !next_inbox)) return set_err(PW_EINVAL, "dataflow ring needs inboxes");
    Launch Lc;
    const bool ghost_on = params->ghost_enabled && sh->gn > 0;  // stage-0 tasks only
    int rc = prepare(sh, *params, tuning, false, 0, ghost_on, Lc, (cudaStream_t)stream, q);
    if (rc) return rc;
    KArgs& A = Lc.A;
    A.df = 1;
    A.df_g = g;
    A.df_N = N;
    for (int c = 0; c <= N; c++) A.df_lo[c] = c == 0 ? 0 : A.df_lo[c - 1] + (int32_t)(q / N + (c - 1 < q % N ? 1 : 0));
    A.df_base[0] = 0;
    for (int st = 0; st < N; st++) {
        const int c = ((g - st) % N + N) % N;
        A.df_base[st + 1] = A.df_base[st] + (A.df_lo[c + 1] - A.df_lo[c]);
    }
    A.df_epoch = epoch;
    A.df_inbox = reinterpret_cast<const unsigned long long*>(inbox);
    A.df_next = reinterpret_cast<unsigned long long*>(next_inbox);
    A.stage = 0;
    A.q0 = 0;
    A.n_tasks = (int32_t)q;
    A.queries = queries;
    if (tl_upload) {
        A.qready = tl_upload->flags;
        A.q_chunk = tl_upload->chunk;
        A.q_epoch = tl_upload->epoch;
    }
    A.entries = nullptr;
    A.forward = nullptr;
    const int64_t k = params->k;
    A.out_ids = shard_ids + (int64_t)g * k;
    A.out_dists = shard_dists + (int64_t)g * k;
    A.out_local = nullptr;
    A.out_stride = (int64_t)N * k;
    A.st32 = stats_i32;
    A.st64 = stats_i64;
    A.st_stride = q;
    if ((stats_i32 == nullptr) != (stats_i64 == nullptr))
        return set_err(PW_EINVAL, "stats_i32 and stats_i64 go together");
    A.st32_stage_stride = 4 * q;  // (N, 4, q)
    A.st64_stage_stride = 6 * q;  // (N, 6, q)
    if (sm_limit > 0) Lc.blocks = std::min(Lc.blocks, sm_limit);
    return launch(sh, Lc, (cudaStream_t)stream);
}

int pw_shard_validate_inter(pw_shard* sh, int64_t n_next) {
    if (!sh) return set_err(PW_EINVAL, "null argument");
    if (!sh->inter) return set_err(PW_EINVAL, "pipelined mode requires inter-shard tables for every shard");
    if (sh->inter_ok_n == n_next) return 0;
    PW_CUDA(cudaSetDevice(sh->device));
    int rc = check_ids(sh->inter, sh->n, n_next, "inter-shard map");
    if (rc) return rc;
    sh->inter_ok_n = n_next;
    return 0;
}

int pw_signal(uint64_t* flag, uint64_t value, void* stream) {
    if (!flag) return set_err(PW_EINVAL, "null argument");
    signal_kernel<<<1, 1, 0, (cudaStream_t)stream>>>(reinterpret_cast<unsigned long long*>(flag), value);
    g_launches++;
    PW_CUDA(cudaGetLastError());
    return 0;
}

int pw_wait(const uint64_t* const* flags, int32_t n, uint64_t value, int32_t* err, void* stream) {
    if (!flags || !err || n < 1 || n > 32) return set_err(PW_EINVAL, "pw_wait needs 1..32 flags and an err flag");
    wait_kernel<<<1, 32, 0, (cudaStream_t)stream>>>(reinterpret_cast<const unsigned long long* const*>(flags), n,
                                                    value, err);
    g_launches++;
    PW_CUDA(cudaGetLastError());
    return 0;
}

int pw_shard_check(pw_shard* sh) {
    if (!sh) return set_err(PW_EINVAL, "null argument");
    if (!sh->counter) return 0;
    PW_CUDA(cudaSetDevice(sh->device));
    return check_err(sh);
}

extern "C" int pw_knn_screen_impl(const float* q, int64_t nq, const float* x, int64_t n, int32_t d,
                                  const float* xn, int64_t self_off, int32_t kc, int32_t* out_ids,
                                  float* out_vals, void* stream, char* msg);

int pw_knn_screen(const float* q, int64_t nq, const float* x, int64_t n, int32_t d, const float* xn,
                  int64_t self_off, int32_t kc, int32_t* out_ids, float* out_vals, void* stream) {
    char msg[256] = {0};
    const int rc = pw_knn_screen_impl(q, nq, x, n, d, xn, self_off, kc, out_ids, out_vals, stream, msg);
    if (rc) return set_err(rc == -1 ? PW_EINVAL : PW_ECUDA, msg);
    return 0;
}

int pw_l2_pairs(const float* a, const float* b, int32_t d, const int64_t* ia, const int64_t* ib, int64_t n,
                float* out, void* stream) {
    if (n <= 0) return 0;
    if (!a || !b || !ia || !ib || !out || d < 1) return set_err(PW_EINVAL, "bad argument");
    L2Plan plan;
    if (!make_plan(d, plan)) return set_err(PW_EINVAL, "dimension too large");
    const int64_t warps = (n + 3) / 4;
    const int blocks = (int)std::min<int64_t>(148 * 16, (warps + 7) / 8);
    l2_pairs_kernel<<<blocks, 256, 0, (cudaStream_t)stream>>>(a, b, d, plan, ia, ib, n, out);
    g_launches++;
    PW_CUDA(cudaGetLastError());
    return 0;
}

int pw_dev_alloc(int64_t bytes, void** out) {
    if (!out || bytes < 0) return set_err(PW_EINVAL, "bad argument");
    *out = nullptr;
    PW_CUDA(cudaMalloc(out, (size_t)std::max<int64_t>(bytes, 1)));
    PW_CUDA(cudaMemset(*out, 0, (size_t)std::max<int64_t>(bytes, 1)));
    return 0;
}
int pw_dev_free(void* ptr) {
    if (ptr) PW_CUDA(cudaFree(ptr));
    return 0;
}
int pw_ipc_get(const void* ptr, void* handle64) {
    static_assert(sizeof(cudaIpcMemHandle_t) == 64, "CUDA IPC handle size");
    if (!ptr || !handle64) return set_err(PW_EINVAL, "null argument");
    cudaIpcMemHandle_t h;
    PW_CUDA(cudaIpcGetMemHandle(&h, const_cast<void*>(ptr)));
    std::memcpy(handle64, &h, sizeof h);
    return 0;
}
int pw_ipc_open(const void* handle64, void** out) {
    if (!handle64 || !out) return set_err(PW_EINVAL, "null argument");
    cudaIpcMemHandle_t h;
    std::memcpy(&h, handle64, sizeof h);
    PW_CUDA(cudaIpcOpenMemHandle(out, h, cudaIpcMemLazyEnablePeerAccess));
    return 0;
}
int pw_ipc_close(void* ptr) {
    if (ptr) PW_CUDA(cudaIpcCloseMemHandle(ptr));
    return 0;
}

int pw_reduce_topk(const int32_t* shard_ids, const float* shard_dists, int64_t q, int32_t n_cand,
                   int32_t k, int32_t* final_ids, float* final_dists, int32_t* err_dev,
                   void* stream) {
    if (q <= 0) return 0;
    cudaStream_t st = (cudaStream_t)stream;
    int32_t* err = err_dev;
    if (!err) {
        PW_CUDA(cudaMallocAsync(&err, sizeof(int32_t), st));
        PW_CUDA(cudaMemsetAsync(err, 0, sizeof(int32_t), st));
    }
    const int n = n_cand;
    const int warps = 4;
    size_t smem = (size_t)warps * n * sizeof(uint64_t);
    if (smem > 48 * 1024)
        PW_CUDA(cudaFuncSetAttribute(reduce_topk_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    int blocks = (int)std::min<int64_t>(4096, (q + warps - 1) / warps);
    reduce_topk_kernel<<<blocks, 32 * warps, smem, st>>>(shard_ids, shard_dists, q, n, k, final_ids,
                                                          final_dists, err);
    g_launches++;
    PW_CUDA(cudaGetLastError());
    if (err_dev) return 0;
    int32_t herr = 0;
    PW_CUDA(cudaMemcpyAsync(&herr, err, sizeof herr, cudaMemcpyDeviceToHost, st));
    PW_CUDA(cudaFreeAsync(err, st));
    PW_CUDA(cudaStreamSynchronize(st));
    if (herr) return set_err(PW_EINVAL, "cannot reduce empty candidate lists");
    return 0;
}

// Grow-only per-device workspace of the host entry points (no allocation
// inside a steady stream of calls, so end-to-end timings measure copies +
// kernels only).  Its mutex serialises every host call that launches on the
// device's shards (pw_run, pw_run_device, pw_search_one): a shard's launch
// workspace (task counter, visited tables) belongs to one launch at a time.
struct RunWs {
    std::mutex mu;
    cudaStream_t st = nullptr;
    char* buf = nullptr;
    size_t cap = 0;
    // logical-shard dataflow ring: one stream per shard, inboxes, run tag
    cudaStream_t ring[8] = {};
    cudaEvent_t ev[9] = {};
    uint64_t* inbox = nullptr;
    size_t inbox_cap = 0;  // u64 words
    uint32_t epoch = 0;
    // overlapped query upload (pw_run): copy stream, chunk flags, call tag
    cudaStream_t cs = nullptr;
    uint32_t* qflags = nullptr;
    size_t qflags_cap = 0;
    uint32_t qepoch = 0;
    // page-locked landing slots of pw_run's error flags (K2's, then one per
    // shard), read with the results instead of one synchronous copy each
    int32_t* hflags = nullptr;
};
RunWs g_ws[64];

// grow-only device buffer of a RunWs (caller holds W.mu)
int ws_reserve(RunWs& W, size_t bytes) {
    if (W.cap >= bytes) return 0;
    if (W.buf) {
        if (W.st) PW_CUDA(cudaStreamSynchronize(W.st));
        cudaFree(W.buf);
    }
    W.buf = nullptr;
    W.cap = 0;
    PW_CUDA(cudaMalloc(&W.buf, bytes));
    W.cap = bytes;
    return 0;
}

// Pipelined path extension over N logical shards of one device as the
// dataflow ring (pipeline.py:308-347): N persistent K1 launches on N
// streams, each capped to SMs/N CTAs so all are resident together; shard g
// runs its (stage, query) tasks stage-major and hands each entry to shard
// g+1 through a device inbox -- no stage barriers, one launch per shard
// instead of N x N stage launches.  Stream-ordered after `st`; `st` waits
// for all of them.
int run_dataflow_local(RunWs& W, pw_shard* const* shards, int32_t N, const pw_params* params,
                       const pw_tuning* tuning, const float* queries, int64_t q, int32_t* shard_ids,
                       float* shard_dists, int32_t* stats_i32, int64_t* stats_i64, cudaStream_t st) {
    for (int g = 0; g < N; g++) {
        if (!W.ring[g]) PW_CUDA(cudaStreamCreateWithFlags(&W.ring[g], cudaStreamNonBlocking));
        if (!W.ev[g]) PW_CUDA(cudaEventCreateWithFlags(&W.ev[g], cudaEventDisableTiming));
    }
    if (!W.ev[8]) PW_CUDA(cudaEventCreateWithFlags(&W.ev[8], cudaEventDisableTiming));
    const int F = (tuning && tuning->forward_count > 0) ? tuning->forward_count : 1;
    const size_t words = (size_t)N * (size_t)q * F;
    if (W.inbox_cap < words) {
        PW_CUDA(cudaStreamSynchronize(st));
        if (W.inbox) cudaFree(W.inbox);
        W.inbox = nullptr;
        W.inbox_cap = 0;
        PW_CUDA(cudaMalloc(&W.inbox, words * sizeof(uint64_t)));
        // tag 0 is never a run's; ordered on st, which the ring streams wait
        // for (a legacy-stream memset is not ordered with them)
        PW_CUDA(cudaMemsetAsync(W.inbox, 0, words * sizeof(uint64_t), st));
        W.inbox_cap = words;
        W.epoch = 0;
    }
    if (++W.epoch == 0) {  // 2^32 runs: re-zero so no stale word can match
        PW_CUDA(cudaStreamSynchronize(st));
        PW_CUDA(cudaMemsetAsync(W.inbox, 0, W.inbox_cap * sizeof(uint64_t), st));
        W.epoch = 1;
    }
    DevInfo* I;
    int rc = dev_info(shards[0]->device, &I);
    if (rc) return rc;
    const int sm_limit = std::max(1, I->sms / N);
    PW_CUDA(cudaEventRecord(W.ev[8], st));
    for (int g = 0; g < N; g++) {
        PW_CUDA(cudaStreamWaitEvent(W.ring[g], W.ev[8], 0));
        rc = pw_search_dataflow(shards[g], params, tuning, queries, q, g, N, W.epoch,
                                W.inbox + (size_t)g * q * F, W.inbox + (size_t)((g + 1) % N) * q * F, shard_ids,
                                shard_dists, stats_i32, stats_i64, sm_limit, W.ring[g]);
        if (rc) return rc;
        PW_CUDA(cudaEventRecord(W.ev[g], W.ring[g]));
    }
    for (int g = 0; g < N; g++) PW_CUDA(cudaStreamWaitEvent(st, W.ev[g], 0));
    return 0;
}

int run_device_impl(RunWs& W, pw_shard* const* shards, int32_t N, const pw_params* params,
                    const pw_tuning* tuning, const float* queries, int64_t q, int32_t mode,
                    int32_t* shard_ids, float* shard_dists, int32_t* final_ids, float* final_dists,
                    int32_t* stats_i32, int64_t* stats_i64, int32_t* entries_a, int32_t* entries_b,
                    int32_t* err_dev, cudaStream_t st) {
    if (N < 1 || !shards) return set_err(PW_EINVAL, "need at least one shard");
    int rc = validate_params(*params);
    if (rc) return rc;
    const int64_t k = params->k;
    if ((rc = pw_init_run(shard_ids, shard_dists, q * N * k, stats_i32, 4 * q * N, stats_i64, 6 * q * N, st)))
        return rc;
    if (mode == PW_MODE_BASELINE) {
        for (int s = 0; s < N; s++) {  // pipeline.py:288-297
            rc = pw_search_stage(shards[s], params, tuning, queries, 0, q, s, nullptr, nullptr,
                                 shard_ids, shard_dists, N, s, stats_i32 + (int64_t)s * 4 * q,
                                 stats_i64 + (int64_t)s * 6 * q, q, st);
            if (rc) return rc;
        }
    } else {
        if (N > 1)
            for (int s = 0; s < N; s++)  // forwarded entries index shard s+1 (pipeline.py:339)
                if ((rc = pw_shard_validate_inter(shards[s], shards[(s + 1) % N]->n))) return rc;
        if (N > 1 && N <= 8 && q >= N) {
            rc = run_dataflow_local(W, shards, N, params, tuning, queries, q, shard_ids, shard_dists, stats_i32,
                                    stats_i64, st);
            if (rc) return rc;
        } else {
            // stage-synchronous schedule (N = 1, or more shards than the
            // dataflow task map holds): chunk c at stage s on shard (c+s)%N
            std::vector<int64_t> lo(N + 1, 0);  // np.array_split(arange(Q), N)
            for (int c = 0; c < N; c++) lo[c + 1] = lo[c] + q / N + (c < q % N ? 1 : 0);
            int32_t* ein = entries_a;
            int32_t* eout = entries_b;
            for (int stage = 0; stage < N; stage++) {  // pipeline.py:344-347
                for (int c = 0; c < N; c++) {
                    int shard = (c + stage) % N;
                    rc = pw_search_stage(shards[shard], params, tuning, queries, lo[c], lo[c + 1] - lo[c],
                                         stage, stage > 0 ? ein : nullptr, stage < N - 1 ? eout : nullptr,
                                         shard_ids, shard_dists, N, shard, stats_i32 + (int64_t)stage * 4 * q,
                                         stats_i64 + (int64_t)stage * 6 * q, q, st);
                    if (rc) return rc;
                }
                std::swap(ein, eout);
            }
        }
    }
    return pw_reduce_topk(shard_ids, shard_dists, q, (int32_t)(N * k), (int32_t)k, final_ids, final_dists,
                          err_dev, st);
}

int pw_run_device(pw_shard* const* shards, int32_t N, const pw_params* params,
                  const pw_tuning* tuning, const float* queries, int64_t q, int32_t mode,
                  int32_t* shard_ids, float* shard_dists, int32_t* final_ids, float* final_dists,
                  int32_t* stats_i32, int64_t* stats_i64, int32_t* entries_a, int32_t* entries_b,
                  void* stream) {
    if (N < 1 || !shards) return set_err(PW_EINVAL, "need at least one shard");
    PW_CUDA(cudaSetDevice(shards[0]->device));
    RunWs& W = g_ws[shards[0]->device];
    std::lock_guard<std::mutex> lk(W.mu);
    // NULL err: K2 synchronises and reports empty lists itself
    return run_device_impl(W, shards, N, params, tuning, queries, q, mode, shard_ids, shard_dists, final_ids,
                           final_dists, stats_i32, stats_i64, entries_a, entries_b, nullptr, (cudaStream_t)stream);
}

int pw_run(pw_shard* const* shards, int32_t N, const pw_params* params, const pw_tuning* tuning,
           const float* queries, int64_t q, int32_t mode, int32_t* shard_ids, float* shard_dists,
           int32_t* final_ids, float* final_dists, int32_t* stats_i32, int64_t* stats_i64,
           int64_t* comm) {
    if (N < 1 || !shards) return set_err(PW_EINVAL, "need at least one shard");
    int rc = validate_params(*params);
    if (rc) return rc;
    const int64_t k = params->k;
    const int32_t d = shards[0]->d;
    for (int s = 0; s < N; s++)
        if (shards[s]->d != d || shards[s]->device != shards[0]->device)
            return set_err(PW_EINVAL, "all shards of one pw_run must share d and device");
    const int dev = shards[0]->device;
    PW_CUDA(cudaSetDevice(dev));
    RunWs& W = g_ws[dev];
    std::lock_guard<std::mutex> lk(W.mu);
    if (!W.st) PW_CUDA(cudaStreamCreateWithFlags(&W.st, cudaStreamNonBlocking));
    cudaStream_t st = W.st;
    const int64_t qq = std::max<int64_t>(q, 1);
    const int64_t F = (tuning && tuning->forward_count > 0) ? tuning->forward_count : 1;
    size_t off = 0;
    auto take = [&](size_t bytes) {
        size_t o = off;
        off += (bytes + 255) / 256 * 256;
        return o;
    };
    size_t o_q = take(sizeof(float) * qq * d), o_sid = take(sizeof(int32_t) * qq * N * k),
           o_sd = take(sizeof(float) * qq * N * k), o_fid = take(sizeof(int32_t) * qq * k),
           o_fd = take(sizeof(float) * qq * k), o_s32 = take(sizeof(int32_t) * qq * N * 4),
           o_s64 = take(sizeof(int64_t) * qq * N * 6), o_ea = take(sizeof(int32_t) * qq * F),
           o_eb = take(sizeof(int32_t) * qq * F), o_err = take(sizeof(int32_t));
    if ((rc = ws_reserve(W, off))) return rc;
    char* b = W.buf;
    float* dq = (float*)(b + o_q);
    int32_t* sid = (int32_t*)(b + o_sid);
    float* sd = (float*)(b + o_sd);
    int32_t* fid = (int32_t*)(b + o_fid);
    float* fd = (float*)(b + o_fd);
    int32_t* s32 = (int32_t*)(b + o_s32);
    int64_t* s64 = (int64_t*)(b + o_s64);
    int32_t* err = (int32_t*)(b + o_err);
    // Query upload overlapped with K1: chunks of kChunk rows on a copy stream,
    // each followed by a stream-ordered flag store (cuStreamWriteValue32) that
    // the kernel polls before reading a row of that chunk.  Every chunk is
    // enqueued before the kernel's launch: a launch that blocks until the
    // kernel ends (a profiler's serialised replay, CUDA_LAUNCH_BLOCKING,
    // a synchronising call between launch and copies) would otherwise leave
    // K1 waiting for copies not yet issued.  Without the driver entry point:
    // one copy ahead of the kernel on the same stream.
    // Chunks grow geometrically (kChunk, 2 kChunk, 4 kChunk, ... rows: chunk c
    // starts at row kChunk (2^c - 1)), so the first rows land within a few
    // microseconds while the whole upload takes few API calls before the
    // launch (6 for 10K queries instead of 20 fixed 512-row chunks: each
    // copy + flag pair costs the host ~5 us, all of it before K1 starts).
    constexpr int32_t kChunk = 256;
    auto chunk_lo = [](int64_t c) { return (int64_t)kChunk * ((1ll << c) - 1); };
    int64_t n_chunks = 0;
    while (chunk_lo(n_chunks) < q) n_chunks++;
    WriteValue32Fn wv = write_value32();
    QUpload up{};
    auto upload_chunk = [&](int64_t c) -> int {
        const int64_t lo = chunk_lo(c), rows = std::min<int64_t>((int64_t)kChunk << c, q - lo);
        PW_CUDA(cudaMemcpyAsync(dq + lo * d, queries + lo * d, sizeof(float) * rows * d, cudaMemcpyHostToDevice,
                                W.cs));
        if (wv(W.cs, (CUdeviceptr)(W.qflags + c), W.qepoch, 0) != CUDA_SUCCESS)
            return set_err(PW_ECUDA, "cuStreamWriteValue32 failed");
        return 0;
    };
    if (wv && q > kChunk) {
        if (!W.cs) PW_CUDA(cudaStreamCreateWithFlags(&W.cs, cudaStreamNonBlocking));
        bool zero = false;
        if (W.qflags_cap < (size_t)n_chunks) {
            if (W.qflags) cudaFree(W.qflags);
            W.qflags = nullptr;
            W.qflags_cap = 0;
            PW_CUDA(cudaMalloc(&W.qflags, sizeof(uint32_t) * n_chunks));
            W.qflags_cap = n_chunks;
            zero = true;
        }
        if (++W.qepoch == 0) {
            W.qepoch = 1;
            zero = true;
        }
        if (zero) {
            // tag 0 is never a call's.  Complete before the kernel can poll: it
            // runs on another stream, and fresh memory may hold any value.
            PW_CUDA(cudaMemsetAsync(W.qflags, 0, sizeof(uint32_t) * W.qflags_cap, W.cs));
            PW_CUDA(cudaStreamSynchronize(W.cs));
        }
        for (int64_t c = 0; c < n_chunks; c++)
            if ((rc = upload_chunk(c))) return rc;
        up = QUpload{W.qflags, kChunk, W.qepoch};
        tl_upload = &up;
    } else {
        PW_CUDA(cudaMemcpyAsync(dq, queries, sizeof(float) * q * d, cudaMemcpyHostToDevice, st));
    }
    PW_CUDA(cudaMemsetAsync(err, 0, sizeof(int32_t), st));
    rc = run_device_impl(W, shards, N, params, tuning, dq, q, mode, sid, sd, fid, fd, s32, s64,
                         (int32_t*)(b + o_ea), (int32_t*)(b + o_eb), err, st);
    tl_upload = nullptr;
    if (!W.hflags) PW_CUDA(cudaMallocHost(&W.hflags, sizeof(int32_t) * (1 + 64)));
    int32_t* hf = W.hflags;
    if (up.flags) PW_CUDA(cudaStreamSynchronize(W.cs));
    if (rc) return rc;
    // the results: one copy when the host buffers form the documented result
    // block (the device workspace holds them in that layout), else six
    char* h0 = reinterpret_cast<char*>(shard_ids);
    const bool block = reinterpret_cast<char*>(shard_dists) == h0 + (o_sd - o_sid) &&
                       reinterpret_cast<char*>(final_ids) == h0 + (o_fid - o_sid) &&
                       reinterpret_cast<char*>(final_dists) == h0 + (o_fd - o_sid) &&
                       reinterpret_cast<char*>(stats_i32) == h0 + (o_s32 - o_sid) &&
                       reinterpret_cast<char*>(stats_i64) == h0 + (o_s64 - o_sid);
    if (block) {
        PW_CUDA(cudaMemcpyAsync(h0, b + o_sid, (o_s64 - o_sid) + sizeof(int64_t) * q * N * 6,
                                cudaMemcpyDeviceToHost, st));
    } else {
        PW_CUDA(cudaMemcpyAsync(shard_ids, sid, sizeof(int32_t) * q * N * k, cudaMemcpyDeviceToHost, st));
        PW_CUDA(cudaMemcpyAsync(shard_dists, sd, sizeof(float) * q * N * k, cudaMemcpyDeviceToHost, st));
        PW_CUDA(cudaMemcpyAsync(final_ids, fid, sizeof(int32_t) * q * k, cudaMemcpyDeviceToHost, st));
        PW_CUDA(cudaMemcpyAsync(final_dists, fd, sizeof(float) * q * k, cudaMemcpyDeviceToHost, st));
        PW_CUDA(cudaMemcpyAsync(stats_i32, s32, sizeof(int32_t) * q * N * 4, cudaMemcpyDeviceToHost, st));
        PW_CUDA(cudaMemcpyAsync(stats_i64, s64, sizeof(int64_t) * q * N * 6, cudaMemcpyDeviceToHost, st));
    }
    PW_CUDA(cudaMemcpyAsync(hf, err, sizeof(int32_t), cudaMemcpyDeviceToHost, st));
    for (int s = 0; s < N && s < 64; s++)
        PW_CUDA(cudaMemcpyAsync(hf + 1 + s, shards[s]->counter + 1, sizeof(int32_t), cudaMemcpyDeviceToHost,
                                st));
    PW_CUDA(cudaStreamSynchronize(st));
    if (up.flags && getenv("PW_UPLOAD_DEBUG")) {
        unsigned long long ph[4];
        PW_CUDA(cudaMemcpy(ph, shards[0]->phase, sizeof ph, cudaMemcpyDeviceToHost));
        std::vector<uint32_t> fl(n_chunks);
        PW_CUDA(cudaMemcpy(fl.data(), W.qflags, sizeof(uint32_t) * n_chunks, cudaMemcpyDeviceToHost));
        fprintf(stderr, "pw_run upload: epoch %u chunks %lld flags[0] %u flags[last] %u | seen %llu want %llu at %llu chunk %llu\n",
                W.qepoch, (long long)n_chunks, fl[0], fl[n_chunks - 1], ph[0], ph[1], ph[2], ph[3]);
    }
    for (int s = 0; s < N; s++)
        if ((s >= 64 || hf[1 + s]) && (rc = check_err(shards[s]))) return rc;
    const int32_t herr = hf[0];
    if (herr) return set_err(PW_EINVAL, "cannot reduce empty candidate lists");
    // comm accounting (pipeline.py:340-341): 4 B per forwarded entry
    std::memset(comm, 0, sizeof(int64_t) * N * N);
    if (mode == PW_MODE_PIPELINED) {
        std::vector<int64_t> lo(N + 1, 0);
        for (int c = 0; c < N; c++) lo[c + 1] = lo[c] + q / N + (c < q % N ? 1 : 0);
        for (int stage = 0; stage < N - 1; stage++)
            for (int c = 0; c < N; c++) comm[(int64_t)stage * N + (c + stage) % N] = 4 * F * (lo[c + 1] - lo[c]);
    }
    return 0;
}

int pw_search_one(pw_shard* sh, int32_t use_ghost, const pw_params* params, const float* query,
                  const int64_t* seeds, int32_t n_seeds, pw_rng* rng, int32_t* out_ids,
                  float* out_dists, int32_t* out_local, pw_search_out* out, int32_t* visit_log,
                  int64_t visit_cap) {
    if (!sh || !params || !rng || !out) return set_err(PW_EINVAL, "null argument");
    const int64_t n = use_ghost ? sh->gn : sh->n;
    for (int i = 0; i < n_seeds; i++)  // search.py:215-217
        if (seeds[i] < 0 || seeds[i] >= n)
            return set_err(PW_EINVAL, "seed " + std::to_string(seeds[i]) + " outside shard of " +
                                          std::to_string(n) + " nodes");
    PW_CUDA(cudaSetDevice(sh->device));
    // The shard's launch workspace (task counter, visited tables, scratch) is
    // shared by every launch on it: searches of one device are serialised on
    // its run stream, under the same lock as pw_run (the reference's search
    // is reentrant and run from thread pools, pipeline.py:352-385).
    RunWs& W = g_ws[sh->device];
    std::lock_guard<std::mutex> lk(W.mu);
    if (!W.st) PW_CUDA(cudaStreamCreateWithFlags(&W.st, cudaStreamNonBlocking));
    cudaStream_t st = W.st;
    Launch Lc;
    int rc = prepare(sh, *params, nullptr, use_ghost != 0, n_seeds, false, Lc, st);
    if (rc) return rc;
    KArgs& A = Lc.A;
    const int64_t k = params->k;
    if (!params->log_visits) visit_cap = 0;
    size_t bytes = 0;
    auto bump = [&](size_t b) {
        size_t o = bytes;
        bytes += (b + 255) / 256 * 256;
        return o;
    };
    size_t o_q = bump(sizeof(float) * sh->d), o_s = bump(sizeof(int64_t) * std::max(n_seeds, 1)),
           o_r = bump(sizeof(Pcg64)), o_id = bump(sizeof(int32_t) * k), o_d = bump(sizeof(float) * k),
           o_l = bump(sizeof(int32_t) * k), o_rec = bump(sizeof(TaskRecord)),
           o_v = bump(sizeof(int32_t) * std::max<int64_t>(visit_cap, 1));
    if ((rc = ws_reserve(W, bytes))) return rc;
    char* buf = W.buf;
    Pcg64 g{rng->state_hi, rng->state_lo, rng->inc_hi, rng->inc_lo, (uint32_t)rng->has_uint32, rng->uinteger};
    PW_CUDA(cudaMemcpyAsync(buf + o_q, query, sizeof(float) * sh->d, cudaMemcpyHostToDevice, st));
    if (n_seeds)
        PW_CUDA(cudaMemcpyAsync(buf + o_s, seeds, sizeof(int64_t) * n_seeds, cudaMemcpyHostToDevice, st));
    PW_CUDA(cudaMemcpyAsync(buf + o_r, &g, sizeof g, cudaMemcpyHostToDevice, st));
    A.stage = 0;
    A.q0 = 0;
    A.n_tasks = 1;
    A.queries = (const float*)(buf + o_q);
    A.seeds = (const int64_t*)(buf + o_s);
    A.n_seeds = n_seeds;
    A.rng_io = (Pcg64*)(buf + o_r);
    A.out_ids = (int32_t*)(buf + o_id);
    A.out_dists = (float*)(buf + o_d);
    A.out_local = (int32_t*)(buf + o_l);
    A.out_stride = k;
    A.rec = (TaskRecord*)(buf + o_rec);
    A.visit_log = visit_cap ? (int32_t*)(buf + o_v) : nullptr;
    A.visit_cap = visit_cap;
    if ((rc = launch(sh, Lc, st))) return rc;
    TaskRecord R;
    PW_CUDA(cudaMemcpyAsync(&R, buf + o_rec, sizeof R, cudaMemcpyDeviceToHost, st));
    PW_CUDA(cudaMemcpyAsync(&g, buf + o_r, sizeof g, cudaMemcpyDeviceToHost, st));
    PW_CUDA(cudaStreamSynchronize(st));
    if ((rc = check_err(sh))) return rc;
    if (R.n_out < 0 || R.n_out > k) return set_err(PW_ECUDA, "search produced no result record");
    PW_CUDA(cudaMemcpyAsync(out_ids, buf + o_id, sizeof(int32_t) * R.n_out, cudaMemcpyDeviceToHost, st));
    PW_CUDA(cudaMemcpyAsync(out_dists, buf + o_d, sizeof(float) * R.n_out, cudaMemcpyDeviceToHost, st));
    if (out_local)
        PW_CUDA(cudaMemcpyAsync(out_local, buf + o_l, sizeof(int32_t) * R.n_out, cudaMemcpyDeviceToHost, st));
    if (visit_cap && visit_log)
        PW_CUDA(cudaMemcpyAsync(visit_log, buf + o_v, sizeof(int32_t) * std::min<int64_t>(R.n_visited, visit_cap),
                                cudaMemcpyDeviceToHost, st));
    PW_CUDA(cudaStreamSynchronize(st));
    out->iterations = R.c[0];
    out->distance_computations = R.c[1];
    out->total_visits = R.c[2];
    out->nodes_expanded = R.c[3];
    out->dgs_skipped = R.c[4];
    out->inserted_total = R.c[5];
    out->converged = R.converged;
    out->retained = R.retained;
    out->n_out = R.n_out;
    out->n_visited = R.n_visited;
    rng->state_hi = g.s_hi;
    rng->state_lo = g.s_lo;
    rng->inc_hi = g.i_hi;
    rng->inc_lo = g.i_lo;
    rng->has_uint32 = (int32_t)g.has32;
    rng->uinteger = g.u32;
    return 0;
}

int pw_phase_cycles(pw_shard* sh, int64_t* out8, int32_t reset) {
    if (!sh || !out8) return set_err(PW_EINVAL, "null argument");
    for (int i = 0; i < 8; i++) out8[i] = 0;
    if (!sh->phase) return 0;
    PW_CUDA(cudaSetDevice(sh->device));
    PW_CUDA(cudaDeviceSynchronize());
    PW_CUDA(cudaMemcpy(out8, sh->phase, sizeof(int64_t) * 8, cudaMemcpyDeviceToHost));
    if (reset) PW_CUDA(cudaMemset(sh->phase, 0, sizeof(unsigned long long) * 8));
    return 0;
}

int pw_launch_config(pw_shard* sh, const pw_params* params, const pw_tuning* tuning,
                     int32_t* out) {
    if (!sh || !params || !out) return set_err(PW_EINVAL, "null argument");
    Launch Lc;
    int rc = prepare(sh, *params, tuning, false, 0, params->ghost_enabled && sh->gn > 0, Lc);
    if (rc) return rc;
    out[0] = Lc.warps_per_block;
    out[1] = Lc.A.warp_bytes;
    out[2] = Lc.A.H;
    out[3] = Lc.A.R;
    out[4] = is_generic(Lc.fn) ? 0 : sh->d;
    out[5] = Lc.blocks;
    return 0;
}

int pw_squared_l2_rows(pw_shard* sh, const int32_t* ids, int64_t n_ids, const float* query,
                       float* out, void* stream) {
    if (!sh) return set_err(PW_EINVAL, "null argument");
    if (n_ids <= 0) return 0;
    L2Plan plan;
    if (!make_plan(sh->d, plan)) return set_err(PW_EINVAL, "dimension too large");
    int spad = (sh->d + 31) / 32 * 32 + 8;
    if (spad - 32 >= sh->d) spad -= 32;
    size_t smem = sizeof(float) * (((sh->d + 3) & ~3) + 4 * spad);
    auto go = [&](auto* tag) -> int {
        using VT_ = std::remove_pointer_t<decltype(tag)>;
        if (smem > 48 * 1024)
            PW_CUDA(cudaFuncSetAttribute(l2_rows_kernel<VT_>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
        int blocks = (int)std::min<int64_t>(4096, (n_ids + 3) / 4);
        l2_rows_kernel<VT_><<<blocks, 32, smem, (cudaStream_t)stream>>>((const VT_*)sh->vec, sh->d, spad, plan, ids, n_ids,
                                                               query, out);
        return 0;
    };
    int rc_ = sh->dtype == PW_DTYPE_U8 ? go((uint8_t*)nullptr) : go((float*)nullptr);
    if (rc_) return rc_;
    g_launches++;
    PW_CUDA(cudaGetLastError());
    return 0;
}

}  // extern "C"

namespace {
__global__ void fill_kernel(float* p, int64_t n, float v) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
        p[i] = v;
}

int pw_fill_inf(float* p, int64_t n, cudaStream_t st) {
    if (n <= 0) return 0;
    fill_kernel<<<(int)std::min<int64_t>(1024, (n + 255) / 256), 256, 0, st>>>(p, n, INFINITY);
    g_launches++;
    PW_CUDA(cudaGetLastError());
    return 0;
}

// A run's output padding (-1 ids, +inf distances) and zeroed stats in one
// launch instead of three memsets and a fill.
__global__ void init_run_kernel(int32_t* ids, float* dists, int64_t n, int32_t* s32, int64_t n32, int64_t* s64,
                                int64_t n64) {
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    const int64_t i0 = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    for (int64_t i = i0; i < n; i += stride) {
        ids[i] = -1;
        dists[i] = INFINITY;
    }
    for (int64_t i = i0; i < n32; i += stride) s32[i] = 0;
    for (int64_t i = i0; i < n64; i += stride) s64[i] = 0;
}

int pw_init_run(int32_t* ids, float* dists, int64_t n, int32_t* s32, int64_t n32, int64_t* s64, int64_t n64,
                cudaStream_t st) {
    const int64_t m = std::max(n, std::max(n32, n64));
    if (m <= 0) return 0;
    init_run_kernel<<<(int)std::min<int64_t>(1024, (m + 255) / 256), 256, 0, st>>>(ids, dists, n, s32, n32, s64, n64);
    g_launches++;
    PW_CUDA(cudaGetLastError());
    return 0;
}
}  // namespace

extern "C" int pw_init_outputs(int32_t* ids, float* dists, int64_t n, int32_t* s32, int64_t n32, int64_t* s64,
                               int64_t n64, void* stream) {
    if ((n > 0 && (!ids || !dists)) || (n32 > 0 && !s32) || (n64 > 0 && !s64))
        return set_err(PW_EINVAL, "null argument");
    return pw_init_run(ids, dists, n, s32, n32, s64, n64, (cudaStream_t)stream);
}
