// pw_crc32c.cu -- CRC-32C (Castagnoli, reflected 0x82F63B78) for the index
// container: shardann/_crc32c.py (crc32c :98-130, combine
// :85-89) and the section checksums of shardann/container.py:96-188.
//
// Device (K3 crc32c_sections_kernel): one launch checksums any number of
// device buffers (the sections of a container already uploaded to HBM).
//   * CRC is linear over GF(2): raw(A||B) = shift(raw(A), |B|) ^ raw(B), where
//     raw is the register with init 0 and no final xor, and shift(c, n) =
//     c * x^(8n) mod P.  So the buffer is cut into 128-byte pieces; lane L of
//     warp w owns pieces w*32+L, +G, +2G, ... (G = 32 * total warps pieces).
//     It folds them into one running register, pre-shifting it across the
//     constant gap to its next piece with a byte-sliced table of
//     b -> b * x^(8*gap) (4 lookups), then shifts its register to the buffer
//     end and atomicXor's it into the result.  The init/final-xor term
//     shift(~0, n) ^ ~0 is xor'ed in once.
//   * A warp's 32 pieces (4 KB) are staged global -> shared with coalesced
//     16-byte cp.async, double-buffered (tile t+1 in flight while tile t is
//     folded), into an XOR-swizzled layout (conflict-free 16-byte reads).
//   * Slicing-by-4 with one private copy of the tables per lane (128 KB):
//     every lookup of lane L hits bank L, so the data-dependent lookups never
//     conflict.  HBM-bound byte work: no tensor cores.
// Host: SSE4.2 crc32 instruction (8 bytes/op), std::thread split + combine
// for large buffers; slicing-by-8 table when SSE4.2 is absent.

#include <cuda_runtime.h>

#include <algorithm>
#include <cstdint>
#include <cstring>
#include <mutex>
#include <string>
#include <thread>
#include <vector>

#if defined(__x86_64__)
#include <cpuid.h>
#endif

#include "../../include/pw_b200.h"

int pw_internal_set_err(int code, const char* msg);
void pw_internal_count_launch();

namespace {

constexpr uint32_t POLY = 0x82F63B78u;
constexpr int PIECE = 128;               // bytes per lane per tile
constexpr int TILE = 32 * PIECE;         // bytes per warp per tile
constexpr int WARPS = 8;                 // warps per CTA
constexpr int CTAS_PER_SM = 1;

// a * b mod P in the reflected domain (bit 31 = x^0); a must be nonzero.
__host__ __device__ inline uint32_t multmodp(uint32_t a, uint32_t b) {
    uint32_t m = 1u << 31, p = 0;
    for (;;) {
        if (a & m) {
            p ^= b;
            if ((a & (m - 1)) == 0) break;
        }
        m >>= 1;
        b = (b & 1) ? (b >> 1) ^ POLY : b >> 1;
    }
    return p;
}

// x^(2^k) mod P for k = 0..63 (x^1 = bit 30)
struct X2N {
    uint32_t t[64];
};
__host__ __device__ inline void make_x2n(X2N& x) {
    uint32_t p = 1u << 30;
    for (int k = 0; k < 64; ++k) {
        x.t[k] = p;
        p = multmodp(p, p);
    }
}
// x^(8n) mod P
__host__ __device__ inline uint32_t x8nmodp(const uint32_t* x2n, uint64_t n) {
    uint32_t p = 1u << 31;
    int k = 3;
    while (n) {
        if (n & 1) p = multmodp(x2n[k & 63], p);
        n >>= 1;
        ++k;
    }
    return p;
}

__host__ __device__ inline uint32_t shift_bytes(const uint32_t* x2n, uint32_t crc, uint64_t n) {
    return n ? multmodp(x8nmodp(x2n, n), crc) : crc;
}

// ---------------------------------------------------------------- device --

struct Sec {
    const uint8_t* ptr;
    int64_t len;
};

__device__ __forceinline__ void cp_async16(void* smem, const void* gmem) {
    unsigned s = (unsigned)__cvta_generic_to_shared(smem);
    asm volatile("cp.async.cg.shared.global.L2::128B [%0], [%1], 16;\n" ::"r"(s), "l"(gmem) : "memory");
}
__device__ __forceinline__ void cp_commit() { asm volatile("cp.async.commit_group;\n" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_wait() { asm volatile("cp.async.wait_group %0;\n" ::"n"(N) : "memory"); }

// Constants the host computes once per grid size (K3Consts, in global memory):
//   GT  4 x 256  b -> b * x^(8*gap) mod P, byte-sliced: the pre-shift between a
//                lane's consecutive pieces (gap = nwarps*TILE - PIECE, constant)
//   GH  4 x 256  b -> b * x^(8*PIECE/2), byte-sliced (the two half-piece chains)
//   XL  32       x^(8*l*PIECE): lane l's piece end -> its warp's tile end
//   XT  nwarps   x^(8*k*TILE):  a warp's last tile end -> the section's tile-grid end
struct K3Consts {
    uint32_t GT[1024];
    uint32_t GH[1024];  // b -> b * x^(8*PIECE/2): joins a piece's two halves
    uint32_t XL[32];
    uint32_t XT[1];  // nwarps entries
};
// Shared memory: LT 4 x 256 x 32 u32 slicing-by-4 tables with one private
// copy per lane (table t = 2p+q, entry e, lane L at byte p*64K + e*256 + q*128
// + 4L, so every lookup of lane L hits bank L: no conflicts, 128 KB), GT/GH
// (8 KB), then the double-buffered staging (WARPS x 2 x TILE, XOR-swizzled).
constexpr size_t K3_LT = 4 * 256 * 32 * 4, K3_GT = 2 * 4 * 256 * 4;
constexpr size_t K3_SMEM = K3_LT + K3_GT + (size_t)WARPS * 2 * TILE;

// a * b mod P for a constant a, branch-free (no divergence across lanes)
__device__ __forceinline__ uint32_t mulc(uint32_t a, uint32_t b) {
    uint32_t p = 0;
#pragma unroll
    for (int i = 31; i >= 0; --i) {
        p ^= (0u - ((a >> i) & 1u)) & b;
        b = (b >> 1) ^ ((0u - (b & 1u)) & POLY);
    }
    return p;
}

// Every section is laid on a grid of TILE-byte tiles that starts at its
// 16-byte-aligned base A <= ptr.  Bytes of the grid outside the section are
// fed as ZEROS: leading zeros leave a raw CRC unchanged, and the trailing Z
// zeros multiply it by x^(8Z), which the host undoes with x^(-8Z)
// (x^-1 = (P - 1) / x).  So every lane folds whole 128-byte pieces, and
// out[s] = raw(section || Z zeros); pw_crc32c_device finishes on the host.
__global__ void __launch_bounds__(WARPS * 32, CTAS_PER_SM)
crc32c_sections_kernel(const Sec* __restrict__ secs, int nsec, const K3Consts* __restrict__ K,
                       uint32_t* __restrict__ out) {
    extern __shared__ __align__(16) uint8_t smem[];
    uint32_t* LT = reinterpret_cast<uint32_t*>(smem);
    uint32_t* GT = reinterpret_cast<uint32_t*>(smem + K3_LT);
    uint8_t* stage = smem + K3_LT + K3_GT;
    const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
    const int64_t warp = (int64_t)blockIdx.x * WARPS + wib;
    const int64_t nwarps = (int64_t)gridDim.x * WARPS;

    uint32_t* T = reinterpret_cast<uint32_t*>(stage);  // compact 4 x 256 first
    for (int i = threadIdx.x; i < 256; i += blockDim.x) {
        uint32_t c = i;
        for (int b = 0; b < 8; ++b) c = (c & 1) ? (c >> 1) ^ POLY : c >> 1;
        T[i] = c;
    }
    for (int i = threadIdx.x; i < 2048; i += blockDim.x) GT[i] = K->GT[i];  // GT then GH
    __syncthreads();
    for (int i = threadIdx.x; i < 256; i += blockDim.x) {
        uint32_t c = T[i];
        for (int t = 1; t < 4; ++t) {
            c = (c >> 8) ^ T[c & 0xff];
            T[t * 256 + i] = c;
        }
    }
    __syncthreads();
    // lane copies: table t = 2p + q, entry e, lane L at byte p*64K + e*256 + q*128 + 4L
    for (int i = threadIdx.x; i < 1024 * 32; i += blockDim.x) {
        const int q = (i >> 5) & 1, e = (i >> 6) & 255, pp = i >> 14;
        LT[i] = T[(2 * pp + q) * 256 + e];
    }
    __syncthreads();

    // one lookup = PRMT (byte k of x into bits 8..15, this lane's 4L into
    // bits 0..7) + LDS at a compile-time table offset
    const uint8_t* Lb = reinterpret_cast<const uint8_t*>(LT);
    const uint32_t l4 = 4u * (uint32_t)lane;
    auto lk = [&](uint32_t x, uint32_t sel, uint32_t toff) -> uint32_t {
        return *reinterpret_cast<const uint32_t*>(Lb + toff + __byte_perm(x, l4, sel));
    };
    auto step4 = [&](uint32_t c, uint32_t w) -> uint32_t {
        const uint32_t x = c ^ w;
        return lk(x, 0x5504, 65536 + 128) ^ lk(x, 0x5514, 65536) ^ lk(x, 0x5524, 128) ^ lk(x, 0x5534, 0);
    };
    auto shift_gap = [&](uint32_t c) -> uint32_t {
        return GT[c & 0xff] ^ GT[256 + ((c >> 8) & 0xff)] ^ GT[512 + ((c >> 16) & 0xff)] ^ GT[768 + (c >> 24)];
    };
    const uint32_t* GH = GT + 1024;
    auto shift_half = [&](uint32_t c) -> uint32_t {
        return GH[c & 0xff] ^ GH[256 + ((c >> 8) & 0xff)] ^ GH[512 + ((c >> 16) & 0xff)] ^ GH[768 + (c >> 24)];
    };
    const uint32_t xl = K->XL[31 - lane];
    uint8_t* buf0 = stage + (size_t)wib * 2 * TILE;
    constexpr int CPP = PIECE / 16;  // 16-byte chunks per piece

    for (int s = 0; s < nsec; ++s) {
        const uint8_t* base = secs[s].ptr;
        const int64_t len = secs[s].len;
        if (len <= 0) continue;
        const uint8_t* A = reinterpret_cast<const uint8_t*>(reinterpret_cast<uintptr_t>(base) & ~(uintptr_t)15);
        const int64_t head = base - A;  // grid bytes before the section (zeros)
        const int64_t span = head + len;
        const int64_t ntiles = (span + TILE - 1) / TILE;
        if (warp >= ntiles) continue;
        // stage tile t into buffer b: chunk h of piece p lands at p*PIECE +
        // ((h ^ (p & (CPP-1))) * 16), so the 8 lanes of a quarter-warp read
        // 16 B from 8 distinct bank groups; grid bytes outside the section are 0
        auto issue = [&](int64_t t, int b) {
            if (t < ntiles) {
                uint8_t* my = buf0 + b * TILE;
                const int64_t t0 = t * TILE;
                if (t0 >= head && t0 + TILE <= span) {  // interior tile: no per-chunk tests
#pragma unroll
                    for (int k = 0; k < TILE / 16 / 32; ++k) {
                        const int c = lane + 32 * k, p = c / CPP, h = c % CPP;
                        cp_async16(my + p * PIECE + ((h ^ (p & (CPP - 1))) << 4), A + t0 + (int64_t)c * 16);
                    }
                } else {
#pragma unroll 1
                    for (int c = lane; c < TILE / 16; c += 32) {
                        const int64_t o = t0 + (int64_t)c * 16;
                        const int p = c / CPP, h = c % CPP;
                        uint8_t* dst = my + p * PIECE + ((h ^ (p & (CPP - 1))) << 4);
                        if (o >= head && o + 16 <= span) {
                            cp_async16(dst, A + o);
                        } else if (o + 16 <= head || o >= span) {
                            *reinterpret_cast<uint4*>(dst) = make_uint4(0u, 0u, 0u, 0u);
                        } else {
                            for (int q = 0; q < 16; ++q) dst[q] = (o + q >= head && o + q < span) ? A[o + q] : 0;
                        }
                    }
                }
            }
            cp_commit();
        };
        uint32_t acc = 0;
        int b = 0;
        int64_t t_last = warp;
        issue(warp, 0);
        for (int64_t t = warp; t < ntiles; t += nwarps, b ^= 1) {
            issue(t + nwarps, b ^ 1);
            cp_wait<1>();
            __syncwarp();
            // two independent chains per lane (ILP): the first half continues
            // the lane's register, the second starts from 0; joined with GH
            const uint8_t* pb = buf0 + b * TILE + lane * PIECE;
            const int sw = lane & (CPP - 1);
            uint32_t a0 = shift_gap(acc), a1 = 0;  // acc == 0 before the first piece
#pragma unroll
            for (int h = 0; h < CPP / 2; ++h) {
                const uint4 v = *reinterpret_cast<const uint4*>(pb + ((h ^ sw) << 4));
                const uint4 w = *reinterpret_cast<const uint4*>(pb + (((h + CPP / 2) ^ sw) << 4));
                a0 = step4(a0, v.x);
                a1 = step4(a1, w.x);
                a0 = step4(a0, v.y);
                a1 = step4(a1, w.y);
                a0 = step4(a0, v.z);
                a1 = step4(a1, w.z);
                a0 = step4(a0, v.w);
                a1 = step4(a1, w.w);
            }
            acc = shift_half(a0) ^ a1;
            t_last = t;
            __syncwarp();
        }
        cp_wait<0>();
        __syncwarp();
        // lane piece end -> warp tile end (XL), xor over the warp, then the
        // warp's last tile end -> the grid end (XT)
        acc = mulc(xl, acc);
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) acc ^= __shfl_xor_sync(0xffffffffu, acc, o);
        if (lane == 0) atomicXor(&out[s], mulc(K->XT[ntiles - 1 - t_last], acc));
    }
}

// ------------------------------------------------------------------ host --

struct HostTables {
    uint32_t t[8][256];
    X2N x;
    HostTables() {
        for (uint32_t i = 0; i < 256; ++i) {
            uint32_t c = i;
            for (int b = 0; b < 8; ++b) c = (c & 1) ? (c >> 1) ^ POLY : c >> 1;
            t[0][i] = c;
        }
        for (int k = 1; k < 8; ++k)
            for (int i = 0; i < 256; ++i) t[k][i] = (t[k - 1][i] >> 8) ^ t[0][t[k - 1][i] & 0xff];
        make_x2n(x);
    }
};
const HostTables& tables() {
    static const HostTables h;
    return h;
}

bool have_sse42() {
#if defined(__x86_64__)
    unsigned a, b, c, d;
    if (!__get_cpuid(1, &a, &b, &c, &d)) return false;
    return (c & bit_SSE4_2) != 0;
#else
    return false;
#endif
}

#if defined(__x86_64__)
__attribute__((target("sse4.2"))) uint32_t raw_sse42(uint32_t c, const uint8_t* p, size_t n) {
    uint64_t c64 = c;
    for (; n && ((uintptr_t)p & 7); --n, ++p) c64 = __builtin_ia32_crc32qi((uint32_t)c64, *p);
    for (; n >= 8; n -= 8, p += 8) {
        uint64_t v;
        std::memcpy(&v, p, 8);
        c64 = __builtin_ia32_crc32di(c64, v);
    }
    for (; n; --n, ++p) c64 = __builtin_ia32_crc32qi((uint32_t)c64, *p);
    return (uint32_t)c64;
}
#endif

uint32_t raw_table(uint32_t c, const uint8_t* p, size_t n) {
    const auto& T = tables().t;
    for (; n && ((uintptr_t)p & 7); --n, ++p) c = (c >> 8) ^ T[0][(c ^ *p) & 0xff];
    for (; n >= 8; n -= 8, p += 8) {
        uint32_t lo, hi;
        std::memcpy(&lo, p, 4);
        std::memcpy(&hi, p + 4, 4);
        lo ^= c;
        c = T[7][lo & 0xff] ^ T[6][(lo >> 8) & 0xff] ^ T[5][(lo >> 16) & 0xff] ^ T[4][lo >> 24] ^
            T[3][hi & 0xff] ^ T[2][(hi >> 8) & 0xff] ^ T[1][(hi >> 16) & 0xff] ^ T[0][hi >> 24];
    }
    for (; n; --n, ++p) c = (c >> 8) ^ T[0][(c ^ *p) & 0xff];
    return c;
}

// standard CRC-32C (init ~0, final ~) of one contiguous range
uint32_t crc_serial(const uint8_t* p, size_t n) {
    static const bool hw = have_sse42();
#if defined(__x86_64__)
    if (hw) return ~raw_sse42(0xffffffffu, p, n);
#endif
    return ~raw_table(0xffffffffu, p, n);
}

// x^(-8n) mod P: x^-1 = (P - 1) / x, reflected (POLY << 1) | 1
uint32_t xinv8n(uint64_t n) {
    uint32_t base = (POLY << 1) | 1u, p = 1u << 31;
    for (int i = 0; i < 3; ++i) base = multmodp(base, base);  // x^-8
    while (n) {
        if (n & 1) p = multmodp(base, p);
        base = multmodp(base, base);
        n >>= 1;
    }
    return p;
}

uint32_t combine(uint32_t c1, uint32_t c2, uint64_t len2) {  // _crc32c.py:85-89
    return shift_bytes(tables().x.t, c1, len2) ^ c2;
}

}  // namespace

extern "C" {

int pw_crc32c(const void* buf, int64_t n, int32_t threads, uint32_t* out) {
    if (!out || n < 0 || (n > 0 && !buf)) return pw_internal_set_err(PW_EINVAL, "pw_crc32c: bad arguments");
    const uint8_t* p = static_cast<const uint8_t*>(buf);
    int nt = threads > 0 ? threads : (int)std::max(1u, std::thread::hardware_concurrency());
    const int64_t min_part = 8 << 20;  // below 8 MB per thread the split does not pay
    nt = (int)std::min<int64_t>(nt, std::max<int64_t>(1, n / min_part));
    if (nt <= 1) {
        *out = crc_serial(p, (size_t)n);
        return PW_OK;
    }
    std::vector<uint32_t> part(nt);
    std::vector<int64_t> lo(nt + 1);
    for (int i = 0; i <= nt; ++i) lo[i] = n * i / nt;
    std::vector<std::thread> pool;
    for (int i = 0; i < nt; ++i)
        pool.emplace_back([&, i] { part[i] = crc_serial(p + lo[i], (size_t)(lo[i + 1] - lo[i])); });
    for (auto& t : pool) t.join();
    uint32_t c = part[0];
    for (int i = 1; i < nt; ++i) c = combine(c, part[i], (uint64_t)(lo[i + 1] - lo[i]));
    *out = c;
    return PW_OK;
}

int pw_crc32c_combine(uint32_t crc1, uint32_t crc2, int64_t len2, uint32_t* out) {
    if (!out || len2 < 0) return pw_internal_set_err(PW_EINVAL, "pw_crc32c_combine: bad arguments");
    *out = combine(crc1, crc2, (uint64_t)len2);
    return PW_OK;
}

int pw_crc32c_device(const void* const* ptrs, const int64_t* lens, int32_t n, uint32_t* out_host,
                     void* stream) {
    if (n < 0 || (n > 0 && (!ptrs || !lens || !out_host)))
        return pw_internal_set_err(PW_EINVAL, "pw_crc32c_device: bad arguments");
    if (n == 0) return PW_OK;
    static std::mutex mu;  // the cached per-device constants
    std::lock_guard<std::mutex> lk(mu);
    for (int i = 0; i < n; ++i)
        if (lens[i] < 0 || (lens[i] > 0 && !ptrs[i]))
            return pw_internal_set_err(PW_EINVAL, "pw_crc32c_device: bad section");
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    auto fail = [](cudaError_t e, const char* what) {
        std::string m = std::string("pw_crc32c_device: ") + what + ": " + cudaGetErrorString(e);
        return pw_internal_set_err(e == cudaErrorMemoryAllocation ? PW_ENOMEM : PW_ECUDA, m.c_str());
    };
    int dev = 0, sms = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    if (dev < 0 || dev >= 64) return pw_internal_set_err(PW_EINVAL, "pw_crc32c_device: device index");
    const int blocks = sms * CTAS_PER_SM;
    const int64_t nwarps = (int64_t)blocks * WARPS;
    // per device, grow-only and reused across calls: the grid-size constants
    // (computed on the host once), the device section table + results, and
    // their page-locked host staging (no allocation or pageable copy per call)
    struct DevWs {
        int64_t nwarps = -1;
        void* consts = nullptr;
        size_t cap = 0;  // sections
        uint8_t* dbuf = nullptr;
        uint8_t* hbuf = nullptr;
        bool attr_set = false;
    };
    static DevWs ws[64];
    DevWs& W = ws[dev];
    cudaError_t e;
    if (W.nwarps != nwarps) {
        const uint32_t* x2n = tables().x.t;
        std::vector<uint32_t> consts(2048 + 32 + nwarps, 0);
        const uint32_t xg = x8nmodp(x2n, (uint64_t)nwarps * TILE - PIECE), xh = x8nmodp(x2n, PIECE / 2);
        for (int i = 0; i < 1024; ++i) {
            consts[i] = multmodp(xg, (uint32_t)(i & 255) << (8 * (i >> 8)));
            consts[1024 + i] = multmodp(xh, (uint32_t)(i & 255) << (8 * (i >> 8)));
        }
        const uint32_t xp = x8nmodp(x2n, PIECE), xt = x8nmodp(x2n, TILE);
        uint32_t c = 1u << 31;
        for (int l = 0; l < 32; ++l, c = multmodp(xp, c)) consts[2048 + l] = c;
        c = 1u << 31;
        for (int64_t k = 0; k < nwarps; ++k, c = multmodp(xt, c)) consts[2080 + k] = c;
        if (W.consts) cudaFree(W.consts);
        W.consts = nullptr;
        W.nwarps = -1;
        if ((e = cudaMalloc(&W.consts, consts.size() * 4)) != cudaSuccess) return fail(e, "alloc");
        if ((e = cudaMemcpy(W.consts, consts.data(), consts.size() * 4, cudaMemcpyHostToDevice)) != cudaSuccess)
            return fail(e, "constants");
        W.nwarps = nwarps;
    }
    const size_t sec_bytes = sizeof(Sec) * n, out_off = (sec_bytes + 15) & ~(size_t)15,
                 out_bytes = sizeof(uint32_t) * n;
    if (W.cap < (size_t)n) {
        if (W.dbuf) cudaFree(W.dbuf);
        if (W.hbuf) cudaFreeHost(W.hbuf);
        W.dbuf = W.hbuf = nullptr;
        W.cap = 0;
        const size_t cap = std::max<size_t>(64, (size_t)n), bytes = ((sizeof(Sec) * cap + 15) & ~(size_t)15) + 4 * cap;
        if ((e = cudaMalloc(&W.dbuf, bytes)) != cudaSuccess) return fail(e, "alloc");
        if ((e = cudaHostAlloc(&W.hbuf, bytes, cudaHostAllocDefault)) != cudaSuccess) return fail(e, "alloc");
        W.cap = cap;
    }
    Sec* h = reinterpret_cast<Sec*>(W.hbuf);
    for (int i = 0; i < n; ++i) h[i] = Sec{static_cast<const uint8_t*>(ptrs[i]), lens[i]};
    Sec* d_secs = reinterpret_cast<Sec*>(W.dbuf);
    uint32_t* d_out = reinterpret_cast<uint32_t*>(W.dbuf + out_off);
    uint32_t* h_out = reinterpret_cast<uint32_t*>(W.hbuf + out_off);
    void* kbuf = W.consts;
    const size_t smem = K3_SMEM;
    if (!W.attr_set) {  // the opt-in shared-memory attribute is per device
        e = cudaFuncSetAttribute(crc32c_sections_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        if (e != cudaSuccess) return fail(e, "smem attribute");
        W.attr_set = true;
    }
    if ((e = cudaMemcpyAsync(d_secs, h, sec_bytes, cudaMemcpyHostToDevice, st)) != cudaSuccess ||
        (e = cudaMemsetAsync(d_out, 0, out_bytes, st)) != cudaSuccess)
        return fail(e, "setup");
    crc32c_sections_kernel<<<blocks, WARPS * 32, smem, st>>>(d_secs, n, static_cast<const K3Consts*>(kbuf),
                                                              d_out);
    if ((e = cudaGetLastError()) != cudaSuccess) return fail(e, "launch");
    pw_internal_count_launch();
    if ((e = cudaMemcpyAsync(h_out, d_out, out_bytes, cudaMemcpyDeviceToHost, st)) != cudaSuccess)
        return fail(e, "readback");
    if ((e = cudaStreamSynchronize(st)) != cudaSuccess) return fail(e, "sync");
    // out = raw(section || Z zeros): undo the Z trailing zeros with x^(-8Z),
    // then apply init/final xor: crc = raw ^ shift(~0, len) ^ ~0
    const uint32_t* x2n = tables().x.t;
    for (int i = 0; i < n; ++i) {
        const int64_t len = lens[i];
        uint32_t raw = 0;
        if (len > 0) {
            const int64_t head = (int64_t)(reinterpret_cast<uintptr_t>(ptrs[i]) & 15);
            const int64_t ntiles = (head + len + TILE - 1) / TILE;
            const uint64_t z = (uint64_t)(ntiles * TILE - head - len);
            raw = z ? multmodp(xinv8n(z), h_out[i]) : h_out[i];
        }
        out_host[i] = raw ^ shift_bytes(x2n, 0xffffffffu, (uint64_t)(len > 0 ? len : 0)) ^ 0xffffffffu;
    }
    return PW_OK;
}

}  // extern "C"
