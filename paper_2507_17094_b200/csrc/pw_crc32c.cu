// pw_crc32c.cu -- CRC-32C (Castagnoli, reflected 0x82F63B78) for the index
// container: shardann/_crc32c.py (crc32c :98-130, combine
// :85-89) and the section checksums of shardann/container.py:96-188.
//
// Device (K3 crc32c_sections_kernel): one launch checksums any number of
// device buffers (the sections of a container already uploaded to HBM).
//   * CRC is linear over GF(2): raw(A||B) = shift(raw(A), |B|) ^ raw(B), where
//     raw is the register with init 0 and no final xor, and shift(c, n) =
//     c * x^(8n) mod P.  So the buffer is cut into 256-byte pieces; lane L of
//     warp w owns pieces w*32+L, +G, +2G, ... (G = 32 * total warps pieces).
//     It folds them into one running register (pre-shifting it across the gap
//     to the next piece by a constant x^(8(G*256-256)) multiply), then shifts
//     its register to the buffer end and atomicXor's it into the result.
//     The init/final-xor term shift(~0, n) ^ ~0 is xor'ed in once.
//   * A warp's 32 pieces (8 KB) are staged global -> shared with coalesced
//     16-byte cp.async into an XOR-swizzled layout (conflict-free 16-byte
//     reads), then each lane runs slicing-by-8 over its piece with the 8 x 256 tables in
//     shared memory.  HBM-bound byte work: no tensor cores.
// Host: SSE4.2 crc32 instruction (8 bytes/op), std::thread split + combine
// for large buffers; slicing-by-8 table when SSE4.2 is absent.

#include <cuda_runtime.h>

#include <algorithm>
#include <cstdint>
#include <cstring>
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
constexpr int PIECE = 256;               // bytes per lane per tile
constexpr int TILE = 32 * PIECE;         // bytes per warp per tile
constexpr int WARPS = 8;                 // warps per CTA
constexpr int CTAS_PER_SM = 2;

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

__device__ __forceinline__ uint32_t step8(const uint32_t* __restrict__ T, uint32_t c, uint64_t v) {
    uint32_t lo = (uint32_t)v ^ c, hi = (uint32_t)(v >> 32);
    return T[7 * 256 + (lo & 0xff)] ^ T[6 * 256 + ((lo >> 8) & 0xff)] ^ T[5 * 256 + ((lo >> 16) & 0xff)] ^
           T[4 * 256 + (lo >> 24)] ^ T[3 * 256 + (hi & 0xff)] ^ T[2 * 256 + ((hi >> 8) & 0xff)] ^
           T[1 * 256 + ((hi >> 16) & 0xff)] ^ T[hi >> 24];
}

__global__ void __launch_bounds__(WARPS * 32, CTAS_PER_SM)
crc32c_sections_kernel(const Sec* __restrict__ secs, int nsec, uint32_t* __restrict__ out) {
    extern __shared__ __align__(16) uint8_t smem[];
    uint32_t* T = reinterpret_cast<uint32_t*>(smem);                 // 8 x 256 slicing tables
    uint32_t* x2n = T + 8 * 256;                                      // 64 entries
    uint8_t* stage = smem + (8 * 256 + 64) * 4;                       // WARPS x 32 x PIECE (swizzled)
    const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
    for (int i = threadIdx.x; i < 256; i += blockDim.x) {
        uint32_t c = i;
        for (int b = 0; b < 8; ++b) c = (c & 1) ? (c >> 1) ^ POLY : c >> 1;
        T[i] = c;
    }
    if (threadIdx.x == 0) {
        X2N x;
        make_x2n(x);
        for (int k = 0; k < 64; ++k) x2n[k] = x.t[k];
    }
    __syncthreads();
    for (int i = threadIdx.x; i < 256; i += blockDim.x) {
        uint32_t c = T[i];
        for (int t = 1; t < 8; ++t) {
            c = (c >> 8) ^ T[c & 0xff];
            T[t * 256 + i] = c;
        }
    }
    __syncthreads();

    const int64_t warp = (int64_t)blockIdx.x * WARPS + wib;
    const int64_t nwarps = (int64_t)gridDim.x * WARPS;
    const uint64_t gap = (uint64_t)nwarps * TILE - PIECE;  // end of a piece -> start of this lane's next
    const uint32_t xgap = x8nmodp(x2n, gap);
    uint8_t* my = stage + (size_t)wib * TILE;

    for (int s = 0; s < nsec; ++s) {
        const uint8_t* base = secs[s].ptr;
        const int64_t len = secs[s].len;
        if (warp == 0 && lane == 0) {  // init/final-xor term: crc = raw ^ shift(~0, len) ^ ~0
            atomicXor(&out[s], shift_bytes(x2n, 0xffffffffu, (uint64_t)len) ^ 0xffffffffu);
        }
        if (len <= 0) continue;
        // tiles are aligned to 16 absolute bytes: A = base rounded down
        const uint8_t* A = reinterpret_cast<const uint8_t*>(reinterpret_cast<uintptr_t>(base) & ~(uintptr_t)15);
        const int64_t head = base - A;  // 0..15 bytes before the section inside tile 0
        const int64_t span = head + len;
        const int64_t ntiles = (span + TILE - 1) / TILE;
        uint32_t acc = 0;
        int64_t pos = -1;  // section offset just past the last byte this lane folded
        for (int64_t t = warp; t < ntiles; t += nwarps) {
            const int64_t t0 = t * TILE;  // offset from A
            // stage: 512 chunks of 16 B, 16 per lane, coalesced; chunk h of piece p
            // lands at p*256 + ((h ^ (p & 15)) * 16) (XOR swizzle: the 8 lanes of
            // a quarter-warp read 16 B from 8 distinct bank groups)
#pragma unroll 4
            for (int c = lane; c < TILE / 16; c += 32) {
                const int64_t o = t0 + (int64_t)c * 16;
                const int p = c / (PIECE / 16), h = c % (PIECE / 16);
                uint8_t* dst = my + p * PIECE + ((h ^ (p & 15)) << 4);
                if (o >= head && o + 16 <= span) {
                    cp_async16(dst, A + o);
                } else if (o + 16 > head && o < span) {
                    for (int b = 0; b < 16; ++b)
                        if (o + b >= head && o + b < span) dst[b] = A[o + b];
                }
            }
            asm volatile("cp.async.wait_all;\n" ::: "memory");
            __syncwarp();
            const int64_t ps = t0 + (int64_t)lane * PIECE;  // piece [ps, ps+PIECE) from A
            const int64_t lo = ps > head ? ps : head, hi = ps + PIECE < span ? ps + PIECE : span;
            if (lo < hi) {
                if (pos >= 0) {
                    const uint64_t g = (uint64_t)((lo - head) - pos);
                    acc = g == gap ? multmodp(xgap, acc) : shift_bytes(x2n, acc, g);
                }
                const uint8_t* pb = my + lane * PIECE;
                const int sw = lane & 15;
                int u = (int)(lo - ps);
                const int ue = (int)(hi - ps);
                for (; u < ue && (u & 15); ++u)
                    acc = (acc >> 8) ^ T[(acc ^ pb[(((u >> 4) ^ sw) << 4) | (u & 15)]) & 0xff];
                for (; u + 16 <= ue; u += 16) {
                    const uint4 v = *reinterpret_cast<const uint4*>(pb + (((u >> 4) ^ sw) << 4));
                    acc = step8(T, acc, (uint64_t)v.x | ((uint64_t)v.y << 32));
                    acc = step8(T, acc, (uint64_t)v.z | ((uint64_t)v.w << 32));
                }
                for (; u < ue; ++u)
                    acc = (acc >> 8) ^ T[(acc ^ pb[(((u >> 4) ^ sw) << 4) | (u & 15)]) & 0xff];
                pos = hi - head;
            }
            __syncwarp();
        }
        if (pos >= 0) atomicXor(&out[s], shift_bytes(x2n, acc, (uint64_t)(len - pos)));
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
    for (int i = 0; i < n; ++i)
        if (lens[i] < 0 || (lens[i] > 0 && !ptrs[i]))
            return pw_internal_set_err(PW_EINVAL, "pw_crc32c_device: bad section");
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    auto fail = [](cudaError_t e, const char* what) {
        std::string m = std::string("pw_crc32c_device: ") + what + ": " + cudaGetErrorString(e);
        return pw_internal_set_err(e == cudaErrorMemoryAllocation ? PW_ENOMEM : PW_ECUDA, m.c_str());
    };
    std::vector<Sec> h(n);
    for (int i = 0; i < n; ++i) h[i] = Sec{static_cast<const uint8_t*>(ptrs[i]), lens[i]};
    const size_t sec_bytes = sizeof(Sec) * n, out_bytes = sizeof(uint32_t) * n;
    void* ws = nullptr;
    cudaError_t e = cudaMallocAsync(&ws, sec_bytes + out_bytes + 16, st);
    if (e != cudaSuccess) return fail(e, "alloc");
    Sec* d_secs = static_cast<Sec*>(ws);
    uint32_t* d_out = reinterpret_cast<uint32_t*>(static_cast<uint8_t*>(ws) + ((sec_bytes + 15) & ~(size_t)15));
    int dev = 0, sms = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    const size_t smem = (8 * 256 + 64) * 4 + (size_t)WARPS * TILE;
    static bool attr_set = false;
    if (!attr_set) {
        e = cudaFuncSetAttribute(crc32c_sections_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        if (e != cudaSuccess) return fail(e, "smem attribute");
        attr_set = true;
    }
    if ((e = cudaMemcpyAsync(d_secs, h.data(), sec_bytes, cudaMemcpyHostToDevice, st)) != cudaSuccess ||
        (e = cudaMemsetAsync(d_out, 0, out_bytes, st)) != cudaSuccess)
        return fail(e, "setup");
    crc32c_sections_kernel<<<sms * CTAS_PER_SM, WARPS * 32, smem, st>>>(d_secs, n, d_out);
    if ((e = cudaGetLastError()) != cudaSuccess) return fail(e, "launch");
    pw_internal_count_launch();
    if ((e = cudaMemcpyAsync(out_host, d_out, out_bytes, cudaMemcpyDeviceToHost, st)) != cudaSuccess)
        return fail(e, "readback");
    cudaFreeAsync(ws, st);
    if ((e = cudaStreamSynchronize(st)) != cudaSuccess) return fail(e, "sync");
    return PW_OK;
}

}  // extern "C"
