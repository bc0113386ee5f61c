// gather_probe.cu -- the achievable HBM bandwidth of K1's access pattern:
// whole rows of `row_bytes` gathered at uniformly random row ids out of a
// table far larger than L2, with as many rows in flight as the SM holds.
// K1's roofline denominator stays the measured copy bandwidth
// (MEASURED_PEAKS.json); this probe says how much of it random row gathers
// can reach at all, i.e. what part of K1's gap is the access pattern itself.
//
// Every warp owns a slice of the id list; 8 lanes cover one row with 16-byte
// loads (LDG.128, L1 bypass), each warp keeps UNROLL rows in flight, and the
// loaded words are XOR-folded into a per-thread value so nothing is dead.
#include <cuda_runtime.h>
#include <stdint.h>

namespace {

template <int UNROLL>
__global__ void __launch_bounds__(512) gather_probe_kernel(const uint4* __restrict__ table, int64_t row_words,
                                                           const int32_t* __restrict__ ids, int64_t n_ids,
                                                           uint32_t* __restrict__ sink) {
    const unsigned lane = threadIdx.x & 31u;
    const int64_t warps = (int64_t)gridDim.x * (blockDim.x >> 5);
    const int64_t gw = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
    const int sub = lane & 7, grp = lane >> 3;  // 4 rows per warp step, 8 lanes per row
    uint32_t acc = 0;
    // rows r = base + 4 * u + grp for u < UNROLL: UNROLL * 4 rows in flight per warp
    for (int64_t base = gw * 4 * UNROLL; base < n_ids; base += warps * 4 * UNROLL) {
        uint4 v[UNROLL][4];
        int64_t rows[UNROLL];
#pragma unroll
        for (int u = 0; u < UNROLL; u++) {
            const int64_t r = base + 4 * u + grp;
            rows[u] = r < n_ids ? (int64_t)ids[r] : -1;
        }
#pragma unroll
        for (int u = 0; u < UNROLL; u++)
#pragma unroll
            for (int c = 0; c < 4; c++) {
                const int64_t w = sub + 8 * c;
                v[u][c] = (rows[u] >= 0 && w < row_words) ? __ldcs(table + rows[u] * row_words + w)
                                                          : make_uint4(0, 0, 0, 0);
            }
#pragma unroll
        for (int u = 0; u < UNROLL; u++)
#pragma unroll
            for (int c = 0; c < 4; c++) acc ^= v[u][c].x ^ v[u][c].y ^ v[u][c].z ^ v[u][c].w;
        // rows longer than 32 x 16 bytes: the remaining chunks
        for (int64_t w0 = 32; w0 < row_words; w0 += 8)
#pragma unroll
            for (int u = 0; u < UNROLL; u++) {
                const int64_t w = w0 + sub;
                if (rows[u] >= 0 && w < row_words) {
                    const uint4 x = __ldcs(table + rows[u] * row_words + w);
                    acc ^= x.x ^ x.y ^ x.z ^ x.w;
                }
            }
    }
    if (acc == 0x9E3779B9u) sink[0] = acc;  // practically never; keeps the loads live
}

}  // namespace

// Gather n_ids rows of row_bytes (multiple of 16) from table (device) at ids
// (device int32); asynchronous on stream.  0 ok, -1 bad argument, -3 CUDA.
extern "C" int pw_gather_probe(const void* table, int64_t row_bytes, const int32_t* ids, int64_t n_ids,
                               uint32_t* sink, int32_t blocks, void* stream) {
    if (!table || !ids || !sink || row_bytes <= 0 || row_bytes % 16 || n_ids <= 0 || blocks <= 0) return -1;
    gather_probe_kernel<4><<<blocks, 512, 0, (cudaStream_t)stream>>>(
        reinterpret_cast<const uint4*>(table), row_bytes / 16, ids, n_ids, sink);
    return cudaGetLastError() == cudaSuccess ? 0 : -3;
}
