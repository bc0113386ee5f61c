// rng_pcg64.cuh -- exact device restatement of the reference's random streams.
//
// shardann/rng.py:26-44 derives one 64-bit seed per (run seed, tag, query id,
// stage) with splitmix64 and feeds it to numpy's PCG64 through SeedSequence.
// Searches draw from it in shardann/search.py:222 (Generator.choice without
// replacement) and shardann/direction.py:105 (Generator.permutation).  This
// header reproduces numpy 2.x's algorithms bit for bit (SeedSequence
// hashmix/mix pool, PCG64 XSL-RR with the buffered 32-bit half, Lemire
// bounded ints, Floyd choice + tail shuffle, masked-rejection permutation) so
// device searches consume exactly the reference's random values.
#pragma once
#include <stdint.h>

#ifdef __CUDACC__
#define PW_HD __host__ __device__ __forceinline__
// cold per-search routines: one out-of-line copy keeps the kernel's hot loop
// inside the instruction caches
#define PW_HD_COLD static __host__ __device__ __noinline__
#else
#define PW_HD inline
#define PW_HD_COLD static inline
#endif

namespace pw {

struct Pcg64 {
    uint64_t s_hi, s_lo;   // 128-bit LCG state
    uint64_t i_hi, i_lo;   // 128-bit increment (odd)
    uint32_t has32;
    uint32_t u32;
};

PW_HD uint64_t mulhi64(uint64_t a, uint64_t b) {
#ifdef __CUDA_ARCH__
    return __umul64hi(a, b);
#else
    return (uint64_t)(((unsigned __int128)a * b) >> 64);
#endif
}

// rng.py:26-31
PW_HD uint64_t splitmix64(uint64_t x) {
    uint64_t z = x + 0x9E3779B97F4A7C15ULL;
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
    return z ^ (z >> 31);
}

// rng.py:34-39 derive_seed(seed, tag, qid, stage)
PW_HD uint64_t derive_seed3(uint64_t seed, uint64_t a, uint64_t b, uint64_t c) {
    uint64_t x = splitmix64(seed);
    x = splitmix64(x ^ a);
    x = splitmix64(x ^ b);
    x = splitmix64(x ^ c);
    return x;
}

// 128-bit LCG step: state = state * M + inc (mod 2^128)
PW_HD void pcg_step(Pcg64& g) {
    const uint64_t M_HI = 2549297995355413924ULL, M_LO = 4865540595714422341ULL;
    uint64_t lo = g.s_lo * M_LO;
    uint64_t hi = mulhi64(g.s_lo, M_LO) + g.s_lo * M_HI + g.s_hi * M_LO;
    uint64_t nlo = lo + g.i_lo;
    hi += g.i_hi + (nlo < lo ? 1u : 0u);
    g.s_lo = nlo;
    g.s_hi = hi;
}

PW_HD uint32_t ss_hashmix(uint32_t v, uint32_t& hc) {
    v ^= hc;
    hc *= 0x931e8875u;
    v *= hc;
    v ^= v >> 16;
    return v;
}
PW_HD uint32_t ss_mix(uint32_t x, uint32_t y) {
    uint32_t r = 0xca01f9ddu * x - 0x4973f715u * y;
    return r ^ (r >> 16);
}

// np.random.PCG64(seed64): SeedSequence(seed64).generate_state(4, uint64)
// then pcg_setseq_128_srandom_r(initstate, initseq).
PW_HD_COLD Pcg64 pcg64_from_seed(uint64_t seed64) {
    uint32_t e0 = (uint32_t)seed64, e1 = (uint32_t)(seed64 >> 32);
    int n_ent = (seed64 >> 32) ? 2 : 1;
    uint32_t pool[4];
    uint32_t hc = 0x43b0d7e5u;
    pool[0] = ss_hashmix(e0, hc);
    pool[1] = ss_hashmix(n_ent > 1 ? e1 : 0u, hc);
    pool[2] = ss_hashmix(0u, hc);
    pool[3] = ss_hashmix(0u, hc);
#pragma unroll
    for (int s = 0; s < 4; s++)
#pragma unroll
        for (int d = 0; d < 4; d++)
            if (s != d) pool[d] = ss_mix(pool[d], ss_hashmix(pool[s], hc));
    uint32_t st[8];
    uint32_t hb = 0x8b51f9ddu;
#pragma unroll
    for (int i = 0; i < 8; i++) {
        uint32_t v = pool[i & 3];
        v ^= hb;
        hb *= 0x58f38dedu;
        v *= hb;
        v ^= v >> 16;
        st[i] = v;
    }
    uint64_t w0 = (uint64_t)st[0] | ((uint64_t)st[1] << 32);
    uint64_t w1 = (uint64_t)st[2] | ((uint64_t)st[3] << 32);
    uint64_t w2 = (uint64_t)st[4] | ((uint64_t)st[5] << 32);
    uint64_t w3 = (uint64_t)st[6] | ((uint64_t)st[7] << 32);
    Pcg64 g;
    // inc = (initseq << 1) | 1 with initseq = w2:w3
    g.i_hi = (w2 << 1) | (w3 >> 63);
    g.i_lo = (w3 << 1) | 1u;
    g.s_hi = 0;
    g.s_lo = 0;
    pcg_step(g);
    // state += initstate (w0:w1)
    uint64_t lo = g.s_lo + w1;
    g.s_hi = g.s_hi + w0 + (lo < g.s_lo ? 1u : 0u);
    g.s_lo = lo;
    pcg_step(g);
    g.has32 = 0;
    g.u32 = 0;
    return g;
}

PW_HD uint64_t pcg_next64(Pcg64& g) {
    pcg_step(g);
    uint64_t x = g.s_hi ^ g.s_lo;
    unsigned rot = (unsigned)(g.s_hi >> 58);
    return (x >> rot) | (x << ((64u - rot) & 63u));
}

PW_HD uint32_t pcg_next32(Pcg64& g) {
    if (g.has32) {
        g.has32 = 0;
        return g.u32;
    }
    uint64_t nx = pcg_next64(g);
    g.has32 = 1;
    g.u32 = (uint32_t)(nx >> 32);
    return (uint32_t)nx;
}

// random_bounded_uint64(off=0, rng, use_masked=false) for rng < 2^32 - 1
// (shard sizes are < 2^31): Lemire with rejection, 32-bit draws.
PW_HD uint32_t bounded_u32(Pcg64& g, uint32_t rng) {
    if (rng == 0) return 0;
    if (rng == 0xFFFFFFFFu) return pcg_next32(g);
    uint32_t excl = rng + 1u;
    uint64_t m = (uint64_t)pcg_next32(g) * excl;
    uint32_t left = (uint32_t)m;
    if (left < excl) {
        uint32_t thr = (0xFFFFFFFFu - rng) % excl;
        while (left < thr) {
            m = (uint64_t)pcg_next32(g) * excl;
            left = (uint32_t)m;
        }
    }
    return (uint32_t)(m >> 32);
}

// random_interval(max) (Generator.shuffle / permutation)
PW_HD uint32_t random_interval(Pcg64& g, uint32_t max) {
    if (max == 0) return 0;
    uint32_t mask = max;
    mask |= mask >> 1; mask |= mask >> 2; mask |= mask >> 4; mask |= mask >> 8; mask |= mask >> 16;
    uint32_t v;
    while ((v = (pcg_next32(g) & mask)) > max) {
    }
    return v;
}

PW_HD uint64_t gen_mask64(uint64_t v) {
    uint64_t m = v;
    m |= m >> 1; m |= m >> 2; m |= m >> 4; m |= m >> 8; m |= m >> 16; m |= m >> 32;
    return m;
}

// Floyd branch of Generator.choice(pop, size, replace=False): `set` is
// (mask+1) uint32 slots (values < 2^31 so 0xFFFFFFFF is the empty marker),
// mask = gen_mask64(uint64(1.2 * size)).  out gets `size` values, then
// _shuffle_int(size, first=1).
PW_HD_COLD Pcg64 choice_floyd(Pcg64 g, uint32_t pop, uint32_t size, uint32_t* set, uint32_t mask,
                               int32_t* out) {
    for (uint32_t i = 0; i <= mask; i++) set[i] = 0xFFFFFFFFu;
    for (uint32_t j = pop - size; j < pop; j++) {
        uint32_t val = bounded_u32(g, j);
        uint32_t loc = val & mask;
        while (set[loc] != 0xFFFFFFFFu && set[loc] != val) loc = (loc + 1) & mask;
        if (set[loc] == 0xFFFFFFFFu) {
            set[loc] = val;
            out[j - pop + size] = (int32_t)val;
        } else {
            loc = j & mask;
            while (set[loc] != 0xFFFFFFFFu) loc = (loc + 1) & mask;
            set[loc] = j;
            out[j - pop + size] = (int32_t)j;
        }
    }
    for (int64_t i = (int64_t)size - 1; i >= 1; i--) {
        uint32_t jj = bounded_u32(g, (uint32_t)i);
        int32_t t = out[jj];
        out[jj] = out[i];
        out[i] = t;
    }
    return g;
}

// Tail-shuffle branch (pop > 10000 and size > pop // 50): partial
// Fisher-Yates of arange(pop) from the top, emulated with a sparse map of the
// touched positions (keys/vals, cap slots, power of 2, keys init 0xFFFFFFFF).
PW_HD uint32_t smap_get(const uint32_t* keys, const uint32_t* vals, uint32_t cmask, uint32_t k) {
    uint32_t h = (k * 0x9E3779B1u) & cmask;
    while (keys[h] != 0xFFFFFFFFu) {
        if (keys[h] == k) return vals[h];
        h = (h + 1) & cmask;
    }
    return k;
}
PW_HD void smap_set(uint32_t* keys, uint32_t* vals, uint32_t cmask, uint32_t k, uint32_t v) {
    uint32_t h = (k * 0x9E3779B1u) & cmask;
    while (keys[h] != 0xFFFFFFFFu && keys[h] != k) h = (h + 1) & cmask;
    keys[h] = k;
    vals[h] = v;
}
PW_HD_COLD Pcg64 choice_tail(Pcg64 g, uint32_t pop, uint32_t size, uint32_t* keys, uint32_t* vals,
                       uint32_t cmask, int32_t* out) {
    for (uint32_t i = 0; i <= cmask; i++) keys[i] = 0xFFFFFFFFu;
    uint32_t first = pop - size > 1 ? pop - size : 1;
    for (int64_t i = (int64_t)pop - 1; i >= (int64_t)first; i--) {
        uint32_t jj = bounded_u32(g, (uint32_t)i);
        uint32_t vi = smap_get(keys, vals, cmask, (uint32_t)i);
        uint32_t vj = smap_get(keys, vals, cmask, jj);
        smap_set(keys, vals, cmask, jj, vi);
        smap_set(keys, vals, cmask, (uint32_t)i, vj);
    }
    for (uint32_t t = 0; t < size; t++) out[t] = (int32_t)smap_get(keys, vals, cmask, pop - size + t);
    return g;
}

PW_HD bool choice_uses_tail(uint32_t pop, uint32_t size) { return pop > 10000u && size > pop / 50u; }

#ifdef __CUDACC__
// ---- warp-parallel Floyd choice (jump-ahead PCG64)
//
// state_k (after k steps of state = A * state + inc) = M_k * s + S_k * inc
// with M_k = A^k and S_k = A^(k-1) + ... + A + 1 (mod 2^128): one 128-bit
// multiply-add per lane replaces a chain of k dependent steps.  `jump` holds
// k = 1..kJumpMax as {M_hi, M_lo, S_hi, S_lo} (pw_abi.cu builds it).
constexpr int kJumpMax = 64;

__device__ __forceinline__ void mul_lo128(uint64_t ah, uint64_t al, uint64_t bh, uint64_t bl, uint64_t& rh,
                                          uint64_t& rl) {
    rl = al * bl;
    rh = __umul64hi(al, bl) + al * bh + ah * bl;
}

__device__ __forceinline__ uint64_t xsl_rr(uint64_t hi, uint64_t lo) {
    const uint64_t x = hi ^ lo;
    const unsigned rot = (unsigned)(hi >> 58);
    return (x >> rot) | (x << ((64u - rot) & 63u));
}

// Lemire draw of bounded_u32(g, rng) from one 32-bit value u: the result, or
// `rej` set when numpy would reject u and draw again.
__device__ __forceinline__ uint32_t lemire_once(uint32_t u, uint32_t rng, bool& rej) {
    const uint32_t excl = rng + 1u;
    const uint64_t m = (uint64_t)u * excl;
    const uint32_t left = (uint32_t)m;
    rej = left < excl && left < (0xFFFFFFFFu - rng) % excl;
    return (uint32_t)(m >> 32);
}

// Generator.choice(pop, size, replace=False) in its Floyd branch, all lanes
// of the warp, bit-exact with choice_floyd.  The 2*size-1 32-bit draws
// (size Floyd values, size-1 for _shuffle_int) come from jump-ahead outputs
// computed in parallel; the result is speculative on the two rare events
// that make numpy's draw sequence data-dependent -- a Lemire rejection (an
// extra draw) and a repeated Floyd value (the j substitution) -- and on
// either one the warp returns g unchanged but for has32 |= 2 (not handled:
// the caller runs the serial restatement).  Otherwise returns the advanced
// generator.  order = false skips the swaps of the final shuffle
// (callers that use the result as a set) but g still advances past its draws.
// buf: >= 128 u32 of warp-private scratch; requires 1 <= size <= 64,
// pop > size and the Floyd branch (!choice_uses_tail).
static __device__ __noinline__ Pcg64 choice_floyd_warp(Pcg64 g, uint32_t pop, uint32_t size, bool order, const uint64_t* jump,
                                  uint32_t* buf, int32_t* out) {
    const unsigned lane = threadIdx.x & 31u;
    const uint32_t K = 2u * size - 1u;               // 32-bit draws
    const uint32_t off = g.has32;                    // draw 0 is the buffered half
    const uint32_t n64 = (K - off + 1u) / 2u;        // 64-bit outputs consumed
    // outputs k = lane, lane + 32 -> buf as little-endian u64 (low half first)
    uint64_t fin_hi = 0, fin_lo = 0;
#pragma unroll
    for (int r = 0; r < 2; r++) {
        const uint32_t k = lane + 32u * r;
        if (k < n64) {
            const uint64_t* J = jump + 4 * (size_t)k;  // entry k+1
            uint64_t mh, ml, ah, al;
            mul_lo128(__ldg(J), __ldg(J + 1), g.s_hi, g.s_lo, mh, ml);
            mul_lo128(__ldg(J + 2), __ldg(J + 3), g.i_hi, g.i_lo, ah, al);
            const uint64_t lo = ml + al;
            const uint64_t hi = mh + ah + (lo < ml ? 1u : 0u);
            reinterpret_cast<uint64_t*>(buf)[k] = xsl_rr(hi, lo);
            if (k == n64 - 1u) {
                fin_hi = hi;
                fin_lo = lo;
            }
        }
    }
    __syncwarp();
    uint32_t v[4];
    bool bad = false;
#pragma unroll
    for (int r = 0; r < 4; r++) {
        const uint32_t t = lane + 32u * r;
        v[r] = 0;
        if (t < K) {
            const uint32_t u = (off && t == 0) ? g.u32 : buf[t - off];
            const uint32_t rng = t < size ? pop - size + t : 2u * size - 1u - t;
            bool rej;
            v[r] = lemire_once(u, rng, rej);
            bad |= rej;
        }
    }
    const uint32_t last_hi = n64 ? buf[2u * n64 - 1u] : g.u32;
    if (__any_sync(0xffffffffu, bad)) {
        g.has32 |= 2u;
        return g;
    }
    __syncwarp();
    // repeated Floyd values (numpy would substitute j): 128-slot hash in buf
    for (uint32_t i = lane; i < 128u; i += 32u) buf[i] = 0xFFFFFFFFu;
    __syncwarp();
    bool dup = false;
#pragma unroll
    for (int r = 0; r < 2; r++) {
        const uint32_t t = lane + 32u * r;
        if (t < size) {
            uint32_t h = (v[r] * 0x9E3779B1u) >> 25;
            for (;;) {
                const uint32_t o = atomicCAS(&buf[h], 0xFFFFFFFFu, v[r]);
                if (o == 0xFFFFFFFFu) break;
                if (o == v[r]) {
                    dup = true;
                    break;
                }
                h = (h + 1u) & 127u;
            }
        }
    }
    if (__any_sync(0xffffffffu, dup)) {
        g.has32 |= 2u;
        return g;
    }
    __syncwarp();
#pragma unroll
    for (int r = 0; r < 2; r++) {
        const uint32_t t = lane + 32u * r;
        if (t < size) out[t] = (int32_t)v[r];
    }
    if (order) {
        // _shuffle_int(size, 1): swap out[i] with out[draw] for i = size-1..1
#pragma unroll
        for (int r = 0; r < 4; r++) {
            const uint32_t t = lane + 32u * r;
            if (t >= size && t < K) buf[t - size] = v[r];
        }
        __syncwarp();
        if (lane == 0)
            for (uint32_t i = size - 1u; i >= 1u; i--) {
                const uint32_t jj = buf[size - 1u - i];
                const int32_t x = out[jj];
                out[jj] = out[i];
                out[i] = x;
            }
    }
    __syncwarp();
    // generator after the last consumed draw (broadcast from its lane)
    if (n64) {
        const int src = (int)((n64 - 1u) & 31u);
        g.s_hi = __shfl_sync(0xffffffffu, fin_hi, src);
        g.s_lo = __shfl_sync(0xffffffffu, fin_lo, src);
        g.u32 = last_hi;
    }
    g.has32 = ((K - off) & 1u) ? 1u : 0u;
    return g;
}
#endif

// Generator.permutation(n) into out[n]
PW_HD_COLD Pcg64 permutation(Pcg64 g, uint32_t n, int32_t* out) {
    for (uint32_t i = 0; i < n; i++) out[i] = (int32_t)i;
    for (int64_t i = (int64_t)n - 1; i >= 1; i--) {
        uint32_t jj = random_interval(g, (uint32_t)i);
        int32_t t = out[jj];
        out[jj] = out[i];
        out[i] = t;
    }
    return g;
}

}  // namespace pw
