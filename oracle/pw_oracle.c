/* pw_oracle.c -- CPU restatement of the reference search path.
 * TEST INFRASTRUCTURE (parity checker / CPU baseline), never the product.
 * See pw_oracle.h for the scope.  Compile with -ffp-contract=off so float
 * arithmetic is the plain IEEE round-to-nearest sequence numpy performs. */
#include "pw_oracle.h"

#include <math.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

typedef unsigned __int128 u128;

static __thread char g_err[256];
const char* orc_last_error(void) { return g_err; }
static int fail(const char* msg) {
    snprintf(g_err, sizeof g_err, "%s", msg);
    return -1;
}

/* ---------------- rng.py:26-39 ---------------- */
uint64_t orc_splitmix64(uint64_t x) {
    uint64_t z = x + 0x9E3779B97F4A7C15ULL;
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
    return z ^ (z >> 31);
}

uint64_t orc_derive_seed(uint64_t seed, const uint64_t* parts, int n_parts) {
    uint64_t x = orc_splitmix64(seed);
    for (int i = 0; i < n_parts; i++) x = orc_splitmix64(x ^ parts[i]);
    return x;
}

/* ---------------- numpy SeedSequence (bit_generator.pyx) ---------------- */
#define SS_INIT_A 0x43b0d7e5u
#define SS_MULT_A 0x931e8875u
#define SS_INIT_B 0x8b51f9ddu
#define SS_MULT_B 0x58f38dedu
#define SS_MIX_L 0xca01f9ddu
#define SS_MIX_R 0x4973f715u

static uint32_t ss_hashmix(uint32_t v, uint32_t* hc) {
    v ^= *hc;
    *hc *= SS_MULT_A;
    v *= *hc;
    v ^= v >> 16;
    return v;
}
static uint32_t ss_mix(uint32_t x, uint32_t y) {
    uint32_t r = SS_MIX_L * x - SS_MIX_R * y;
    r ^= r >> 16;
    return r;
}

/* PCG64(seed64): SeedSequence(seed64).generate_state(4, uint64) then
 * pcg_setseq_128_srandom_r(initstate, initseq) (numpy pcg64.c). */
void orc_pcg64_seed(uint64_t seed64, orc_pcg64* g) {
    uint32_t ent[2];
    int n_ent;
    if (seed64 == 0) { ent[0] = 0; n_ent = 1; }
    else if ((seed64 >> 32) == 0) { ent[0] = (uint32_t)seed64; n_ent = 1; }
    else { ent[0] = (uint32_t)seed64; ent[1] = (uint32_t)(seed64 >> 32); n_ent = 2; }
    uint32_t pool[4];
    uint32_t hc = SS_INIT_A;
    for (int i = 0; i < 4; i++) pool[i] = ss_hashmix(i < n_ent ? ent[i] : 0u, &hc);
    for (int s = 0; s < 4; s++)
        for (int d = 0; d < 4; d++)
            if (s != d) pool[d] = ss_mix(pool[d], ss_hashmix(pool[s], &hc));
    uint32_t st[8];
    uint32_t hb = SS_INIT_B;
    for (int i = 0; i < 8; i++) {
        uint32_t v = pool[i % 4];
        v ^= hb;
        hb *= SS_MULT_B;
        v *= hb;
        v ^= v >> 16;
        st[i] = v;
    }
    uint64_t w[4];
    for (int i = 0; i < 4; i++) w[i] = (uint64_t)st[2 * i] | ((uint64_t)st[2 * i + 1] << 32);
    u128 initstate = ((u128)w[0] << 64) | w[1];
    u128 initseq = ((u128)w[2] << 64) | w[3];
    const u128 mult = ((u128)2549297995355413924ULL << 64) | 4865540595714422341ULL;
    u128 inc = (initseq << 1) | 1;
    u128 state = 0;
    state = state * mult + inc;
    state += initstate;
    state = state * mult + inc;
    g->state_hi = (uint64_t)(state >> 64);
    g->state_lo = (uint64_t)state;
    g->inc_hi = (uint64_t)(inc >> 64);
    g->inc_lo = (uint64_t)inc;
    g->has_uint32 = 0;
    g->uinteger = 0;
}

uint64_t orc_pcg64_next64(orc_pcg64* g) {
    const u128 mult = ((u128)2549297995355413924ULL << 64) | 4865540595714422341ULL;
    u128 state = ((u128)g->state_hi << 64) | g->state_lo;
    u128 inc = ((u128)g->inc_hi << 64) | g->inc_lo;
    state = state * mult + inc;
    g->state_hi = (uint64_t)(state >> 64);
    g->state_lo = (uint64_t)state;
    uint64_t x = g->state_hi ^ g->state_lo;
    unsigned rot = (unsigned)(g->state_hi >> 58);
    return (x >> rot) | (x << ((64 - rot) & 63));
}

uint32_t orc_pcg64_next32(orc_pcg64* g) {
    if (g->has_uint32) {
        g->has_uint32 = 0;
        return g->uinteger;
    }
    uint64_t nx = orc_pcg64_next64(g);
    g->has_uint32 = 1;
    g->uinteger = (uint32_t)(nx >> 32);
    return (uint32_t)nx;
}

/* random_bounded_uint64(off=0, rng, mask=0, use_masked=0) (distributions.c) */
static uint64_t bounded_u64(orc_pcg64* g, uint64_t rng) {
    if (rng == 0) return 0;
    if (rng <= 0xFFFFFFFFULL) {
        if (rng == 0xFFFFFFFFULL) return orc_pcg64_next32(g);
        uint32_t rng_excl = (uint32_t)rng + 1u;
        uint64_t m = (uint64_t)orc_pcg64_next32(g) * rng_excl;
        uint32_t left = (uint32_t)m;
        if (left < rng_excl) {
            uint32_t thr = (uint32_t)(0xFFFFFFFFu - (uint32_t)rng) % rng_excl;
            while (left < thr) {
                m = (uint64_t)orc_pcg64_next32(g) * rng_excl;
                left = (uint32_t)m;
            }
        }
        return m >> 32;
    }
    if (rng == 0xFFFFFFFFFFFFFFFFULL) return orc_pcg64_next64(g);
    /* bounded_lemire_uint64 */
    uint64_t rng_excl = rng + 1;
    u128 m = (u128)orc_pcg64_next64(g) * rng_excl;
    uint64_t left = (uint64_t)m;
    if (left < rng_excl) {
        uint64_t thr = (0xFFFFFFFFFFFFFFFFULL - rng) % rng_excl;
        while (left < thr) {
            m = (u128)orc_pcg64_next64(g) * rng_excl;
            left = (uint64_t)m;
        }
    }
    return (uint64_t)(m >> 64);
}

/* random_interval (distributions.c), used by Generator.shuffle/permutation */
static uint64_t random_interval(orc_pcg64* g, uint64_t max) {
    if (max == 0) return 0;
    uint64_t mask = max;
    mask |= mask >> 1; mask |= mask >> 2; mask |= mask >> 4;
    mask |= mask >> 8; mask |= mask >> 16; mask |= mask >> 32;
    uint64_t v;
    if (max <= 0xFFFFFFFFULL) {
        while ((v = (orc_pcg64_next32(g) & mask)) > max) {}
    } else {
        while ((v = (orc_pcg64_next64(g) & mask)) > max) {}
    }
    return v;
}

static void shuffle_int(orc_pcg64* g, int64_t n, int64_t first, int64_t* data) {
    for (int64_t i = n - 1; i >= first; i--) {
        int64_t j = (int64_t)bounded_u64(g, (uint64_t)i);
        int64_t t = data[j];
        data[j] = data[i];
        data[i] = t;
    }
}

static uint64_t gen_mask(uint64_t v) {
    uint64_t m = v;
    m |= m >> 1; m |= m >> 2; m |= m >> 4; m |= m >> 8; m |= m >> 16; m |= m >> 32;
    return m;
}

/* sparse map for the tail-shuffle branch (positions -> values) */
typedef struct { int64_t* keys; int64_t* vals; uint64_t mask; } smap;
static int64_t smap_get(smap* s, int64_t k) {
    uint64_t h = ((uint64_t)k * 0x9E3779B97F4A7C15ULL) & s->mask;
    while (s->keys[h] != -1) {
        if (s->keys[h] == k) return s->vals[h];
        h = (h + 1) & s->mask;
    }
    return k;
}
static void smap_set(smap* s, int64_t k, int64_t v) {
    uint64_t h = ((uint64_t)k * 0x9E3779B97F4A7C15ULL) & s->mask;
    while (s->keys[h] != -1 && s->keys[h] != k) h = (h + 1) & s->mask;
    s->keys[h] = k;
    s->vals[h] = v;
}

/* Generator.choice(pop, size, replace=False, shuffle=True) (_generator.pyx). */
int orc_choice(orc_pcg64* g, int64_t pop, int64_t size, int64_t* out) {
    if (size > pop || size < 0) return fail("Cannot take a larger sample than population when replace is False");
    if (size == 0) return 0;
    if (pop > 10000 && size > pop / 50) {
        /* tail shuffle of arange(pop): _shuffle_int(pop, max(pop-size,1)); idx[pop-size:] */
        int64_t first = pop - size > 1 ? pop - size : 1;
        uint64_t cap = gen_mask((uint64_t)(4 * size + 8)) + 1;
        smap s;
        s.keys = (int64_t*)malloc(cap * sizeof(int64_t));
        s.vals = (int64_t*)malloc(cap * sizeof(int64_t));
        s.mask = cap - 1;
        for (uint64_t i = 0; i < cap; i++) s.keys[i] = -1;
        for (int64_t i = pop - 1; i >= first; i--) {
            int64_t j = (int64_t)bounded_u64(g, (uint64_t)i);
            int64_t vi = smap_get(&s, i), vj = smap_get(&s, j);
            smap_set(&s, j, vi);
            smap_set(&s, i, vj);
        }
        for (int64_t t = 0; t < size; t++) out[t] = smap_get(&s, pop - size + t);
        free(s.keys);
        free(s.vals);
        return 0;
    }
    /* Floyd's algorithm with a linear-probing set, then shuffle */
    uint64_t set_size = (uint64_t)(1.2 * (double)size);
    uint64_t mask = gen_mask(set_size);
    uint64_t* hs = (uint64_t*)malloc((mask + 1) * sizeof(uint64_t));
    for (uint64_t i = 0; i <= mask; i++) hs[i] = ~0ULL;
    for (int64_t j = pop - size; j < pop; j++) {
        uint64_t val = bounded_u64(g, (uint64_t)j);
        uint64_t loc = val & mask;
        while (hs[loc] != ~0ULL && hs[loc] != val) loc = (loc + 1) & mask;
        if (hs[loc] == ~0ULL) {
            hs[loc] = val;
            out[j - pop + size] = (int64_t)val;
        } else {
            loc = (uint64_t)j & mask;
            while (hs[loc] != ~0ULL) loc = (loc + 1) & mask;
            hs[loc] = (uint64_t)j;
            out[j - pop + size] = j;
        }
    }
    free(hs);
    shuffle_int(g, size, 1, out);
    return 0;
}

/* Generator.permutation(n) = shuffle(arange(n)) with random_interval. */
void orc_permutation(orc_pcg64* g, int64_t n, int64_t* out) {
    for (int64_t i = 0; i < n; i++) out[i] = i;
    for (int64_t i = n - 1; i >= 1; i--) {
        int64_t j = (int64_t)random_interval(g, (uint64_t)i);
        int64_t t = out[j];
        out[j] = out[i];
        out[i] = t;
    }
}

/* ---------------- data.py:70-79 squared_l2 ---------------- */
/* numpy pairwise_sum for float32 (loops_utils.h.src), PW_BLOCKSIZE 128 */
static float pairwise_sum(const float* a, int64_t n) {
    if (n < 8) {
        float res = 0.f;
        for (int64_t i = 0; i < n; i++) res += a[i];
        return res;
    }
    if (n <= 128) {
        float r[8];
        for (int t = 0; t < 8; t++) r[t] = a[t];
        int64_t i;
        for (i = 8; i < n - (n % 8); i += 8)
            for (int t = 0; t < 8; t++) r[t] += a[i + t];
        float res = ((r[0] + r[1]) + (r[2] + r[3])) + ((r[4] + r[5]) + (r[6] + r[7]));
        for (; i < n; i++) res += a[i];
        return res;
    }
    int64_t n2 = n / 2;
    n2 -= n2 % 8;
    return pairwise_sum(a, n2) + pairwise_sum(a + n2, n - n2);
}

static float sq_l2_row(const float* x, const float* q, int32_t d, float* tmp) {
    for (int32_t t = 0; t < d; t++) {
        float df = x[t] - q[t];
        tmp[t] = df * df;
    }
    return pairwise_sum(tmp, d);
}

/* Inner-product distance (BASELINE C5; NOT in the reference -- parity
 * unpinned, restated here so the device metric has a CPU checker):
 * -(pairwise_sum(x * q)) with the same float32 pairwise order, no FMA. */
static float neg_ip_row(const float* x, const float* q, int32_t d, float* tmp) {
    for (int32_t t = 0; t < d; t++) tmp[t] = x[t] * q[t];
    return -pairwise_sum(tmp, d);
}

static float metric_row(int32_t metric, const float* x, const float* q, int32_t d, float* tmp) {
    return metric == 1 ? neg_ip_row(x, q, d, tmp) : sq_l2_row(x, q, d, tmp);
}

void orc_squared_l2(const float* points, int64_t rows, int32_t d, const float* q, float* out) {
    float* tmp = (float*)malloc(sizeof(float) * (size_t)(d > 0 ? d : 1));
    for (int64_t r = 0; r < rows; r++) out[r] = sq_l2_row(points + r * d, q, d, tmp);
    free(tmp);
}

/* ---------------- direction.py ---------------- */
static int32_t words_per_vector(int32_t d) { return (d + 31) / 32; }

/* direction.py:28-38 pack_sign_bits (little-endian bit order within u32) */
void orc_pack_sign_bits(const uint8_t* bits, int64_t rows, int32_t d, uint32_t* out) {
    int32_t w = words_per_vector(d);
    for (int64_t r = 0; r < rows; r++) {
        for (int32_t k = 0; k < w; k++) out[r * w + k] = 0;
        for (int32_t t = 0; t < d; t++)
            if (bits[r * d + t]) out[r * w + t / 32] |= 1u << (t % 32);
    }
}

/* direction.py:72-76 */
int32_t orc_keep_count(int32_t j, double discard_ratio) {
    int32_t v = (int32_t)((1.0 - discard_ratio) * (double)j + 0.5);
    return v > 1 ? v : 1;
}

/* direction.py:90-100 */
int32_t orc_in_cooldown(int32_t iteration, int32_t max_iter, double cooldown_ratio) {
    int32_t start = max_iter - (int32_t)floor(cooldown_ratio * (double)max_iter + 1e-9);
    return iteration >= start;
}

/* ---------------- search.py ---------------- */
typedef struct { float d; int32_t id; } pair_t;

static int pair_cmp(const void* a, const void* b) {
    const pair_t* x = (const pair_t*)a;
    const pair_t* y = (const pair_t*)b;
    if (x->d < y->d) return -1;
    if (x->d > y->d) return 1;
    return (x->id > y->id) - (x->id < y->id);
}

/* growable open-addressing set of non-negative int64 (the visited set of
 * search.py:167, kept sparse so huge shards cost nothing per search) */
typedef struct { int64_t* slots; uint64_t mask; int64_t count; } iset;
static void iset_init(iset* s, uint64_t cap) {
    uint64_t c = 16;
    while (c < cap) c <<= 1;
    s->slots = (int64_t*)malloc(c * sizeof(int64_t));
    for (uint64_t i = 0; i < c; i++) s->slots[i] = -1;
    s->mask = c - 1;
    s->count = 0;
}
static void iset_free(iset* s) { free(s->slots); }
static uint64_t ihash(int64_t k) { return (uint64_t)k * 0x9E3779B97F4A7C15ULL >> 17; }
static int iset_has(const iset* s, int64_t k) {
    uint64_t h = ihash(k) & s->mask;
    while (s->slots[h] != -1) {
        if (s->slots[h] == k) return 1;
        h = (h + 1) & s->mask;
    }
    return 0;
}
static void iset_grow(iset* s);
static int iset_add(iset* s, int64_t k) { /* 1 if newly added */
    if ((uint64_t)(s->count + 1) * 2 > s->mask + 1) iset_grow(s);
    uint64_t h = ihash(k) & s->mask;
    while (s->slots[h] != -1) {
        if (s->slots[h] == k) return 0;
        h = (h + 1) & s->mask;
    }
    s->slots[h] = k;
    s->count++;
    return 1;
}
static void iset_grow(iset* s) {
    iset n;
    iset_init(&n, (s->mask + 1) * 2);
    for (uint64_t i = 0; i <= s->mask; i++)
        if (s->slots[i] != -1) iset_add(&n, s->slots[i]);
    iset_free(s);
    *s = n;
}

typedef struct {
    int32_t l;
    int32_t qlen;
    pair_t* q;      /* queue sorted by (dist, id) */
    uint8_t* qexp;  /* expanded flag per queue entry */
    pair_t* tmpq;
    uint8_t* tmpe;
    pair_t* inc;    /* incoming buffer */
} queue_t;

/* search.py:170-190 merge_and_sort: new ids are never queued nor repeated
 * (batch is unique and queued ids are visited), so the merge reduces to
 * sorted(queue + sorted(incoming))[:l]. */
static int32_t merge_and_sort(queue_t* Q, pair_t* inc, int32_t n_inc) {
    qsort(inc, (size_t)n_inc, sizeof(pair_t), pair_cmp);
    int32_t a = 0, b = 0, o = 0, inserted = 0;
    while (o < Q->l && (a < Q->qlen || b < n_inc)) {
        int take_q;
        if (a >= Q->qlen) take_q = 0;
        else if (b >= n_inc) take_q = 1;
        else take_q = pair_cmp(&Q->q[a], &inc[b]) < 0;
        if (take_q) {
            Q->tmpq[o] = Q->q[a];
            Q->tmpe[o] = Q->qexp[a];
            a++;
        } else {
            Q->tmpq[o] = inc[b];
            Q->tmpe[o] = 0;
            b++;
            inserted++;
        }
        o++;
    }
    pair_t* t = Q->q; Q->q = Q->tmpq; Q->tmpq = t;
    uint8_t* te = Q->qexp; Q->qexp = Q->tmpe; Q->tmpe = te;
    Q->qlen = o;
    return inserted;
}

int orc_search(const orc_graph* ctx, const float* query, const orc_params* p,
               const int64_t* seeds, int32_t n_seeds, orc_pcg64* rng,
               int32_t* out_ids, float* out_dists, int32_t* out_local,
               orc_result* res, int32_t* visit_log, int64_t visit_cap) {
    const int64_t n = ctx->n;
    const int32_t d = ctx->d, j = ctx->j;
    if (n == 0) return fail("empty graph");
    if (p->selection == 1 && p->discard_ratio > 0.0 && ctx->direction == NULL)
        return fail("direction table required for direction-guided selection");
    for (int32_t i = 0; i < n_seeds; i++)
        if (seeds[i] < 0 || seeds[i] >= n) {
            snprintf(g_err, sizeof g_err, "seed %lld outside shard of %lld nodes",
                     (long long)seeds[i], (long long)n);
            return -1;
        }
    memset(res, 0, sizeof *res);
    orc_counters* c = &res->c;
    /* search.py:289 */
    int64_t cap = p->buffer_cap ? p->buffer_cap : ((int64_t)p->m > (int64_t)p->r * j ? p->m : (int64_t)p->r * j);
    const int64_t want = p->m < n ? p->m : n;
    const int fill_random = p->seed_mode == 1 || n_seeds == 0;

    /* search.py:207-227 _initial_batch */
    int64_t bcap = (int64_t)p->r * (j > 0 ? j : 1);
    if (bcap < want) bcap = want;
    int64_t* batch = (int64_t*)malloc(sizeof(int64_t) * (size_t)(bcap + 1));
    int64_t nb = 0;
    {
        iset taken;
        iset_init(&taken, 2 * (uint64_t)(n_seeds + want) + 16);
        for (int32_t i = 0; i < n_seeds && nb < want; i++)
            if (iset_add(&taken, seeds[i])) batch[nb++] = seeds[i];
        if (fill_random && nb < want) {
            int64_t* ch = (int64_t*)malloc(sizeof(int64_t) * (size_t)want);
            if (orc_choice(rng, n, want, ch)) { free(ch); iset_free(&taken); free(batch); return -1; }
            for (int64_t i = 0; i < want && nb < want; i++)
                if (!iset_has(&taken, ch[i])) batch[nb++] = ch[i];
            free(ch);
        }
        iset_free(&taken);
    }

    iset visited;
    iset_init(&visited, 4096);
    queue_t Q;
    Q.l = p->l;
    Q.qlen = 0;
    Q.q = (pair_t*)malloc(sizeof(pair_t) * (size_t)p->l);
    Q.tmpq = (pair_t*)malloc(sizeof(pair_t) * (size_t)p->l);
    Q.qexp = (uint8_t*)malloc((size_t)p->l);
    Q.tmpe = (uint8_t*)malloc((size_t)p->l);
    pair_t* inc = (pair_t*)malloc(sizeof(pair_t) * (size_t)(bcap + 1));
    float* tmp = (float*)malloc(sizeof(float) * (size_t)(d > 0 ? d : 1));
    int32_t W = words_per_vector(d);
    uint32_t* qbits = (uint32_t*)malloc(sizeof(uint32_t) * (size_t)(W > 0 ? W : 1));
    int64_t* rows = (int64_t*)malloc(sizeof(int64_t) * (size_t)((int64_t)p->r * (j > 0 ? j : 1) + 1));
    int32_t* cnt = (int32_t*)malloc(sizeof(int32_t) * (size_t)(j > 0 ? j : 1));
    int64_t* slots = (int64_t*)malloc(sizeof(int64_t) * (size_t)(j > 0 ? j : 1));
    int32_t* parents = (int32_t*)malloc(sizeof(int32_t) * (size_t)p->r);

    int converged = 0;
    for (int32_t it = 0; it < p->max_iter; it++) {
        c->iterations++;
        /* Step 3 (search.py:300-309) */
        int32_t n_new = 0;
        for (int64_t b = 0; b < nb; b++) {
            int64_t v = batch[b];
            if (iset_has(&visited, v)) continue;
            inc[n_new].d = metric_row(p->metric, ctx->vectors + v * d, query, d, tmp);
            inc[n_new].id = (int32_t)v;
            n_new++;
        }
        int32_t inserted = 0;
        if (n_new) {
            for (int32_t t = 0; t < n_new; t++) {
                iset_add(&visited, inc[t].id);
                if (p->log_visits && visit_log && res->n_visited < visit_cap)
                    visit_log[res->n_visited++] = inc[t].id;
            }
            c->distance_computations += n_new;
            inserted = merge_and_sort(&Q, inc, n_new);
            c->inserted_total += inserted;
        }
        if (inserted == 0) { converged = 1; break; }
        if (it == p->max_iter - 1) break;
        /* Step 4 (search.py:316-321) select_parents / mark_expanded */
        int32_t np_ = 0;
        for (int32_t t = 0; t < Q.qlen && np_ < p->r; t++)
            if (!Q.qexp[t]) { parents[np_++] = Q.q[t].id; Q.qexp[t] = 1; }
        if (np_ == 0) { converged = 1; break; }
        c->nodes_expanded += np_;
        /* _expand (search.py:235-266) */
        int prune = p->selection != 0 && p->discard_ratio > 0.0 &&
                    !orc_in_cooldown(it, p->max_iter, p->cooldown_ratio);
        int32_t nsel = j;
        int64_t nrows = 0;
        if (prune) {
            int32_t n_keep = orc_keep_count(j, p->discard_ratio);
            nsel = n_keep < j ? n_keep : j;
            for (int32_t pi = 0; pi < np_; pi++) {
                const int32_t* arow = ctx->adj + (int64_t)parents[pi] * j;
                if (p->selection == 1) {
                    const float* xp = ctx->vectors + (int64_t)parents[pi] * d;
                    for (int32_t w = 0; w < W; w++) qbits[w] = 0;
                    for (int32_t t = 0; t < d; t++)
                        if (query[t] >= xp[t]) qbits[t / 32] |= 1u << (t % 32);
                    const uint32_t* dr = ctx->direction + (int64_t)parents[pi] * j * W;
                    for (int32_t s = 0; s < j; s++) {
                        int32_t diff = 0;
                        for (int32_t w = 0; w < W; w++) diff += __builtin_popcount(dr[s * W + w] ^ qbits[w]);
                        cnt[s] = d - diff;
                    }
                    /* stable argsort(-counts)[:n_keep]: count desc, slot asc */
                    for (int32_t s = 0; s < j; s++) {
                        int32_t rank = 0;
                        for (int32_t o = 0; o < j; o++)
                            if (cnt[o] > cnt[s] || (cnt[o] == cnt[s] && o < s)) rank++;
                        slots[rank] = s;
                    }
                } else {
                    orc_permutation(rng, j, slots);
                }
                for (int32_t s = 0; s < nsel; s++) rows[nrows++] = arow[slots[s]];
            }
            c->dgs_skipped += (int64_t)np_ * (j - n_keep);
        } else {
            for (int32_t pi = 0; pi < np_; pi++) {
                const int32_t* arow = ctx->adj + (int64_t)parents[pi] * j;
                for (int32_t s = 0; s < j; s++) rows[nrows++] = arow[s];
            }
        }
        (void)nsel;
        /* _ordered_unique(rows)[:cap] */
        nb = 0;
        {
            iset seen;
            iset_init(&seen, 2 * (uint64_t)nrows + 16);
            for (int64_t t = 0; t < nrows && nb < cap; t++)
                if (iset_add(&seen, rows[t])) batch[nb++] = rows[t];
            iset_free(&seen);
        }
        c->total_visits += nb;
    }

    /* search.py:323-335 */
    int32_t nk = Q.qlen < p->k ? Q.qlen : p->k;
    for (int32_t t = 0; t < nk; t++) {
        out_local[t] = Q.q[t].id;
        out_ids[t] = ctx->global_ids[Q.q[t].id];
        out_dists[t] = p->metric == 1 ? Q.q[t].d : sqrtf(Q.q[t].d);  /* search.py:325 (L2) */
    }
    res->n_out = nk;
    res->converged = converged;
    res->retained = Q.qlen;

    iset_free(&visited);
    free(Q.q); free(Q.tmpq); free(Q.qexp); free(Q.tmpe);
    free(inc); free(tmp); free(qbits); free(rows); free(cnt); free(slots); free(parents);
    free(batch);
    return 0;
}

/* pipeline.py:158-184 */
int orc_ghost_stage(const orc_shard* sh, const float* query, const orc_params* p,
                    orc_pcg64* rng, int32_t* entry, orc_counters* c) {
    if (!sh->has_ghost) return fail("ghost index absent for this shard");
    orc_params gp = *p;
    gp.k = 1;
    gp.max_iter = p->ghost_max_iter;
    gp.selection = 0;
    gp.discard_ratio = 0.0;
    gp.ghost_enabled = 0;
    gp.log_visits = 0;
    gp.buffer_cap = 0;
    int32_t id, loc;
    float dist;
    orc_result r;
    if (orc_search(&sh->ghost, query, &gp, NULL, 0, rng, &id, &dist, &loc, &r, NULL, 0)) return -1;
    *entry = id;
    *c = r.c;
    return 0;
}

/* pipeline.py:187-196: lexsort((ids, dists)) over valid entries */
static int pair_cmp_sqrt(const void* a, const void* b) { return pair_cmp(a, b); }
int orc_reduce_topk(const int32_t* ids, const float* dists, int64_t n, int32_t k,
                    int32_t* out_ids, float* out_dists) {
    pair_t* v = (pair_t*)malloc(sizeof(pair_t) * (size_t)(n > 0 ? n : 1));
    int64_t m = 0;
    for (int64_t i = 0; i < n; i++)
        if (ids[i] >= 0) { v[m].d = dists[i]; v[m].id = ids[i]; m++; }
    if (m == 0) { free(v); return fail("cannot reduce empty candidate lists"); }
    qsort(v, (size_t)m, sizeof(pair_t), pair_cmp_sqrt);
    int32_t o = (int32_t)(m < k ? m : k);
    for (int32_t t = 0; t < o; t++) { out_ids[t] = v[t].id; out_dists[t] = v[t].d; }
    free(v);
    return o;
}

/* pipeline.py:213-247 _Run.search_one, writing into the stage arrays. */
typedef struct {
    const orc_shard* shards;
    int32_t n_shards;
    const float* queries;
    int64_t q;
    int32_t d;
    const orc_params* p;
    int32_t* shard_ids;
    float* shard_dists;
    int32_t* s32;
    int64_t* s64;
} run_t;

#define TAG_SEARCH 4
#define TAG_GHOST_SEARCH 5

/* stage >= 1 parameters (opt-in late budgets; the reference uses p itself) */
static orc_params stage_params(const orc_params* p, int32_t stage) {
    orc_params q = *p;
    if (stage > 0 && p->late_l > 0) q.l = p->late_l;
    if (stage > 0 && p->late_max_iter > 0) q.max_iter = p->late_max_iter;
    return q;
}

static int32_t fwd_count(const orc_params* p) { return p->forward_count > 0 ? p->forward_count : 1; }

static int search_one(run_t* R, int64_t qid, int32_t shard, int32_t stage, int has_seed,
                      const int64_t* entry_in, int32_t* top_local) {
    const orc_params ps = stage_params(R->p, stage);
    const orc_params* p = &ps;
    const int32_t F = fwd_count(R->p);
    const orc_shard* sh = &R->shards[shard];
    const float* query = R->queries + qid * R->d;
    const int64_t Q = R->q;
    int32_t* it32 = R->s32 + (int64_t)stage * 4 * Q;
    int64_t* it64 = R->s64 + (int64_t)stage * 4 * Q;
    int64_t seeds_buf[8 * (1 + 512)];
    int64_t* seeds = seeds_buf;
    int32_t n_seeds = 0;
    if (has_seed)
        for (int32_t f = 0; f < F; f++) seeds[n_seeds++] = entry_in[f];
    if (p->ghost_enabled && !has_seed && sh->has_ghost) {
        uint64_t parts[3] = {TAG_GHOST_SEARCH, (uint64_t)qid, (uint64_t)stage};
        orc_pcg64 g;
        orc_pcg64_seed(orc_derive_seed(p->seed, parts, 3), &g);
        int32_t e;
        orc_counters gc;
        if (orc_ghost_stage(sh, query, p, &g, &e, &gc)) return -1;
        seeds[n_seeds++] = e;
        it32[1 * Q + qid] += (int32_t)gc.iterations;
        it64[0 * Q + qid] += gc.distance_computations;
        it64[1 * Q + qid] += gc.total_visits;
    }
    if (n_seeds && p->seed_mode == 0) {
        /* [e] + adj[e] (pipeline.py:229-231); F entries: [e_0..e_F-1] + adj[e_0] + ... */
        int32_t j = sh->main.j;
        int64_t e[8];
        const int32_t ne = n_seeds;
        for (int32_t f = 0; f < ne; f++) e[f] = seeds[f];
        if ((int64_t)ne * (1 + j) > 8 * (1 + 512)) seeds = (int64_t*)malloc(sizeof(int64_t) * (size_t)(ne * (1 + j)));
        for (int32_t f = 0; f < ne; f++) seeds[f] = e[f];
        for (int32_t f = 0; f < ne; f++)
            for (int32_t t = 0; t < j; t++) seeds[ne + f * j + t] = sh->main.adj[e[f] * j + t];
        n_seeds = ne * (1 + j);
    }
    uint64_t parts[3] = {TAG_SEARCH, (uint64_t)qid, (uint64_t)stage};
    orc_pcg64 g;
    orc_pcg64_seed(orc_derive_seed(p->seed, parts, 3), &g);
    int32_t k = p->k;
    int32_t ids[4096], loc[4096];
    float dists[4096];
    int32_t* pid = ids; int32_t* ploc = loc; float* pd = dists;
    if (k > 4096) {
        pid = (int32_t*)malloc(sizeof(int32_t) * k);
        ploc = (int32_t*)malloc(sizeof(int32_t) * k);
        pd = (float*)malloc(sizeof(float) * k);
    }
    orc_result r;
    int rc = orc_search(&sh->main, query, p, seeds, n_seeds, &g, pid, pd, ploc, &r, NULL, 0);
    if (seeds != seeds_buf) free(seeds);
    if (rc == 0) {
        it32[0 * Q + qid] += (int32_t)r.c.iterations;
        it64[0 * Q + qid] += r.c.distance_computations;
        it64[1 * Q + qid] += r.c.total_visits;
        it64[2 * Q + qid] += r.c.inserted_total;
        it32[2 * Q + qid] += r.retained;
        it64[3 * Q + qid] += r.c.dgs_skipped;
        it32[3 * Q + qid] = r.converged;
        int64_t base = (qid * R->n_shards + shard) * (int64_t)k;
        for (int32_t t = 0; t < r.n_out; t++) {
            R->shard_ids[base + t] = pid[t];
            R->shard_dists[base + t] = pd[t];
        }
        /* top-F local ids (short lists repeat their last entry) */
        for (int32_t f = 0; f < F; f++) top_local[f] = r.n_out ? ploc[f < r.n_out ? f : r.n_out - 1] : -1;
    }
    if (pid != ids) { free(pid); free(ploc); free(pd); }
    return rc;
}

int orc_run_stage(const orc_shard* shard, const float* queries, int64_t q_total, int64_t q0,
                  int64_t n, const orc_params* p, int32_t stage, const int32_t* entries_in,
                  int32_t* forward_out, int32_t* shard_ids, float* shard_dists, int32_t n_cols,
                  int32_t col, int32_t* stats_i32, int64_t* stats_i64, int32_t threads) {
    /* the per-query dispatcher indexes shards[shard]; present this one shard at
     * index `col` of a virtual array so search_one's output column is col */
    orc_shard* arr = (orc_shard*)calloc((size_t)n_cols, sizeof(orc_shard));
    arr[col] = *shard;
    /* search_one writes stats at [stage*4*Q]: point the bases so stage maps to row 0 */
    run_t R = {arr, n_cols, queries, q_total, shard->main.d, p, shard_ids, shard_dists,
               stats_i32 - (int64_t)stage * 4 * q_total, stats_i64 - (int64_t)stage * 4 * q_total};
#ifdef _OPENMP
    if (threads > 0) omp_set_num_threads(threads);
#else
    (void)threads;
#endif
    volatile int err = 0;
    char errbuf[256] = {0};
#pragma omp parallel for schedule(dynamic, 4)
    for (int64_t qi = q0; qi < q0 + n; qi++) {
        if (err) continue;
        const int32_t F = fwd_count(p);
        int32_t tl[8] = {-1, -1, -1, -1, -1, -1, -1, -1};
        int64_t ein[8] = {0};
        if (entries_in)
            for (int32_t f = 0; f < F; f++) ein[f] = entries_in[qi * F + f];
        if (search_one(&R, qi, col, stage, entries_in != NULL, ein, tl)) {
#pragma omp critical
            { err = 1; snprintf(errbuf, sizeof errbuf, "%s", g_err); }
            continue;
        }
        if (forward_out)
            for (int32_t f = 0; f < F; f++) forward_out[qi * F + f] = shard->inter_map[tl[f]];
    }
    free(arr);
    if (err) { snprintf(g_err, sizeof g_err, "%s", errbuf); return -1; }
    return 0;
}

int orc_run(const orc_shard* shards, int32_t n_shards, const float* queries, int64_t q,
            const orc_params* p, int32_t mode, int32_t threads,
            int32_t* shard_ids, float* shard_dists, int32_t* final_ids, float* final_dists,
            int32_t* stats_i32, int64_t* stats_i64, int64_t* comm) {
    const int32_t N = n_shards, k = p->k;
    if (mode == 1 && N > 1)
        for (int32_t s = 0; s < N; s++)
            if (!shards[s].inter_map) return fail("pipelined mode requires inter-shard tables for every shard");
    run_t R = {shards, N, queries, q, shards[0].main.d, p, shard_ids, shard_dists, stats_i32, stats_i64};
    for (int64_t i = 0; i < q * N * k; i++) { shard_ids[i] = -1; shard_dists[i] = INFINITY; }
    memset(stats_i32, 0, sizeof(int32_t) * (size_t)(N * 4 * q));
    memset(stats_i64, 0, sizeof(int64_t) * (size_t)(N * 4 * q));
    memset(comm, 0, sizeof(int64_t) * (size_t)(N * N));
#ifdef _OPENMP
    if (threads > 0) omp_set_num_threads(threads);
#else
    (void)threads;
#endif
    volatile int err = 0;
    char errbuf[256] = {0};
    if (mode == 0) {
        /* pipeline.py:288-304: shard s, stage s, no seeds */
        for (int32_t s = 0; s < N; s++) {
#pragma omp parallel for schedule(dynamic, 4)
            for (int64_t qi = 0; qi < q; qi++) {
                if (err) continue;
                int32_t tl[8];
                if (search_one(&R, qi, s, s, 0, NULL, tl)) {
#pragma omp critical
                    { err = 1; snprintf(errbuf, sizeof errbuf, "%s", g_err); }
                }
            }
        }
    } else {
        /* pipeline.py:327-347: chunks = array_split(arange(Q), N) */
        int64_t* lo = (int64_t*)malloc(sizeof(int64_t) * (size_t)(N + 1));
        int64_t base = q / N, extra = q % N;
        lo[0] = 0;
        for (int32_t c = 0; c < N; c++) lo[c + 1] = lo[c] + base + (c < extra ? 1 : 0);
        const int32_t F = fwd_count(p);
        int64_t* entries = (int64_t*)malloc(sizeof(int64_t) * (size_t)(q > 0 ? q * F : 1));
        for (int32_t stage = 0; stage < N; stage++) {
            for (int32_t c = 0; c < N; c++) {
                int32_t shard = (c + stage) % N;
                int forward = stage < N - 1;
#pragma omp parallel for schedule(dynamic, 4)
                for (int64_t qi = lo[c]; qi < lo[c + 1]; qi++) {
                    if (err) continue;
                    int32_t tl[8] = {-1, -1, -1, -1, -1, -1, -1, -1};
                    if (search_one(&R, qi, shard, stage, stage > 0, entries + qi * F, tl)) {
#pragma omp critical
                        { err = 1; snprintf(errbuf, sizeof errbuf, "%s", g_err); }
                        continue;
                    }
                    if (forward)
                        for (int32_t f = 0; f < F; f++) entries[qi * F + f] = shards[shard].inter_map[tl[f]];
                }
                if (forward) comm[(int64_t)stage * N + shard] = 4 * F * (lo[c + 1] - lo[c]);
            }
        }
        free(lo);
        free(entries);
    }
    if (err) { snprintf(g_err, sizeof g_err, "%s", errbuf); return -1; }
    /* pipeline.py:249-267 finish */
    for (int64_t i = 0; i < q * k; i++) { final_ids[i] = -1; final_dists[i] = INFINITY; }
    for (int64_t qi = 0; qi < q; qi++) {
        int rc = orc_reduce_topk(shard_ids + qi * N * k, shard_dists + qi * N * k, (int64_t)N * k, k,
                                 final_ids + qi * k, final_dists + qi * k);
        if (rc < 0) return -1;
    }
    return 0;
}

/* ------------------------------------------------------------------ CRC-32C
 * _crc32c.py:17-29 _make_tables (table 0: eight reflected shifts of the byte
 * by polynomial 0x82F63B78) and :32-37 _update_serial (one table step per
 * byte).  The reference's lane/GF(2)-stitch path for large buffers
 * (_crc32c.py:98-130) computes the same function; this restatement keeps the
 * plain serial definition so it checks both. */
uint32_t orc_crc32c_update(uint32_t state, const uint8_t* buf, int64_t n) {
    static uint32_t tab[256];
    static int ready = 0;
    if (!ready) {
        for (uint32_t i = 0; i < 256; ++i) {
            uint32_t c = i;
            for (int b = 0; b < 8; ++b) c = (c & 1u) ? (c >> 1) ^ 0x82F63B78u : c >> 1;
            tab[i] = c;
        }
        ready = 1;
    }
    for (int64_t i = 0; i < n; ++i) state = (state >> 8) ^ tab[(state ^ buf[i]) & 0xFFu];
    return state;
}
