/*
 * dgz_inputs/gen.c -- seeded synthetic INPUT generators shared by the oracle side and the
 * CUDA side.  This file holds none of the method's arithmetic:
 * no Philox, no Floyd sampling, no frontier union, no gather.  It only produces
 *   - a CSR graph with Poisson(lambda) out-degrees and uniform endpoints
 *     (SURVEY.md section 8(d) "Concrete synthetic inputs"; SPEC.md S:60-66 generate_graph),
 *   - a feature table filled with random bits keyed by the 8-byte word index, so that a wrong
 *     row or word cannot compare equal (SURVEY.md section 8(c) "What pins each part"),
 *   - the epoch permutation of node IDs that defines global batch j's seeds
 *     (section 3.4 data parallel; SPEC.md S:123-126 minibatch_stream),
 *   - a per-batch 64-bit sampler seed.
 * All functions are deterministic in their arguments and independent of the thread count.
 */
#include <stdint.h>
#include <string.h>
#include <math.h>
#ifdef _OPENMP
#include <omp.h>
#endif

static inline uint64_t sm64(uint64_t x) {
    x += 0x9E3779B97F4A7C15ull;
    x = (x ^ (x >> 30)) * 0xBF58476D1CE4E5B9ull;
    x = (x ^ (x >> 27)) * 0x94D049BB133111EBull;
    return x ^ (x >> 31);
}
/* keyed hash of (seed, stream, index) */
static inline uint64_t hk(uint64_t seed, uint64_t stream, uint64_t i) {
    return sm64(sm64(seed ^ (stream * 0xD1B54A32D192ED03ull)) ^ i);
}
/* uniform double in [0,1) */
static inline double u01(uint64_t h) { return (double)(h >> 11) * (1.0 / 9007199254740992.0); }

enum { ST_DEG = 1, ST_COL = 2, ST_TABLE = 3, ST_PERM = 4, ST_RNG = 5, ST_EPOCH = 6 };

int dgz_gen_abi_version(void) { return 1; }

/* Thread count of the OpenMP generators (torchrun sets OMP_NUM_THREADS=1 per rank). */
void dgz_gen_set_threads(int n) {
#ifdef _OPENMP
    if (n > 0) omp_set_num_threads(n);
#else
    (void)n;
#endif
}

/* Poisson(lambda) by inverse CDF with the pmf recursion, in double. lambda <= 700. */
static int64_t poisson_inv(double lam, double u) {
    double p = exp(-lam), c = p;
    int64_t k = 0;
    while (u >= c && k < 100000) {
        k++;
        p *= lam / (double)k;
        c += p;
        if (p == 0.0 && (double)k > lam) break;
    }
    return k;
}

/* off[0..n] (int64). Degrees ~ Poisson(lam) capped at n (no self-loop rule; duplicate
 * endpoints allowed: SPEC S:97 keeps duplicate edges as distinct slots). Returns E. */
int64_t dgz_gen_offsets(int64_t n, double lam, uint64_t seed, int64_t* off) {
    if (n <= 0 || !off || lam < 0 || lam > 700) return -1;
    off[0] = 0;
#pragma omp parallel for schedule(static)
    for (int64_t u = 0; u < n; u++) {
        int64_t d = poisson_inv(lam, u01(hk(seed, ST_DEG, (uint64_t)u)));
        off[u + 1] = d;
    }
    for (int64_t u = 0; u < n; u++) off[u + 1] += off[u];
    return off[n];
}

/* col[e] uniform in [0,n) by multiply-high of a 64-bit hash of the edge slot index. */
void dgz_gen_cols32(int64_t n, int64_t e_total, uint64_t seed, int32_t* col) {
#pragma omp parallel for schedule(static)
    for (int64_t e = 0; e < e_total; e++)
        col[e] = (int32_t)(((__uint128_t)hk(seed, ST_COL, (uint64_t)e) * (uint64_t)n) >> 64);
}
void dgz_gen_cols64(int64_t n, int64_t e_total, uint64_t seed, int64_t* col) {
#pragma omp parallel for schedule(static)
    for (int64_t e = 0; e < e_total; e++)
        col[e] = (int64_t)(((__uint128_t)hk(seed, ST_COL, (uint64_t)e) * (uint64_t)n) >> 64);
}

/* Fill bytes [0, nbytes) of a table buffer: byte b holds byte (b % 8) (little endian) of
 * hk(seed, ST_TABLE, b / 8).  Keyed by absolute byte position in the table, so row r, byte k
 * is a function of (r*R + k) only. */
void dgz_gen_fill(uint8_t* p, int64_t nbytes, uint64_t seed) {
    int64_t nw = nbytes / 8;
#pragma omp parallel for schedule(static)
    for (int64_t w = 0; w < nw; w++) {
        uint64_t v = hk(seed, ST_TABLE, (uint64_t)w);
        memcpy(p + 8 * w, &v, 8);
    }
    if (nbytes % 8) {
        uint64_t v = hk(seed, ST_TABLE, (uint64_t)nw);
        memcpy(p + 8 * nw, &v, (size_t)(nbytes % 8));
    }
}

/* count finite fp32 values, uniform on the 2^-23 grid of [-1, 1): value i = (top 24 bits of
 * hk(seed, ST_TABLE + 100, i)) / 2^23 - 1, exact in fp32 (for consumers that do arithmetic on rows,
 * at sizes numpy's generator is too slow for, e.g. the 56.9 GB config-4 table). */
void dgz_gen_fill_f32(float* p, int64_t count, uint64_t seed) {
#pragma omp parallel for schedule(static)
    for (int64_t i = 0; i < count; i++)
        p[i] = (float)(hk(seed, ST_TABLE + 100, (uint64_t)i) >> 40) * (1.0f / 8388608.0f) - 1.0f;
}

/* Keyed bijection on [0, n) (6-round Feistel network on 2h bits with cycle walking). */
static uint64_t feistel_perm(uint64_t x, uint64_t n, uint64_t key) {
    int bits = 2;
    while ((1ull << bits) < n) bits++;
    if (bits & 1) bits++;
    int h = bits / 2;
    uint64_t mask = (1ull << h) - 1;
    do {
        uint64_t l = x >> h, r = x & mask;
        for (int round = 0; round < 6; round++) {
            uint64_t nl = r;
            r = l ^ (hk(key, ST_PERM, ((uint64_t)round << 58) ^ r) & mask);
            l = nl;
        }
        x = (l << h) | r;
    } while (x >= n);
    return x;
}

/* Global batch j of batch size b over a node set of size n: epoch e = j / ceil(n/b), the
 * epoch permutation perm_e, seeds = perm_e[b*jj : min(b*(jj+1), n)] with jj = j mod ceil(n/b).
 * Writes up to b seeds, returns the count (last batch of an epoch may be short). */
int64_t dgz_gen_batch_seeds(int64_t n, int64_t b, uint64_t seed, int64_t j, int64_t* out) {
    if (n <= 0 || b <= 0 || j < 0 || !out) return -1;
    int64_t nb = (n + b - 1) / b;
    int64_t e = j / nb, jj = j % nb;
    int64_t lo = jj * b, hi = lo + b < n ? lo + b : n;
    uint64_t key = hk(seed, ST_EPOCH, (uint64_t)e);
    for (int64_t i = lo; i < hi; i++) out[i - lo] = (int64_t)feistel_perm((uint64_t)i, (uint64_t)n, key);
    return hi - lo;
}

/* Per-batch 64-bit sampler seed (the caller passes it to both sampler implementations). */
uint64_t dgz_gen_batch_rng_seed(uint64_t seed, int64_t j) { return hk(seed, ST_RNG, (uint64_t)j); }

/* n uniformly random row IDs in [0, rows) (duplicates possible) for gather-only sweeps. */
void dgz_gen_random_ids(int64_t rows, int64_t n, uint64_t seed, int64_t* out) {
#pragma omp parallel for schedule(static)
    for (int64_t i = 0; i < n; i++)
        out[i] = (int64_t)(((__uint128_t)hk(seed, ST_COL + 100, (uint64_t)i) * (uint64_t)rows) >> 64);
}

/* n DISTINCT row IDs in [0, rows): a keyed permutation prefix (n <= rows). */
void dgz_gen_distinct_ids(int64_t rows, int64_t n, uint64_t seed, int64_t* out) {
#pragma omp parallel for schedule(static)
    for (int64_t i = 0; i < n; i++) out[i] = (int64_t)feistel_perm((uint64_t)i, (uint64_t)rows, seed ^ 0xA5A5ull);
}

/* Skewed ("power-law") endpoints for the hot-row cache experiments:
 * rank = floor(n * u^alpha) (alpha > 1 concentrates edges on low ranks: the top fraction x of
 * ranks receives a share x^(1/alpha) of the edges), mapped to a node ID by a keyed permutation so
 * that hot nodes are scattered over the table. */
void dgz_gen_cols32_skewed(int64_t n, int64_t e_total, uint64_t seed, double alpha, int32_t* col) {
    const uint64_t key = hk(seed, ST_PERM + 100, 0);
#pragma omp parallel for schedule(static)
    for (int64_t e = 0; e < e_total; e++) {
        double u = u01(hk(seed, ST_COL, (uint64_t)e));
        int64_t r = (int64_t)((double)n * pow(u, alpha));
        if (r >= n) r = n - 1;
        col[e] = (int32_t)feistel_perm((uint64_t)r, (uint64_t)n, key);
    }
}
