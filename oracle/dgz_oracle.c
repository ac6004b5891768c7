/*
 * ORACLE -- TEST INFRASTRUCTURE ONLY.
 *
 * A plain, slow, single-threaded CPU implementation of what the hot path computes:
 * layered uniform neighbour sampling and the sparse feature row gather.  Only tests/,
 * __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference legs may load it.
 * It shares no code, header, table or constant generator with the CUDA path
 * (paper_2103_03330_b200/csrc) and does not include include/dgz.h.
 *
 * Citations: "P:n" = /root/reference/PAPER.md line n, "S:n" = SPEC.md line n; the readings
 * of silent or garbled passages are listed in DESIGN.md section "Readings" (R1..R17).
 *
 * Pins (tests/test_oracle_*.py): Philox4x32-10 known-answer vectors (Random123), Floyd
 * uniformity by exact enumeration, brute-force invariants on tiny graphs (membership,
 * cardinality min(f, deg), frontier prefix, uniqueness), SPEC special cases,
 * gather == numpy.take and == table[id] byte for byte.
 */
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

/* ------------------------------------------------------------------------------------------
 * Philox4x32-10 (Salmon et al., SC'11 "Parallel random numbers: as easy as 1, 2, 3").
 * The paper names no RNG; reading R11 fixes this counter-based generator.
 * ------------------------------------------------------------------------------------------ */
void oracle_philox4x32_10(const uint32_t ctr_in[4], const uint32_t key_in[2], uint32_t out[4]) {
    uint32_t c0 = ctr_in[0], c1 = ctr_in[1], c2 = ctr_in[2], c3 = ctr_in[3];
    uint32_t k0 = key_in[0], k1 = key_in[1];
    for (int round = 0; round < 10; round++) {
        if (round > 0) { k0 += 0x9E3779B9u; k1 += 0xBB67AE85u; }
        uint64_t p0 = (uint64_t)0xD2511F53u * (uint64_t)c0;
        uint64_t p1 = (uint64_t)0xCD9E8D57u * (uint64_t)c2;
        uint32_t hi0 = (uint32_t)(p0 >> 32), lo0 = (uint32_t)p0;
        uint32_t hi1 = (uint32_t)(p1 >> 32), lo1 = (uint32_t)p1;
        uint32_t n0 = hi1 ^ c1 ^ k0;
        uint32_t n1 = lo1;
        uint32_t n2 = hi0 ^ c3 ^ k1;
        uint32_t n3 = lo0;
        c0 = n0; c1 = n1; c2 = n2; c3 = n3;
    }
    out[0] = c0; out[1] = c1; out[2] = c2; out[3] = c3;
}

/* r(t) for node u at hop k: word 0 of Philox4x32-10 with counter (t, k, lo32 u, hi32 u) and
 * key (lo32 seed, hi32 seed)  (reading R11). */
static uint32_t draw(uint64_t rng_seed, int hop, int64_t u, uint32_t t) {
    uint32_t ctr[4] = {t, (uint32_t)hop, (uint32_t)((uint64_t)u & 0xffffffffu), (uint32_t)((uint64_t)u >> 32)};
    uint32_t key[2] = {(uint32_t)(rng_seed & 0xffffffffu), (uint32_t)(rng_seed >> 32)};
    uint32_t o[4];
    oracle_philox4x32_10(ctr, key, o);
    return o[0];
}

static int cmp_i64(const void* a, const void* b) {
    int64_t x = *(const int64_t*)a, y = *(const int64_t*)b;
    return (x > y) - (x < y);
}

/* ------------------------------------------------------------------------------------------
 * Uniform selection of min(f, d) distinct CSR slots of a node of degree d
 * ("uniformly random selection"; without replacement; reading R7).
 * d <= f: all slots 0..d-1 in CSR order.  d > f: Robert Floyd's algorithm
 *   S = {}; for t = 0..f-1: j = d - f + t; x = floor(r(t) * (j+1) / 2^32);
 *           if x in S then insert j else insert x
 * then the positions are S in ascending order.  Returns the count.
 * ------------------------------------------------------------------------------------------ */
int64_t oracle_select_positions(int64_t d, int32_t f, uint64_t rng_seed, int hop, int64_t u, int64_t* pos) {
    if (d <= 0 || f <= 0) return 0;
    if (d <= f) {
        for (int64_t p = 0; p < d; p++) pos[p] = p;
        return d;
    }
    int64_t count = 0;
    for (int32_t t = 0; t < f; t++) {
        int64_t j = d - f + t;
        uint64_t r = draw(rng_seed, hop, u, (uint32_t)t);
        int64_t x = (int64_t)((r * (uint64_t)(j + 1)) >> 32);
        int found = 0;
        for (int64_t q = 0; q < count; q++)
            if (pos[q] == x) { found = 1; break; }
        pos[count++] = found ? j : x;
    }
    qsort(pos, (size_t)count, sizeof(int64_t), cmp_i64);
    return count;
}

typedef struct { int64_t key; int64_t idx; } kv_t;
static int cmp_kv(const void* a, const void* b) {
    const kv_t* x = (const kv_t*)a; const kv_t* y = (const kv_t*)b;
    if (x->key != y->key) return (x->key > y->key) - (x->key < y->key);
    return (x->idx > y->idx) - (x->idx < y->idx);
}

static int64_t col_at(const void* col, int col_is64, int64_t e) {
    return col_is64 ? ((const int64_t*)col)[e] : (int64_t)((const int32_t*)col)[e];
}

/* ------------------------------------------------------------------------------------------
 * Layered uniform neighbour sampling (section 2.2; readings R7-R11).
 *   F_0 = seeds with duplicates removed, first occurrence kept.
 *   hop k = 0..L-1 with f = fanouts[k] (fanouts[0] is the seeds' hop, reading R8):
 *     every u in F_k (in order) selects min(f, deg u) neighbour slots (above);
 *     new = sorted unique(all selected IDs) minus F_k;  F_{k+1} = F_k ++ new  (R9, R10).
 *   U = F_L is the gather list (seeds included).
 * Outputs (caller-allocated):
 *   U[ucap]            frontier-prefix unique IDs,
 *   sizes[L+1]         |F_0| .. |F_L|,
 *   nbr (optional)     hop k block at sum_{i<k} sizes[i]*fanouts[i]: |F_k| x f_k sampled IDs,
 *                      row-major, unused tail slots = -1,
 *   cnt (optional)     hop k block at sum_{i<k} sizes[i]: count per frontier node,
 *   local (optional)   same layout as nbr: position in U of each sampled ID, -1 padded.
 * Returns 0 ok, 1 invalid argument, 3 capacity too small, 4 seed out of range.
 * ------------------------------------------------------------------------------------------ */
int oracle_sample_uniform(int64_t n_nodes, const int64_t* off, const void* col, int col_is64,
                          const int64_t* seeds, int64_t n_seeds, const int32_t* fanouts, int L,
                          uint64_t rng_seed, int64_t* U, int64_t ucap, int64_t* sizes,
                          int64_t* nbr, int64_t nbr_cap, int32_t* cnt, int64_t cnt_cap,
                          int32_t* local) {
    if (n_nodes <= 0 || !off || !col || (n_seeds > 0 && !seeds) || L < 0 || !U || !sizes) return 1;
    for (int k = 0; k < L; k++) if (fanouts[k] < 0) return 1;
    for (int64_t i = 0; i < n_seeds; i++) if (seeds[i] < 0 || seeds[i] >= n_nodes) return 4;

    /* F_0: seeds, first occurrence kept */
    kv_t* sk = (kv_t*)malloc(sizeof(kv_t) * (size_t)(n_seeds > 0 ? n_seeds : 1));
    for (int64_t i = 0; i < n_seeds; i++) { sk[i].key = seeds[i]; sk[i].idx = i; }
    qsort(sk, (size_t)n_seeds, sizeof(kv_t), cmp_kv);
    char* keep = (char*)calloc((size_t)(n_seeds > 0 ? n_seeds : 1), 1);
    for (int64_t p = 0; p < n_seeds; p++)
        if (p == 0 || sk[p].key != sk[p - 1].key) keep[sk[p].idx] = 1;
    int64_t nF = 0;
    for (int64_t i = 0; i < n_seeds; i++) if (keep[i]) {
        if (nF >= ucap) { free(sk); free(keep); return 3; }
        U[nF++] = seeds[i];
    }
    free(sk); free(keep);
    sizes[0] = nF;

    int64_t nbr_base = 0, cnt_base = 0;
    int64_t* pos = NULL;
    int32_t fmax = 0;
    for (int k = 0; k < L; k++) if (fanouts[k] > fmax) fmax = fanouts[k];
    pos = (int64_t*)malloc(sizeof(int64_t) * (size_t)(fmax > 0 ? fmax : 1));

    for (int k = 0; k < L; k++) {
        int32_t f = fanouts[k];
        int64_t nk = nF;
        if (nbr && nbr_base + nk * (int64_t)f > nbr_cap) { free(pos); return 3; }
        if (cnt && cnt_base + nk > cnt_cap) { free(pos); return 3; }
        int64_t* cand = (int64_t*)malloc(sizeof(int64_t) * (size_t)(nk * (int64_t)f > 0 ? nk * (int64_t)f : 1));
        int64_t nc = 0;
        for (int64_t i = 0; i < nk; i++) {
            int64_t u = U[i];
            int64_t d = off[u + 1] - off[u];
            int64_t c = oracle_select_positions(d, f, rng_seed, k, u, pos);
            for (int64_t q = 0; q < c; q++) {
                int64_t s = col_at(col, col_is64, off[u] + pos[q]);
                cand[nc++] = s;
                if (nbr) nbr[nbr_base + i * f + q] = s;
            }
            if (nbr) for (int64_t q = c; q < f; q++) nbr[nbr_base + i * f + q] = -1;
            if (cnt) cnt[cnt_base + i] = (int32_t)c;
        }
        /* new = sorted unique(cand) \ F_k */
        qsort(cand, (size_t)nc, sizeof(int64_t), cmp_i64);
        int64_t* fs = (int64_t*)malloc(sizeof(int64_t) * (size_t)(nk > 0 ? nk : 1));
        memcpy(fs, U, sizeof(int64_t) * (size_t)nk);
        qsort(fs, (size_t)nk, sizeof(int64_t), cmp_i64);
        for (int64_t p = 0; p < nc; p++) {
            if (p > 0 && cand[p] == cand[p - 1]) continue;
            if (bsearch(&cand[p], fs, (size_t)nk, sizeof(int64_t), cmp_i64)) continue;
            if (nF >= ucap) { free(cand); free(fs); free(pos); return 3; }
            U[nF++] = cand[p];
        }
        free(cand); free(fs);
        sizes[k + 1] = nF;
        nbr_base += nk * (int64_t)f;
        cnt_base += nk;
    }
    free(pos);

    /* local positions of the sampled IDs in U (the sub-graph "block" of P:248) */
    if (local && nbr) {
        kv_t* pu = (kv_t*)malloc(sizeof(kv_t) * (size_t)(nF > 0 ? nF : 1));
        for (int64_t i = 0; i < nF; i++) { pu[i].key = U[i]; pu[i].idx = i; }
        qsort(pu, (size_t)nF, sizeof(kv_t), cmp_kv);
        for (int64_t e = 0; e < nbr_base; e++) {
            if (nbr[e] < 0) { local[e] = -1; continue; }
            kv_t probe = {nbr[e], -1};
            /* lower bound */
            int64_t lo = 0, hi = nF;
            while (lo < hi) { int64_t mid = (lo + hi) / 2; if (cmp_kv(&pu[mid], &probe) < 0) lo = mid + 1; else hi = mid; }
            local[e] = (int32_t)pu[lo].idx;
        }
        free(pu);
    }
    return 0;
}

/* ------------------------------------------------------------------------------------------
 * Row gather: out[r*R + b] = table[idx[r]*R + b] for 0 <= r < n, 0 <= b < R
 * (Listing 2 last line "dst[dstOffset] = src[srcOffset]"; S:200-208 reference_gather;
 * the circular shift only permutes which thread copies which element).
 * Out-of-range IDs leave their output row untouched; the return value counts them.
 * ------------------------------------------------------------------------------------------ */
int64_t oracle_gather(const uint8_t* table, int64_t rows, int64_t row_bytes, const int64_t* idx,
                      int64_t n, uint8_t* out) {
    int64_t bad = 0;
    for (int64_t r = 0; r < n; r++) {
        int64_t id = idx[r];
        if (id < 0 || id >= rows) { bad++; continue; }
        memcpy(out + r * row_bytes, table + id * row_bytes, (size_t)row_bytes);
    }
    return bad;
}
