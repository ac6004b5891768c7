/*
 * A plain C program using libdgz through include/dgz.h only (no Python, no PyTorch):
 * allocate + fill a host table, register it, build a CSR on the host, sample one
 * minibatch on the GPU, gather its rows by zero-copy in address order
 * (dgz_gather_perm), and compare every gathered byte with table[U[r]] computed here with memcmp.
 *
 *   ./c_abi_gather [rows] [dim]        exit 0 = bit-exact, 1 = mismatch, 2 = error
 */
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#include "dgz.h"

#define CHECK(x)                                                                      \
    do {                                                                              \
        dgz_status _s = (x);                                                          \
        if (_s != DGZ_OK) {                                                           \
            fprintf(stderr, "%s failed: %d %s\n", #x, (int)_s, dgz_last_error());     \
            return 2;                                                                 \
        }                                                                             \
    } while (0)

static uint64_t mix(uint64_t x) {
    x += 0x9E3779B97F4A7C15ull;
    x = (x ^ (x >> 30)) * 0xBF58476D1CE4E5B9ull;
    x = (x ^ (x >> 27)) * 0x94D049BB133111EBull;
    return x ^ (x >> 31);
}

int main(int argc, char** argv) {
    const int64_t rows = argc > 1 ? atoll(argv[1]) : 20000;
    const int64_t dim = argc > 2 ? atoll(argv[2]) : 100;
    const int64_t R = dim * 4;
    const int32_t fanouts[2] = {10, 5};
    const int64_t n_seeds = 512;

    /* host table + CSR (random, 8 out-edges per node) */
    void* table = NULL;
    CHECK(dgz_host_alloc(NULL, (size_t)(rows * R), 1, DGZ_HOST_HUGEPAGE, &table));
    for (int64_t i = 0; i < rows * R / 8; i++) ((uint64_t*)table)[i] = mix((uint64_t)i);
    int64_t* off = (int64_t*)malloc(sizeof(int64_t) * (rows + 1));
    int32_t* col = (int32_t*)malloc(sizeof(int32_t) * rows * 8);
    for (int64_t u = 0; u <= rows; u++) off[u] = 8 * u;
    for (int64_t e = 0; e < rows * 8; e++) col[e] = (int32_t)(mix(e ^ 0xABCDull) % (uint64_t)rows);
    int64_t seeds[512];
    for (int64_t i = 0; i < n_seeds; i++) seeds[i] = (int64_t)((i * 7919) % rows);

    dgz_table t;
    CHECK(dgz_register_table(table, rows, dim, DGZ_F32, 0, &t));

    int64_t *d_off, *d_seeds, *d_ids, *d_sizes, *d_sorted, *d_pos;
    int32_t* d_col;
    int64_t bounds[3], be, ce;
    size_t ws_bytes;
    void* d_ws;
    uint8_t* d_out;
    CHECK(dgz_sample_bounds(rows, n_seeds, fanouts, 2, bounds, &be, &ce));
    CHECK(dgz_sample_workspace_bytes(rows, n_seeds, &ws_bytes));
    if (cudaMalloc((void**)&d_off, sizeof(int64_t) * (rows + 1)) || cudaMalloc((void**)&d_col, sizeof(int32_t) * rows * 8) ||
        cudaMalloc((void**)&d_seeds, sizeof(seeds)) || cudaMalloc((void**)&d_ids, sizeof(int64_t) * bounds[2]) ||
        cudaMalloc((void**)&d_sorted, sizeof(int64_t) * bounds[2]) || cudaMalloc((void**)&d_pos, sizeof(int64_t) * bounds[2]) ||
        cudaMalloc((void**)&d_sizes, sizeof(int64_t) * 3) || cudaMalloc(&d_ws, ws_bytes) ||
        cudaMalloc((void**)&d_out, (size_t)(bounds[2] * R))) {
        fprintf(stderr, "cudaMalloc failed\n");
        return 2;
    }
    cudaMemcpy(d_off, off, sizeof(int64_t) * (rows + 1), cudaMemcpyHostToDevice);
    cudaMemcpy(d_col, col, sizeof(int32_t) * rows * 8, cudaMemcpyHostToDevice);
    cudaMemcpy(d_seeds, seeds, sizeof(seeds), cudaMemcpyHostToDevice);

    dgz_csr csr = {rows, d_off, d_col, 0, 0};
    dgz_sample_out so;
    memset(&so, 0, sizeof(so));
    so.ids = d_ids;
    so.ids_cap = bounds[2];
    so.sizes_dev = d_sizes;
    so.workspace = d_ws;
    so.workspace_bytes = ws_bytes;
    so.ids_sorted = d_sorted;
    so.ids_sorted_pos = d_pos;
    CHECK(dgz_sample_uniform(&csr, d_seeds, n_seeds, fanouts, 2, 0x1234u, &so, NULL));
    CHECK(dgz_gather_perm(t, d_sorted, d_pos, bounds[2], d_sizes + 2, d_out, NULL, NULL));
    CHECK(dgz_check_errors(t, NULL));

    int64_t sizes[3];
    cudaMemcpy(sizes, d_sizes, sizeof(sizes), cudaMemcpyDeviceToHost);
    const int64_t n = sizes[2];
    int64_t* U = (int64_t*)malloc(sizeof(int64_t) * n);
    uint8_t* out = (uint8_t*)malloc((size_t)(n * R));
    cudaMemcpy(U, d_ids, sizeof(int64_t) * n, cudaMemcpyDeviceToHost);
    cudaMemcpy(out, d_out, (size_t)(n * R), cudaMemcpyDeviceToHost);
    int64_t bad = 0;
    for (int64_t r = 0; r < n; r++)
        if (U[r] < 0 || U[r] >= rows || memcmp(out + r * R, (uint8_t*)table + U[r] * R, (size_t)R)) bad++;
    printf("c_abi_gather: |F| = %lld %lld %lld, %lld rows x %lld B, %lld mismatches, %llu kernels\n", (long long)sizes[0],
           (long long)sizes[1], (long long)sizes[2], (long long)n, (long long)R, (long long)bad,
           (unsigned long long)dgz_kernel_launches());
    CHECK(dgz_unregister_table(t));
    CHECK(dgz_host_free(table, (size_t)(rows * R)));
    return bad ? 1 : 0;
}
