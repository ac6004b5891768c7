// HBM row cache construction: slot map + shard rows.
// The cached gather itself is the SEGMENT kernel with CACHED = true (gather.cu).
#include "internal.h"

namespace {

__global__ void slot_scatter_kernel(const int64_t* __restrict__ hot, int64_t n_hot, int64_t rows, int32_t* __restrict__ slot,
                                    int* __restrict__ err) {
    for (int64_t c = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; c < n_hot; c += int64_t(gridDim.x) * blockDim.x) {
        const int64_t id = hot[c];
        if (id < 0 || id >= rows) atomicOr(err, 1);
        else slot[id] = (int32_t)c;
    }
}

// shard g's list of table IDs: hot[g], hot[g + G], hot[g + 2G], ...
__global__ void strided_ids_kernel(const int64_t* __restrict__ hot, int64_t n_hot, int G, int g, int64_t* __restrict__ out) {
    const int64_t m = (n_hot - g + G - 1) / G;
    for (int64_t k = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; k < m; k += int64_t(gridDim.x) * blockDim.x) out[k] = hot[g + k * G];
}

}  // namespace

using namespace dgz;

extern "C" dgz_status dgz_cache_fill(dgz_table t, const int64_t* hot_ids_dev, int64_t n_hot, const dgz_cache_view* cache,
                                     dgz_stream stream) {
    return dgz_cache_fill_local(t, hot_ids_dev, n_hot, cache, -1, stream);
}

extern "C" dgz_status dgz_cache_fill_local(dgz_table t, const int64_t* hot_ids_dev, int64_t n_hot, const dgz_cache_view* cache,
                                           int32_t local_shard, dgz_stream stream) {
    DGZ_REQUIRE(t && cache && cache->slot_map, "dgz_cache_fill: null argument");
    DGZ_REQUIRE(cache->n_shards >= 1 && cache->n_shards <= DGZ_MAX_CACHE_SHARDS, "dgz_cache_fill: n_shards %d", cache->n_shards);
    DGZ_REQUIRE(n_hot >= 0 && n_hot <= t->rows && n_hot < (int64_t(1) << 31), "dgz_cache_fill: n_hot %lld", (long long)n_hot);
    DGZ_REQUIRE(n_hot == 0 || hot_ids_dev, "dgz_cache_fill: null hot_ids");
    DGZ_REQUIRE(local_shard >= -1 && local_shard < cache->n_shards, "dgz_cache_fill: local_shard %d of %d", local_shard,
                cache->n_shards);
    for (int g = 0; g < cache->n_shards; ++g)
        DGZ_REQUIRE(cache->shards[g] || n_hot == 0 || (local_shard >= 0 && g != local_shard), "dgz_cache_fill: null shard %d", g);
    cudaStream_t s = (cudaStream_t)stream;
    int* err = dgz_table_flag(t);
    if (!err) { set_error("dgz_cache_fill: cannot allocate the device flag"); return DGZ_ERR_CUDA; }
    DGZ_CUDA(cudaMemsetAsync(cache->slot_map, 0xff, sizeof(int32_t) * (size_t)t->rows, s));  // all -1
    if (n_hot == 0) return DGZ_OK;
    const int grid = (int)((n_hot + 255) / 256 < 148 * 8 ? (n_hot + 255) / 256 : 148 * 8);
    slot_scatter_kernel<<<grid, 256, 0, s>>>(hot_ids_dev, n_hot, t->rows, cache->slot_map, err);
    dgz::count_launch();
    const int G = cache->n_shards;
    if (G == 1) {   // (local_shard is -1 or 0)
        return dgz_gather_impl(t, hot_ids_dev, 1, nullptr, n_hot, nullptr, cache->shards[0], nullptr, s, nullptr);
    }
    int64_t* tmp = nullptr;
    const int64_t m = (n_hot + G - 1) / G;
    DGZ_CUDA(cudaMallocAsync((void**)&tmp, sizeof(int64_t) * (size_t)m, s));
    dgz_status st = DGZ_OK;
    for (int g = 0; g < G && st == DGZ_OK; ++g) {
        if (local_shard >= 0 && g != local_shard) continue;   // filled by the rank that owns it
        const int64_t mg = (n_hot - g + G - 1) / G;
        if (mg <= 0) continue;
        strided_ids_kernel<<<grid, 256, 0, s>>>(hot_ids_dev, n_hot, G, g, tmp);
        dgz::count_launch();
        st = dgz_gather_impl(t, tmp, 1, nullptr, mg, nullptr, cache->shards[g], nullptr, s, nullptr);
    }
    cudaFreeAsync(tmp, s);
    if (st != DGZ_OK) return st;
    return launch_check("dgz_cache_fill");
}

// ---- device memory and CUDA IPC for cache shards owned by other ranks (NVLink peer loads) ----
static_assert(sizeof(cudaIpcMemHandle_t) == sizeof(dgz_ipc_handle), "dgz_ipc_handle must hold a cudaIpcMemHandle_t");

extern "C" dgz_status dgz_device_alloc(size_t bytes, void** out) {
    DGZ_REQUIRE(out && bytes > 0, "dgz_device_alloc: null out or zero bytes");
    *out = nullptr;
    DGZ_CUDA(cudaMalloc(out, bytes));
    return DGZ_OK;
}

extern "C" dgz_status dgz_device_free(void* p) {
    if (p) DGZ_CUDA(cudaFree(p));
    return DGZ_OK;
}

extern "C" dgz_status dgz_ipc_get_handle(void* dev_ptr, dgz_ipc_handle* out) {
    DGZ_REQUIRE(dev_ptr && out, "dgz_ipc_get_handle: null argument");
    cudaIpcMemHandle_t h;
    DGZ_CUDA(cudaIpcGetMemHandle(&h, dev_ptr));
    memcpy(out->bytes, &h, sizeof(h));
    return DGZ_OK;
}

extern "C" dgz_status dgz_ipc_open(const dgz_ipc_handle* handle, void** out) {
    DGZ_REQUIRE(handle && out, "dgz_ipc_open: null argument");
    *out = nullptr;
    cudaIpcMemHandle_t h;
    memcpy(&h, handle->bytes, sizeof(h));
    DGZ_CUDA(cudaIpcOpenMemHandle(out, h, cudaIpcMemLazyEnablePeerAccess));
    return DGZ_OK;
}

extern "C" dgz_status dgz_ipc_close(void* dev_ptr) {
    DGZ_REQUIRE(dev_ptr, "dgz_ipc_close: null pointer");
    DGZ_CUDA(cudaIpcCloseMemHandle(dev_ptr));
    return DGZ_OK;
}
