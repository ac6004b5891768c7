// Address ordering of an arbitrary ID list for dgz_gather_perm.
//
// The sampler emits its gather list already in address order (from its frontier bitmap).  For an
// arbitrary caller list (duplicates allowed) this radix-sorts (id, position) pairs on the device,
// using only the bits that can differ (ids < max_id), so that any gather can be issued in table
// order and scattered back: out[pos[k]] = table[ids_sorted[k]].
#include <cub/device/device_radix_sort.cuh>

#include "internal.h"

namespace {

__global__ void iota_kernel(int64_t* __restrict__ p, int64_t n) {
    for (int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < n; i += int64_t(gridDim.x) * blockDim.x) p[i] = i;
}

int bits_for(int64_t max_id) {
    int b = 1;
    while (b < 63 && (int64_t(1) << b) < max_id) ++b;
    return b;
}

inline size_t al256(size_t x) { return (x + 255) & ~size_t(255); }

}  // namespace

using namespace dgz;

extern "C" dgz_status dgz_order_workspace_bytes(int64_t n, size_t* bytes) {
    DGZ_REQUIRE(n >= 0 && n < (int64_t(1) << 31) && bytes, "dgz_order_workspace_bytes: need 0 <= n < 2^31");
    size_t tmp = 0;
    cudaError_t e = cub::DeviceRadixSort::SortPairs(nullptr, tmp, (const int64_t*)nullptr, (int64_t*)nullptr, (const int64_t*)nullptr,
                                                    (int64_t*)nullptr, (int)(n > 0 ? n : 1), 0, 63);
    if (e != cudaSuccess) return cuda_fail(e, "cub::DeviceRadixSort::SortPairs (size query)");
    *bytes = al256(8 * (size_t)(n > 0 ? n : 1)) + al256(tmp);
    return DGZ_OK;
}

extern "C" dgz_status dgz_order_ids(const int64_t* ids_dev, int64_t n, int64_t max_id, int64_t* ids_sorted, int64_t* pos,
                                    void* workspace, size_t workspace_bytes, dgz_stream stream) {
    DGZ_REQUIRE(n >= 0 && n < (int64_t(1) << 31), "dgz_order_ids: need 0 <= n < 2^31");
    if (n == 0) return DGZ_OK;
    DGZ_REQUIRE(ids_dev && ids_sorted && pos && workspace && max_id >= 1, "dgz_order_ids: null argument or max_id < 1");
    size_t need = 0;
    dgz_status st = dgz_order_workspace_bytes(n, &need);
    if (st != DGZ_OK) return st;
    DGZ_REQUIRE(workspace_bytes >= need, "dgz_order_ids: workspace %zu < %zu bytes", workspace_bytes, need);
    cudaStream_t s = (cudaStream_t)stream;
    int64_t* iota = (int64_t*)workspace;
    void* tmp = (uint8_t*)workspace + al256(8 * (size_t)n);
    size_t tmp_bytes = workspace_bytes - al256(8 * (size_t)n);
    int grid = (int)((n + 255) / 256);
    if (grid > 148 * 8) grid = 148 * 8;
    iota_kernel<<<grid, 256, 0, s>>>(iota, n);
    dgz::count_launch();
    // IDs outside [0, max_id) keep their order among themselves (sign and high bits included
    // whenever max_id needs them); the gather later reports them as RANGE faults
    cudaError_t e = cub::DeviceRadixSort::SortPairs(tmp, tmp_bytes, ids_dev, ids_sorted, iota, pos, (int)n, 0, bits_for(max_id), s);
    if (e != cudaSuccess) return cuda_fail(e, "cub::DeviceRadixSort::SortPairs");
    dgz::count_launch();  // CUB's onesweep sort is counted as one launch (it issues a few)
    return launch_check("dgz_order_ids");
}
