// Internal helpers shared by the libdgz translation units (not part of the ABI).
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>
#include <string.h>

#include "dgz.h"

namespace dgz {

void set_error(const char* fmt, ...);
dgz_status cuda_fail(cudaError_t e, const char* what);

#define DGZ_CUDA(call)                                                 \
    do {                                                               \
        cudaError_t _e = (call);                                       \
        if (_e != cudaSuccess) return ::dgz::cuda_fail(_e, #call);     \
    } while (0)

#define DGZ_REQUIRE(cond, ...)                                         \
    do {                                                               \
        if (!(cond)) { ::dgz::set_error(__VA_ARGS__); return DGZ_ERR_INVALID; } \
    } while (0)

inline dgz_status launch_check(const char* what) {
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return cuda_fail(e, what);
    return DGZ_OK;
}

int sm_count_of_current_device();
void count_launch();  // every kernel launch of libdgz increments dgz_kernel_launches()

// Shared-memory carveout requested for a kernel (cudaFuncAttributePreferredSharedMemoryCarveout, set once per
// kernel).  Gathers (kCarveoutGather): the maximum shared memory by default (DGZ_CARVEOUT=<percent> to change
// it, -1 = the driver's choice).  An SM runs CTAs of kernels whose carveouts differ only after it drains and
// reconfigures, so a gather with the driver's small-smem carveout keeps a shared-memory-heavy consumer (the a7
// layer: ~196 KiB per SM) off every SM it occupies (a one-warp spin kernel on 64 SMs
// stretched the layer 1.46x with the driver's carveout, 1.01x with the maximum); the gathers' line loads
// bypass L1, so the smaller L1 costs them nothing.  Sampler kernels (kCarveoutSampler): the driver's choice
// by default (DGZ_SAMPLER_CARVEOUT to change it) -- their random CSR reads use L1 (maximum carveout: 0.29 ->
// 0.34 ms per config-4 minibatch).
constexpr int kCarveoutGather = 0, kCarveoutSampler = 1;
int carveout_pct(int cls);
void apply_carveout(const void* kernel, int cls = kCarveoutGather);

}  // namespace dgz

struct dgz_table_s {
    const uint8_t* host;      // caller's pointer to row 0
    const uint8_t* dev;       // device-visible pointer to row 0
    int64_t rows, dim, row_bytes;
    int32_t elem_bytes;
    int32_t device;
    uint32_t flags;
    void* reg_base;           // page-aligned base that this handle registered (nullptr if none)
    size_t reg_bytes;
    int64_t gpu_mem_delta;
    double register_seconds;
    int* err_flag[64];        // per-device RANGE flag (device memory), lazily allocated
    uint64_t managed_devs;    // DGZ_REG_MANAGED: devices already advised AccessedBy (bit d = device d)
};

// gather.cu
dgz_status dgz_gather_impl(dgz_table t, const void* idx, int idx_is64, const int64_t* dst_pos, int64_t n,
                           const int64_t* n_dev, void* out, const dgz_gather_cfg* cfg, cudaStream_t stream,
                           const dgz_cache_view* cache);
int* dgz_table_flag(dgz_table t);
// hostvmm.cu: 1 = inside a DGZ_HOST_VMM allocation (access granted to the current device), 0 = not,
// negative = -dgz_status
int dgz_vmm_register(const void* p, size_t bytes);  // flag for the current device (allocates on first use)
