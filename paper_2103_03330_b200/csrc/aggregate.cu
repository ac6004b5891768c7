// Stand-in GraphSAGE mean aggregation (the consumer of step a7; P:554-555 fig:singlegpu).
// It exists to occupy the GPU while the next minibatch is gathered on a side stream, so that
// the exposed fetch time can be measured.  One warp per destination node,
// lanes across the feature dimension; fp32 accumulation.
#include "internal.h"

namespace {

__global__ void __launch_bounds__(256)
aggregate_mean_kernel(const float* __restrict__ x, int64_t dim, const int32_t* __restrict__ nbr, const int32_t* __restrict__ cnt,
                      int fanout, const int64_t* __restrict__ n_dst_dev, int64_t n_dst_max, float* __restrict__ y, int repeat) {
    int64_t n = n_dst_max;
    if (n_dst_dev) {
        const int64_t m = *n_dst_dev;
        n = m < n ? m : n;
    }
    const int lane = threadIdx.x & 31;
    const int64_t w = (int64_t(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
    const int64_t nw = (int64_t(gridDim.x) * blockDim.x) >> 5;
    for (int rep = 0; rep < repeat; ++rep) {
        for (int64_t i = w; i < n; i += nw) {
            const int c = cnt[i];
            const float inv = 1.0f / (float)(1 + c);
            for (int64_t d = lane; d < dim; d += 32) {
                float acc = x[i * dim + d];
                for (int q = 0; q < c; ++q) acc += x[(int64_t)nbr[i * fanout + q] * dim + d];
                y[i * dim + d] = acc * inv;
            }
        }
    }
}

}  // namespace

using namespace dgz;

extern "C" dgz_status dgz_aggregate_mean(const float* x, int64_t dim, const int32_t* nbr_local, const int32_t* cnt, int32_t fanout,
                                         const int64_t* n_dst_dev, int64_t n_dst_max, float* y, int32_t repeat, int32_t sm_count,
                                         int32_t ctas_per_sm, dgz_stream stream) {
    DGZ_REQUIRE(x && nbr_local && cnt && y && dim >= 1 && fanout >= 0 && n_dst_max >= 0 && repeat >= 1,
                "dgz_aggregate_mean: bad arguments");
    if (n_dst_max == 0) return DGZ_OK;
    const int nsm = sm_count_of_current_device();
    const int k = (sm_count > 0 && sm_count < nsm) ? sm_count : nsm;
    // ctas_per_sm == 0: non-persistent grid (one CTA per 8 destination nodes, each CTA lives a few
    // microseconds, like training kernels), launched `repeat` times: a high-priority fetch stream
    // gets SM slots within microseconds.  ctas_per_sm > 0: a persistent grid of k * ctas_per_sm
    // CTAs doing all repeats in one launch (occupies its slots for the whole call).
    int64_t blocks = (n_dst_max * 32 + 255) / 256;
    if (ctas_per_sm > 0) {
        const int64_t cap = (int64_t)k * ctas_per_sm;
        if (blocks > cap) blocks = cap;
        aggregate_mean_kernel<<<(int)blocks, 256, 0, (cudaStream_t)stream>>>(x, dim, nbr_local, cnt, fanout, n_dst_dev, n_dst_max, y,
                                                                            repeat);
        dgz::count_launch();
    } else {
        for (int r = 0; r < repeat; ++r) {
            aggregate_mean_kernel<<<(int)blocks, 256, 0, (cudaStream_t)stream>>>(x, dim, nbr_local, cnt, fanout, n_dst_dev, n_dst_max,
                                                                                y, 1);
            dgz::count_launch();
        }
    }
    return launch_check("aggregate_mean_kernel");
}
