// PCIe zero-copy probes: the streaming-read ceiling of GPU-initiated loads
// over the link, and the round-trip time of one dependent load (the paper's Little's-law
// inputs).
#include "internal.h"

namespace {

__device__ __forceinline__ uint4 ld_zc(uint64_t p) {
    uint4 r;
    asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];" : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w) : "l"(p));
    return r;
}

// the same load with an L2 prefetch-size hint (PTX .L2::64B / ::128B / ::256B): does the L2 then
// fetch 256 B from system memory per miss (fewer, larger PCIe reads)?
template <int PF>
__device__ __forceinline__ uint4 ld_zc_pf(uint64_t p) {
    uint4 r;
    if constexpr (PF == 256)
        asm volatile("ld.global.nc.L1::no_allocate.L2::256B.v4.u32 {%0,%1,%2,%3}, [%4];"
                     : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w) : "l"(p));
    else if constexpr (PF == 128)
        asm volatile("ld.global.nc.L1::no_allocate.L2::128B.v4.u32 {%0,%1,%2,%3}, [%4];"
                     : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w) : "l"(p));
    else if constexpr (PF == 64)
        asm volatile("ld.global.nc.L1::no_allocate.L2::64B.v4.u32 {%0,%1,%2,%3}, [%4];"
                     : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w) : "l"(p));
    else
        r = ld_zc(p);
    return r;
}

template <int U, int PF = 0>
__global__ void __launch_bounds__(1024, 1) stream_kernel(const uint8_t* __restrict__ src, int64_t chunks, uint64_t* sink) {
    const int lane = threadIdx.x & 31;
    const int64_t w = (int64_t(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
    const int64_t nw = (int64_t(gridDim.x) * blockDim.x) >> 5;
    uint32_t acc = 0;
    for (int64_t c0 = w * 32 * U; c0 < chunks; c0 += nw * 32 * U) {
        uint4 v[U];
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const int64_t c = c0 + u * 32 + lane;
            if (c < chunks) v[u] = ld_zc_pf<PF>((uint64_t)src + (uint64_t)c * 16);
            else v[u] = make_uint4(0, 0, 0, 0);
        }
#pragma unroll
        for (int u = 0; u < U; ++u) acc ^= v[u].x ^ v[u].y ^ v[u].z ^ v[u].w;
    }
    if (acc == 0x9E3779B9u) atomicAdd((unsigned long long*)sink, 1ull);  // keeps the loads live
}

// random-row read probe: each warp reads U rows of R bytes (16 B per lane per step) at the given IDs
// with all U rows' loads issued before any is consumed; XOR-folded, nothing written -- the read-only
// ceiling of random row traffic (the a7 layer's pattern) at a given number of rows in flight
template <int U>
__global__ void __launch_bounds__(1024) rows_kernel(const uint8_t* __restrict__ src, int64_t R, const int64_t* __restrict__ ids,
                                                    int64_t n, uint64_t* sink) {
    const int lane = threadIdx.x & 31;
    const int64_t w = (int64_t(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
    const int64_t nw = (int64_t(gridDim.x) * blockDim.x) >> 5;
    uint32_t acc = 0;
    for (int64_t r0 = w * U; r0 < n; r0 += nw * U) {
        for (int64_t b = (int64_t)lane * 16; b < R; b += 512) {
            uint4 v[U];
#pragma unroll
            for (int u = 0; u < U; ++u) {
                const int64_t r = r0 + u;
                v[u] = r < n ? __ldg(reinterpret_cast<const uint4*>(src + __ldg(ids + r) * R + b)) : make_uint4(0, 0, 0, 0);
            }
#pragma unroll
            for (int u = 0; u < U; ++u) acc ^= v[u].x ^ v[u].y ^ v[u].z ^ v[u].w;
        }
    }
    if (acc == 0x9E3779B9u) atomicAdd((unsigned long long*)sink, 1ull);
}

__global__ void chase_kernel(const int64_t* __restrict__ src, int64_t steps, uint64_t* cycles) {
    int64_t p = 0;
    const long long t0 = clock64();
    for (int64_t s = 0; s < steps; ++s) {
        int64_t nx;
        asm volatile("ld.global.cv.s64 %0, [%1];" : "=l"(nx) : "l"(src + p));
        p = nx;
    }
    const long long t1 = clock64();
    cycles[0] = (uint64_t)(t1 - t0);
    cycles[1] = (uint64_t)p;
}

// pure-ALU load: dependent FMA chains, no memory traffic (interference experiments)
__global__ void spin_kernel(int64_t iters, float* sink) {
    float a = threadIdx.x * 1e-3f, b = 1.0001f, c = 0.9999f;
    for (int64_t i = 0; i < iters; ++i) {
        a = fmaf(a, b, c);
        b = fmaf(b, c, a * 1e-9f);
    }
    if (a == 1234.5f) sink[0] = b;
}

}  // namespace

using namespace dgz;

extern "C" dgz_status dgz_probe_spin(int32_t ctas, int32_t threads, int64_t iters, float* sink_dev, dgz_stream stream) {
    DGZ_REQUIRE(ctas > 0 && threads > 0 && threads <= 1024 && iters >= 0 && sink_dev, "dgz_probe_spin: bad args");
    dgz::apply_carveout((const void*)spin_kernel);
    spin_kernel<<<ctas, threads, 0, (cudaStream_t)stream>>>(iters, sink_dev);
    dgz::count_launch();
    return launch_check("spin_kernel");
}

extern "C" dgz_status dgz_probe_stream(const void* src_dev, int64_t bytes, int32_t sm_count, int32_t warps, int32_t unroll,
                                       uint64_t* sink_dev, dgz_stream stream) {
    DGZ_REQUIRE(src_dev && sink_dev && bytes > 0 && bytes % 16 == 0 && ((uintptr_t)src_dev % 16) == 0, "dgz_probe_stream: bad args");
    const int nsm = sm_count_of_current_device();
    const int k = (sm_count > 0 && sm_count < nsm) ? sm_count : nsm;
    if (warps <= 0 || warps > 32) warps = 32;
    cudaStream_t s = (cudaStream_t)stream;
    const int64_t chunks = bytes / 16;
    switch (unroll) {
        case 1: stream_kernel<1><<<k, warps * 32, 0, s>>>((const uint8_t*)src_dev, chunks, sink_dev); dgz::count_launch(); break;
        case 2: stream_kernel<2><<<k, warps * 32, 0, s>>>((const uint8_t*)src_dev, chunks, sink_dev); dgz::count_launch(); break;
        case 4: stream_kernel<4><<<k, warps * 32, 0, s>>>((const uint8_t*)src_dev, chunks, sink_dev); dgz::count_launch(); break;
        case 16: stream_kernel<16><<<k, warps * 32, 0, s>>>((const uint8_t*)src_dev, chunks, sink_dev); dgz::count_launch(); break;
        default: stream_kernel<8><<<k, warps * 32, 0, s>>>((const uint8_t*)src_dev, chunks, sink_dev); dgz::count_launch(); break;
    }
    return launch_check("stream_kernel");
}

extern "C" dgz_status dgz_probe_stream_hint(const void* src_dev, int64_t bytes, int32_t sm_count, int32_t warps,
                                            int32_t l2_prefetch_bytes, uint64_t* sink_dev, dgz_stream stream) {
    DGZ_REQUIRE(src_dev && sink_dev && bytes > 0 && bytes % 16 == 0 && ((uintptr_t)src_dev % 16) == 0,
                "dgz_probe_stream_hint: bad args");
    const int nsm = sm_count_of_current_device();
    const int k = (sm_count > 0 && sm_count < nsm) ? sm_count : nsm;
    if (warps <= 0 || warps > 32) warps = 32;
    cudaStream_t s = (cudaStream_t)stream;
    const int64_t chunks = bytes / 16;
    switch (l2_prefetch_bytes) {
        case 64: stream_kernel<8, 64><<<k, warps * 32, 0, s>>>((const uint8_t*)src_dev, chunks, sink_dev); break;
        case 128: stream_kernel<8, 128><<<k, warps * 32, 0, s>>>((const uint8_t*)src_dev, chunks, sink_dev); break;
        case 256: stream_kernel<8, 256><<<k, warps * 32, 0, s>>>((const uint8_t*)src_dev, chunks, sink_dev); break;
        default: stream_kernel<8, 0><<<k, warps * 32, 0, s>>>((const uint8_t*)src_dev, chunks, sink_dev); break;
    }
    dgz::count_launch();
    return launch_check("stream_kernel (hint)");
}

extern "C" dgz_status dgz_probe_rows(const void* src_dev, int64_t row_bytes, const int64_t* ids_dev, int64_t n, int32_t sm_count,
                                     int32_t warps, int32_t rows_in_flight, uint64_t* sink_dev, dgz_stream stream) {
    DGZ_REQUIRE(src_dev && ids_dev && sink_dev && n > 0 && row_bytes > 0 && row_bytes % 16 == 0 && ((uintptr_t)src_dev % 16) == 0,
                "dgz_probe_rows: bad args");
    const int nsm = sm_count_of_current_device();
    const int k = (sm_count > 0 && sm_count < nsm) ? sm_count : nsm;
    if (warps <= 0 || warps > 32) warps = 32;
    cudaStream_t s = (cudaStream_t)stream;
    const uint8_t* src = (const uint8_t*)src_dev;
    switch (rows_in_flight) {
        case 1: rows_kernel<1><<<k, warps * 32, 0, s>>>(src, row_bytes, ids_dev, n, sink_dev); break;
        case 2: rows_kernel<2><<<k, warps * 32, 0, s>>>(src, row_bytes, ids_dev, n, sink_dev); break;
        case 4: rows_kernel<4><<<k, warps * 32, 0, s>>>(src, row_bytes, ids_dev, n, sink_dev); break;
        case 16: rows_kernel<16><<<k, warps * 32, 0, s>>>(src, row_bytes, ids_dev, n, sink_dev); break;
        default: rows_kernel<8><<<k, warps * 32, 0, s>>>(src, row_bytes, ids_dev, n, sink_dev); break;
    }
    dgz::count_launch();
    return launch_check("rows_kernel");
}

extern "C" dgz_status dgz_probe_chase(const void* src_dev, int64_t steps, uint64_t* cycles_dev, dgz_stream stream) {
    DGZ_REQUIRE(src_dev && cycles_dev && steps > 0, "dgz_probe_chase: bad args");
    chase_kernel<<<1, 1, 0, (cudaStream_t)stream>>>((const int64_t*)src_dev, steps, cycles_dev); dgz::count_launch();
    return launch_check("chase_kernel");
}
