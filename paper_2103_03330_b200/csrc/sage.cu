// Stand-in GraphSAGE layer (the consumer of step a7; SURVEY 8(a) a7 "mean over each dst node's
// sampled neighbours of the gathered rows, then a small GEMM"; P:554-555 fig:singlegpu
// for the layer itself):
//
//   h[i, :] = (x[i, :] + sum_{q < cnt[i]} x[nbr_local[i*fanout + q], :]) * (1 / (1 + cnt[i]))   fp32
//   y[i, :] = bf16(h[i, :]) . W^T            W: [hidden, dim] bf16 (nn.Linear layout), y fp32
//
// One CTA owns a tile of 128 destination nodes (the UMMA M):
//   1. sixteen warps compute h for the tile from HBM (fp32, the same sequential order as
//      dgz_aggregate_mean, so h is bit-identical to it), round it to bf16 and write it into shared
//      memory as the K-major A operand (core-matrix layout, SWIZZLE_NONE);
//   2. one thread issues tcgen05.mma.cta_group::1.kind::f16 (M = 128, N = hidden, K = 16 per
//      instruction, fp32 accumulate) with A and W from shared memory and D in tensor memory, and
//      commits to an mbarrier;
//   3. the sixteen warps read D back with tcgen05.ld (warp w: TMEM lanes 32(w%4).., 16-column chunks
//      w/4 + 4c), stage each chunk in shared memory (64 B swizzle) and the TMA writes it to y.
// W is staged once per resident CTA in the same core-matrix layout (B operand, K-major), by cp.async
// while the first tile is summed; the K dimension is zero-padded to a multiple of 16 and chunked when
// wider than the shared-memory budget.  Two CTAs share an SM (TMEM columns and a 56-register budget are
// sized for it: 32 warps per SM keep the random row reads in flight, and a one-warp gather CTA still fits
// beside them); tiles come from a per-launch row counter, the second CTA of an SM starting half a tile
// behind.  Measured on a config-4 last-hop block (tools/consumer_roofline.py): 4.32 TB/s of algorithmic
// bytes (0.66 of HBM; 3.75 TB/s with one tile per CTA and the warps' own stores); the mean alone
// (dgz_aggregate_mean) 3.32 TB/s.
#include "internal.h"

#include <cuda.h>
#include <cuda_bf16.h>
#include <stdlib.h>

#include <atomic>
#include <mutex>

namespace {

constexpr int kTileM = 128;
constexpr int kThreads = 512;   // 16 warps
constexpr int kWarps = kThreads / 32;

// Core-matrix K-major layout of an [rows x Kp] bf16 operand (SWIZZLE_NONE, "interleave"):
// element (r, k) at (r/8)*SBO + (k/8)*LBO + (r%8)*16 + (k%8)*2 with LBO = 128 B (the K-adjacent
// 8x16 B core matrix) and SBO = Kp*16 B (the next 8 rows).
__device__ __forceinline__ uint32_t core_off(int r, int k, int Kp) {
    return (uint32_t)((r >> 3) * (Kp * 16) + (k >> 3) * 128 + (r & 7) * 16 + (k & 7) * 2);
}

__device__ __forceinline__ uint64_t smem_desc(uint32_t saddr, int Kp) {
    // bits 0-13 start >> 4, 16-29 LBO >> 4, 32-45 SBO >> 4, 46-47 version 1 (sm_100),
    // 49-51 base offset 0, 52 LBO mode 0, 61-63 layout 0 = SWIZZLE_NONE
    uint64_t d = 0;
    d |= (uint64_t)((saddr >> 4) & 0x3FFF);
    d |= (uint64_t)((128u >> 4) & 0x3FFF) << 16;
    d |= (uint64_t)(((uint32_t)(Kp * 16) >> 4) & 0x3FFF) << 32;
    d |= (uint64_t)1 << 46;
    return d;
}

// kind::f16 instruction descriptor: D fp32, A/B bf16, both K-major, N >> 3, M >> 4.
__host__ __device__ constexpr uint32_t instr_desc(int M, int N) {
    return (1u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(M >> 4) << 24);
}

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

__device__ __forceinline__ void mbar_wait(uint32_t bar, uint32_t phase) {
    asm volatile(
        "{\n\t.reg .pred P;\n"
        "WAIT_%=:\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 P, [%0], %1;\n\t"
        "@!P bra WAIT_%=;\n}\n" ::"r"(bar),
        "r"(phase)
        : "memory");
}

struct RowRef {
    int64_t i;
    int c;
    float inv;
    int32_t my_nbr;   // lane q holds the q-th sampled position (q < 32)
    bool live;
};

__device__ __forceinline__ RowRef row_ref(int64_t i, int64_t n, const int32_t* __restrict__ cnt, const int32_t* __restrict__ nbr,
                                          int fanout, int lane) {
    RowRef r;
    r.i = i;
    r.live = i < n;
    // cnt and the nbr row are loaded independently (positions past cnt are never used)
    r.c = r.live ? __ldg(cnt + i) : 0;
    r.my_nbr = (r.live && lane < fanout) ? __ldg(nbr + i * fanout + lane) : 0;
    r.inv = 1.0f / (1.0f + (float)r.c);
    return r;
}

__device__ __forceinline__ uint2 pack_bf16(float4 s, float inv) {
    __nv_bfloat162 lo = __floats2bfloat162_rn(s.x * inv, s.y * inv), hi = __floats2bfloat162_rn(s.z * inv, s.w * inv);
    uint2 pk;
    pk.x = *reinterpret_cast<uint32_t*>(&lo);
    pk.y = *reinterpret_cast<uint32_t*>(&hi);
    return pk;
}

__device__ __forceinline__ float4 ld4(const float* p) { return __ldg(reinterpret_cast<const float4*>(p)); }

__device__ __forceinline__ void add4(float4& a, const float4& b) {
    a.x += b.x;
    a.y += b.y;
    a.z += b.z;
    a.w += b.w;
}

// x[i] + sum_q x[nbr_q] at columns k0..k0+3 of NR rows at once (dim % 4 == 0, x 16 B aligned): the
// positions of a batch of B neighbours per row are shuffled out first, then all the batch's loads
// issue, then the adds run per row in q order.  Every guard is warp-uniform (cnt is per row).
template <int NR, int B>
__device__ __forceinline__ void sum_vec(const float* __restrict__ x, int dim, int k0, const RowRef (&A)[NR],
                                        const int32_t* __restrict__ nbr, int fanout, float4 (&s)[NR]) {
    const float4 z = make_float4(0.f, 0.f, 0.f, 0.f);
    int cm = 0;
#pragma unroll
    for (int r = 0; r < NR; ++r) {
        const bool on = A[r].live && k0 < dim;
        s[r] = on ? ld4(x + A[r].i * (int64_t)dim + k0) : z;
        cm = A[r].c > cm ? A[r].c : cm;
    }
    for (int q0 = 0; q0 < cm; q0 += B) {
        int32_t j[NR][B];
#pragma unroll
        for (int r = 0; r < NR; ++r)
#pragma unroll
            for (int q = 0; q < B; ++q) {
                const int qq = q0 + q;
                j[r][q] = 0;
                if (qq < A[r].c) j[r][q] = qq < 32 ? __shfl_sync(0xffffffffu, A[r].my_nbr, qq & 31) : nbr[A[r].i * fanout + qq];
            }
        float4 v[NR][B];
#pragma unroll
        for (int r = 0; r < NR; ++r)
#pragma unroll
            for (int q = 0; q < B; ++q)
                v[r][q] = (A[r].live && k0 < dim && q0 + q < A[r].c) ? ld4(x + (int64_t)j[r][q] * dim + k0) : z;
#pragma unroll
        for (int r = 0; r < NR; ++r)
#pragma unroll
            for (int q = 0; q < B; ++q)
                if (q0 + q < A[r].c) add4(s[r], v[r][q]);
    }
}

template <int NR, int BATCH>
__global__ void __maxnreg__(56)
sage_mean_linear_kernel(const float* __restrict__ x, int dim, int Kc, int nchunk, const int32_t* __restrict__ nbr,
                        const int32_t* __restrict__ cnt, int fanout, const int64_t* __restrict__ n_dst_dev, int64_t n_dst_max,
                        const __nv_bfloat16* __restrict__ w, int N, uint32_t tmem_cols, float* __restrict__ y, int repeat,
                        bool x_vec, bool w_vec, unsigned long long* __restrict__ sched,
                        const __grid_constant__ CUtensorMap tmap_y, bool tma_y) {
    extern __shared__ __align__(1024) uint8_t smem[];
    uint8_t* sB = smem;                                   // [N x Kc] bf16, core-matrix K-major (one K chunk of W)
    uint8_t* sA = smem + (size_t)N * Kc * 2;              // [128 x Kc] bf16 (the same K chunk of the means)
    uint64_t* bar = reinterpret_cast<uint64_t*>(sA + (size_t)kTileM * Kc * 2);
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bar + 1);
    int64_t* s_start = reinterpret_cast<int64_t*>(bar + 2);    // dynamic schedule: the grabbed rows' start
    int32_t* s_rows = reinterpret_cast<int32_t*>(bar + 3);     // ... their count, and the first grab's size

    int64_t n = n_dst_max;
    if (n_dst_dev) {
        const int64_t m = *n_dst_dev;
        n = m < n ? m : n;
    }
    const int64_t tiles = (n + kTileM - 1) / kTileM;
    // Dynamic schedule (sched != nullptr): CTAs grab row ranges from a counter, 128 rows at a time,
    // except that the second CTA to arrive on an SM starts with 64 -- that puts the two CTAs of an SM
    // half a mean phase apart, so one's MMA + epilogue runs while the other loads rows (in step, the
    // phases added up: DESIGN.md section 4).  The first grab happens before any setup, so a CTA that
    // finds no rows left leaves at once.
    int64_t it_static = 0;
    if (sched) {
        if (threadIdx.x == 0) {
            uint32_t smid;
            asm volatile("mov.u32 %0, %%smid;" : "=r"(smid));
            const unsigned long long slot = atomicAdd(sched + 1 + (smid & 255), 1ull);
            const int want = (slot & 1) ? kTileM / 2 : kTileM;
            *s_start = (int64_t)atomicAdd(sched, (unsigned long long)want);
            *s_rows = want;
        }
        __syncthreads();
        if (*s_start >= n) return;
    } else if ((int64_t)blockIdx.x >= tiles) {
        return;   // whole CTA leaves before any TMEM / barrier use
    }

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;

    // --- setup: barrier, TMEM columns, W into shared memory -----------------------------------
    if (threadIdx.x == 0) {
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(bar)));
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_slot)),
                     "r"(tmem_cols));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    // W's columns [kc0, kc0 + Kc) into sB: cp.async for whole 16 B pieces, zero padding past dim
    auto load_w = [&](int kc0) {
        for (int c = threadIdx.x; c < N * (Kc >> 3); c += kThreads) {   // one 16 B piece (8 k) per step
            const int r = c / (Kc >> 3), kl = (c % (Kc >> 3)) * 8, kg = kc0 + kl;
            if (w_vec && kg + 8 <= dim) {
                asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(smem_u32(sB + core_off(r, kl, Kc))),
                             "l"(w + (int64_t)r * dim + kg)
                             : "memory");
            } else {
                __align__(16) __nv_bfloat16 v[8];
#pragma unroll
                for (int e = 0; e < 8; ++e) v[e] = (kg + e < dim) ? w[(int64_t)r * dim + kg + e] : __float2bfloat16_rn(0.0f);
                *reinterpret_cast<uint4*>(sB + core_off(r, kl, Kc)) = *reinterpret_cast<const uint4*>(v);
            }
        }
        asm volatile("cp.async.commit_group;" ::: "memory");
    };
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    const uint32_t tmem = *tmem_slot;
    bool w_resident = false;   // one chunk: W stays in shared memory for every tile of the CTA
    const uint32_t bar_a = smem_u32(bar);
    const uint32_t idesc = instr_desc(kTileM, N);
    const uint32_t a_base = smem_u32(sA), b_base = smem_u32(sB);
    uint32_t phase = 0;

    bool grabbed = sched != nullptr;   // the first range is already in s_start / s_rows
    for (int rep = 0; rep < repeat; ++rep) {
        it_static = 0;
        while (true) {
          int64_t r0, lim;   // rows [r0, lim) of this tile
          if (sched) {
              if (!grabbed) {
                  if (threadIdx.x == 0) *s_start = (int64_t)atomicAdd(sched, (unsigned long long)kTileM), *s_rows = kTileM;
                  __syncthreads();
              }
              grabbed = false;
              r0 = *s_start;
              if (r0 >= n) break;
              lim = r0 + *s_rows < n ? r0 + *s_rows : n;
          } else {
              const int64_t tile = blockIdx.x + it_static * gridDim.x;
              ++it_static;
              if (tile >= tiles) break;
              r0 = tile * kTileM;
              lim = r0 + kTileM < n ? r0 + kTileM : n;
          }
          for (int ci = 0; ci < nchunk; ++ci) {
            const int kc0 = ci * Kc;
            const bool load = !w_resident;   // W's chunk ci (every chunk, every tile, when K is chunked)
            if (load) load_w(kc0);
            // --- 1. h for 128 rows, columns [kc0, kc0 + Kc) -> bf16 A (warp per row, lane per 4 features)
            if (x_vec) {
                // one row per warp at a time, up to kBatch neighbour rows in flight (loads of a batch
                // issued before its adds; the adds run in q order, so h stays bit-identical to
                // dgz_aggregate_mean); the next row's count and positions load meanwhile
                RowRef A[NR];
#pragma unroll
                for (int r = 0; r < NR; ++r) A[r] = row_ref(r0 + warp + r * kWarps, lim, cnt, nbr, fanout, lane);
                for (int rr = warp; rr < kTileM; rr += NR * kWarps) {
                    RowRef An[NR];
#pragma unroll
                    for (int r = 0; r < NR; ++r) An[r] = A[r];
                    if (rr + NR * kWarps < kTileM) {
#pragma unroll
                        for (int r = 0; r < NR; ++r)
                            An[r] = row_ref(r0 + rr + (NR + r) * kWarps, lim, cnt, nbr, fanout, lane);
                    }
                    for (int kb = 0; kb < Kc; kb += 128) {
                        const int kl = kb + lane * 4;
                        float4 sa[NR];
                        sum_vec<NR, BATCH>(x, dim, kc0 + kl, A, nbr, fanout, sa);
                        if (kl < Kc) {
#pragma unroll
                            for (int r = 0; r < NR; ++r)
                                *reinterpret_cast<uint2*>(sA + core_off(rr + r * kWarps, kl, Kc)) = pack_bf16(sa[r], A[r].inv);
                        }
                    }
#pragma unroll
                    for (int r = 0; r < NR; ++r) A[r] = An[r];
                }
            } else {
                for (int rr = warp; rr < kTileM; rr += kWarps) {   // scalar loads (dim % 4 != 0 or unaligned x)
                    const RowRef A = row_ref(r0 + rr, lim, cnt, nbr, fanout, lane);
                    for (int kb = 0; kb < Kc; kb += 128) {
                        const int kl = kb + lane * 4, k0 = kc0 + kl;
                        float v[4] = {0.f, 0.f, 0.f, 0.f};
                        if (A.live) {
                            const float* xi = x + A.i * (int64_t)dim;
#pragma unroll
                            for (int e = 0; e < 4; ++e)
                                if (k0 + e < dim) v[e] = xi[k0 + e];
                            for (int q = 0; q < A.c; ++q) {
                                const int32_t j = q < 32 ? __shfl_sync(0xffffffffu, A.my_nbr, q) : nbr[A.i * fanout + q];
                                const float* xj = x + (int64_t)j * dim;
#pragma unroll
                                for (int e = 0; e < 4; ++e)
                                    if (k0 + e < dim) v[e] += xj[k0 + e];
                            }
                        }
                        if (kl < Kc)
                            *reinterpret_cast<uint2*>(sA + core_off(rr, kl, Kc)) = pack_bf16(make_float4(v[0], v[1], v[2], v[3]), A.inv);
                    }
                }
            }
            if (load) {   // this thread's W pieces have landed
                asm volatile("cp.async.wait_all;" ::: "memory");
                w_resident = nchunk == 1;
            }
            // generic-proxy stores -> visible to the tensor core (async proxy)
            asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
            __syncthreads();
            // --- 2. one thread issues the MMAs: D[tmem] (+)= A . B^T over Kc / 16 steps ---------------
            if (threadIdx.x == 0) {
                asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
                for (int s = 0; s < (Kc >> 4); ++s) {
                    const uint64_t ad = smem_desc(a_base + s * 256, Kc), bd = smem_desc(b_base + s * 256, Kc);
                    const uint32_t acc = (ci > 0 || s > 0) ? 1u : 0u;
                    asm volatile(
                        "{\n\t.reg .pred p;\n\t"
                        "setp.ne.b32 p, %4, 0;\n\t"
                        "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}\n" ::"r"(tmem),
                        "l"(ad), "l"(bd), "r"(idesc), "r"(acc));
                }
                asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(bar_a)
                             : "memory");
            }
            // the MMAs have read A and B: both may be overwritten (next chunk) and D is complete (last chunk)
            mbar_wait(bar_a, phase);
            phase ^= 1;
            asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
            if (ci + 1 < nchunk) {
                asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
                __syncthreads();   // every warp past the wait before anyone rewrites A / B
            }
          }
            // --- 3. epilogue: TMEM -> registers -> y.  Warp w reads TMEM lanes 32(w%4).. (its rows)
            if (Kc >= 128) {
                // 16-column chunks staged through the (now free) A buffer, 2 KiB per warp, so each
                // store instruction writes 8 rows x 64 contiguous bytes instead of 32 rows x 16 B
                const int quarter = warp & 3, group = warp >> 2;
                uint8_t* stage = sA + warp * 2048;
                const int64_t row0 = r0 + quarter * 32;
                for (int col = group * 16; col < N; col += 16 * (kWarps / 4)) {
                    uint32_t v[16];
                    const uint32_t taddr = tmem + ((uint32_t)(quarter * 32) << 16) + (uint32_t)col;
                    asm volatile(
                        "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
                        : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]),
                          "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15])
                        : "r"(taddr));
                    asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
                    const bool tma = tma_y && row0 + 32 <= lim;   // the warp's 32 rows all live: one TMA store
                    if (tma && lane == 0)   // the previous chunk's TMA store has read the staging buffer
                        asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
                    __syncwarp();
                    const int sw = (lane >> 1) & 3;   // 16 B-chunk swizzle (= the TMA's 64 B swizzle): conflict-free
#pragma unroll
                    for (int c = 0; c < 4; ++c)
                        *reinterpret_cast<uint4*>(stage + lane * 64 + ((c ^ sw) * 16)) =
                            make_uint4(v[4 * c], v[4 * c + 1], v[4 * c + 2], v[4 * c + 3]);
                    if (tma) {
                        // [32 rows x 16 fp32] box of y written by the TMA engine from the staging buffer
                        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
                        __syncwarp();
                        if (lane == 0) {
                            asm volatile(
                                "cp.async.bulk.tensor.2d.global.shared::cta.bulk_group [%0, {%1, %2}], [%3];" ::"l"(&tmap_y),
                                "r"(col), "r"((int32_t)row0), "r"(smem_u32(stage))
                                : "memory");
                            asm volatile("cp.async.bulk.commit_group;" ::: "memory");
                        }
                        continue;
                    }
                    __syncwarp();
#pragma unroll
                    for (int it = 0; it < 4; ++it) {
                        const int idx = it * 32 + lane, r = idx >> 2, c = idx & 3;
                        const uint4 val = *reinterpret_cast<const uint4*>(stage + r * 64 + ((c ^ ((r >> 1) & 3)) * 16));
                        if (row0 + r < lim) *reinterpret_cast<uint4*>(y + (row0 + r) * (int64_t)N + col + c * 4) = val;
                    }
                    __syncwarp();
                }
                if (tma_y && lane == 0)   // staging (= A) is rewritten by the next tile
                    asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
                __syncwarp();
            } else {
                const int quarter = warp & 3, group = warp >> 2;   // direct: 8-column chunks
                const int64_t row = r0 + quarter * 32 + lane;
                for (int col = group * 8; col < N; col += 8 * (kWarps / 4)) {
                    uint32_t v[8];
                    const uint32_t taddr = tmem + ((uint32_t)(quarter * 32) << 16) + (uint32_t)col;
                    asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                                 : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]),
                                   "=r"(v[7])
                                 : "r"(taddr));
                    asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
                    if (row < lim) {
                        float4* dst = reinterpret_cast<float4*>(y + row * (int64_t)N + col);
                        dst[0] = make_float4(__uint_as_float(v[0]), __uint_as_float(v[1]), __uint_as_float(v[2]),
                                             __uint_as_float(v[3]));
                        dst[1] = make_float4(__uint_as_float(v[4]), __uint_as_float(v[5]), __uint_as_float(v[6]),
                                             __uint_as_float(v[7]));
                    }
                }
            }
            // TMEM reads done and A free before the next tile's writes / MMAs
            asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
            __syncthreads();
        }
    }
    if (tma_y && lane == 0) asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");   // y written
    if (warp == 0) {
        asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(tmem_cols));
    }
}

}  // namespace

using namespace dgz;

// K chunk of the operands in shared memory: all of K when (hidden + 128) x K bf16 fits the budget of two
// CTAs per SM (112 KiB), else the largest multiple of 128 that does (>= 128 for hidden <= 256); the
// kernel then accumulates the chunks in TMEM, re-staging W's chunk for every tile.
static int64_t sage_chunk(int64_t dim, int64_t hidden) {
    const int64_t Kp = (dim + 15) / 16 * 16, budget = 112 * 1024 - 48;
    if ((hidden + kTileM) * Kp * 2 <= budget) return Kp;
    int64_t kc = budget / ((hidden + kTileM) * 2) / 128 * 128;
    return kc < 128 ? 128 : kc;
}

// Per-launch schedule slots for the dynamic tile schedule: a row counter and 256 per-SM arrival
// counters, in a ring of kSchedSlots per device allocated once; each launch takes the next slot and
// zeroes it on its own stream (as the gather's work counters).
static constexpr int kSchedSlots = 1024, kSchedWords = 1 + 256;
static unsigned long long* sched_slot(int dev) {
    static std::mutex mu;
    static unsigned long long* ring[64] = {};
    static std::atomic<uint32_t> next[64];
    if (dev < 0 || dev >= 64) return nullptr;
    {
        std::lock_guard<std::mutex> g(mu);
        if (!ring[dev]) {
            unsigned long long* p = nullptr;
            cudaStreamCaptureMode m = cudaStreamCaptureModeRelaxed;
            cudaThreadExchangeStreamCaptureMode(&m);
            const cudaError_t e = cudaMalloc((void**)&p, sizeof(unsigned long long) * kSchedSlots * kSchedWords);
            cudaThreadExchangeStreamCaptureMode(&m);
            if (e != cudaSuccess) return nullptr;
            ring[dev] = p;
        }
    }
    return ring[dev] + (size_t)(next[dev].fetch_add(1, std::memory_order_relaxed) % kSchedSlots) * kSchedWords;
}

// y as a TMA tensor ([rows][hidden] fp32, box 32 rows x 16 columns, 64 B swizzle = the staging layout)
static bool make_y_map(CUtensorMap* m, float* y, int64_t rows, int64_t hidden) {
    using Enc = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*, const cuuint64_t*,
                             const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                             CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
    static Enc enc = [] {
        void* p = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) != cudaSuccess ||
            q != cudaDriverEntryPointSuccess)
            return (Enc) nullptr;
        return reinterpret_cast<Enc>(p);
    }();
    if (!enc || rows <= 0 || rows > (int64_t(1) << 31)) return false;
    const cuuint64_t dims[2] = {(cuuint64_t)hidden, (cuuint64_t)rows};
    const cuuint64_t strides[1] = {(cuuint64_t)hidden * 4};
    const cuuint32_t box[2] = {16, 32}, estr[2] = {1, 1};
    return enc(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, y, dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
               CU_TENSOR_MAP_SWIZZLE_64B, CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

extern "C" dgz_status dgz_sage_workspace(int64_t dim, int64_t hidden, int64_t* smem_bytes, int32_t* tmem_cols) {
    DGZ_REQUIRE(dim >= 1 && hidden >= 1, "dgz_sage_workspace: dim and hidden must be >= 1");
    uint32_t cols = 32;
    while (cols < (uint32_t)hidden && cols < 512) cols <<= 1;
    if (smem_bytes) *smem_bytes = (hidden + kTileM) * sage_chunk(dim, hidden) * 2 + 48;
    if (tmem_cols) *tmem_cols = (int32_t)cols;
    return DGZ_OK;
}

extern "C" dgz_status dgz_sage_mean_linear(const float* x, int64_t dim, const int32_t* nbr_local, const int32_t* cnt,
                                           int32_t fanout, const int64_t* n_dst_dev, int64_t n_dst_max, const void* w_bf16,
                                           int64_t hidden, float* y, int32_t repeat, int32_t sm_count, int32_t ctas_per_sm,
                                           dgz_stream stream) {
    DGZ_REQUIRE(x && nbr_local && cnt && w_bf16 && y && dim >= 1 && fanout >= 0 && n_dst_max >= 0 && repeat >= 1,
                "dgz_sage_mean_linear: bad arguments");
    DGZ_REQUIRE(hidden >= 16 && hidden <= 256 && hidden % 16 == 0,
                "dgz_sage_mean_linear: hidden must be a multiple of 16 in [16, 256] (UMMA N with M = 128)");
    DGZ_REQUIRE(((uintptr_t)y & 15) == 0, "dgz_sage_mean_linear: y must be 16-byte aligned");
    DGZ_REQUIRE(((uintptr_t)w_bf16 & 1) == 0 && ((uintptr_t)x & 3) == 0, "dgz_sage_mean_linear: misaligned x or W");
    if (n_dst_max == 0) return DGZ_OK;
    int64_t need = 0;
    int32_t cols = 0;
    dgz_sage_workspace(dim, hidden, &need, &cols);
    const int64_t Kp = (dim + 15) / 16 * 16, Kc = sage_chunk(dim, hidden), nchunk = (Kp + Kc - 1) / Kc;
    DGZ_REQUIRE(dim < (int64_t(1) << 30), "dgz_sage_mean_linear: dim too large");
    // at most 512 / cols (>= 2) CTAs per SM may hold TMEM at once; the 56-register cap (2 x 512 x 56 of
    // the 64 K registers) already limits the kernel to 2 CTAs per SM, and leaves room for one warp of a
    // co-running gather (4 K registers) -- so shared memory is not padded: the gather's CTA fits beside two
    // of these (2 x 97 KiB for dim 128 / hidden 256; K is chunked to stay within that)
    const int64_t smem = need;
    // one row per warp at a time, neighbours loaded in batches of 6 (fanout <= 6: the whole row in one
    // batch) or 8; measured on the config-4 last hop (fanout 5): 1 x 6 0.193 ms, 1 x 8 0.197, two rows per
    // warp (2 x 4, 2 x 6) 0.209 / 0.238 -- they spill at the 64-register budget of 2 CTAs per SM
    auto kern = fanout <= 6 ? sage_mean_linear_kernel<1, 6> : sage_mean_linear_kernel<1, 8>;
    DGZ_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    const int nsm = sm_count_of_current_device();
    const int k = (sm_count > 0 && sm_count < nsm) ? sm_count : nsm;
    const int64_t tiles = (n_dst_max + kTileM - 1) / kTileM;
    int64_t blocks = tiles;
    cudaStream_t s = (cudaStream_t)stream;
    const bool x_vec = (dim % 4 == 0) && (((uintptr_t)x & 15) == 0);   // float4 row loads
    const bool w_vec = (dim % 8 == 0) && (((uintptr_t)w_bf16 & 15) == 0);   // 16 B W loads
    const __nv_bfloat16* w = reinterpret_cast<const __nv_bfloat16*>(w_bf16);
    int dev = 0;
    DGZ_CUDA(cudaGetDevice(&dev));
    // the dynamic schedule needs one pass over the rows per launch (repeat 1); DGZ_SAGE_STATIC=1 turns it off
    static const bool force_static = getenv("DGZ_SAGE_STATIC") != nullptr;
    auto sched_for = [&](int reps) -> unsigned long long* {
        if (force_static || reps != 1) return nullptr;
        unsigned long long* p = sched_slot(dev);
        if (p && cudaMemsetAsync(p, 0, sizeof(unsigned long long) * kSchedWords, s) != cudaSuccess) return nullptr;
        return p;
    };
    // TMA stores of y for the staged epilogue (K chunk >= 128); DGZ_SAGE_NO_TMA=1 keeps the warps' stores
    static const bool no_tma = getenv("DGZ_SAGE_NO_TMA") != nullptr;
    CUtensorMap ymap;
    memset(&ymap, 0, sizeof(ymap));
    const bool tma_y = !no_tma && Kc >= 128 && make_y_map(&ymap, y, n_dst_max, hidden);
    if (ctas_per_sm > 0) {
        const int64_t c = (int64_t)k * ctas_per_sm;
        if (blocks > c) blocks = c;
        kern<<<(int)blocks, kThreads, smem, s>>>(x, (int)dim, (int)Kc, (int)nchunk, nbr_local, cnt, fanout, n_dst_dev,
                                                 n_dst_max, w, (int)hidden, (uint32_t)cols, y, repeat, x_vec, w_vec,
                                                 sched_for(repeat), ymap, tma_y);
        dgz::count_launch();
    } else {
        for (int r = 0; r < repeat; ++r) {
            kern<<<(int)blocks, kThreads, smem, s>>>(x, (int)dim, (int)Kc, (int)nchunk, nbr_local, cnt, fanout,
                                                     n_dst_dev, n_dst_max, w, (int)hidden, (uint32_t)cols, y, 1, x_vec, w_vec,
                                                     sched_for(1), ymap, tma_y);
            dgz::count_launch();
        }
    }
    return launch_check("sage_mean_linear_kernel");
}
