// BULK gather variant: the TMA engine copies whole rows from the mapped host table into a
// shared-memory ring (cp.async.bulk ... mbarrier::complete_tx), consumer warps move them to
// HBM.  One bulk copy per row covers the row's 16 B-aligned span (sectors are fetched whole
// anyway), so the number of bytes in flight per SM is set by the ring size, not by registers:
// the B200 way to keep many PCIe reads outstanding from very few SMs (step a6; NEXT-3 in
// SURVEY 8(f)).  Result identical to the SEGMENT kernel (same closed form).
#include "internal.h"

namespace {

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}
__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t* bar, uint32_t tx) {
    asm volatile("mbarrier.arrive.expect_tx.release.cta.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(tx)
                 : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
    asm volatile("mbarrier.arrive.release.cta.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
    uint32_t done = 0;
    do {
        asm volatile(
            "{\n .reg .pred p;\n mbarrier.try_wait.parity.acquire.cta.shared::cta.b64 p, [%1], %2;\n selp.u32 %0, 1, 0, p;\n}\n"
            : "=r"(done)
            : "r"(smem_u32(bar)), "r"(parity)
            : "memory");
    } while (!done);
}
__device__ __forceinline__ void bulk_g2s(void* dst_smem, uint64_t src, uint32_t bytes, uint64_t* bar) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(smem_u32(dst_smem)),
        "l"(src), "r"(bytes), "r"(smem_u32(bar))
        : "memory");
}

template <int SW>
struct piece_t;
template <> struct piece_t<16> { using T = uint4; };
template <> struct piece_t<8> { using T = uint2; };
template <> struct piece_t<4> { using T = uint32_t; };
template <> struct piece_t<2> { using T = uint16_t; };
template <> struct piece_t<1> { using T = uint8_t; };

// smem layout: [full mbarriers x S][empty mbarriers x S][pad to 128 B][S slots]
template <int SW, typename IdxT>
__global__ void __launch_bounds__(1024, 1)
gather_bulk_kernel(const uint8_t* __restrict__ src, int64_t rows, int64_t R, const IdxT* __restrict__ idx,
                   const int64_t* __restrict__ dst_pos, int64_t n_cap, const int64_t* __restrict__ n_dev,
                   uint8_t* __restrict__ dst, int* __restrict__ err, int S, int slot_bytes, int blocked) {
    extern __shared__ __align__(128) uint8_t smem[];
    uint64_t* full = reinterpret_cast<uint64_t*>(smem);
    uint64_t* empty = full + S;
    uint8_t* slots = smem + (((size_t)S * 16 + 127) & ~size_t(127));

    int64_t n = n_cap;
    if (n_dev) {
        const int64_t m = *n_dev;
        n = m < n_cap ? m : n_cap;
    }
    const uint64_t base = reinterpret_cast<uint64_t>(src);
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int nwarps = blockDim.x >> 5;
    // S is a multiple of nconsumers (launch_bulk): job j and job j + S (same slot) then run on the
    // same consumer warp, so a consumer never waits on a slot's full barrier more than one phase
    // ahead of it -- the parity wait of use u cannot be satisfied by phase u - 2 (ABA)
    const int nconsumers = nwarps - 1 < S ? nwarps - 1 : S;
    if (threadIdx.x == 0) {
        for (int s = 0; s < S; ++s) {
            mbar_init(&full[s], 1);
            mbar_init(&empty[s], 1);
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    // rows of this CTA: blocked = the contiguous range [first, first + njobs), else the
    // row-cyclic set first + j * gridDim.x; job j uses slot j % S
    int64_t first, stride, njobs;
    if (blocked) {
        const int64_t per = (n + gridDim.x - 1) / gridDim.x;
        first = int64_t(blockIdx.x) * per;
        stride = 1;
        njobs = first < n ? min(per, n - first) : 0;
    } else {
        first = blockIdx.x;
        stride = gridDim.x;
        njobs = first < n ? (n - 1 - first) / stride + 1 : 0;
    }

    if (warp == 0) {
        // producer warp: per round, lanes l < step issue jobs j0 + l (step <= S, so a slot is used
        // at most once per round); __syncwarp keeps every lane in the same round, so an
        // empty-barrier wait is never more than one phase ahead (parity waits are ABA-safe)
        const int step = S < 32 ? S : 32;
        for (int64_t j0 = 0; j0 < njobs; j0 += step) {
            const int64_t j = j0 + lane;
            if (lane < step && j < njobs) {
                const int s = (int)(j % S);
                const int64_t use = j / S;
                if (use > 0) {
                    mbar_wait(&empty[s], (uint32_t)((use - 1) & 1));
                    // the consumers' generic-proxy reads of this slot precede the next async-proxy
                    // (TMA) write into it
                    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
                }
                const int64_t r = first + j * stride;
                const int64_t id = (int64_t)idx[r];
                if (id < 0 || id >= rows) {
                    atomicOr(err, 1);
                    mbar_arrive(&full[s]);
                } else {
                    const uint64_t a = base + (uint64_t)id * (uint64_t)R;
                    const uint64_t a16 = a & ~uint64_t(15);
                    const uint32_t span = (uint32_t)(((a + (uint64_t)R + 15) & ~uint64_t(15)) - a16);
                    mbar_arrive_expect_tx(&full[s], span);
                    bulk_g2s(slots + (size_t)s * slot_bytes, a16, span, &full[s]);
                }
            }
            __syncwarp();
        }
    } else if (warp - 1 < nconsumers) {
        using P = typename piece_t<SW>::T;
        for (int64_t j = warp - 1; j < njobs; j += nconsumers) {
            const int s = (int)(j % S);
            const int64_t r = first + j * stride;
            // the consumer re-derives the row's 16 B phase from its ID (no shared metadata:
            // the only shared-memory traffic is the TMA-written slot, ordered by the mbarriers)
            const int64_t id = (int64_t)idx[r];
            mbar_wait(&full[s], (uint32_t)((j / S) & 1));
            if (id >= 0 && id < rows) {
                const int off = (int)((base + (uint64_t)id * (uint64_t)R) & 15u);
                const uint8_t* sp = slots + (size_t)s * slot_bytes + off;
                uint8_t* dp = dst + (dst_pos ? dst_pos[r] : r) * R;
                for (int64_t q = (int64_t)lane * SW; q < R; q += 32 * SW)
                    *reinterpret_cast<P*>(dp + q) = *reinterpret_cast<const P*>(sp + q);
            }
            __syncwarp();
            if (lane == 0) mbar_arrive(&empty[s]);
        }
    }
}

template <int SW, typename IdxT>
cudaError_t launch_bulk(const dgz_table_s* t, const IdxT* idx, const int64_t* dst_pos, int64_t n, const int64_t* n_dev, uint8_t* out,
                        int* err, int blocks, int threads, int blocked, cudaStream_t s) {
    const int slot_bytes = (int)(((t->row_bytes + 32 + 127) / 128) * 128);
    const int max_smem = 227 * 1024;
    int S = (max_smem - 256) / (slot_bytes + 16);
    if (S > 1024) S = 1024;
    if (S < 2) return cudaErrorInvalidValue;
    // consumers = min(warps - 1, S), and S rounded down to a multiple of them (see the kernel)
    const int nc = threads / 32 - 1 < S ? threads / 32 - 1 : S;
    S = S / nc * nc;
    const size_t smem = (((size_t)S * 16 + 127) & ~size_t(127)) + (size_t)S * slot_bytes;
    cudaError_t e = cudaFuncSetAttribute(gather_bulk_kernel<SW, IdxT>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    dgz::apply_carveout((const void*)gather_bulk_kernel<SW, IdxT>);
    gather_bulk_kernel<SW, IdxT><<<blocks, threads, smem, s>>>(t->dev, t->rows, t->row_bytes, idx, dst_pos, n, n_dev, out, err, S,
                                                               slot_bytes, blocked); dgz::count_launch();
    return cudaGetLastError();
}

template <typename IdxT>
cudaError_t launch_bulk_sw(int sw, const dgz_table_s* t, const IdxT* idx, const int64_t* dst_pos, int64_t n, const int64_t* n_dev,
                           uint8_t* out, int* err, int blocks, int threads, int blocked, cudaStream_t s) {
    switch (sw) {
        case 16: return launch_bulk<16>(t, idx, dst_pos, n, n_dev, out, err, blocks, threads, blocked, s);
        case 8: return launch_bulk<8>(t, idx, dst_pos, n, n_dev, out, err, blocks, threads, blocked, s);
        case 4: return launch_bulk<4>(t, idx, dst_pos, n, n_dev, out, err, blocks, threads, blocked, s);
        case 2: return launch_bulk<2>(t, idx, dst_pos, n, n_dev, out, err, blocks, threads, blocked, s);
        default: return launch_bulk<1>(t, idx, dst_pos, n, n_dev, out, err, blocks, threads, blocked, s);
    }
}

}  // namespace

dgz_status dgz_gather_bulk(const dgz_table_s* t, const void* idx, int idx_is64, const int64_t* dst_pos, int64_t n,
                           const int64_t* n_dev, void* out, int* err, int sms, int warps, int blocked, cudaStream_t s) {
    using namespace dgz;
    DGZ_REQUIRE(t->row_bytes <= 64 * 1024, "BULK gather: rows above 64 KiB are not supported");
    if (warps < 2) warps = 2;
    // the SW store width must divide the row, the table base and the output base: the slot
    // keeps the source's 16 B phase, so the smem read address is SW-aligned as well
    const uint64_t x = (uint64_t)t->row_bytes | ((uint64_t)(uintptr_t)t->dev & 15u) | ((uint64_t)(uintptr_t)out & 15u) | 16u;
    const int sw = (int)(x & (~x + 1));
    cudaError_t e;
    if (idx_is64)
        e = launch_bulk_sw<int64_t>(sw, t, (const int64_t*)idx, dst_pos, n, n_dev, (uint8_t*)out, err, sms, warps * 32, blocked, s);
    else
        e = launch_bulk_sw<int32_t>(sw, t, (const int32_t*)idx, dst_pos, n, n_dev, (uint8_t*)out, err, sms, warps * 32, blocked, s);
    if (e != cudaSuccess) return cuda_fail(e, "bulk gather launch");
    return DGZ_OK;
}
