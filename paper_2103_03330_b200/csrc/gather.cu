// Sparse feature gather over PCIe zero-copy (step a4, the hot path).
//
//   out[r*R + b] = table[idx[r]*R + b]     (Listing 2; closed form)
//
// SEGMENT kernel (the product).  The paper's circular shift (fig:auto_alignment)
// exists so that a warp's loads start on 128 B line boundaries and every PCIe read request
// carries as many useful bytes as possible.  On sm_100a we get the same goal directly, per
// row: a row that starts at byte a and has R bytes touches L = ceil(((a mod 128) + R) / 128)
// lines, and the kernel issues exactly one warp-cooperative 128 B-aligned segment load per
// line (8 lanes x 16 B, LDG.E.128), i.e. the per-row minimum number of PCIe reads (SURVEY
// 8(a) a4').  A warp owns 32 rows at a time; lane i loads row i's ID, computes its line count,
// and a warp inclusive scan turns the 32 rows into a flat list of line tasks; each warp load
// instruction serves 4 line tasks (4 groups of 8 lanes), U instructions are issued back to
// back before any store so that 4*U lines per warp are in flight over PCIe.  Loads are always
// 16 B and line aligned (whatever the row alignment: sectors are fetched whole anyway);
// stores go to HBM in the widest piece SW in {16,8,4,2,1} that divides R and both base
// addresses, so no byte outside the row is ever written and no shared-memory realignment is
// needed.  HBM stores of a warp instruction are contiguous per line group (coalesced).
//
// NAIVE / SHIFT kernels: the paper's Listing 2 without / with the circular shift stage, one
// element per thread (ablations for the fig:alignment_measurement analogue).  The shift
// aligns to 128 BYTES (W = 128 / sizeof(T) elements; reading R3) with 64-bit offsets (R4).
#include <atomic>
#include <mutex>

#include "internal.h"

namespace {

__device__ __forceinline__ uint4 ld_zc_v4(uint64_t p) {
    uint4 r;
    asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];"
                 : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w)
                 : "l"(p));
    return r;
}
__device__ __forceinline__ uint4 ld_zc_v4_hint(uint64_t p, uint64_t pol) {
    uint4 r;
    asm volatile("ld.global.nc.L1::no_allocate.L2::cache_hint.v4.u32 {%0,%1,%2,%3}, [%4], %5;"
                 : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w)
                 : "l"(p), "l"(pol));
    return r;
}
__device__ __forceinline__ uint64_t l2_evict_first_policy() {
    uint64_t pol;
    asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
    return pol;
}
__device__ __forceinline__ void st_g(uint64_t d, uint4 v) {
    asm volatile("st.global.v4.u32 [%0], {%1,%2,%3,%4};" ::"l"(d), "r"(v.x), "r"(v.y), "r"(v.z), "r"(v.w) : "memory");
}
__device__ __forceinline__ void st_g_cs(uint64_t d, uint4 v) {  // streaming store: evict-first in L2
    asm volatile("st.global.cs.v4.u32 [%0], {%1,%2,%3,%4};" ::"l"(d), "r"(v.x), "r"(v.y), "r"(v.z), "r"(v.w) : "memory");
}
__device__ __forceinline__ void st_g(uint64_t d, uint2 v) {
    asm volatile("st.global.v2.u32 [%0], {%1,%2};" ::"l"(d), "r"(v.x), "r"(v.y) : "memory");
}
__device__ __forceinline__ void st_g32(uint64_t d, uint32_t v) { asm volatile("st.global.u32 [%0], %1;" ::"l"(d), "r"(v) : "memory"); }
__device__ __forceinline__ void st_g16(uint64_t d, uint32_t v) {
    asm volatile("st.global.u16 [%0], %1;" ::"l"(d), "h"((unsigned short)v) : "memory");
}
__device__ __forceinline__ void st_g8(uint64_t d, uint32_t v) {
    asm volatile("st.global.u8 [%0], %1;" ::"l"(d), "h"((unsigned short)(v & 0xff)) : "memory");
}

template <int SW>
__device__ __forceinline__ void store_pieces(uint64_t d, const uint4& v, int lo, int hi, bool cs = false) {
    // store bytes [lo, hi) of the 16-byte chunk v (lo, hi multiples of SW) at global address d + byte
    if constexpr (SW == 16) {
        if (cs) st_g_cs(d, v);
        else st_g(d, v);
    } else if constexpr (SW == 8) {
        if (lo <= 0 && hi >= 8) st_g(d, make_uint2(v.x, v.y));
        if (lo <= 8 && hi >= 16) st_g(d + 8, make_uint2(v.z, v.w));
    } else if constexpr (SW == 4) {
        const uint32_t w[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
        for (int p = 0; p < 4; ++p)
            if (p * 4 >= lo && p * 4 < hi) st_g32(d + 4 * p, w[p]);
    } else if constexpr (SW == 2) {
        const uint32_t w[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
        for (int p = 0; p < 8; ++p)
            if (p * 2 >= lo && p * 2 < hi) st_g16(d + 2 * p, w[p >> 1] >> (16 * (p & 1)));
    } else {
        const uint32_t w[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
        for (int p = 0; p < 16; ++p)
            if (p >= lo && p < hi) st_g8(d + p, w[p >> 2] >> (8 * (p & 3)));
    }
}

// HBM row cache: slot[id] >= 0 -> the row lives in shard (slot % G) at
// row (slot / G) (local HBM, or a peer GPU's HBM mapped into this address space).
struct CacheArgs {
    const int32_t* slot;
    int32_t G;
    const uint8_t* shard[DGZ_MAX_CACHE_SHARDS];
};

template <int SW, int U, bool MERGE, bool CACHED, typename IdxT>
__global__ void __launch_bounds__(512, 1)
gather_segment_kernel(const uint8_t* __restrict__ src, int64_t rows, int64_t R, const IdxT* __restrict__ idx,
                      const int64_t* __restrict__ dst_pos, int64_t n_cap, const int64_t* __restrict__ n_dev,
                      uint8_t* __restrict__ dst, int* __restrict__ err, int blocked, const CacheArgs ca, int hints,
                      unsigned long long* __restrict__ ctr) {
    int64_t n = n_cap;
    if (n_dev) {
        const int64_t m = *n_dev;
        n = m < n_cap ? m : n_cap;
    }
    const int lane = threadIdx.x & 31;
    const int g = lane >> 3;
    const int sub = lane & 7;
    const uint64_t base = reinterpret_cast<uint64_t>(src);
    const uint64_t dbase = reinterpret_cast<uint64_t>(dst);
    // cache hints (DGZ_GATHER_FLAG_STREAM_STORES / _EVICT_FIRST_LOADS): keep the streamed rows from
    // displacing the GPU page-table lines the MMU walks for the zero-copy loads
    const bool cs_stores = hints & 1;
    const bool ef_loads = hints & 2;
    const uint64_t pol = ef_loads ? l2_evict_first_policy() : 0;

    // Schedule of 32-row batches.  Interleaved: warp w of the grid takes batches w, w + W, ...
    // Blocked (translation-aware): CTA c owns a contiguous range of batches and its warps
    // interleave inside it, so each SM walks its own address range monotonically when the
    // index list is sorted (one GPU TLB miss per 2 MiB region per SM instead of per row).
    const int64_t nb = (n + 31) >> 5;
    const int wid = threadIdx.x >> 5;
    const int wpc = blockDim.x >> 5;
    int64_t bcur, bend, bstep;
    if (blocked) {
        const int64_t per = (nb + gridDim.x - 1) / gridDim.x;
        bcur = int64_t(blockIdx.x) * per + wid;
        bend = min(nb, int64_t(blockIdx.x + 1) * per);
        bstep = wpc;
    } else {
        bcur = int64_t(blockIdx.x) * wpc + wid;
        bend = nb;
        bstep = int64_t(gridDim.x) * wpc;
    }

    // Software-pipelined index loads: IDs two batches ahead, the cache slot (which depends on the
    // ID) one batch ahead, the destination row one batch ahead -- none of them stalls the PCIe
    // loads of the current batch.
    auto load_id = [&](int64_t bb) -> int64_t {
        const int64_t rr = (bb << 5) + lane;
        return (bb < bend && rr < n) ? (int64_t)idx[rr] : -1;
    };
    auto load_dp = [&](int64_t bb) -> int64_t {
        const int64_t rr = (bb << 5) + lane;
        return (bb < bend && rr < n) ? (dst_pos ? dst_pos[rr] : rr) : -1;
    };
    auto load_slot = [&](int64_t id) -> int32_t {
        if constexpr (CACHED) return (id >= 0 && id < rows) ? ca.slot[id] : -1;
        return -1;
    };
    // Batch order: static (warp w takes w, w + W, ...) or, with a work counter (ctr != nullptr,
    // DGZ_GATHER_FLAG_DYNAMIC), grabbed in ascending order by whichever warp is free -- the sorted
    // list is still swept as one narrow window, and warps on SMs that walk the page tables faster
    // take more batches instead of every warp waiting for the slowest SM at the end.
    const bool dyn = ctr != nullptr && !blocked;
    auto grab = [&]() -> int64_t {
        unsigned long long v = 0;
        if (lane == 0) v = atomicAdd(ctr, 1ull);
        return (int64_t)__shfl_sync(0xffffffffu, v, 0);
    };
    int64_t bn1, bn2;   // the next two batches of this warp (index loads run ahead on them)
    if (dyn) {
        bcur = grab();
        bn1 = grab();
        bn2 = grab();
    } else {
        bn1 = bcur + bstep;
        bn2 = bcur + 2 * bstep;
    }
    int64_t id_n1 = load_id(bcur), id_n2 = load_id(bn1);
    int64_t dp_n1 = load_dp(bcur);
    int32_t sl_n1 = load_slot(id_n1);

    unsigned long long pend = 0;   // lane 0's grab for the batch after bn2, in flight during this batch
    for (; bcur < bend; bcur = bn1, bn1 = bn2, bn2 = dyn ? (int64_t)__shfl_sync(0xffffffffu, pend, 0) : bn2 + bstep) {
        if (dyn && lane == 0) pend = atomicAdd(ctr, 1ull);   // consumed only at the loop's end: no stall
        const int64_t b0 = bcur << 5;
        const int64_t r = b0 + lane;
        int64_t id = id_n1;
        const int64_t drow = dp_n1;
        const int32_t slot = sl_n1;
        id_n1 = id_n2;
        sl_n1 = load_slot(id_n1);
        dp_n1 = load_dp(bn1);
        id_n2 = load_id(bn2);
        if (r < n && (id < 0 || id >= rows)) {
            atomicOr(err, 1);
            id = -1;
        }
        if (r >= n) id = -1;
        uint64_t a = base + (uint64_t)(id < 0 ? 0 : id) * (uint64_t)R;
        if constexpr (CACHED) {
            if (id >= 0 && slot >= 0)
                a = reinterpret_cast<uint64_t>(ca.shard[slot % ca.G]) + (uint64_t)(slot / ca.G) * (uint64_t)R;
        }
        const uint64_t l0 = a & ~uint64_t(127);
        int nl = id < 0 ? 0 : (int)((a + (uint64_t)R - l0 + 127) >> 7);
        // MERGE (sorted lists, R >= 128): a row that starts where the previous row of the batch
        // ends shares that row's last 128 B line; the line is fetched once (by the previous row's
        // task) and stored to both rows -- one PCIe read per distinct line of the batch, which is
        // never more than Listing 2's flat enumeration either (SURVEY 8(a) a4')
        unsigned mmask = 0;
        if constexpr (MERGE) {
            const uint64_t a_prev = __shfl_up_sync(0xffffffffu, a, 1);
            const int64_t id_prev = __shfl_up_sync(0xffffffffu, id, 1);
            const bool mp = lane > 0 && id >= 0 && id_prev >= 0 && a_prev + (uint64_t)R == a && (a & 127u) != 0;
            mmask = __ballot_sync(0xffffffffu, mp);
            nl -= mp ? 1 : 0;
        }
        int incl = nl;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const int v = __shfl_up_sync(0xffffffffu, incl, o);
            if (lane >= o) incl += v;
        }
        const int excl = incl - nl;
        const int T = __shfl_sync(0xffffffffu, incl, 31);

        for (int t0 = 0; t0 < T; t0 += 4 * U) {
            uint4 v[U];
            int pk[U];  // (offset of the chunk in its row + 128) << 5 | row lane, or -1 if idle
#pragma unroll
            for (int u = 0; u < U; ++u) {
                const int tb = t0 + 4 * u;
                const unsigned m0 = __ballot_sync(0xffffffffu, incl <= tb);
                const unsigned m1 = __ballot_sync(0xffffffffu, incl <= tb + 1);
                const unsigned m2 = __ballot_sync(0xffffffffu, incl <= tb + 2);
                const unsigned m3 = __ballot_sync(0xffffffffu, incl <= tb + 3);
                const unsigned m = g == 0 ? m0 : (g == 1 ? m1 : (g == 2 ? m2 : m3));
                const int t = tb + g;
                const int rho = __popc(m);  // first lane whose inclusive count exceeds t
                const int sl = rho < 32 ? rho : 31;
                const uint64_t ar = __shfl_sync(0xffffffffu, a, sl);
                const int er = __shfl_sync(0xffffffffu, excl, sl);
                // chunk = 16 B piece `sub` of line (t - er) of the row's 128 B-aligned segment list
                // (shifted by one line when the row's first line was merged into the previous row)
                const int line = t - er + (MERGE ? (int)((mmask >> sl) & 1u) : 0);
                const int q = (int)(ar & 127u);               // row start offset within its first line
                const int cq = line * 128 + sub * 16 - q;      // chunk start relative to the row start
                const bool nxt = MERGE && sl < 31 && ((mmask >> (sl + 1)) & 1u);
                const bool act = (t < T) && (cq + 16 > 0) && (cq < (int)R || nxt);
                pk[u] = act ? (((cq + 128) << 5) | sl) : -1;
                if (act) v[u] = ef_loads ? ld_zc_v4_hint(ar + (uint64_t)(int64_t)cq, pol) : ld_zc_v4(ar + (uint64_t)(int64_t)cq);
            }
#pragma unroll
            for (int u = 0; u < U; ++u) {
                const int sl = pk[u] & 31;
                const int64_t dr = __shfl_sync(0xffffffffu, drow, sl);
                int64_t dr2 = 0;
                if constexpr (MERGE) dr2 = __shfl_sync(0xffffffffu, drow, sl < 31 ? sl + 1 : 31);
                if (pk[u] >= 0) {
                    const int cq = (pk[u] >> 5) - 128;
                    if (cq < (int)R) {
                        const uint64_t d = dbase + (uint64_t)dr * (uint64_t)R + (uint64_t)(int64_t)cq;
                        store_pieces<SW>(d, v[u], cq < 0 ? -cq : 0, (int)R - cq > 16 ? 16 : (int)R - cq, cs_stores);
                    }
                    if constexpr (MERGE) {
                        // bytes past this row's end belong to the next row when it was merged
                        const bool nxt = sl < 31 && ((mmask >> (sl + 1)) & 1u);
                        if (nxt && cq + 16 > (int)R) {
                            const int lo2 = (int)R - cq > 0 ? (int)R - cq : 0;
                            const uint64_t d2 = dbase + (uint64_t)dr2 * (uint64_t)R + (uint64_t)(int64_t)(cq - (int)R);
                            store_pieces<SW>(d2, v[u], lo2, 16, cs_stores);
                        }
                    }
                }
            }
        }
    }
}

// Listing 2, one element per thread; SHIFT adds the circular-shift stage.
template <typename T, bool SHIFT, typename IdxT>
__global__ void __launch_bounds__(512)
gather_elem_kernel(const T* __restrict__ src, int64_t rows, int64_t F, const IdxT* __restrict__ idx, int64_t n_cap,
                   const int64_t* __restrict__ n_dev, T* __restrict__ dst, int* __restrict__ err) {
    int64_t n = n_cap;
    if (n_dev) {
        const int64_t m = *n_dev;
        n = m < n_cap ? m : n_cap;
    }
    constexpr int64_t W = 128 / sizeof(T);  // 128 bytes in elements (reading R3)
    const int64_t num = n * F;
    for (int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < num; i += int64_t(gridDim.x) * blockDim.x) {
        const int64_t dst_idx = i / F;
        const int64_t offset = i % F;  // reading R1 (P:406-407 garbled)
        const int64_t id = (int64_t)idx[dst_idx];
        if (id < 0 || id >= rows) {
            if (offset == 0) atomicOr(err, 1);
            continue;
        }
        const int64_t dst_start = dst_idx * F;
        const int64_t src_start = id * F;
        int64_t dst_off = offset + dst_start;
        int64_t src_off = offset + src_start;
        if (SHIFT && F > W && (F % W)) {
            int64_t diff = (dst_start - src_start) % W;
            diff = diff < 0 ? diff + W : diff;
            dst_off += diff;
            src_off += diff;
            if (src_off < src_start) {
                dst_off += F;
                src_off += F;
            } else if (src_off >= src_start + F) {
                dst_off -= F;
                src_off -= F;
            }
        }
        dst[dst_off] = src[src_off];
    }
}

struct SegLaunch {
    const CacheArgs* cache;
    int flags;
    const int64_t* dst_pos;
    int64_t n;
    const int64_t* n_dev;
    uint8_t* out;
    int* err;
    int blocks, threads, blocked;
    cudaStream_t s;
    unsigned long long* ctr;   // zeroed work counter (DGZ_GATHER_FLAG_DYNAMIC) or nullptr
};

inline int hints_of(int flags) {
    return ((flags & DGZ_GATHER_FLAG_STREAM_STORES) ? 1 : 0) | ((flags & DGZ_GATHER_FLAG_EVICT_FIRST_LOADS) ? 2 : 0);
}

template <int SW, int U, bool MERGE, typename IdxT>
void launch_segment_k(const dgz_table_s* t, const IdxT* idx, const SegLaunch& L) {
    dgz::apply_carveout(L.cache ? (const void*)gather_segment_kernel<SW, U, MERGE, true, IdxT>
                                : (const void*)gather_segment_kernel<SW, U, MERGE, false, IdxT>);
    if (L.cache) {
        gather_segment_kernel<SW, U, MERGE, true, IdxT><<<L.blocks, L.threads, 0, L.s>>>(
            t->dev, t->rows, t->row_bytes, idx, L.dst_pos, L.n, L.n_dev, L.out, L.err, L.blocked, *L.cache, hints_of(L.flags),
            L.ctr);
    } else {
        gather_segment_kernel<SW, U, MERGE, false, IdxT><<<L.blocks, L.threads, 0, L.s>>>(
            t->dev, t->rows, t->row_bytes, idx, L.dst_pos, L.n, L.n_dev, L.out, L.err, L.blocked, CacheArgs{}, hints_of(L.flags),
            L.ctr);
    }
    dgz::count_launch();
}

template <int SW, typename IdxT>
cudaError_t launch_segment(const dgz_table_s* t, const IdxT* idx, const SegLaunch& L) {
    // merging shared boundary lines pays only for address-sorted lists of rows >= 128 B
    const bool merge = L.dst_pos != nullptr && t->row_bytes >= 128 && !(L.flags & DGZ_GATHER_FLAG_NO_MERGE);
    const bool deep = L.flags & DGZ_GATHER_FLAG_DEEP;
    if (deep) {
        if (merge) launch_segment_k<SW, 16, true>(t, idx, L);
        else launch_segment_k<SW, 16, false>(t, idx, L);
    } else {
        if (merge) launch_segment_k<SW, 8, true>(t, idx, L);
        else launch_segment_k<SW, 8, false>(t, idx, L);
    }
    return cudaGetLastError();
}

template <typename IdxT>
cudaError_t launch_segment_sw(int sw, const dgz_table_s* t, const IdxT* idx, const SegLaunch& L) {
    switch (sw) {
        case 16: return launch_segment<16>(t, idx, L);
        case 8: return launch_segment<8>(t, idx, L);
        case 4: return launch_segment<4>(t, idx, L);
        case 2: return launch_segment<2>(t, idx, L);
        default: return launch_segment<1>(t, idx, L);
    }
}

template <bool SHIFT, typename IdxT>
cudaError_t launch_elem(const dgz_table_s* t, const IdxT* idx, int64_t n, const int64_t* n_dev, void* out, int* err, int blocks,
                        cudaStream_t s) {
    switch (t->elem_bytes) {
        case 4:
            dgz::apply_carveout((const void*)gather_elem_kernel<uint32_t, SHIFT, IdxT>);
            gather_elem_kernel<uint32_t, SHIFT, IdxT><<<blocks, 512, 0, s>>>((const uint32_t*)t->dev, t->rows, t->dim, idx, n, n_dev,
                                                                           (uint32_t*)out, err); dgz::count_launch();
            break;
        case 2:
            dgz::apply_carveout((const void*)gather_elem_kernel<uint16_t, SHIFT, IdxT>);
            gather_elem_kernel<uint16_t, SHIFT, IdxT><<<blocks, 512, 0, s>>>((const uint16_t*)t->dev, t->rows, t->dim, idx, n, n_dev,
                                                                           (uint16_t*)out, err); dgz::count_launch();
            break;
        default:
            dgz::apply_carveout((const void*)gather_elem_kernel<uint8_t, SHIFT, IdxT>);
            gather_elem_kernel<uint8_t, SHIFT, IdxT><<<blocks, 512, 0, s>>>((const uint8_t*)t->dev, t->rows, t->dim, idx, n, n_dev,
                                                                          (uint8_t*)out, err); dgz::count_launch();
    }
    return cudaGetLastError();
}

}  // namespace

using namespace dgz;

dgz_status dgz_gather_bulk(const dgz_table_s* t, const void* idx, int idx_is64, const int64_t* dst_pos, int64_t n,
                           const int64_t* n_dev, void* out, int* err, int sms, int warps, int blocked, cudaStream_t s);

// Launch shape of a gather: the caller's cfg where given, else the measured defaults (DESIGN.md
// section 5).  Shared by the gathers and dgz_gather_plan (which reports it).
struct LaunchPlan {
    int variant, k, warps, cps, flags, blocked;
};

static LaunchPlan plan_launch(const dgz_table_s* t, int64_t n, bool sorted_path, const dgz_gather_cfg* cfg, bool cache) {
    const int nsm = sm_count_of_current_device();
    int variant = cfg ? cfg->variant : DGZ_GATHER_AUTO;
    if (variant == DGZ_GATHER_AUTO) variant = DGZ_GATHER_SEGMENT;
    const bool bounded = cfg && cfg->sm_count > 0;
    // Defaults measured on B200.  Unsorted lists: the whole GPU keeps as
    // many rows in flight as possible to ride out GPU address-translation misses.  Sorted lists
    // (dgz_gather_perm): a narrow in-flight window (1-2 warps per SM, 16 line loads per lane,
    // shaped by row width and sparsity below) keeps translations local and still covers the PCIe
    // bandwidth-delay product; it also leaves SMs free.
    int k = bounded ? (cfg->sm_count < nsm ? cfg->sm_count : nsm) : nsm;
    const bool hbm_table = t->flags & DGZ_REG_DEVICE;   // HBM-resident: latency-bound, wants many warps
    // HBM-resident tables (All-in-GPU): 8 warps x 8 CTAs per SM (explore31: 2.94 TB/s of rows =
    // 91 % of the HBM copy bandwidth counting reads and writes, in frontier order)
    int warps = (cfg && cfg->warps_per_cta > 0) ? cfg->warps_per_cta
                                                : (variant == DGZ_GATHER_BULK ? 8 : ((sorted_path && !hbm_table) ? 2 :
                                                                                     (hbm_table ? 8 : 16)));
    int flags = cfg ? cfg->flags : 0;
    if (sorted_path && !hbm_table && !bounded && !(cfg && cfg->warps_per_cta > 0) &&
        (flags & ~(DGZ_GATHER_FLAG_NO_MERGE | DGZ_GATHER_FLAG_STREAM_STORES | DGZ_GATHER_FLAG_EVICT_FIRST_LOADS |
                   DGZ_GATHER_FLAG_DYNAMIC)) == 0) {
        flags |= DGZ_GATHER_FLAG_DEEP;
        if (variant == DGZ_GATHER_SEGMENT && (t->flags & DGZ_REG_MANAGED)) {
            // managed host table (2 MiB GPU pages, no page-walk bound; DESIGN.md 5.1,
            // tools/managed_shape_sweep.py): rows of one line are bound by the link's request rate
            // and want one warp per SM; rows of >= 2 lines reach the link with 4 (256 B random rows
            // 48.1 -> 50.9 GB/s, 512 B 49.1 -> 51.0; cached gather, 20 % of the power-law graph in
            // HBM: 103.5 -> 117.2 GB/s effective, tools/cache_managed_shapes.py)
            const int64_t lines = (t->row_bytes + 127) / 128;
            k = nsm;
            warps = lines >= 2 ? 4 : 1;
        } else if (variant == DGZ_GATHER_SEGMENT && !cache) {
            // Translation-bound regime (explore19-22): below ~1 KiB per row
            // the rate is set by GPU page walks, and it peaks with FEWER rows (distinct pages) in
            // flight than the 2-warps-per-SM shape that dense 512 B minibatches want.  Measured rule
            // (each warp keeps 64 line tasks in flight): rows >= 1 KiB or dense rows of >= 4 lines
            // (< 80 KiB apart): 2 warps per SM; sparse (> 150 KiB apart): one warp on half the SMs;
            // otherwise one warp per SM.
            const int64_t lines = (t->row_bytes + 127) / 128;
            const double gap = (double)t->rows * (double)t->row_bytes / (double)n;
            if (lines >= 8 || (lines >= 4 && gap < 80.0 * 1024.0)) {
                k = nsm;
                warps = 2;
            } else if (gap > 150.0 * 1024.0) {
                k = nsm / 2 > 0 ? nsm / 2 : 1;
                warps = 1;
            } else {
                k = nsm;
                warps = 1;
            }
        } else if (variant == DGZ_GATHER_SEGMENT && cache) {
            // cached gather: the rows left for PCIe are the sparse part of the list (the hot rows
            // come from HBM), i.e. the translation-bound regime -- one warp per SM (explore30:
            // 5 % / 20 % cached on the power-law graph, 54 -> 67 / 78 -> 91 GB/s effective)
            k = nsm;
            warps = 1;
        }
    }
    const int max_warps = variant == DGZ_GATHER_SEGMENT ? 16 : 32;  // SEGMENT: <= 512 threads (128 regs)
    if (warps > max_warps) warps = max_warps;
    int cps = (cfg && cfg->ctas_per_sm > 0) ? cfg->ctas_per_sm : (hbm_table ? 8 : 1);
    if (warps * cps > 64) cps = 64 / warps > 0 ? 64 / warps : 1;
    const int sched = cfg ? cfg->schedule : DGZ_SCHED_AUTO;
    const int blocked = sched == DGZ_SCHED_BLOCKED;
    return LaunchPlan{variant, k, warps, cps, flags, blocked};
}

// Work counters of DGZ_GATHER_FLAG_DYNAMIC launches: a ring of kWorkCounters 8-byte slots per
// device, allocated on first use and kept for the process.  Each launch takes the next slot and
// zeroes it on its own stream, so launches on one stream are ordered, and launches on different
// streams collide only if kWorkCounters of them are in flight at once.
static constexpr int kWorkCounters = 4096;

static unsigned long long* work_counter_slot(int dev) {
    static std::mutex mu;
    static unsigned long long* ring[64] = {};
    static std::atomic<uint32_t> next[64];
    if (dev < 0 || dev >= 64) { set_error("dgz_gather: device %d out of range", dev); return nullptr; }
    {
        std::lock_guard<std::mutex> g(mu);
        if (!ring[dev]) {
            unsigned long long* p = nullptr;
            // allowed even while the caller's stream is being captured into a CUDA graph
            cudaStreamCaptureMode m = cudaStreamCaptureModeRelaxed;
            cudaThreadExchangeStreamCaptureMode(&m);
            const cudaError_t e = cudaMalloc((void**)&p, sizeof(unsigned long long) * kWorkCounters);
            cudaThreadExchangeStreamCaptureMode(&m);
            if (e != cudaSuccess) { cuda_fail(e, "cudaMalloc (work counters)"); return nullptr; }
            ring[dev] = p;
        }
    }
    return ring[dev] + (next[dev].fetch_add(1, std::memory_order_relaxed) % kWorkCounters);
}

dgz_status dgz_gather_impl(dgz_table t, const void* idx, int idx_is64, const int64_t* dst_pos, int64_t n, const int64_t* n_dev,
                           void* out, const dgz_gather_cfg* cfg, cudaStream_t s, const dgz_cache_view* cache) {
    DGZ_REQUIRE(t, "dgz_gather: null table");
    DGZ_REQUIRE(n >= 0, "dgz_gather: n < 0");
    if (n == 0) return DGZ_OK;
    DGZ_REQUIRE(idx && out, "dgz_gather: null idx or out");
    DGZ_REQUIRE(((uintptr_t)out % (uintptr_t)t->elem_bytes) == 0, "dgz_gather: out not aligned to the element size");
    {
        const uint8_t* o = (const uint8_t*)out;
        const uint8_t* tb = t->host;
        const uint8_t* te = t->host + t->rows * t->row_bytes;
        DGZ_REQUIRE(o + n * t->row_bytes <= tb || o >= te, "dgz_gather: out aliases the table");
    }
    int dev = 0;
    DGZ_CUDA(cudaGetDevice(&dev));
    if (dev != t->device && (t->flags & DGZ_REG_VMM_BACKED)) {
        // VMM host memory is mapped only into the devices granted access: grant this one on
        // demand (a no-op once granted) instead of letting the kernel touch an unmapped address
        const int g = dgz_vmm_register(t->host, (size_t)t->rows * (size_t)t->row_bytes);
        if (g != 1) {
            if (g < 0) return (dgz_status)(-g);
            set_error("dgz_gather: VMM table not accessible from device %d", dev);
            return DGZ_ERR_STATE;
        }
    } else if (dev != t->device && (t->flags & DGZ_REG_MANAGED)) {
        // managed memory is mapped only into the devices advised AccessedBy: add this one on its
        // first gather (the bit is set after the advice succeeded; a race only repeats the advice)
        const uint64_t bit = dev < 64 ? uint64_t(1) << dev : 0;
        if (!(__atomic_load_n(&t->managed_devs, __ATOMIC_ACQUIRE) & bit)) {
            DGZ_CUDA(cudaMemAdvise(t->host, (size_t)t->rows * (size_t)t->row_bytes, cudaMemAdviseSetAccessedBy, dev));
            __atomic_fetch_or(&t->managed_devs, bit, __ATOMIC_RELEASE);
        }
    } else if (dev != t->device && !(t->flags & DGZ_REG_PORTABLE)) {
        set_error("dgz_gather: table registered on device %d without DGZ_REG_PORTABLE, current device %d", t->device, dev);
        return DGZ_ERR_STATE;
    }
    int* err = dgz_table_flag(t);
    if (!err) { set_error("dgz_gather: cannot allocate the device flag"); return DGZ_ERR_CUDA; }
    const LaunchPlan P = plan_launch(t, n, dst_pos != nullptr, cfg, cache != nullptr);
    const int variant = P.variant, k = P.k, warps = P.warps, cps = P.cps, flags = P.flags, blocked = P.blocked;
    DGZ_REQUIRE(!dst_pos || variant == DGZ_GATHER_SEGMENT || variant == DGZ_GATHER_BULK,
                "dgz_gather: destination permutation needs the SEGMENT or BULK variant");

    cudaError_t e = cudaSuccess;
    if (variant == DGZ_GATHER_SEGMENT) {
        DGZ_REQUIRE(t->row_bytes < (int64_t(1) << 25), "dgz_gather: rows of 32 MiB or more are not supported");
        int64_t batches = (n + 31) / 32;
        int64_t blocks = (int64_t)k * cps;
        int64_t need = (batches + warps - 1) / warps;
        if (blocks > need) blocks = need;
        uint64_t x = (uint64_t)t->row_bytes | ((uint64_t)(uintptr_t)t->dev & 15u) | ((uint64_t)(uintptr_t)out & 15u) | 16u;
        CacheArgs ca{};
        if (cache) {
            DGZ_REQUIRE(cache->slot_map && cache->n_shards >= 1 && cache->n_shards <= DGZ_MAX_CACHE_SHARDS,
                        "dgz_gather_cached: bad cache view");
            ca.slot = cache->slot_map;
            ca.G = cache->n_shards;
            for (int g = 0; g < ca.G; ++g) {
                DGZ_REQUIRE(cache->shards[g], "dgz_gather_cached: null shard %d", g);
                ca.shard[g] = (const uint8_t*)cache->shards[g];
                x |= (uint64_t)(uintptr_t)cache->shards[g] & 15u;   // stores must suit every source base
            }
        }
        const int sw = (int)(x & (~x + 1));
        unsigned long long* ctr = nullptr;
        if (flags & DGZ_GATHER_FLAG_DYNAMIC) {
            // the work counter: one 8-byte slot of a per-device ring allocated once, zeroed in
            // stream order before the launch (no allocation per launch, no pool attribute change)
            ctr = work_counter_slot(dev);
            if (!ctr) return DGZ_ERR_CUDA;
            DGZ_CUDA(cudaMemsetAsync(ctr, 0, sizeof(unsigned long long), s));
        }
        SegLaunch L{cache ? &ca : nullptr, flags, dst_pos, n, n_dev, (uint8_t*)out, err, (int)blocks, warps * 32, blocked, s, ctr};
        if (idx_is64)
            e = launch_segment_sw<int64_t>(sw, t, (const int64_t*)idx, L);
        else
            e = launch_segment_sw<int32_t>(sw, t, (const int32_t*)idx, L);
    } else if (variant == DGZ_GATHER_NAIVE || variant == DGZ_GATHER_SHIFT) {
        int64_t blocks = (int64_t)k * 4;
        const bool sh = variant == DGZ_GATHER_SHIFT;
        if (idx_is64)
            e = sh ? launch_elem<true>(t, (const int64_t*)idx, n, n_dev, out, err, (int)blocks, s)
                   : launch_elem<false>(t, (const int64_t*)idx, n, n_dev, out, err, (int)blocks, s);
        else
            e = sh ? launch_elem<true>(t, (const int32_t*)idx, n, n_dev, out, err, (int)blocks, s)
                   : launch_elem<false>(t, (const int32_t*)idx, n, n_dev, out, err, (int)blocks, s);
    } else if (variant == DGZ_GATHER_BULK) {
        return dgz_gather_bulk(t, idx, idx_is64, dst_pos, n, n_dev, out, err, k, warps, blocked, s);
    } else {
        set_error("dgz_gather: unknown variant %d", variant);
        return DGZ_ERR_INVALID;
    }
    if (e != cudaSuccess) return cuda_fail(e, "gather kernel launch");
    return DGZ_OK;
}

extern "C" dgz_status dgz_order_workspace_bytes(int64_t n, size_t* bytes);
extern "C" dgz_status dgz_order_ids(const int64_t* ids_dev, int64_t n, int64_t max_id, int64_t* ids_sorted, int64_t* pos,
                                    void* workspace, size_t workspace_bytes, dgz_stream stream);

// Fetch in table order: sort (id, position) on the device, gather in address order and scatter
// back (GPU address translation of 4 KiB host pages bounds random rows on
// large tables).  Scratch comes from the stream-ordered allocator (pooled, non-blocking).
static dgz_status gather_ordered(dgz_table t, const int64_t* idx, int64_t n, void* out, const dgz_gather_cfg* cfg,
                                 cudaStream_t s) {
    size_t ws = 0;
    dgz_status st = dgz_order_workspace_bytes(n, &ws);
    if (st != DGZ_OK) return st;
    const size_t arr = ((size_t)n * 8 + 255) & ~size_t(255);
    uint8_t* mem = nullptr;
    DGZ_CUDA(cudaMallocAsync((void**)&mem, 2 * arr + ws, s));
    int64_t* srt = (int64_t*)mem;
    int64_t* pos = (int64_t*)(mem + arr);
    st = dgz_order_ids(idx, n, t->rows, srt, pos, mem + 2 * arr, ws, (dgz_stream)s);
    if (st == DGZ_OK) st = dgz_gather_impl(t, srt, 1, pos, n, nullptr, out, cfg, s, nullptr);
    cudaFreeAsync(mem, s);
    return st;
}

static bool want_order(const dgz_table_s* t, int64_t n) {
    // large host tables only: below a few GiB the GPU's translation caches cover the table
    return !(t->flags & DGZ_REG_DEVICE) && n >= (int64_t(1) << 16) && n < (int64_t(1) << 31) &&
           (double)t->rows * (double)t->row_bytes >= 4.0 * (1 << 30);
}

extern "C" dgz_status dgz_gather(dgz_table t, const int64_t* idx_dev, int64_t n, void* out_dev, dgz_stream stream) {
    if (t && idx_dev && out_dev && want_order(t, n)) return gather_ordered(t, idx_dev, n, out_dev, nullptr, (cudaStream_t)stream);
    return dgz_gather_impl(t, idx_dev, 1, nullptr, n, nullptr, out_dev, nullptr, (cudaStream_t)stream, nullptr);
}

extern "C" dgz_status dgz_gather_i32(dgz_table t, const int32_t* idx_dev, int64_t n, void* out_dev, dgz_stream stream) {
    return dgz_gather_impl(t, idx_dev, 0, nullptr, n, nullptr, out_dev, nullptr, (cudaStream_t)stream, nullptr);
}

extern "C" dgz_status dgz_gather_ex(dgz_table t, const int64_t* idx_dev, int64_t n, const int64_t* n_dev, void* out_dev,
                                    const dgz_gather_cfg* cfg, dgz_stream stream) {
    if (cfg && (cfg->flags & DGZ_GATHER_FLAG_ORDER)) {
        DGZ_REQUIRE(t && idx_dev && out_dev && !n_dev && n >= 0 && n < (int64_t(1) << 31),
                    "dgz_gather_ex: DGZ_GATHER_FLAG_ORDER needs a host-known n < 2^31 and no n_dev");
        DGZ_REQUIRE(cfg->variant == DGZ_GATHER_AUTO || cfg->variant == DGZ_GATHER_SEGMENT || cfg->variant == DGZ_GATHER_BULK,
                    "dgz_gather_ex: DGZ_GATHER_FLAG_ORDER needs the SEGMENT or BULK variant");
        if (n == 0) return DGZ_OK;
        dgz_gather_cfg c2 = *cfg;
        c2.flags &= ~DGZ_GATHER_FLAG_ORDER;
        return gather_ordered(t, idx_dev, n, out_dev, &c2, (cudaStream_t)stream);
    }
    return dgz_gather_impl(t, idx_dev, 1, nullptr, n, n_dev, out_dev, cfg, (cudaStream_t)stream, nullptr);
}

extern "C" dgz_status dgz_gather_perm(dgz_table t, const int64_t* idx_dev, const int64_t* dst_pos_dev, int64_t n,
                                      const int64_t* n_dev, void* out_dev, const dgz_gather_cfg* cfg, dgz_stream stream) {
    DGZ_REQUIRE(dst_pos_dev || n == 0, "dgz_gather_perm: null dst_pos");
    return dgz_gather_impl(t, idx_dev, 1, dst_pos_dev, n, n_dev, out_dev, cfg, (cudaStream_t)stream, nullptr);
}

extern "C" dgz_status dgz_gather_cached(dgz_table t, const dgz_cache_view* cache, const int64_t* idx_dev, const int64_t* dst_pos_dev,
                                        int64_t n, const int64_t* n_dev, void* out_dev, const dgz_gather_cfg* cfg, dgz_stream stream) {
    DGZ_REQUIRE(cache, "dgz_gather_cached: null cache view");
    DGZ_REQUIRE(!cfg || cfg->variant == DGZ_GATHER_AUTO || cfg->variant == DGZ_GATHER_SEGMENT,
                "dgz_gather_cached: only the SEGMENT variant reads the cache");
    return dgz_gather_impl(t, idx_dev, 1, dst_pos_dev, n, n_dev, out_dev, cfg, (cudaStream_t)stream, cache);
}

extern "C" dgz_status dgz_gather_plan(dgz_table t, int64_t n, int32_t sorted, const dgz_gather_cfg* cfg, dgz_gather_cfg* plan,
                                      int32_t* ctas) {
    DGZ_REQUIRE(t && plan && n > 0, "dgz_gather_plan: null table/plan or n <= 0");
    const LaunchPlan P = plan_launch(t, n, sorted != 0, cfg, false);
    plan->variant = P.variant;
    plan->sm_count = P.k;
    plan->warps_per_cta = P.warps;
    plan->ctas_per_sm = P.cps;
    plan->schedule = P.blocked ? DGZ_SCHED_BLOCKED : DGZ_SCHED_INTERLEAVED;
    plan->flags = P.flags;
    if (ctas) {
        int64_t blocks = (int64_t)P.k * P.cps;
        if (P.variant == DGZ_GATHER_SEGMENT) {
            const int64_t need = ((n + 31) / 32 + P.warps - 1) / P.warps;
            if (blocks > need) blocks = need;
        }
        *ctas = (int32_t)blocks;
    }
    return DGZ_OK;
}
