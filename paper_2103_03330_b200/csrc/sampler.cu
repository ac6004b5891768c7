// Layered uniform neighbour sampling on the GPU (steps a2-a3; section 2.2).
//
//   F_0 = seeds (first occurrence kept)
//   hop k: each u in F_k selects min(f_k, deg u) distinct CSR slots (Floyd; r(t) = Philox word 0
//          with counter (t, k, lo32 u, hi32 u), key = rng_seed; reading R11), and
//          F_{k+1} = F_k ++ sorted(unique(selected) \ F_k)            (readings R9-R10)
//
// B200 design: the frontier set F_k is a bitmap over all N nodes in HBM (N/8 bytes: 14 MB for
// the papers100M-shaped graph).  Selected IDs are OR-ed into a candidate bitmap; ONE single-pass
// compaction over the two bitmaps (per 4096-word chunk: popcount, decoupled look-back for the
// chunk's prefix, emit) yields the new IDs already sorted and de-duplicated, with no sort and no
// hash table.  A minibatch is 1 + 2L (+1 sorted, +1 local positions) kernel launches.  Every size that
// depends on the data (|F_k|) stays on the device: kernels read it from sizes_dev, so the whole
// minibatch (sampling + gather) is enqueued without a host round trip and can be graph-captured.
#include <cub/block/block_reduce.cuh>
#include <cub/block/block_scan.cuh>

#include "internal.h"

namespace {

constexpr int kChunkWords = 4096;   // bitmap words per chunk (131072 node IDs)
constexpr int kChunkThreads = 256;  // 16 words per thread
constexpr int kWordsPerThread = kChunkWords / kChunkThreads;
constexpr int kSeedChunk = 4096;    // seeds per chunk in the seed compaction

// ---------------------------------------------------------------------------------------------
// Philox4x32-10 (Salmon, Moraes, Dror, Shaw, SC'11); returns output word 0.
// ---------------------------------------------------------------------------------------------
__device__ __forceinline__ uint32_t philox4x32_10_w0(uint32_t c0, uint32_t c1, uint32_t c2, uint32_t c3, uint32_t k0, uint32_t k1) {
#pragma unroll
    for (int r = 0; r < 10; ++r) {
        if (r) {
            k0 += 0x9E3779B9u;
            k1 += 0xBB67AE85u;
        }
        const uint32_t lo0 = 0xD2511F53u * c0, hi0 = __umulhi(0xD2511F53u, c0);
        const uint32_t lo1 = 0xCD9E8D57u * c2, hi1 = __umulhi(0xCD9E8D57u, c2);
        const uint32_t n0 = hi1 ^ c1 ^ k0, n2 = hi0 ^ c3 ^ k1;
        c0 = n0;
        c1 = lo1;
        c2 = n2;
        c3 = lo0;
    }
    return c0;
}

template <typename ColT>
__global__ void __launch_bounds__(256)
hop_sample_kernel(const int64_t* __restrict__ off, const ColT* __restrict__ cols, const int64_t* __restrict__ U,
                  const int64_t* __restrict__ sizes, int k, int f, uint32_t key0, uint32_t key1,
                  const uint64_t* __restrict__ key_dev, int64_t* __restrict__ nbr, int32_t* __restrict__ cnt,
                  uint32_t* __restrict__ cand) {
    const int64_t nk = sizes[k];
    if (key_dev) {  // device-resident sampler seed (CUDA-graph replays update it in place)
        const uint64_t kk = *key_dev;
        key0 = (uint32_t)(kk & 0xffffffffu);
        key1 = (uint32_t)(kk >> 32);
    }
    uint32_t pos[DGZ_MAX_FANOUT];
    for (int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < nk; i += int64_t(gridDim.x) * blockDim.x) {
        const int64_t u = U[i];
        const int64_t o0 = off[u];
        const int64_t d = off[u + 1] - o0;
        int c;
        if (d <= f) {
            c = (int)d;
            for (int q = 0; q < c; ++q) pos[q] = (uint32_t)q;
        } else {
            // Floyd: for t < f, j = d - f + t, x = floor(r(t) (j+1) / 2^32); take j if x taken
            c = f;
            for (int t = 0; t < f; ++t) {
                const uint64_t j = (uint64_t)(d - f + t);
                const uint32_t r = philox4x32_10_w0((uint32_t)t, (uint32_t)k, (uint32_t)((uint64_t)u & 0xffffffffu),
                                                    (uint32_t)((uint64_t)u >> 32), key0, key1);
                uint32_t x = (uint32_t)(((uint64_t)r * (j + 1)) >> 32);
                bool taken = false;
                for (int q = 0; q < t; ++q) taken |= (pos[q] == x);
                pos[t] = taken ? (uint32_t)j : x;
            }
            // ascending order (insertion sort, f <= 64)
            for (int a = 1; a < c; ++a) {
                const uint32_t v = pos[a];
                int b = a - 1;
                while (b >= 0 && pos[b] > v) {
                    pos[b + 1] = pos[b];
                    --b;
                }
                pos[b + 1] = v;
            }
        }
        // column loads batched 8 at a time ahead of their uses: independent loads in flight per
        // thread (a zero-copy CSR in host memory pays one PCIe round trip per batch, not per slot)
        for (int q0 = 0; q0 < c; q0 += 8) {
            int64_t sv[8];
#pragma unroll
            for (int e = 0; e < 8; ++e)
                if (q0 + e < c) sv[e] = (int64_t)cols[o0 + pos[q0 + e]];
#pragma unroll
            for (int e = 0; e < 8; ++e) {
                if (q0 + e < c) {
                    const int64_t s = sv[e];
                    if (nbr) nbr[i * f + q0 + e] = s;
                    atomicOr(&cand[s >> 5], 1u << (s & 31));
                }
            }
        }
        if (nbr)
            for (int q = c; q < f; ++q) nbr[i * f + q] = -1;
        if (cnt) cnt[i] = c;
    }
}

// exclusive scan of chunk sums (one block); *total_out = (base ? *base : 0) + sum
__global__ void __launch_bounds__(1024)
scan_chunks_kernel(const int64_t* __restrict__ sums, int64_t nchunks, int64_t* __restrict__ offs, const int64_t* base,
                   int64_t* total_out) {
    using BS = cub::BlockScan<int64_t, 1024>;
    __shared__ typename BS::TempStorage tmp;
    __shared__ int64_t carry;
    if (threadIdx.x == 0) carry = 0;
    __syncthreads();
    for (int64_t t0 = 0; t0 < nchunks; t0 += 1024) {
        const int64_t i = t0 + threadIdx.x;
        const int64_t v = i < nchunks ? sums[i] : 0;
        int64_t ex, agg;
        BS(tmp).ExclusiveSum(v, ex, agg);
        if (i < nchunks) offs[i] = carry + ex;
        __syncthreads();
        if (threadIdx.x == 0) carry += agg;
        __syncthreads();
    }
    if (threadIdx.x == 0) *total_out = (base ? *base : 0) + carry;
}

// ---- seeds: F_0 = seeds with the first occurrence of each ID kept -----------------------------
__global__ void seeds_mark_kernel(const int64_t* __restrict__ seeds, int64_t n, int64_t N, int32_t* __restrict__ pos, int* err) {
    for (int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < n; i += int64_t(gridDim.x) * blockDim.x) {
        const int64_t s = seeds[i];
        if (s < 0 || s >= N) atomicOr(err, 1);
        else pos[s] = 0x7fffffff;
    }
}
__global__ void seeds_min_kernel(const int64_t* __restrict__ seeds, int64_t n, int64_t N, int32_t* __restrict__ pos) {
    for (int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < n; i += int64_t(gridDim.x) * blockDim.x) {
        const int64_t s = seeds[i];
        if (s >= 0 && s < N) atomicMin(&pos[s], (int32_t)i);
    }
}
__device__ __forceinline__ bool seed_kept(const int64_t* seeds, int64_t i, int64_t n, int64_t N, const int32_t* pos) {
    if (i >= n) return false;
    const int64_t s = seeds[i];
    return s >= 0 && s < N && pos[s] == (int32_t)i;
}
__global__ void __launch_bounds__(256)
seeds_count_kernel(const int64_t* __restrict__ seeds, int64_t n, int64_t N, const int32_t* __restrict__ pos, int64_t* sums) {
    using BR = cub::BlockReduce<int, 256>;
    __shared__ typename BR::TempStorage tmp;
    int c = 0;
    for (int q = threadIdx.x; q < kSeedChunk; q += 256) c += seed_kept(seeds, int64_t(blockIdx.x) * kSeedChunk + q, n, N, pos);
    const int tot = BR(tmp).Sum(c);
    if (threadIdx.x == 0) sums[blockIdx.x] = tot;
}
__global__ void __launch_bounds__(256)
seeds_emit_kernel(const int64_t* __restrict__ seeds, int64_t n, int64_t N, const int32_t* __restrict__ pos,
                  const int64_t* __restrict__ offs, int64_t* __restrict__ U, uint32_t* __restrict__ front) {
    using BS = cub::BlockScan<int, 256>;
    __shared__ typename BS::TempStorage tmp;
    __shared__ int64_t run;
    if (threadIdx.x == 0) run = offs[blockIdx.x];
    __syncthreads();
    for (int q0 = 0; q0 < kSeedChunk; q0 += 256) {
        const int64_t i = int64_t(blockIdx.x) * kSeedChunk + q0 + threadIdx.x;
        const bool keep = seed_kept(seeds, i, n, N, pos);
        int ex, agg;
        BS(tmp).ExclusiveSum((int)keep, ex, agg);
        if (keep) {
            const int64_t s = seeds[i];
            U[run + ex] = s;
            atomicOr(&front[s >> 5], 1u << (s & 31));
        }
        __syncthreads();
        if (threadIdx.x == 0) run += agg;
        __syncthreads();
    }
}

// ---- fused single-pass compaction (decoupled look-back) ---------------------------------------
// One launch per hop instead of count + scan + emit: each 4096-word chunk takes a ticket (so a
// chunk only ever waits for chunks that already started), publishes its popcount, looks back
// over its predecessors' published aggregates / inclusive prefixes, and emits its IDs in order.
// MODE_NEW: the new IDs of hop k (cand & ~front) are appended to U at sizes[k] + prefix, their
//           positions recorded in pos[], front |= cand, cand = 0; the last chunk writes sizes[k+1].
// MODE_ALL: all IDs of the final frontier in ascending order with their positions in U.
constexpr int MODE_NEW = 0, MODE_ALL = 1;
constexpr unsigned long long kFlagAgg = 1ull << 62, kFlagIncl = 2ull << 62, kValMask = (1ull << 62) - 1;

template <int MODE>
__global__ void __launch_bounds__(kChunkThreads)
bitmap_compact_kernel(uint32_t* __restrict__ front, uint32_t* __restrict__ cand, unsigned long long* __restrict__ status,
                      unsigned* __restrict__ ticket, int64_t nchunks, int64_t* __restrict__ sizes, int k, int64_t* __restrict__ U,
                      int32_t* __restrict__ pos, int64_t* __restrict__ sorted, int64_t* __restrict__ sorted_pos) {
    using BS = cub::BlockScan<int, kChunkThreads>;
    using BR = cub::BlockReduce<int, kChunkThreads>;
    __shared__ union {
        typename BS::TempStorage scan;
        typename BR::TempStorage reduce;
    } tmp;
    __shared__ int chunk_s;
    __shared__ long long prefix_s;
    if (threadIdx.x == 0) chunk_s = (int)atomicAdd(ticket, 1u);
    __syncthreads();
    const int chunk = chunk_s;
    // word r*256 + t of the chunk goes to thread t: coalesced loads, and the IDs of a sparse or
    // dense region are spread over all threads when they are emitted
    const int64_t wbase = int64_t(chunk) * kChunkWords + threadIdx.x;
    uint32_t nw[kWordsPerThread];
    int c = 0;
#pragma unroll
    for (int r = 0; r < kWordsPerThread; ++r) {
        const int64_t w = wbase + r * kChunkThreads;
        if (MODE == MODE_NEW) {
            const uint32_t a = cand[w], b = front[w];
            nw[r] = a & ~b;
            if (a) {
                front[w] = a | b;
                cand[w] = 0;
            }
        } else {
            nw[r] = front[w];
        }
        c += __popc(nw[r]);
    }
    const int agg_t0 = BR(tmp.reduce).Sum(c);   // valid in thread 0
    if (threadIdx.x < 32) {
        // warp-parallel decoupled look-back: 32 predecessors per step, newest first
        const int lane = threadIdx.x;
        const int agg = __shfl_sync(0xffffffffu, agg_t0, 0);
        if (lane == 0) atomicExch(&status[chunk], (chunk == 0 ? kFlagIncl : kFlagAgg) | (unsigned long long)agg);
        long long prefix = 0;
        for (int j_hi = chunk - 1; j_hi >= 0; j_hi -= 32) {
            const int j = j_hi - lane;
            unsigned long long v = j >= 0 ? atomicAdd(&status[j], 0ull) : kFlagIncl;
            while (__any_sync(0xffffffffu, (v & ~kValMask) == 0)) {   // started (ticket order), not yet published
                if ((v & ~kValMask) == 0) v = atomicAdd(&status[j], 0ull);
            }
            const unsigned incl = __ballot_sync(0xffffffffu, (v & ~kValMask) == kFlagIncl);
            const int stop = incl ? __ffs(incl) - 1 : 31;                // newest inclusive prefix ends the walk
            long long val = lane <= stop ? (long long)(v & kValMask) : 0;
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) val += __shfl_down_sync(0xffffffffu, val, o);
            prefix += __shfl_sync(0xffffffffu, val, 0);
            if (incl) break;
        }
        if (lane == 0) {
            if (chunk > 0) atomicExch(&status[chunk], kFlagIncl | (unsigned long long)(prefix + agg));
            prefix_s = prefix;
            if (MODE == MODE_NEW && chunk == nchunks - 1) sizes[k + 1] = sizes[k] + prefix + agg;
        }
    }
    __syncthreads();
    int64_t run = (MODE == MODE_NEW ? sizes[k] : 0) + prefix_s;
#pragma unroll
    for (int r = 0; r < kWordsPerThread; ++r) {
        const int cnt = __popc(nw[r]);
        int ex, ragg;
        BS(tmp.scan).ExclusiveSum(cnt, ex, ragg);
        int64_t p = run + ex;
        uint32_t bits = nw[r];
        const int64_t w = wbase + r * kChunkThreads;
        while (bits) {
            const int b = __ffs(bits) - 1;
            const int64_t id = w * 32 + b;
            if (MODE == MODE_NEW) {
                U[p] = id;
                pos[id] = (int32_t)p;
            } else {
                sorted[p] = id;
                sorted_pos[p] = pos[id];
            }
            ++p;
            bits &= bits - 1;
        }
        run += ragg;
        __syncthreads();  // BlockScan storage reuse
    }
}

// F_0 for up to kSmallSeeds seeds in one block: first occurrence kept, positions recorded
constexpr int kSmallSeeds = 4096;  // 32 KiB of dynamic shared memory: no opt-in attribute needed
__global__ void __launch_bounds__(1024)
seeds_small_kernel(const int64_t* __restrict__ seeds, int n, int64_t N, int64_t* __restrict__ U, uint32_t* __restrict__ front,
                   int32_t* __restrict__ pos, int64_t* __restrict__ sizes, int* __restrict__ err) {
    // one block, O(n): the first occurrence of each seed wins an atomicMin on its entry of the
    // position map (pos[] is scratch here; it receives the seed's position in U at the end)
    extern __shared__ int64_t sh[];
    using BS = cub::BlockScan<int, 1024>;
    __shared__ typename BS::TempStorage tmp;
    __shared__ int run;
    for (int i = threadIdx.x; i < n; i += 1024) {
        const int64_t v = seeds[i];
        const bool ok = v >= 0 && v < N;
        if (!ok) atomicOr(err, 1);
        sh[i] = ok ? v : -1;
        if (ok) pos[v] = 0x7fffffff;
    }
    if (threadIdx.x == 0) run = 0;
    __syncthreads();
    for (int i = threadIdx.x; i < n; i += 1024)
        if (sh[i] >= 0) atomicMin(&pos[sh[i]], i);
    __syncthreads();
    for (int i = threadIdx.x; i < n; i += 1024)      // keep flag: the sign bit of sh[i] (-1 = dropped)
        if (sh[i] >= 0 && pos[sh[i]] != i) sh[i] = -1;
    __syncthreads();
    for (int i0 = 0; i0 < n; i0 += 1024) {
        const int i = i0 + threadIdx.x;
        const bool keep = i < n && sh[i] >= 0;
        int ex, agg;
        BS(tmp).ExclusiveSum((int)keep, ex, agg);
        if (keep) {
            const int64_t v = sh[i];
            const int p = run + ex;
            U[p] = v;
            pos[v] = p;
            atomicOr(&front[v >> 5], 1u << (v & 31));
        }
        __syncthreads();
        if (threadIdx.x == 0) run += agg;
        __syncthreads();
    }
    if (threadIdx.x == 0) sizes[0] = run;
}

__global__ void posmap_range_kernel(const int64_t* __restrict__ U, const int64_t* __restrict__ sizes, int32_t* __restrict__ pos) {
    const int64_t n = sizes[0];
    for (int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < n; i += int64_t(gridDim.x) * blockDim.x) pos[U[i]] = (int32_t)i;
}

// positions in U of every sampled ID, all hops in one launch
struct HopTable {
    int64_t start[DGZ_MAX_LAYERS + 1];  // element offset of hop k's block (bound-based layout)
    int32_t f[DGZ_MAX_LAYERS];
    int32_t L;
};
__global__ void local_all_kernel(const int64_t* __restrict__ nbr, const int64_t* __restrict__ sizes, const HopTable ht,
                                 const int32_t* __restrict__ pos, int32_t* __restrict__ local) {
    const int64_t total = ht.start[ht.L];
    for (int64_t e = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; e < total; e += int64_t(gridDim.x) * blockDim.x) {
        int k = 0;
        while (k + 1 < ht.L && e >= ht.start[k + 1]) ++k;
        if (ht.f[k] == 0 || e - ht.start[k] >= sizes[k] * ht.f[k]) continue;  // beyond this hop's |F_k|
        const int64_t v = nbr[e];
        local[e] = v < 0 ? -1 : pos[v];
    }
}

// ---- workspace layout ----------------------------------------------------------------------
struct Layout {
    int64_t nwords_pad, nchunks, seed_chunks;
    size_t o_front, o_cand, o_status, o_ticket, o_zero_end, o_csum, o_coff, o_ssum, o_soff, o_pos, o_err, total;
};
inline size_t al(size_t x) { return (x + 255) & ~size_t(255); }
Layout layout(int64_t N, int64_t max_seeds) {
    Layout l{};
    const int64_t nwords = (N + 31) / 32;
    l.nchunks = (nwords + kChunkWords - 1) / kChunkWords;
    l.nwords_pad = l.nchunks * kChunkWords;
    l.seed_chunks = (max_seeds + kSeedChunk - 1) / kSeedChunk;
    if (l.seed_chunks < 1) l.seed_chunks = 1;
    size_t o = 0;
    l.o_err = o; o = al(o + 8);  // first: dgz_sample_check finds it without the layout
    l.o_front = o; o = al(o + 4 * (size_t)l.nwords_pad);
    l.o_cand = o; o = al(o + 4 * (size_t)l.nwords_pad);
    l.o_status = o; o = al(o + 8 * (size_t)l.nchunks * (DGZ_MAX_LAYERS + 1));   // one look-back array per compaction
    l.o_ticket = o; o = al(o + 4 * (DGZ_MAX_LAYERS + 1));
    l.o_zero_end = o;                                                            // everything above is zeroed per call
    l.o_csum = o; o = al(o + 8 * ((size_t)l.nchunks + 1));
    l.o_coff = o; o = al(o + 8 * (size_t)l.nchunks);
    l.o_ssum = o; o = al(o + 8 * (size_t)l.seed_chunks);
    l.o_soff = o; o = al(o + 8 * (size_t)l.seed_chunks);
    l.o_pos = o; o = al(o + 4 * (size_t)N);
    l.total = o;
    return l;
}

int grid_for(int64_t work, int threads) {
    const int nsm = dgz::sm_count_of_current_device();
    int64_t b = (work + threads - 1) / threads;
    const int64_t cap = (int64_t)(nsm > 0 ? nsm : 148) * 8;
    if (b > cap) b = cap;
    if (b < 1) b = 1;
    return (int)b;
}

}  // namespace

using namespace dgz;

extern "C" dgz_status dgz_sample_bounds(int64_t n_nodes, int64_t n_seeds, const int32_t* fanouts, int n_layers, int64_t* bounds,
                                        int64_t* blocks_elems, int64_t* cnt_elems) {
    DGZ_REQUIRE(n_nodes >= 1 && n_seeds >= 0 && n_layers >= 0 && n_layers <= DGZ_MAX_LAYERS && (n_layers == 0 || fanouts),
                "dgz_sample_bounds: bad arguments");
    int64_t b = n_seeds, be = 0, ce = 0;
    int64_t cur = b < n_nodes ? b : n_nodes;
    if (bounds) bounds[0] = cur;
    for (int k = 0; k < n_layers; ++k) {
        DGZ_REQUIRE(fanouts[k] >= 0 && fanouts[k] <= DGZ_MAX_FANOUT, "dgz_sample_bounds: fanout %d out of [0, %d]", fanouts[k],
                    DGZ_MAX_FANOUT);
        be += cur * fanouts[k];
        ce += cur;
        b = b > (int64_t(1) << 40) ? b : b * (1 + fanouts[k]);
        cur = b < n_nodes ? b : n_nodes;
        if (bounds) bounds[k + 1] = cur;
    }
    if (blocks_elems) *blocks_elems = be;
    if (cnt_elems) *cnt_elems = ce;
    return DGZ_OK;
}

extern "C" dgz_status dgz_sample_workspace_bytes(int64_t n_nodes, int64_t max_seeds, size_t* bytes) {
    DGZ_REQUIRE(n_nodes >= 1 && n_nodes < (int64_t(1) << 31) && max_seeds >= 0 && bytes,
                "dgz_sample_workspace_bytes: need 1 <= n_nodes < 2^31");
    *bytes = layout(n_nodes, max_seeds).total;
    return DGZ_OK;
}

extern "C" dgz_status dgz_sample_uniform(const dgz_csr* csr, const int64_t* seeds_dev, int64_t n_seeds, const int32_t* fanouts,
                                         int n_layers, uint64_t rng_seed, const dgz_sample_out* out, dgz_stream stream) {
    DGZ_REQUIRE(csr && out, "dgz_sample_uniform: null csr/out");
    const int64_t N = csr->n_nodes;
    DGZ_REQUIRE(N >= 1 && N < (int64_t(1) << 31) && csr->offsets, "dgz_sample_uniform: bad csr");  // cols may be NULL when E == 0
    DGZ_REQUIRE(n_seeds >= 0 && (n_seeds == 0 || seeds_dev), "dgz_sample_uniform: bad seeds");
    DGZ_REQUIRE(n_seeds < (int64_t(1) << 31), "dgz_sample_uniform: too many seeds");
    DGZ_REQUIRE(n_layers >= 0 && n_layers <= DGZ_MAX_LAYERS && (n_layers == 0 || fanouts), "dgz_sample_uniform: bad layers");
    int64_t bounds[DGZ_MAX_LAYERS + 1], be = 0, ce = 0;
    dgz_status st = dgz_sample_bounds(N, n_seeds, fanouts, n_layers, bounds, &be, &ce);
    if (st != DGZ_OK) return st;
    DGZ_REQUIRE(out->ids && out->ids_cap >= bounds[n_layers], "dgz_sample_uniform: ids capacity %lld < bound %lld",
                (long long)out->ids_cap, (long long)bounds[n_layers]);
    DGZ_REQUIRE(out->sizes_dev, "dgz_sample_uniform: sizes_dev is required");
    DGZ_REQUIRE(!out->nbr || out->blocks_cap >= be, "dgz_sample_uniform: nbr capacity %lld < %lld", (long long)out->blocks_cap,
                (long long)be);
    DGZ_REQUIRE(!out->nbr_local || (out->nbr && out->blocks_cap >= be), "dgz_sample_uniform: nbr_local needs nbr");
    DGZ_REQUIRE(!out->cnt || out->cnt_cap >= ce, "dgz_sample_uniform: cnt capacity");
    DGZ_REQUIRE(!out->ids_sorted == !out->ids_sorted_pos, "dgz_sample_uniform: ids_sorted and ids_sorted_pos go together");
    const Layout l = layout(N, n_seeds);
    DGZ_REQUIRE(out->workspace && out->workspace_bytes >= l.total, "dgz_sample_uniform: workspace %zu < %zu bytes",
                out->workspace_bytes, l.total);
    DGZ_REQUIRE(((uintptr_t)out->workspace & 255) == 0, "dgz_sample_uniform: workspace must be 256-byte aligned");

    cudaStream_t s = (cudaStream_t)stream;
    uint8_t* ws = (uint8_t*)out->workspace;
    uint32_t* front = (uint32_t*)(ws + l.o_front);
    uint32_t* cand = (uint32_t*)(ws + l.o_cand);
    int64_t* csum = (int64_t*)(ws + l.o_csum);
    int64_t* coff = (int64_t*)(ws + l.o_coff);
    int64_t* ssum = (int64_t*)(ws + l.o_ssum);
    int64_t* soff = (int64_t*)(ws + l.o_soff);
    int32_t* pos = (int32_t*)(ws + l.o_pos);
    int* err = (int*)(ws + l.o_err);
    int64_t* sizes = out->sizes_dev;

    unsigned long long* status = (unsigned long long*)(ws + l.o_status);
    unsigned* tickets = (unsigned*)(ws + l.o_ticket);
    for (const void* k : {(const void*)seeds_small_kernel, (const void*)seeds_mark_kernel, (const void*)seeds_min_kernel,
                          (const void*)seeds_count_kernel, (const void*)scan_chunks_kernel, (const void*)seeds_emit_kernel,
                          (const void*)posmap_range_kernel, (const void*)hop_sample_kernel<int64_t>,
                          (const void*)hop_sample_kernel<int32_t>, (const void*)bitmap_compact_kernel<MODE_NEW>,
                          (const void*)bitmap_compact_kernel<MODE_ALL>, (const void*)local_all_kernel})
        dgz::apply_carveout(k, dgz::kCarveoutSampler);   // internal.h
    DGZ_CUDA(cudaMemsetAsync(ws, 0, l.o_zero_end, s));  // error word, bitmaps, look-back state
    // F_0 (pos[] of every ID of U is written where the ID is emitted)
    if (n_seeds > 0 && n_seeds <= kSmallSeeds) {
        seeds_small_kernel<<<1, 1024, sizeof(int64_t) * (size_t)n_seeds, s>>>(seeds_dev, (int)n_seeds, N, out->ids, front, pos, sizes,
                                                                            err);
        dgz::count_launch();
    } else if (n_seeds > 0) {
        const int gs = grid_for(n_seeds, 256);
        const int sc = (int)((n_seeds + kSeedChunk - 1) / kSeedChunk);
        seeds_mark_kernel<<<gs, 256, 0, s>>>(seeds_dev, n_seeds, N, pos, err); dgz::count_launch();
        seeds_min_kernel<<<gs, 256, 0, s>>>(seeds_dev, n_seeds, N, pos); dgz::count_launch();
        seeds_count_kernel<<<sc, 256, 0, s>>>(seeds_dev, n_seeds, N, pos, ssum); dgz::count_launch();
        scan_chunks_kernel<<<1, 1024, 0, s>>>(ssum, sc, soff, nullptr, sizes); dgz::count_launch();
        seeds_emit_kernel<<<sc, 256, 0, s>>>(seeds_dev, n_seeds, N, pos, soff, out->ids, front); dgz::count_launch();
        posmap_range_kernel<<<gs, 256, 0, s>>>(out->ids, sizes, pos); dgz::count_launch();
    } else {
        DGZ_CUDA(cudaMemsetAsync(sizes, 0, 8, s));
    }
    int64_t nbr_off = 0, cnt_off = 0;
    const uint32_t k0 = (uint32_t)(rng_seed & 0xffffffffu), k1 = (uint32_t)(rng_seed >> 32);
    HopTable ht{};
    ht.L = n_layers;
    for (int k = 0; k < n_layers; ++k) {
        const int f = fanouts[k];
        int64_t* nbr_k = out->nbr ? out->nbr + nbr_off : nullptr;
        int32_t* cnt_k = out->cnt ? out->cnt + cnt_off : nullptr;
        const int gh = grid_for(bounds[k], 256);
        if (csr->cols_is64)
            hop_sample_kernel<int64_t><<<gh, 256, 0, s>>>(csr->offsets, (const int64_t*)csr->cols, out->ids, sizes, k, f, k0, k1,
                                                          out->rng_seed_dev, nbr_k, cnt_k, cand);
        else
            hop_sample_kernel<int32_t><<<gh, 256, 0, s>>>(csr->offsets, (const int32_t*)csr->cols, out->ids, sizes, k, f, k0, k1,
                                                          out->rng_seed_dev, nbr_k, cnt_k, cand);
        dgz::count_launch();
        bitmap_compact_kernel<MODE_NEW><<<(int)l.nchunks, kChunkThreads, 0, s>>>(
            front, cand, status + (size_t)k * l.nchunks, tickets + k, l.nchunks, sizes, k, out->ids, pos, nullptr, nullptr);
        dgz::count_launch();
        ht.start[k] = nbr_off;
        ht.f[k] = f;
        nbr_off += bounds[k] * f;
        cnt_off += bounds[k];
    }
    ht.start[n_layers] = nbr_off;
    if (out->ids_sorted) {
        // the final frontier bitmap holds exactly U: compact it in ascending ID order
        bitmap_compact_kernel<MODE_ALL><<<(int)l.nchunks, kChunkThreads, 0, s>>>(
            front, cand, status + (size_t)n_layers * l.nchunks, tickets + n_layers, l.nchunks, sizes, n_layers, nullptr, pos,
            out->ids_sorted, out->ids_sorted_pos);
        dgz::count_launch();
    }
    if (out->nbr_local && nbr_off > 0) {
        local_all_kernel<<<grid_for(nbr_off, 256), 256, 0, s>>>(out->nbr, sizes, ht, pos, out->nbr_local);
        dgz::count_launch();
    }
    st = launch_check("dgz_sample_uniform kernels");
    if (st != DGZ_OK) return st;
    if (out->sizes_host)
        DGZ_CUDA(cudaMemcpyAsync(out->sizes_host, sizes, sizeof(int64_t) * (n_layers + 1), cudaMemcpyDeviceToHost, s));
    return DGZ_OK;
}

extern "C" dgz_status dgz_sample_check(const dgz_sample_out* out, dgz_stream stream) {
    DGZ_REQUIRE(out && out->workspace && out->workspace_bytes >= 8, "dgz_sample_check: null out/workspace");
    int h = 0;
    DGZ_CUDA(cudaMemcpyAsync(&h, out->workspace, sizeof(int), cudaMemcpyDeviceToHost, (cudaStream_t)stream));
    DGZ_CUDA(cudaStreamSynchronize((cudaStream_t)stream));
    if (h) { set_error("dgz_sample_uniform: a seed was outside [0, n_nodes)"); return DGZ_ERR_RANGE; }
    return DGZ_OK;
}
