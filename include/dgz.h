/*
 * dgz.h -- C ABI of libdgz: direct GPU zero-copy feature gather for GCN minibatches on B200.
 *
 * The operations follow arXiv 2103.03330 (PyTorch-Direct); "P:n" is /root/reference/PAPER.md
 * line n, "S:n" is SPEC.md line n.  The boundary is described in DESIGN.md section 1.
 *
 * Conventions for every entry point
 *   - Returns a dgz_status.  No exception crosses the ABI and nothing calls exit().
 *   - DGZ_ERR_INVALID: bad argument, detected synchronously before any work is enqueued.
 *   - DGZ_ERR_CUDA: a CUDA runtime call failed; dgz_last_error() has the CUDA error string.
 *   - DGZ_ERR_NOMEM: host allocation / pinning failed.
 *   - DGZ_ERR_RANGE: an index was out of range.  Device-side range faults are latched in a
 *     device flag and reported by dgz_check_errors (the offending row is skipped, the CUDA
 *     context is never faulted).
 *   - DGZ_ERR_STATE: the call is not valid in the current state (e.g. wrong device).
 *   - dgz_last_error() returns a thread-local message describing the last failure.
 *   - "device" pointers are CUDA device (or UVA-mapped) addresses owned by the caller;
 *     "host" pointers are ordinary process addresses.  Streams are cudaStream_t (NULL =
 *     legacy default stream).  All enqueuing calls are asynchronous on that stream.
 */
#ifndef DGZ_H
#define DGZ_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define DGZ_ABI_VERSION 1

#if defined(__GNUC__)
#define DGZ_API __attribute__((visibility("default")))
#else
#define DGZ_API
#endif

typedef enum {
    DGZ_OK = 0,
    DGZ_ERR_INVALID = 1,
    DGZ_ERR_CUDA = 2,
    DGZ_ERR_NOMEM = 3,
    DGZ_ERR_RANGE = 4,
    DGZ_ERR_STATE = 5
} dgz_status;

/* Element types of the feature table: 4 / 2 / 2 / 1 bytes.  The gather moves bytes only and
 * never does floating-point arithmetic on them (NaN payloads are preserved; reading R17). */
typedef enum { DGZ_F32 = 0, DGZ_F16 = 1, DGZ_BF16 = 2, DGZ_U8 = 3 } dgz_dtype;

typedef struct CUstream_st* dgz_stream; /* == cudaStream_t */
typedef struct dgz_table_s* dgz_table;  /* opaque registration handle */

DGZ_API int dgz_abi_version(void);
DGZ_API const char* dgz_last_error(void);
/* Number of SMs of the current device (148 on B200), or -1. */
DGZ_API int dgz_device_sm_count(void);
/* Number of CUDA kernels libdgz has launched in this process (all threads, all devices). */
DGZ_API uint64_t dgz_kernel_launches(void);

/* ==========================================================================================
 * Host table manager (B1).  The paper shares one host feature table between the per-GPU
 * processes by allocating Linux shared memory first and registering it in every process
 * (section 3.4, Listing 3).
 * ========================================================================================== */
#define DGZ_HOST_HUGEPAGE 1u /* madvise(MADV_HUGEPAGE) on the mapping */
#define DGZ_HOST_POPULATE 2u /* pre-fault every page at creation */
#define DGZ_HOST_CUDA_PINNED 8u /* cudaHostAlloc(Mapped | Portable): driver-allocated pinned memory
                                   (single process; not shareable by name) */
#define DGZ_HOST_HUGETLB_2M 16u /* anonymous MAP_HUGETLB 2 MiB pages (needs vm.nr_hugepages) */
#define DGZ_HOST_HUGETLB_1G 32u /* anonymous MAP_HUGETLB 1 GiB pages */
#define DGZ_HOST_NUMA_INTERLEAVE 64u /* mbind(MPOL_INTERLEAVE) over the allowed NUMA nodes before first
                                        touch (a no-op on one node): multi-socket boxes whose G GPUs all
                                        read the one shared table (SURVEY 7 "host aggregate"); a hint:
                                        if the kernel refuses it the mapping keeps first-touch placement */
#define DGZ_HOST_VMM 4u      /* CUDA VMM host allocation (cuMemCreate on host NUMA node 0): pinned,
                                CPU-accessible, mapped into the current GPU at the same address (with
                                2 MiB allocation granularity; the GPU still translated it at 4 KiB pages
                                on the measured boxes).  Needs a CUDA device;
                                shm_name must be NULL (share it across processes with dgz_host_export /
                                dgz_host_import). */

#define DGZ_HOST_MANAGED 128u /* CUDA managed memory kept in HOST memory: cudaMallocManaged +
                                 cudaMemAdviseSetPreferredLocation(CPU) before first touch, so the CPU
                                 fills it in place and it never migrates; dgz_register_table then maps
                                 it for the GPU (cudaMemAdviseSetAccessedBy) and the gather reads it by
                                 zero-copy like a registered table.  The driver maps such memory with
                                 large GPU pages, so sparse rows are not bound by the GPU page walks a
                                 cudaHostRegister'd table pays per 64 KiB.
                                 Needs a CUDA device; shm_name must be NULL (managed memory is not
                                 shareable across processes: one copy per process). */

/* Number of NUMA nodes this process may allocate on (cpuset Mems_allowed; 1 when unknown). */
DGZ_API int dgz_host_numa_nodes(void);
/* Map `bytes` of host memory.  shm_name == NULL: private anonymous mapping.  Otherwise a POSIX
 * shared-memory object (/dev/shm/<name>): create != 0 creates/truncates it to `bytes`,
 * create == 0 opens an existing object of at least `bytes` bytes.  A name containing a second '/'
 * is a file path instead (a file on a tmpfs / hugetlbfs mount, or /proc/<pid>/fd/<n> naming
 * another process's memfd), opened with open(2) -- for boxes whose /dev/shm is too small for the
 * table; it must be shmem-backed for cudaHostRegister to pin it.  *ptr receives a page-aligned
 * address.  The caller releases it with dgz_host_free.  dgz_host_unlink removes the name
 * (shm_unlink / unlink; a no-op for /proc/<pid>/fd paths). */
DGZ_API dgz_status dgz_host_alloc(const char* shm_name, size_t bytes, int create, uint32_t flags, void** ptr);
DGZ_API dgz_status dgz_host_free(void* ptr, size_t bytes);
DGZ_API dgz_status dgz_host_unlink(const char* shm_name);
/* POSIX file descriptor of a DGZ_HOST_VMM allocation (ptr = the address dgz_host_alloc returned);
 * pass it to another process (SCM_RIGHTS / pidfd_getfd) and map it there with dgz_host_import.
 * The caller closes the fd. */
DGZ_API dgz_status dgz_host_export(void* ptr, int* fd);
/* Map an exported DGZ_HOST_VMM allocation into this process, accessible by the CPU and the current
 * device.  `bytes` must be the size the exporter passed to dgz_host_alloc (the whole allocation is
 * mapped).  Release with dgz_host_free. */
DGZ_API dgz_status dgz_host_import(int fd, size_t bytes, void** ptr);

/* ==========================================================================================
 * Table registration (step a1).  The paper's "unified tensor": cudaHostRegister page-locks
 * the caller's host table and cudaHostGetDevicePointer maps it into the GPU address space so
 * that kernels read it by zero-copy over PCIe, with no copy (section 3.1, tab:tensor).
 * ========================================================================================== */
#define DGZ_REG_PORTABLE 1u  /* cudaHostRegisterPortable: valid on every device of this process */
#define DGZ_REG_READONLY 2u  /* cudaHostRegisterReadOnly when the device supports it */
#define DGZ_REG_NO_PIN 4u    /* memory is already page-locked (e.g. cudaHostAlloc): map only */
#define DGZ_REG_DEVICE 16u    /* (reported) a device-resident table wrapped by dgz_wrap_device_table */
#define DGZ_REG_VMM_BACKED 8u /* (reported in dgz_table_info.flags) the table lies in a DGZ_HOST_VMM
                                 allocation: no cudaHostRegister, mapped by the VMM allocation itself */
#define DGZ_REG_MANAGED 32u   /* (reported) the table lies in CUDA managed memory (e.g. DGZ_HOST_MANAGED):
                                 no cudaHostRegister; registration advises AccessedBy(current device)
                                 so the GPU reads the host-resident pages through its own mapping, and a
                                 gather on another device adds that device on first use */

/* host_ptr: row 0 of a row-major, unpadded rows x dim table of `dtype` elements in host
 * memory (any alignment; unaligned bases are a first-class case, S:37 base_offset).  The caller
 * owns the memory and must keep it alive and unmodified-in-size until dgz_unregister_table.
 * Registers on the CURRENT device.  rows >= 1, dim >= 1.  A span whose pages are ALL already
 * registered (by another table or by the caller) is mapped, not re-pinned; a span that only
 * partly overlaps an existing registration (e.g. two tables sharing a boundary page) is refused
 * with DGZ_ERR_STATE, because cudaHostRegister cannot extend a registration (probed at the first
 * and last byte and every 64 MiB between).  A DGZ_REG_VMM_BACKED table is granted to another
 * device on that device's first gather. */
DGZ_API dgz_status dgz_register_table(const void* host_ptr, int64_t rows, int64_t dim, dgz_dtype dtype,
                              uint32_t flags, dgz_table* out);
DGZ_API dgz_status dgz_unregister_table(dgz_table t);
/* A handle for a table already resident in device memory (HBM), read by the same gather kernels:
 * the paper's "All-in-GPU" reference point, and the source of cache shards.  The
 * caller owns the memory; dgz_unregister_table releases only the handle. */
DGZ_API dgz_status dgz_wrap_device_table(const void* dev_ptr, int64_t rows, int64_t dim, dgz_dtype dtype, dgz_table* out);

typedef struct {
    const void* dev_ptr;     /* device-visible address of row 0 */
    int64_t rows, dim, row_bytes;
    int32_t elem_bytes;
    int32_t device;          /* device the registration was made on */
    int32_t base_mod128;     /* (address of row 0) mod 128: the misalignment of the table */
    int32_t flags;
    int64_t pinned_bytes;    /* page-rounded span that was registered by this handle */
    int64_t gpu_mem_delta;   /* device memory consumed by the mapping (~bytes/512) */
    double register_seconds; /* wall time of cudaHostRegister */
} dgz_table_info;
DGZ_API dgz_status dgz_table_get_info(dgz_table t, dgz_table_info* info);

/* ==========================================================================================
 * Sparse feature gather (step a4, the hot path).
 *   out[r*R + b] = table[idx[r]*R + b]   for 0 <= r < n, 0 <= b < R = dim * elem_bytes
 * (Listing 2, last line "dst[dstOffset] = src[srcOffset]"; the circular shift and
 * the segment plan only change which thread copies which byte).  Each row is
 * fetched as its 128 B-aligned line segments (one PCIe read per line the row touches, the
 * per-row minimum).  Byte-exact; duplicates allowed; n == 0 is a no-op.
 * idx_dev: device int64 (or int32 for *_i32) [n].  out_dev: device [n x R] bytes, aligned to
 * the element size, not aliasing the table.  IDs < 0 or >= rows: the row is skipped (its
 * output bytes are left unchanged) and the table's RANGE flag is latched (dgz_check_errors).
 * ========================================================================================== */
DGZ_API dgz_status dgz_gather(dgz_table t, const int64_t* idx_dev, int64_t n, void* out_dev, dgz_stream stream);
/* (dgz_gather on a host table of >= 4 GiB with n >= 65536 rows fetches in table-address order --
 * device radix sort + dgz_gather_perm, scratch from cudaMallocAsync -- because GPU address
 * translation of 4 KiB host pages bounds random rows there; the result is identical.) */
DGZ_API dgz_status dgz_gather_i32(dgz_table t, const int32_t* idx_dev, int64_t n, void* out_dev, dgz_stream stream);

typedef enum {
    DGZ_GATHER_AUTO = 0,    /* = SEGMENT */
    DGZ_GATHER_SEGMENT = 1, /* 128 B-segment plan, 16 B vector loads, warp-cooperative rows */
    DGZ_GATHER_NAIVE = 2,   /* ablation K1n: one element per thread, no alignment */
    DGZ_GATHER_SHIFT = 3,   /* ablation: Listing 2 circular shift, one element per thread */
    DGZ_GATHER_BULK = 4     /* cp.async.bulk (TMA engine) row copies via shared memory */
} dgz_gather_variant;

typedef enum {
    DGZ_SCHED_AUTO = 0,        /* = INTERLEAVED (measured best on B200) */
    DGZ_SCHED_INTERLEAVED = 1, /* warp w of the grid takes 32-row batches w, w + W, ... */
    DGZ_SCHED_BLOCKED = 2      /* CTA c owns a contiguous range of batches (translation-aware:
                                  with a sorted index list each SM walks its own address range) */
} dgz_gather_schedule;

typedef struct {
    int32_t variant;       /* dgz_gather_variant */
    int32_t sm_count;      /* 0 = default grid; k > 0 bounds the persistent grid to k CTAs, one
                              per SM (the B200 analogue of the paper's MPS X%, step a6) */
    int32_t warps_per_cta; /* 0 = default */
    int32_t ctas_per_sm;   /* 0 = default (1) */
    int32_t schedule;      /* dgz_gather_schedule */
    int32_t flags;         /* DGZ_GATHER_FLAG_* (SEGMENT variant) */
} dgz_gather_cfg;
#define DGZ_GATHER_FLAG_NO_MERGE 1       /* dgz_gather_perm: do not merge the 128 B line two
                                            table-adjacent rows share (default: merged, R >= 128) */
#define DGZ_GATHER_FLAG_DEEP 2           /* 16 instead of 8 line loads in flight per lane */
#define DGZ_GATHER_FLAG_ORDER 4          /* dgz_gather_ex: fetch in table-address order (sort on the
                                            device, gather, scatter back); same result */
#define DGZ_GATHER_FLAG_STREAM_STORES 8  /* SEGMENT: HBM stores as st.global.cs (evict-first in L2) */
#define DGZ_GATHER_FLAG_EVICT_FIRST_LOADS 16 /* SEGMENT: zero-copy loads under an L2 evict_first policy */
#define DGZ_GATHER_FLAG_DYNAMIC 32       /* SEGMENT: warps take 32-row batches from a work counter (in
                                            ascending order) instead of a static interleave; the 8-byte
                                            counter is a slot of a per-device ring of 4096 allocated once
                                            (cudaMalloc on first use) and zeroed on the launch's stream;
                                            at most 4096 such launches may be in flight at once across
                                            streams */

/* The launch a gather of n rows would use (sorted != 0: dgz_gather_perm / the fetcher's sorted
 * path) with `cfg` (NULL = defaults): the resolved variant, SM count, warps per CTA, CTAs per SM,
 * schedule and flags in *plan, and the grid size in *ctas (optional).  No GPU work. */
DGZ_API dgz_status dgz_gather_plan(dgz_table t, int64_t n, int32_t sorted, const dgz_gather_cfg* cfg, dgz_gather_cfg* plan,
                                   int32_t* ctas);
/* As dgz_gather, with an optional device-resident row count: when n_dev != NULL the kernel
 * gathers min(*n_dev, n) rows (n is the capacity), so a gather can follow the sampler on the
 * same stream without a host round trip.  cfg may be NULL (defaults). */
DGZ_API dgz_status dgz_gather_ex(dgz_table t, const int64_t* idx_dev, int64_t n, const int64_t* n_dev,
                         void* out_dev, const dgz_gather_cfg* cfg, dgz_stream stream);

/* Gather in a caller-chosen processing order: out[dst_pos[k]] = table[idx[k]] for k < n (or
 * < min(n, *n_dev)).  With idx sorted by address and dst_pos its inverse permutation this is
 * the same result as dgz_gather on the unsorted list, fetched in table order (each SM walks a
 * contiguous address range: far fewer GPU address-translation misses on tables of tens of GB;
 * DESIGN.md section 5).  dst_pos must be a permutation of [0, n) (else rows may overlap). */
DGZ_API dgz_status dgz_gather_perm(dgz_table t, const int64_t* idx_dev, const int64_t* dst_pos_dev, int64_t n,
                                   const int64_t* n_dev, void* out_dev, const dgz_gather_cfg* cfg, dgz_stream stream);

/* ==========================================================================================
 * HBM row cache.  The paper found page-granular UVM caching "nearly
 * useless" for irregular accesses; a ROW-granular cache of the most-referenced rows in
 * HBM is a different design: on skewed graphs it removes their PCIe reads entirely.  The cache is
 * a slot map (device int32 [rows], -1 = not cached) and G shards: slot s lives at row s / G of
 * shard s % G.  Shards may be this GPU's HBM or peer GPUs' HBM mapped into this process (NVLink
 * peer loads); all are caller-owned device memory of ceil(capacity / G) x row_bytes bytes.
 * ========================================================================================== */
#define DGZ_MAX_CACHE_SHARDS 8
typedef struct {
    int32_t* slot_map;    /* device int32 [table rows] */
    int32_t n_shards;     /* 1 <= G <= DGZ_MAX_CACHE_SHARDS */
    int32_t reserved;
    void* shards[DGZ_MAX_CACHE_SHARDS];
} dgz_cache_view;

/* Build: slot_map[hot_ids[c]] = c for c < n_hot, every other entry -1, and shard (c % G) row
 * (c / G) = table row hot_ids[c] (fetched by zero-copy).  hot_ids: device int64 [n_hot], distinct
 * and in range (DGZ_ERR_RANGE is latched in the table flag otherwise).  One-time setup: may
 * allocate temporary device memory. */
DGZ_API dgz_status dgz_cache_fill(dgz_table t, const int64_t* hot_ids_dev, int64_t n_hot, const dgz_cache_view* cache,
                                  dgz_stream stream);
/* dgz_cache_fill for a cache sharded across ranks (one process per GPU):
 * builds the full slot map on the current device but fetches only shard `local_shard` (this rank's
 * HBM); the other shards of `cache` may be NULL here and are filled by their owners (map them with
 * dgz_ipc_open before gathering, and order the fills before the first gather, e.g. by a barrier).
 * local_shard = -1: every shard, as dgz_cache_fill. */
DGZ_API dgz_status dgz_cache_fill_local(dgz_table t, const int64_t* hot_ids_dev, int64_t n_hot, const dgz_cache_view* cache,
                                        int32_t local_shard, dgz_stream stream);
/* Device memory for shards and CUDA IPC handles to map another rank's shard into this process:
 * on a different GPU of the box the mapping is a peer mapping and the cached gather reads it by
 * NVLink loads (peer access enabled lazily); on the same GPU it is plain HBM.  dgz_ipc_open's
 * pointer stays valid until dgz_ipc_close; the owner must not free the shard before that. */
typedef struct { unsigned char bytes[64]; } dgz_ipc_handle;
DGZ_API dgz_status dgz_device_alloc(size_t bytes, void** out);
DGZ_API dgz_status dgz_device_free(void* dev_ptr);
DGZ_API dgz_status dgz_ipc_get_handle(void* dev_ptr, dgz_ipc_handle* out);
DGZ_API dgz_status dgz_ipc_open(const dgz_ipc_handle* handle, void** out);
DGZ_API dgz_status dgz_ipc_close(void* dev_ptr);
/* As dgz_gather_perm (dst_pos_dev may be NULL: identity), reading cached rows from HBM and the
 * others by zero-copy from the table: out[dst_pos[k]] = table[idx[k]] either way (byte-exact). */
DGZ_API dgz_status dgz_gather_cached(dgz_table t, const dgz_cache_view* cache, const int64_t* idx_dev,
                                     const int64_t* dst_pos_dev, int64_t n, const int64_t* n_dev, void* out_dev,
                                     const dgz_gather_cfg* cfg, dgz_stream stream);

/* Address order of an arbitrary device ID list (duplicates allowed): ids_sorted[k] ascending and
 * pos[k] its position in ids_dev -- the inputs of dgz_gather_perm, so that any gather can be
 * fetched in table order (the sampler emits these for its own list).  IDs are compared on their
 * low ceil(log2(max_id)) bits (pass max_id = table rows); out-of-range IDs still appear exactly
 * once and are reported by the gather.  ids_sorted/pos: device int64 [n]; workspace: device
 * scratch of dgz_order_workspace_bytes(n) bytes.  n < 2^31. */
DGZ_API dgz_status dgz_order_workspace_bytes(int64_t n, size_t* bytes);
DGZ_API dgz_status dgz_order_ids(const int64_t* ids_dev, int64_t n, int64_t max_id, int64_t* ids_sorted, int64_t* pos,
                                 void* workspace, size_t workspace_bytes, dgz_stream stream);

/* Synchronises `stream`, reads and clears the table's device RANGE flag for the current
 * device: DGZ_ERR_RANGE if any gather since the last check met an out-of-range ID. */
DGZ_API dgz_status dgz_check_errors(dgz_table t, dgz_stream stream);

/* ==========================================================================================
 * Layered uniform neighbour sampling on the GPU (steps a2-a3; section 2.2).
 *   F_0 = seeds (duplicates dropped, first occurrence kept)
 *   hop k = 0..L-1, f = fanouts[k]: every u in F_k selects min(f, deg u) distinct CSR slots
 *     uniformly without replacement (Floyd's algorithm, r(t) = word 0 of Philox4x32-10 with
 *     counter (t, k, lo32 u, hi32 u) and key (lo32 rng_seed, hi32 rng_seed); reading R11);
 *     new = sorted unique(selected IDs) \ F_k;  F_{k+1} = F_k ++ new  (readings R9-R10)
 *   ids = F_L, the gather list (seeds included).
 * The result depends only on (csr, seeds, fanouts, rng_seed): not on grid, device or timing.
 * ========================================================================================== */
typedef struct {
    int64_t n_nodes;
    const int64_t* offsets; /* device-accessible [n_nodes + 1], offsets[0] = 0, non-decreasing */
    const void* cols;       /* device-accessible [offsets[n_nodes]] int32 or int64 node IDs < n_nodes
                               (NULL if no edges).  Either HBM, or host memory registered with
                               dgz_register_table (its dgz_table_info.dev_ptr): the sampler then reads
                               the CSR by zero-copy loads over PCIe (a CSR that
                               does not fit HBM); the result is the same either way.  The caller
                               owns both arrays; they must outlive the call's stream work. */
    int32_t cols_is64;
    int32_t reserved;
} dgz_csr;

#define DGZ_MAX_FANOUT 64
#define DGZ_MAX_LAYERS 8

typedef struct {
    int64_t* ids;          /* device [ids_cap] >= bounds[L]: frontier-prefix unique IDs */
    int64_t ids_cap;
    int64_t* sizes_dev;    /* device [L + 1]: |F_0| .. |F_L| (required) */
    int64_t* sizes_host;   /* optional pinned host [L + 1]: async copy of sizes_dev */
    int64_t* nbr;          /* optional device: hop k block at sum_{i<k} bounds[i]*fanouts[i],
                              bounds[k] x fanouts[k] row-major sampled IDs, unused slots -1 */
    int32_t* nbr_local;    /* optional device, layout of nbr: position of the ID in ids */
    int32_t* cnt;          /* optional device: hop k block at sum_{i<k} bounds[i]: counts */
    int64_t blocks_cap;    /* elements available in nbr / nbr_local */
    int64_t cnt_cap;       /* elements available in cnt */
    void* workspace;       /* device scratch of dgz_sample_workspace_bytes() bytes; not */
    size_t workspace_bytes;/* shared between calls that may run concurrently */
    int64_t* ids_sorted;   /* optional device [ids_cap]: the IDs of `ids` in ascending order */
    int64_t* ids_sorted_pos; /* optional device [ids_cap] (with ids_sorted): position in `ids` of
                              each sorted ID -- the inputs of dgz_gather_perm */
    const uint64_t* rng_seed_dev; /* optional device uint64 [1]: when set, the sampler reads its
                              seed here and ignores `rng_seed` (a captured CUDA graph can then be
                              replayed for a new minibatch by updating seeds and this word) */
} dgz_sample_out;

/* bounds[k] = min(n_nodes, n_seeds * prod_{i<k}(1 + fanouts[i])) for k = 0..L; also the
 * element counts the optional block outputs need.  Any pointer may be NULL. */
DGZ_API dgz_status dgz_sample_bounds(int64_t n_nodes, int64_t n_seeds, const int32_t* fanouts, int n_layers,
                             int64_t* bounds, int64_t* blocks_elems, int64_t* cnt_elems);
DGZ_API dgz_status dgz_sample_workspace_bytes(int64_t n_nodes, int64_t max_seeds, size_t* bytes);
/* seeds_dev: device int64 [n_seeds], each in [0, n_nodes) (else DGZ_ERR_RANGE is latched in
 * the workspace and reported by dgz_sample_check; offending seeds are dropped).
 * fanouts: HOST int32 [n_layers], 0 <= f <= DGZ_MAX_FANOUT, n_layers <= DGZ_MAX_LAYERS. */
DGZ_API dgz_status dgz_sample_uniform(const dgz_csr* csr, const int64_t* seeds_dev, int64_t n_seeds,
                              const int32_t* fanouts, int n_layers, uint64_t rng_seed,
                              const dgz_sample_out* out, dgz_stream stream);
/* Synchronises `stream`; DGZ_ERR_RANGE if a seed was out of range in the last call. */
DGZ_API dgz_status dgz_sample_check(const dgz_sample_out* out, dgz_stream stream);

/* ==========================================================================================
 * Stand-in GraphSAGE mean aggregation (consumer, step a7; P:554-555 fig:singlegpu): for dst
 * node i < *n_dst_dev (bounded by n_dst_max):
 *   y[i, :] = (x[i, :] + sum_{c < cnt[i]} x[nbr_local[i*fanout + c], :]) / (1 + cnt[i])
 * over fp32 rows x [*, dim].  `repeat` re-runs the aggregation to scale the consumer's work
 * (T_c ~ T_g for the overlap measurement).  ctas_per_sm == 0: `repeat` launches of a
 * non-persistent grid (one 256-thread CTA per 8 destination nodes; short-lived CTAs, like training
 * kernels, so a co-running fetch gets SM slots quickly).  ctas_per_sm > 0: one persistent launch of
 * ctas_per_sm x sm_count CTAs (sm_count 0 = all) that holds its slots for the whole call.
 * Not on the parity path.
 * ========================================================================================== */
DGZ_API dgz_status dgz_aggregate_mean(const float* x, int64_t dim, const int32_t* nbr_local, const int32_t* cnt,
                              int32_t fanout, const int64_t* n_dst_dev, int64_t n_dst_max, float* y,
                              int32_t repeat, int32_t sm_count, int32_t ctas_per_sm, dgz_stream stream);

/* ==========================================================================================
 * Stand-in GraphSAGE layer (consumer, step a7: "mean over each dst node's sampled neighbours of
 * the gathered rows, then a small GEMM" -- SURVEY 8(a) a7; P:554-555 fig:singlegpu; the layer
 * P:224-229).  For dst node i < min(*n_dst_dev, n_dst_max):
 *   h[i, :] = (x[i, :] + sum_{q < cnt[i]} x[nbr_local[i*fanout + q], :]) * (1 / (1 + cnt[i]))
 *             (fp32, q in order: bit-identical to dgz_aggregate_mean)
 *   y[i, n] = sum_k bf16(h[i, k]) * w[n*dim + k]    fp32 accumulation on the tensor cores
 * x: fp32 [*, dim] device rows (the gathered minibatch), 4-byte aligned; w: bf16 [hidden, dim]
 * device, row-major (nn.Linear weight layout), 2-byte aligned; y: fp32 [n_dst, hidden] device,
 * 16-byte aligned, rows >= n_dst untouched.  hidden: a multiple of 16 in [16, 256]; any dim (K is
 * staged in chunks of up to (112 KiB / ((hidden + 128) x 2)) columns, accumulated in TMEM; dim 128 /
 * hidden 256: one chunk, 96 KiB).  h is rounded
 * to bf16 (round to nearest even) before the product: |y - h.W^T| <= 2^-8 sum_k |h_k w_nk| plus
 * fp32 accumulation error.  repeat / sm_count / ctas_per_sm as for dgz_aggregate_mean.  Async on
 * `stream`; n_dst_max == 0 is a no-op.  Errors: DGZ_ERR_INVALID (arguments, sizes), DGZ_ERR_CUDA.
 * ========================================================================================== */
DGZ_API dgz_status dgz_sage_mean_linear(const float* x, int64_t dim, const int32_t* nbr_local, const int32_t* cnt,
                              int32_t fanout, const int64_t* n_dst_dev, int64_t n_dst_max, const void* w_bf16,
                              int64_t hidden, float* y, int32_t repeat, int32_t sm_count, int32_t ctas_per_sm,
                              dgz_stream stream);
/* Shared-memory bytes (one K chunk of both bf16 operands) and TMEM columns one dgz_sage_mean_linear CTA uses. */
DGZ_API dgz_status dgz_sage_workspace(int64_t dim, int64_t hidden, int64_t* smem_bytes, int32_t* tmem_cols);

/* ==========================================================================================
 * In-process SM partition (step a6): the paper's MPS X% / (100-X)% split done with
 * CUDA green contexts.  The current device's SMs are split into a fetch group of at least
 * `fetch_sms` SMs (rounded up to the hardware granularity: multiples of 8 on sm_90+, finer with
 * DGZ_PARTITION_FINE) and a compute group with the rest; each group gets one non-blocking stream.
 * Kernels launched on a group's stream run only on that group's SMs.  Device memory of the
 * primary context is usable from both.  Destroy after all work on the streams has finished.
 * ========================================================================================== */
typedef struct dgz_partition_s* dgz_partition;
#define DGZ_PARTITION_FINE 1u   /* CU_DEV_SM_RESOURCE_SPLIT_IGNORE_SM_COSCHEDULING: finer SM counts */
#define DGZ_PARTITION_SPREAD 2u /* fetch SMs taken evenly across the device (all GPCs) from the
                                   finest split; the compute group gets every other SM */
/* Explicit SM sets: the device's SMs as the smallest groups a green-context split allows (in the
 * driver's order; *sms_per_group SMs each), and a partition whose fetch side is exactly the listed
 * groups (the compute side gets the rest).  Which SMs a translation-bound gather runs on changes
 * its rate at a fixed SM count; these entry points let a caller measure and
 * pick them. */
DGZ_API dgz_status dgz_partition_group_count(int32_t* n_groups, int32_t* sms_per_group);
DGZ_API dgz_status dgz_partition_create_groups(const int32_t* fetch_groups, int32_t n_fetch_groups, int32_t fetch_priority,
                                               dgz_partition* out);
DGZ_API dgz_status dgz_partition_create(int32_t fetch_sms, int32_t fetch_priority, uint32_t flags, dgz_partition* out);
DGZ_API dgz_status dgz_partition_get(dgz_partition p, dgz_stream* fetch_stream, dgz_stream* compute_stream,
                                     int32_t* fetch_sms, int32_t* compute_sms);
/* Another non-blocking stream on group 0 (fetch) or 1 (compute) of the partition, e.g. so that the
 * sampler of step j+1 runs on the fetch SMs beside the gather of step j (a5).  Owned by the
 * partition: destroyed by dgz_partition_destroy. */
DGZ_API dgz_status dgz_partition_stream(dgz_partition p, int32_t group, int32_t priority, dgz_stream* out);
DGZ_API dgz_status dgz_partition_destroy(dgz_partition p);

/* ==========================================================================================
 * PCIe probes (the zero-copy ceiling and the round-trip time).
 * ========================================================================================== */
/* Streaming zero-copy read of `bytes` (multiple of 16) from a mapped host pointer with 16 B
 * loads, `warps` warps on each of `sm_count` SMs, each warp keeping `unroll` loads in flight.
 * A checksum is written to *sink_dev so the loads cannot be elided. */
/* As dgz_probe_stream (unroll 8) with the loads' L2 prefetch-size hint set to l2_prefetch_bytes
 * (0 = none, 64, 128, 256): whether GPU-initiated sysmem reads can be made larger than a line. */
DGZ_API dgz_status dgz_probe_stream_hint(const void* src_dev, int64_t bytes, int32_t sm_count, int32_t warps,
                                         int32_t l2_prefetch_bytes, uint64_t* sink_dev, dgz_stream stream);
DGZ_API dgz_status dgz_probe_stream(const void* src_dev, int64_t bytes, int32_t sm_count, int32_t warps,
                            int32_t unroll, uint64_t* sink_dev, dgz_stream stream);
/* Dependent-load chain of `steps` hops through a mapped host array of int64 "next" offsets;
 * writes cycles_dev[0] = total cycles, cycles_dev[1] = final offset (one thread;
 * RTT = cycles / steps / SM clock).  cycles_dev: device uint64 [2]. */
/* Pure-ALU load (dependent FMA chains, no memory traffic): `ctas` x `threads` threads spin for
 * `iters` iterations.  Used to separate SM-issue from memory-system interference in the overlap
 * experiments.  sink_dev: device float [1]. */
DGZ_API dgz_status dgz_probe_spin(int32_t ctas, int32_t threads, int64_t iters, float* sink_dev, dgz_stream stream);
/* Random-row read probe (the a7 layer's access pattern): reads rows ids_dev[0..n) of row_bytes bytes
 * (a multiple of 16) from the device-accessible src_dev, rows_in_flight (1, 2, 4, 8, 16) rows per warp
 * issued before any is consumed, on sm_count SMs x warps warps; writes nothing but a sink word.  For
 * the HBM ceiling of random row reads. */
DGZ_API dgz_status dgz_probe_rows(const void* src_dev, int64_t row_bytes, const int64_t* ids_dev, int64_t n, int32_t sm_count,
                                  int32_t warps, int32_t rows_in_flight, uint64_t* sink_dev, dgz_stream stream);
DGZ_API dgz_status dgz_probe_chase(const void* src_dev, int64_t steps, uint64_t* cycles_dev, dgz_stream stream);

#ifdef __cplusplus
}
#endif
#endif /* DGZ_H */
