// libdgz: error state, host table manager (B1) and table registration (step a1).
//   Registration = the paper's "unified tensor" (section 3.1): cudaHostRegister
//   page-locks the caller's table, cudaHostGetDevicePointer maps it for zero-copy access.
//   Shared host memory across per-GPU processes = P:616-627 section 3.4 (Listing 3).
#include <errno.h>
#include <fcntl.h>
#include <stdarg.h>
#include <sys/mman.h>
#include <sys/stat.h>
#include <time.h>
#include <unistd.h>

#include <atomic>
#include <mutex>
#include <map>
#include <vector>

#include <sys/syscall.h>
#include <unistd.h>

#include "internal.h"

namespace dgz {

static thread_local char g_err[512] = "";

void set_error(const char* fmt, ...) {
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(g_err, sizeof(g_err), fmt, ap);
    va_end(ap);
}

dgz_status cuda_fail(cudaError_t e, const char* what) {
    set_error("%s: %s (%s)", what, cudaGetErrorString(e), cudaGetErrorName(e));
    // the failure is reported here: clear the runtime's last-error state so a non-sticky error
    // (e.g. an invalid IPC handle) does not resurface in the next call's launch check
    (void)cudaGetLastError();
    return DGZ_ERR_CUDA;
}

int sm_count_of_current_device() {
    int dev = 0, n = 0;
    if (cudaGetDevice(&dev) != cudaSuccess) return -1;
    if (cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess) return -1;
    return n;
}

static std::atomic<uint64_t> g_launches{0};
void count_launch() { g_launches.fetch_add(1, std::memory_order_relaxed); }

int carveout_pct(int cls) {
    static const int gather_pct = [] {
        const char* e = getenv("DGZ_CARVEOUT");
        return e ? atoi(e) : (int)cudaSharedmemCarveoutMaxShared;
    }();
    static const int sampler_pct = [] {
        const char* e = getenv("DGZ_SAMPLER_CARVEOUT");
        return e ? atoi(e) : -1;
    }();
    return cls == kCarveoutSampler ? sampler_pct : gather_pct;
}

void apply_carveout(const void* kernel, int cls) {
    const int pct = carveout_pct(cls);
    if (pct < 0) return;
    int dev = 0;
    if (cudaGetDevice(&dev) != cudaSuccess) return;
    static std::mutex mu;
    static std::vector<std::pair<const void*, int>> done;   // (kernel, device): the attribute is per device
    std::lock_guard<std::mutex> lk(mu);
    for (const auto& k : done)
        if (k.first == kernel && k.second == dev) return;
    cudaFuncSetAttribute(kernel, cudaFuncAttributePreferredSharedMemoryCarveout, pct);
    done.emplace_back(kernel, dev);
}

static double now_s() {
    timespec ts;
    clock_gettime(CLOCK_MONOTONIC, &ts);
    return ts.tv_sec + 1e-9 * ts.tv_nsec;
}

}  // namespace dgz

using namespace dgz;

static std::mutex g_pinned_mu;
static std::map<uintptr_t, size_t> g_pinned;  // cudaHostAlloc'ed host tables -> bytes
static std::map<uintptr_t, size_t> g_mapped;  // hugetlb mappings -> mapped (rounded) bytes
static std::map<uintptr_t, size_t> g_managed; // DGZ_HOST_MANAGED allocations -> bytes

dgz_status dgz_vmm_alloc(size_t bytes, void** ptr);
int dgz_vmm_free(void* ptr);
int dgz_vmm_register(const void* p, size_t bytes);

extern "C" int dgz_abi_version(void) { return DGZ_ABI_VERSION; }
extern "C" const char* dgz_last_error(void) { return g_err; }
extern "C" int dgz_device_sm_count(void) { return sm_count_of_current_device(); }
extern "C" uint64_t dgz_kernel_launches(void) { return g_launches.load(); }

// ---------------------------------------------------------------------------------------------
// Host table manager
// ---------------------------------------------------------------------------------------------
// NUMA nodes this process may allocate on, as a bit mask: the cpuset's Mems_allowed_list from
// /proc/self/status (a container may restrict it), else /sys/devices/system/node/online; lists
// look like "0-1" or "0,2-3".
static int numa_online_mask(unsigned long* mask, int max_nodes) {
    char line[512] = {0};
    bool found = false;
    if (FILE* st = fopen("/proc/self/status", "r")) {
        char buf[512];
        while (fgets(buf, sizeof buf, st)) {
            if (strncmp(buf, "Mems_allowed_list:", 18) == 0) {
                const char* v = buf + 18;
                while (*v == ' ' || *v == '\t') ++v;
                strncpy(line, v, sizeof line - 1);
                found = true;
                break;
            }
        }
        fclose(st);
    }
    if (!found) {
        FILE* f = fopen("/sys/devices/system/node/online", "r");
        if (!f) return 1;   // no NUMA information: treat as one node
        if (!fgets(line, sizeof line, f)) line[0] = 0;
        fclose(f);
    }
    int count = 0;
    for (char* tok = strtok(line, ",\n"); tok; tok = strtok(nullptr, ",\n")) {
        int lo = 0, hi = 0;
        if (sscanf(tok, "%d-%d", &lo, &hi) < 2) hi = lo = atoi(tok);
        for (int n = lo; n <= hi && n < max_nodes; ++n) {
            mask[n / (8 * sizeof(unsigned long))] |= 1ul << (n % (8 * sizeof(unsigned long)));
            ++count;
        }
    }
    return count > 0 ? count : 1;
}

extern "C" int dgz_host_numa_nodes(void) {
    unsigned long mask[16] = {0};
    return numa_online_mask(mask, 16 * 8 * (int)sizeof(unsigned long));
}

extern "C" dgz_status dgz_host_alloc(const char* shm_name, size_t bytes, int create, uint32_t flags, void** ptr) {
    DGZ_REQUIRE(ptr && bytes > 0, "dgz_host_alloc: null ptr or zero size");
    *ptr = nullptr;
    if (flags & DGZ_HOST_VMM) {
        DGZ_REQUIRE(!shm_name, "dgz_host_alloc: DGZ_HOST_VMM allocations are shared with dgz_host_export, not by name");
        return dgz_vmm_alloc(bytes, ptr);
    }
    if (flags & DGZ_HOST_MANAGED) {
        DGZ_REQUIRE(!shm_name, "dgz_host_alloc: DGZ_HOST_MANAGED memory cannot be named (not shareable across processes)");
        void* p = nullptr;
        cudaError_t e = cudaMallocManaged(&p, bytes, cudaMemAttachGlobal);
        if (e != cudaSuccess) return cuda_fail(e, "cudaMallocManaged");
        // before the first touch: the CPU's writes then place every page in host memory, and no GPU
        // access migrates it (the GPU gets a mapping at registration, dgz_register_table)
        e = cudaMemAdvise(p, bytes, cudaMemAdviseSetPreferredLocation, cudaCpuDeviceId);
        if (e != cudaSuccess) {
            cudaFree(p);
            return cuda_fail(e, "cudaMemAdvise(PreferredLocation = CPU)");
        }
        std::lock_guard<std::mutex> g(g_pinned_mu);
        g_managed[(uintptr_t)p] = bytes;
        *ptr = p;
        return DGZ_OK;
    }
    if (flags & DGZ_HOST_CUDA_PINNED) {
        DGZ_REQUIRE(!shm_name, "dgz_host_alloc: DGZ_HOST_CUDA_PINNED memory cannot be named");
        void* p = nullptr;
        cudaError_t e = cudaHostAlloc(&p, bytes, cudaHostAllocMapped | cudaHostAllocPortable);
        if (e != cudaSuccess) return cuda_fail(e, "cudaHostAlloc");
        std::lock_guard<std::mutex> g(g_pinned_mu);
        g_pinned[(uintptr_t)p] = bytes;
        *ptr = p;
        return DGZ_OK;
    }
    void* p = MAP_FAILED;
    if (!shm_name) {
        int extra = 0;
        size_t huge = 0;
        if (flags & DGZ_HOST_HUGETLB_2M) { extra = MAP_HUGETLB | (21 << MAP_HUGE_SHIFT); huge = size_t(1) << 21; }
        if (flags & DGZ_HOST_HUGETLB_1G) { extra = MAP_HUGETLB | (30 << MAP_HUGE_SHIFT); huge = size_t(1) << 30; }
        const size_t mapped = huge ? (bytes + huge - 1) / huge * huge : bytes;   // munmap needs the huge-page multiple
        p = mmap(nullptr, mapped, PROT_READ | PROT_WRITE, MAP_PRIVATE | MAP_ANONYMOUS | extra, -1, 0);
        if (p != MAP_FAILED && huge) {
            std::lock_guard<std::mutex> g(g_pinned_mu);
            g_mapped[(uintptr_t)p] = mapped;
        }
    } else {
        DGZ_REQUIRE(shm_name[0] == '/', "dgz_host_alloc: shm name must start with '/'");
        // "/name": a POSIX shared-memory object (/dev/shm).  A name with a second '/' is a file
        // path on a tmpfs / hugetlbfs (or /proc/<pid>/fd/<n> of another process's memfd): the
        // fallback when /dev/shm is too small to hold the table
        const bool path = strchr(shm_name + 1, '/') != nullptr;
        int fd = path ? open(shm_name, O_RDWR | (create ? O_CREAT : 0), 0600)
                      : shm_open(shm_name, O_RDWR | (create ? O_CREAT : 0), 0600);
        if (fd < 0) { set_error("%s(%s): %s", path ? "open" : "shm_open", shm_name, strerror(errno)); return DGZ_ERR_NOMEM; }
        if (create) {
            if (ftruncate(fd, (off_t)bytes) != 0) {
                set_error("ftruncate(%s, %zu): %s", shm_name, bytes, strerror(errno));
                close(fd);
                return DGZ_ERR_NOMEM;
            }
        } else {
            struct stat st;
            if (fstat(fd, &st) != 0 || (size_t)st.st_size < bytes) {
                set_error("shm object %s smaller than %zu bytes", shm_name, bytes);
                close(fd);
                return DGZ_ERR_INVALID;
            }
        }
        p = mmap(nullptr, bytes, PROT_READ | PROT_WRITE, MAP_SHARED, fd, 0);
        close(fd);
    }
    if (p == MAP_FAILED) { set_error("mmap(%zu): %s", bytes, strerror(errno)); return DGZ_ERR_NOMEM; }
    if (flags & DGZ_HOST_NUMA_INTERLEAVE) {
        // pages are placed round-robin over the online NUMA nodes at first touch (for a /dev/shm
        // object this sets the object's shared policy): on a multi-socket box the G ranks' random
        // reads then spread over every socket's memory controllers instead of the filling rank's
        const int max_nodes = 1024;
        unsigned long mask[max_nodes / (8 * sizeof(unsigned long))] = {0};
        if (numa_online_mask(mask, max_nodes) > 1) {
            const int mpol_interleave = 3;   // MPOL_INTERLEAVE (linux/mempolicy.h)
            // a placement hint, not a requirement: if the kernel refuses it the mapping keeps the
            // default first-touch policy (and dgz_last_error says why)
            if (syscall(SYS_mbind, p, bytes, mpol_interleave, mask, (unsigned long)max_nodes, 0u) != 0)
                set_error("mbind(MPOL_INTERLEAVE, %zu bytes) ignored: %s", bytes, strerror(errno));
        }
    }
    if (flags & DGZ_HOST_HUGEPAGE) madvise(p, bytes, MADV_HUGEPAGE);
    if (flags & DGZ_HOST_POPULATE) {
        volatile uint8_t* b = (volatile uint8_t*)p;
        long pg = sysconf(_SC_PAGESIZE);
        for (size_t off = 0; off < bytes; off += (size_t)pg) b[off] = b[off];
    }
    *ptr = p;
    return DGZ_OK;
}

extern "C" dgz_status dgz_host_free(void* ptr, size_t bytes) {
    DGZ_REQUIRE(ptr && bytes > 0, "dgz_host_free: null ptr or zero size");
    if (dgz_vmm_free(ptr) == 1) return DGZ_OK;
    {
        std::lock_guard<std::mutex> g(g_pinned_mu);
        if (g_pinned.erase((uintptr_t)ptr)) {
            cudaError_t e = cudaFreeHost(ptr);
            if (e != cudaSuccess) return cuda_fail(e, "cudaFreeHost");
            return DGZ_OK;
        }
        if (g_managed.erase((uintptr_t)ptr)) {
            cudaError_t e = cudaFree(ptr);
            if (e != cudaSuccess) return cuda_fail(e, "cudaFree (managed)");
            return DGZ_OK;
        }
    }
    {
        std::lock_guard<std::mutex> g(g_pinned_mu);
        auto it = g_mapped.find((uintptr_t)ptr);
        if (it != g_mapped.end()) {
            bytes = it->second;
            g_mapped.erase(it);
        }
    }
    if (munmap(ptr, bytes) != 0) { set_error("munmap: %s", strerror(errno)); return DGZ_ERR_INVALID; }
    return DGZ_OK;
}

extern "C" dgz_status dgz_host_unlink(const char* shm_name) {
    DGZ_REQUIRE(shm_name, "dgz_host_unlink: null name");
    if (strncmp(shm_name, "/proc/", 6) == 0) return DGZ_OK;   // a memfd: gone with its last reference
    const int r = strchr(shm_name + 1, '/') ? unlink(shm_name) : shm_unlink(shm_name);
    if (r != 0 && errno != ENOENT) {
        set_error("shm_unlink(%s): %s", shm_name, strerror(errno));
        return DGZ_ERR_INVALID;
    }
    return DGZ_OK;
}

// ---------------------------------------------------------------------------------------------
// Registration
// ---------------------------------------------------------------------------------------------
static int elem_bytes_of(dgz_dtype d) {
    switch (d) {
        case DGZ_F32: return 4;
        case DGZ_F16: return 2;
        case DGZ_BF16: return 2;
        case DGZ_U8: return 1;
    }
    return 0;
}

static bool is_cuda_pinned(const void* p) {
    std::lock_guard<std::mutex> g(g_pinned_mu);
    auto it = g_pinned.upper_bound((uintptr_t)p);
    if (it == g_pinned.begin()) return false;
    --it;
    return (uintptr_t)p >= it->first && (uintptr_t)p < it->first + it->second;
}

extern "C" dgz_status dgz_register_table(const void* host_ptr, int64_t rows, int64_t dim, dgz_dtype dtype,
                                         uint32_t flags, dgz_table* out) {
    DGZ_REQUIRE(out, "dgz_register_table: null out");
    *out = nullptr;
    DGZ_REQUIRE(host_ptr, "dgz_register_table: null host_ptr");
    DGZ_REQUIRE(rows >= 1 && dim >= 1, "dgz_register_table: rows=%lld dim=%lld", (long long)rows, (long long)dim);
    int eb = elem_bytes_of(dtype);
    DGZ_REQUIRE(eb > 0, "dgz_register_table: unknown dtype %d", (int)dtype);
    DGZ_REQUIRE(dim <= (int64_t(1) << 40) / eb && rows <= (int64_t(1) << 62) / (dim * eb),
                "dgz_register_table: table too large");
    DGZ_REQUIRE(((uintptr_t)host_ptr % eb) == 0, "dgz_register_table: host_ptr not aligned to the element size");

    dgz_table t = new (std::nothrow) dgz_table_s();
    if (!t) { set_error("out of memory"); return DGZ_ERR_NOMEM; }
    t->host = (const uint8_t*)host_ptr;
    t->rows = rows;
    t->dim = dim;
    t->elem_bytes = eb;
    t->row_bytes = dim * eb;
    t->flags = flags;
    cudaError_t e = cudaGetDevice(&t->device);
    if (e != cudaSuccess) { delete t; return cuda_fail(e, "cudaGetDevice"); }

    const size_t bytes = (size_t)rows * (size_t)t->row_bytes;
    const uintptr_t pg = (uintptr_t)sysconf(_SC_PAGESIZE);
    uintptr_t lo = (uintptr_t)host_ptr & ~(pg - 1);
    uintptr_t hi = ((uintptr_t)host_ptr + bytes + pg - 1) & ~(pg - 1);

    size_t free0 = 0, free1 = 0, total = 0;
    cudaMemGetInfo(&free0, &total);
    double t0 = now_s();
    const int vmm = dgz_vmm_register(host_ptr, bytes);
    if (vmm < 0) {
        delete t;
        return (dgz_status)(-vmm);
    }
    cudaPointerAttributes pa{};
    const bool managed = vmm != 1 && cudaPointerGetAttributes(&pa, host_ptr) == cudaSuccess && pa.type == cudaMemoryTypeManaged;
    cudaGetLastError();
    if (vmm == 1) {
        t->flags |= DGZ_REG_NO_PIN | DGZ_REG_VMM_BACKED;  // CUDA VMM host memory: already mapped
    } else if (managed) {
        // CUDA managed memory: no page locking by us; the current device gets a mapping of the pages
        // where they are (host memory for DGZ_HOST_MANAGED), read by the gather like a registered table
        t->flags |= DGZ_REG_NO_PIN | DGZ_REG_MANAGED;
        e = cudaMemAdvise(host_ptr, bytes, cudaMemAdviseSetAccessedBy, t->device);
        if (e != cudaSuccess) {
            delete t;
            return cuda_fail(e, "cudaMemAdvise(AccessedBy)");
        }
        if (t->device >= 0 && t->device < 64) t->managed_devs = uint64_t(1) << t->device;
    } else if (!(flags & DGZ_REG_NO_PIN) && !is_cuda_pinned(host_ptr)) {
        unsigned int rf = cudaHostRegisterMapped;
        if (flags & DGZ_REG_PORTABLE) rf |= cudaHostRegisterPortable;
        if (flags & DGZ_REG_READONLY) {
            int ro = 0;
            cudaDeviceGetAttribute(&ro, cudaDevAttrHostRegisterReadOnlySupported, t->device);
            if (ro) rf |= cudaHostRegisterReadOnly;
        }
        e = cudaHostRegister((void*)lo, hi - lo, rf);
        if (e == cudaErrorHostMemoryAlreadyRegistered) {
            cudaGetLastError();
            // pages already registered by someone else: map only -- if the WHOLE span is
            // registered.  cudaHostRegister refuses a range that overlaps a registration at all,
            // so a partial overlap would leave the rest unpinned and unmapped: probe the first
            // and last byte and every 64 MiB between, and refuse the table otherwise.
            bool covered = true;
            const uintptr_t a0 = (uintptr_t)host_ptr, a1 = (uintptr_t)host_ptr + bytes - 1;
            for (uintptr_t a = a0;; a += (uintptr_t(64) << 20)) {
                const uintptr_t q = a < a1 ? a : a1;
                void* dp = nullptr;
                if (cudaHostGetDevicePointer(&dp, (void*)q, 0) != cudaSuccess) {
                    cudaGetLastError();
                    covered = false;
                    break;
                }
                if (q == a1) break;
            }
            if (!covered) {
                delete t;
                set_error("dgz_register_table: [%p, +%zu) partly overlaps an existing host registration; "
                          "register a span that shares no page with another registration",
                          host_ptr, bytes);
                return DGZ_ERR_STATE;
            }
        } else if (e != cudaSuccess) {
            delete t;
            return cuda_fail(e, "cudaHostRegister");
        } else {
            t->reg_base = (void*)lo;
            t->reg_bytes = hi - lo;
        }
    }
    t->register_seconds = now_s() - t0;
    void* dptr = (void*)host_ptr;  // VMM / managed memory: one VA for the CPU and every GPU
    e = (vmm == 1 || managed) ? cudaSuccess : cudaHostGetDevicePointer(&dptr, (void*)host_ptr, 0);
    if (e != cudaSuccess) {
        if (t->reg_base) cudaHostUnregister(t->reg_base);
        delete t;
        return cuda_fail(e, "cudaHostGetDevicePointer");
    }
    cudaMemGetInfo(&free1, &total);
    t->gpu_mem_delta = (int64_t)free0 - (int64_t)free1;
    t->dev = (const uint8_t*)dptr;
    *out = t;
    return DGZ_OK;
}

extern "C" dgz_status dgz_wrap_device_table(const void* dev_ptr, int64_t rows, int64_t dim, dgz_dtype dtype, dgz_table* out) {
    DGZ_REQUIRE(out && dev_ptr && rows >= 1 && dim >= 1, "dgz_wrap_device_table: bad arguments");
    *out = nullptr;
    const int eb = elem_bytes_of(dtype);
    DGZ_REQUIRE(eb > 0 && ((uintptr_t)dev_ptr % eb) == 0, "dgz_wrap_device_table: bad dtype or alignment");
    dgz_table t = new (std::nothrow) dgz_table_s();
    if (!t) { set_error("out of memory"); return DGZ_ERR_NOMEM; }
    t->host = t->dev = (const uint8_t*)dev_ptr;
    t->rows = rows;
    t->dim = dim;
    t->elem_bytes = eb;
    t->row_bytes = dim * eb;
    t->flags = DGZ_REG_NO_PIN | DGZ_REG_DEVICE;
    cudaError_t e = cudaGetDevice(&t->device);
    if (e != cudaSuccess) { delete t; return cuda_fail(e, "cudaGetDevice"); }
    *out = t;
    return DGZ_OK;
}

extern "C" dgz_status dgz_unregister_table(dgz_table t) {
    DGZ_REQUIRE(t, "dgz_unregister_table: null table");
    dgz_status st = DGZ_OK;
    for (int d = 0; d < 64; d++) {
        if (t->err_flag[d]) {
            int cur = 0;
            cudaGetDevice(&cur);
            cudaSetDevice(d);
            cudaFree(t->err_flag[d]);
            cudaSetDevice(cur);
        }
    }
    if (t->reg_base) {
        cudaError_t e = cudaHostUnregister(t->reg_base);
        if (e != cudaSuccess) st = cuda_fail(e, "cudaHostUnregister");
    }
    delete t;
    return st;
}

extern "C" dgz_status dgz_table_get_info(dgz_table t, dgz_table_info* info) {
    DGZ_REQUIRE(t && info, "dgz_table_get_info: null argument");
    info->dev_ptr = t->dev;
    info->rows = t->rows;
    info->dim = t->dim;
    info->row_bytes = t->row_bytes;
    info->elem_bytes = t->elem_bytes;
    info->device = t->device;
    info->base_mod128 = (int32_t)((uintptr_t)t->dev & 127);
    info->flags = (int32_t)t->flags;
    info->pinned_bytes = (int64_t)t->reg_bytes;
    info->gpu_mem_delta = t->gpu_mem_delta;
    info->register_seconds = t->register_seconds;
    return DGZ_OK;
}

static std::mutex g_flag_mu;

int* dgz_table_flag(dgz_table t) {
    int dev = 0;
    if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= 64) return nullptr;
    std::lock_guard<std::mutex> g(g_flag_mu);
    if (!t->err_flag[dev]) {
        int* f = nullptr;
        if (cudaMalloc(&f, sizeof(int)) != cudaSuccess) return nullptr;
        if (cudaMemset(f, 0, sizeof(int)) != cudaSuccess) { cudaFree(f); return nullptr; }
        t->err_flag[dev] = f;
    }
    return t->err_flag[dev];
}

extern "C" dgz_status dgz_check_errors(dgz_table t, dgz_stream stream) {
    DGZ_REQUIRE(t, "dgz_check_errors: null table");
    int* f = dgz_table_flag(t);
    if (!f) { set_error("dgz_check_errors: cannot allocate the device flag"); return DGZ_ERR_CUDA; }
    int h = 0;
    DGZ_CUDA(cudaMemcpyAsync(&h, f, sizeof(int), cudaMemcpyDeviceToHost, (cudaStream_t)stream));
    DGZ_CUDA(cudaMemsetAsync(f, 0, sizeof(int), (cudaStream_t)stream));
    DGZ_CUDA(cudaStreamSynchronize((cudaStream_t)stream));
    if (h) { set_error("gather met an index outside [0, rows)"); return DGZ_ERR_RANGE; }
    return DGZ_OK;
}
