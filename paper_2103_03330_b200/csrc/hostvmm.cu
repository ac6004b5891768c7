// Host feature table through the CUDA virtual-memory-management API (B1, B200-native variant).
//
// The paper pins an existing host buffer with cudaHostRegister.  On this B200 box
// that mapping uses 4 KiB GPU pages (the mapping costs bytes/512 of HBM, exactly the paper's
// 1/512), and random 512 B rows over a 57 GB table are then limited by address
// translation, not by PCIe.  cuMemCreate with a HOST_NUMA location gives
// pinned host memory with a 2 MiB allocation granularity, CPU-accessible at the same virtual
// address and exportable as a POSIX fd so that every per-GPU process can map the same pages
// (the role Linux shm + per-process registration plays in P:616-627).  It was built to get
// large GPU pages for sysmem; on the measured boxes the GPU still translated it at 4 KiB
// (same 111 MB mapping cost, same random-row rate as cudaHostRegister: DESIGN.md section 5,
// include/dgz.h DGZ_HOST_VMM), so it is an alternative allocator, not a faster one.
#include <cuda.h>
#include <unistd.h>

#include <map>
#include <mutex>

#include "internal.h"

namespace {

struct Drv {
    bool ok = false;
    decltype(&cuMemGetAllocationGranularity) granularity = nullptr;
    decltype(&cuMemCreate) create = nullptr;
    decltype(&cuMemAddressReserve) reserve = nullptr;
    decltype(&cuMemMap) map = nullptr;
    decltype(&cuMemSetAccess) set_access = nullptr;
    decltype(&cuMemUnmap) unmap = nullptr;
    decltype(&cuMemAddressFree) addr_free = nullptr;
    decltype(&cuMemRelease) release = nullptr;
    decltype(&cuMemExportToShareableHandle) export_handle = nullptr;
    decltype(&cuMemImportFromShareableHandle) import_handle = nullptr;
    decltype(&cuGetErrorString) err_string = nullptr;
};

template <typename F>
bool load(const char* name, F& f) {
    cudaDriverEntryPointQueryResult q;
    void* p = nullptr;
    if (cudaGetDriverEntryPoint(name, &p, cudaEnableDefault, &q) != cudaSuccess || q != cudaDriverEntryPointSuccess || !p) return false;
    f = reinterpret_cast<F>(p);
    return true;
}

Drv& drv() {
    static Drv d;
    static std::once_flag once;
    std::call_once(once, [] {
        d.ok = load("cuMemGetAllocationGranularity", d.granularity) && load("cuMemCreate", d.create) &&
               load("cuMemAddressReserve", d.reserve) && load("cuMemMap", d.map) && load("cuMemSetAccess", d.set_access) &&
               load("cuMemUnmap", d.unmap) && load("cuMemAddressFree", d.addr_free) && load("cuMemRelease", d.release) &&
               load("cuMemExportToShareableHandle", d.export_handle) && load("cuMemImportFromShareableHandle", d.import_handle) &&
               load("cuGetErrorString", d.err_string);
    });
    return d;
}

struct Alloc {
    size_t bytes;  // mapped (granularity-rounded) size
    CUmemGenericAllocationHandle h;
    uint64_t dev_mask;  // devices granted access
};
std::mutex g_mu;
std::map<uintptr_t, Alloc> g_allocs;

dgz_status cu_fail(CUresult r, const char* what) {
    const char* s = nullptr;
    if (drv().err_string) drv().err_string(r, &s);
    dgz::set_error("%s: CUresult %d (%s)", what, (int)r, s ? s : "?");
    return r == CUDA_ERROR_OUT_OF_MEMORY ? DGZ_ERR_NOMEM : DGZ_ERR_CUDA;
}

CUmemAllocationProp host_prop() {
    CUmemAllocationProp p = {};
    p.type = CU_MEM_ALLOCATION_TYPE_PINNED;
    p.location.type = CU_MEM_LOCATION_TYPE_HOST_NUMA;
    p.location.id = 0;
    p.requestedHandleTypes = CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR;
    return p;
}

dgz_status grant(uintptr_t va, size_t bytes, int dev, bool host) {
    CUmemAccessDesc d[2] = {};
    int n = 0;
    if (host) {
        d[n].location.type = CU_MEM_LOCATION_TYPE_HOST_NUMA;
        d[n].location.id = 0;
        d[n].flags = CU_MEM_ACCESS_FLAGS_PROT_READWRITE;
        ++n;
    }
    d[n].location.type = CU_MEM_LOCATION_TYPE_DEVICE;
    d[n].location.id = dev;
    d[n].flags = CU_MEM_ACCESS_FLAGS_PROT_READWRITE;
    ++n;
    CUresult r = drv().set_access((CUdeviceptr)va, bytes, d, n);
    if (r != CUDA_SUCCESS) return cu_fail(r, "cuMemSetAccess");
    return DGZ_OK;
}

dgz_status map_handle(CUmemGenericAllocationHandle h, size_t bytes, size_t gran, void** ptr) {
    int dev = 0;
    DGZ_CUDA(cudaGetDevice(&dev));
    CUdeviceptr va = 0;
    CUresult r = drv().reserve(&va, bytes, gran, 0, 0);
    if (r != CUDA_SUCCESS) return cu_fail(r, "cuMemAddressReserve");
    r = drv().map(va, bytes, 0, h, 0);
    if (r != CUDA_SUCCESS) {
        drv().addr_free(va, bytes);
        return cu_fail(r, "cuMemMap");
    }
    dgz_status st = grant((uintptr_t)va, bytes, dev, true);
    if (st != DGZ_OK) {
        drv().unmap(va, bytes);
        drv().addr_free(va, bytes);
        return st;
    }
    std::lock_guard<std::mutex> g(g_mu);
    g_allocs[(uintptr_t)va] = Alloc{bytes, h, uint64_t(1) << dev};
    *ptr = (void*)va;
    return DGZ_OK;
}

}  // namespace

// ---- used by api.cu ---------------------------------------------------------------------------
dgz_status dgz_vmm_alloc(size_t bytes, void** ptr) {
    if (!drv().ok) { dgz::set_error("CUDA VMM driver entry points unavailable"); return DGZ_ERR_CUDA; }
    int dev = 0;
    DGZ_CUDA(cudaGetDevice(&dev));
    int sup = 0;
    cudaDeviceGetAttribute(&sup, (cudaDeviceAttr)CU_DEVICE_ATTRIBUTE_HOST_NUMA_VIRTUAL_MEMORY_MANAGEMENT_SUPPORTED, dev);
    if (!sup) { dgz::set_error("device %d does not support HOST_NUMA VMM allocations", dev); return DGZ_ERR_STATE; }
    CUmemAllocationProp p = host_prop();
    size_t gran = 0;
    CUresult r = drv().granularity(&gran, &p, CU_MEM_ALLOC_GRANULARITY_RECOMMENDED);
    if (r != CUDA_SUCCESS) return cu_fail(r, "cuMemGetAllocationGranularity");
    const size_t sz = (bytes + gran - 1) / gran * gran;
    CUmemGenericAllocationHandle h = 0;
    r = drv().create(&h, sz, &p, 0);
    if (r != CUDA_SUCCESS) return cu_fail(r, "cuMemCreate(HOST_NUMA)");
    dgz_status st = map_handle(h, sz, gran, ptr);
    if (st != DGZ_OK) drv().release(h);
    return st;
}

// 1 = ptr is a VMM host allocation (freed), 0 = not ours, <0 = error status
int dgz_vmm_free(void* ptr) {
    Alloc a;
    {
        std::lock_guard<std::mutex> g(g_mu);
        auto it = g_allocs.find((uintptr_t)ptr);
        if (it == g_allocs.end()) return 0;
        a = it->second;
        g_allocs.erase(it);
    }
    drv().unmap((CUdeviceptr)ptr, a.bytes);
    drv().addr_free((CUdeviceptr)ptr, a.bytes);
    drv().release(a.h);
    return 1;
}

// If [p, p+bytes) lies inside a VMM host allocation: grant the current device access and return
// 1; 0 if not a VMM allocation; negative dgz_status on failure.
int dgz_vmm_register(const void* p, size_t bytes) {
    int dev = 0;
    if (cudaGetDevice(&dev) != cudaSuccess) return -DGZ_ERR_CUDA;
    uintptr_t base = 0;
    Alloc a{};
    {
        std::lock_guard<std::mutex> g(g_mu);
        auto it = g_allocs.upper_bound((uintptr_t)p);
        if (it == g_allocs.begin()) return 0;
        --it;
        if ((uintptr_t)p < it->first || (uintptr_t)p + bytes > it->first + it->second.bytes) return 0;
        base = it->first;
        a = it->second;
    }
    if (a.dev_mask & (uint64_t(1) << dev)) return 1;
    dgz_status st = grant(base, a.bytes, dev, false);
    if (st != DGZ_OK) return -(int)st;
    std::lock_guard<std::mutex> g(g_mu);
    g_allocs[base].dev_mask |= uint64_t(1) << dev;
    return 1;
}

using namespace dgz;

extern "C" dgz_status dgz_host_export(void* ptr, int* fd) {
    DGZ_REQUIRE(ptr && fd, "dgz_host_export: null argument");
    Alloc a;
    {
        std::lock_guard<std::mutex> g(g_mu);
        auto it = g_allocs.find((uintptr_t)ptr);
        DGZ_REQUIRE(it != g_allocs.end(), "dgz_host_export: not a DGZ_HOST_VMM allocation");
        a = it->second;
    }
    int f = -1;
    CUresult r = drv().export_handle(&f, a.h, CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR, 0);
    if (r != CUDA_SUCCESS) return cu_fail(r, "cuMemExportToShareableHandle");
    *fd = f;
    return DGZ_OK;
}

extern "C" dgz_status dgz_host_import(int fd, size_t bytes, void** ptr) {
    DGZ_REQUIRE(ptr && fd >= 0 && bytes > 0, "dgz_host_import: bad argument");
    if (!drv().ok) { set_error("CUDA VMM driver entry points unavailable"); return DGZ_ERR_CUDA; }
    CUmemAllocationProp p = host_prop();
    size_t gran = 0;
    CUresult r = drv().granularity(&gran, &p, CU_MEM_ALLOC_GRANULARITY_RECOMMENDED);
    if (r != CUDA_SUCCESS) return cu_fail(r, "cuMemGetAllocationGranularity");
    const size_t sz = (bytes + gran - 1) / gran * gran;
    CUmemGenericAllocationHandle h = 0;
    r = drv().import_handle(&h, (void*)(intptr_t)fd, CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR);
    if (r != CUDA_SUCCESS) return cu_fail(r, "cuMemImportFromShareableHandle");
    dgz_status st = map_handle(h, sz, gran, ptr);
    if (st != DGZ_OK) drv().release(h);
    return st;
}
