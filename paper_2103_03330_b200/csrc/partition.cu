// In-process SM partitioning with CUDA green contexts (step a6).
//
// The paper gives the zero-copy producer X% of the SMs and training (100-X)% by running them in
// separate processes under MPS, and notes "it would be more elegant if the resource limitation
// can be configured in the user CUDA code".  Green contexts do exactly that: the
// device's SMs are split into a fetch group and a compute group, and each group gets a stream;
// kernels launched on a stream run only on its group's SMs, so a fetch never waits for a compute
// kernel's CTAs to retire and vice versa (the serialisation of P:741-745, fig:mps_eval).
#include <cuda.h>

#include <mutex>
#include <vector>

#include "internal.h"

namespace {

struct GDrv {
    bool ok = false;
    decltype(&cuDeviceGet) device_get = nullptr;
    decltype(&cuDeviceGetDevResource) get_resource = nullptr;
    decltype(&cuDevSmResourceSplitByCount) split = nullptr;
    decltype(&cuDevResourceGenerateDesc) gen_desc = nullptr;
    decltype(&cuGreenCtxCreate) create = nullptr;
    decltype(&cuGreenCtxDestroy) destroy = nullptr;
    decltype(&cuGreenCtxStreamCreate) stream_create = nullptr;
    decltype(&cuStreamDestroy) stream_destroy = nullptr;
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

GDrv& gdrv() {
    static GDrv d;
    static std::once_flag once;
    std::call_once(once, [] {
        d.ok = load("cuDeviceGet", d.device_get) && load("cuDeviceGetDevResource", d.get_resource) &&
               load("cuDevSmResourceSplitByCount", d.split) && load("cuDevResourceGenerateDesc", d.gen_desc) &&
               load("cuGreenCtxCreate", d.create) && load("cuGreenCtxDestroy", d.destroy) &&
               load("cuGreenCtxStreamCreate", d.stream_create) && load("cuStreamDestroy", d.stream_destroy) &&
               load("cuGetErrorString", d.err_string);
    });
    return d;
}

dgz_status gfail(CUresult r, const char* what) {
    const char* s = nullptr;
    if (gdrv().err_string) gdrv().err_string(r, &s);
    dgz::set_error("%s: CUresult %d (%s)", what, (int)r, s ? s : "?");
    return DGZ_ERR_CUDA;
}

}  // namespace

struct dgz_partition_s {
    CUgreenCtx g[2] = {nullptr, nullptr};
    CUstream s[2] = {nullptr, nullptr};
    int sms[2] = {0, 0};
    std::vector<CUstream> extra;   // dgz_partition_stream
};

using namespace dgz;

extern "C" dgz_status dgz_partition_create(int32_t fetch_sms, int32_t fetch_priority, uint32_t flags, dgz_partition* out) {
    DGZ_REQUIRE(out && fetch_sms > 0, "dgz_partition_create: bad arguments");
    *out = nullptr;
    if (!gdrv().ok) { set_error("green-context driver entry points unavailable"); return DGZ_ERR_CUDA; }
    int dev = 0;
    DGZ_CUDA(cudaGetDevice(&dev));
    DGZ_CUDA(cudaFree(nullptr));  // make sure the primary context exists
    CUdevice cd;
    CUresult r = gdrv().device_get(&cd, dev);
    if (r != CUDA_SUCCESS) return gfail(r, "cuDeviceGet");
    CUdevResource all;
    r = gdrv().get_resource(cd, &all, CU_DEV_RESOURCE_TYPE_SM);
    if (r != CUDA_SUCCESS) return gfail(r, "cuDeviceGetDevResource");
    DGZ_REQUIRE((unsigned)fetch_sms < all.sm.smCount, "dgz_partition_create: fetch_sms %d >= %u SMs", fetch_sms, all.sm.smCount);
    dgz_partition p = new dgz_partition_s();
    if (flags & DGZ_PARTITION_SPREAD) {
        // split the device into the smallest groups the hardware allows, then take every
        // (ngroups / m)-th group for the fetch side: its SMs are spread over the GPCs (per-GPC
        // address-translation resources matter for zero-copy gathers)
        const unsigned use = CU_DEV_SM_RESOURCE_SPLIT_IGNORE_SM_COSCHEDULING;
        unsigned int ng = 0;
        CUdevResource rem;
        r = gdrv().split(nullptr, &ng, &all, nullptr, use, 1);
        if (r != CUDA_SUCCESS || ng == 0) { delete p; return gfail(r, "cuDevSmResourceSplitByCount(query)"); }
        std::vector<CUdevResource> groups(ng);
        r = gdrv().split(groups.data(), &ng, &all, &rem, use, 1);
        if (r != CUDA_SUCCESS) { delete p; return gfail(r, "cuDevSmResourceSplitByCount"); }
        const unsigned per = groups[0].sm.smCount ? groups[0].sm.smCount : 1;
        unsigned m = ((unsigned)fetch_sms + per - 1) / per;
        if (m >= ng) m = ng - 1;
        std::vector<char> pick(ng, 0);
        for (unsigned i = 0; i < m; ++i) pick[(size_t)i * ng / m] = 1;
        std::vector<CUdevResource> sel[2];
        for (unsigned i = 0; i < ng; ++i) sel[pick[i] ? 0 : 1].push_back(groups[i]);
        if (rem.sm.smCount) sel[1].push_back(rem);
        for (int i = 0; i < 2; ++i) {
            CUdevResourceDesc desc;
            r = gdrv().gen_desc(&desc, sel[i].data(), (unsigned)sel[i].size());
            if (r == CUDA_SUCCESS) r = gdrv().create(&p->g[i], desc, cd, CU_GREEN_CTX_DEFAULT_STREAM);
            if (r == CUDA_SUCCESS) r = gdrv().stream_create(&p->s[i], p->g[i], CU_STREAM_NON_BLOCKING, i == 0 ? fetch_priority : 0);
            if (r != CUDA_SUCCESS) {
                dgz_status st = gfail(r, "green context creation");
                dgz_partition_destroy(p);
                return st;
            }
            int c = 0;
            for (auto& g : sel[i]) c += (int)g.sm.smCount;
            p->sms[i] = c;
        }
        *out = p;
        return DGZ_OK;
    }
    CUdevResource grp, rem;
    unsigned int nb = 1;
    const unsigned use = (flags & DGZ_PARTITION_FINE) ? CU_DEV_SM_RESOURCE_SPLIT_IGNORE_SM_COSCHEDULING : 0;
    r = gdrv().split(&grp, &nb, &all, &rem, use, (unsigned)fetch_sms);
    if (r != CUDA_SUCCESS) { delete p; return gfail(r, "cuDevSmResourceSplitByCount"); }
    if (!(nb == 1 && rem.sm.smCount > 0)) {
        delete p;
        set_error("dgz_partition_create: split gave %u groups, remainder %u SMs", nb, rem.sm.smCount);
        return DGZ_ERR_INVALID;
    }
    CUdevResource* res[2] = {&grp, &rem};
    for (int i = 0; i < 2; ++i) {
        CUdevResourceDesc desc;
        r = gdrv().gen_desc(&desc, res[i], 1);
        if (r == CUDA_SUCCESS) r = gdrv().create(&p->g[i], desc, cd, CU_GREEN_CTX_DEFAULT_STREAM);
        if (r == CUDA_SUCCESS) r = gdrv().stream_create(&p->s[i], p->g[i], CU_STREAM_NON_BLOCKING, i == 0 ? fetch_priority : 0);
        if (r != CUDA_SUCCESS) {
            dgz_status st = gfail(r, "green context creation");
            dgz_partition_destroy(p);
            return st;
        }
        p->sms[i] = (int)res[i]->sm.smCount;
    }
    *out = p;
    return DGZ_OK;
}

// The device's SMs as the smallest groups a green-context split allows (in the driver's order).
static dgz_status min_groups(CUdevice* cd, std::vector<CUdevResource>& groups, CUdevResource* rem) {
    int dev = 0;
    DGZ_CUDA(cudaGetDevice(&dev));
    DGZ_CUDA(cudaFree(nullptr));
    CUresult r = gdrv().device_get(cd, dev);
    if (r != CUDA_SUCCESS) return gfail(r, "cuDeviceGet");
    CUdevResource all;
    r = gdrv().get_resource(*cd, &all, CU_DEV_RESOURCE_TYPE_SM);
    if (r != CUDA_SUCCESS) return gfail(r, "cuDeviceGetDevResource");
    const unsigned use = CU_DEV_SM_RESOURCE_SPLIT_IGNORE_SM_COSCHEDULING;
    unsigned int ng = 0;
    r = gdrv().split(nullptr, &ng, &all, nullptr, use, 1);
    if (r != CUDA_SUCCESS || ng == 0) return gfail(r, "cuDevSmResourceSplitByCount(query)");
    groups.resize(ng);
    r = gdrv().split(groups.data(), &ng, &all, rem, use, 1);
    if (r != CUDA_SUCCESS) return gfail(r, "cuDevSmResourceSplitByCount");
    groups.resize(ng);
    return DGZ_OK;
}

extern "C" dgz_status dgz_partition_group_count(int32_t* n_groups, int32_t* sms_per_group) {
    DGZ_REQUIRE(n_groups && sms_per_group, "dgz_partition_group_count: null argument");
    if (!gdrv().ok) { set_error("green-context driver entry points unavailable"); return DGZ_ERR_CUDA; }
    CUdevice cd;
    std::vector<CUdevResource> groups;
    CUdevResource rem;
    dgz_status st = min_groups(&cd, groups, &rem);
    if (st != DGZ_OK) return st;
    *n_groups = (int32_t)groups.size();
    *sms_per_group = groups.empty() ? 0 : (int32_t)groups[0].sm.smCount;
    return DGZ_OK;
}

extern "C" dgz_status dgz_partition_create_groups(const int32_t* fetch_groups, int32_t n_fetch_groups, int32_t fetch_priority,
                                                  dgz_partition* out) {
    DGZ_REQUIRE(out && fetch_groups && n_fetch_groups > 0, "dgz_partition_create_groups: bad arguments");
    *out = nullptr;
    if (!gdrv().ok) { set_error("green-context driver entry points unavailable"); return DGZ_ERR_CUDA; }
    CUdevice cd;
    std::vector<CUdevResource> groups;
    CUdevResource rem;
    dgz_status st = min_groups(&cd, groups, &rem);
    if (st != DGZ_OK) return st;
    const int ng = (int)groups.size();
    std::vector<char> pick(ng, 0);
    for (int i = 0; i < n_fetch_groups; ++i) {
        DGZ_REQUIRE(fetch_groups[i] >= 0 && fetch_groups[i] < ng && !pick[fetch_groups[i]],
                    "dgz_partition_create_groups: group %d invalid or repeated (%d groups)", fetch_groups[i], ng);
        pick[fetch_groups[i]] = 1;
    }
    DGZ_REQUIRE(n_fetch_groups < ng || rem.sm.smCount > 0, "dgz_partition_create_groups: nothing left for compute");
    dgz_partition p = new dgz_partition_s();
    std::vector<CUdevResource> sel[2];
    for (int i = 0; i < ng; ++i) sel[pick[i] ? 0 : 1].push_back(groups[i]);
    if (rem.sm.smCount) sel[1].push_back(rem);
    for (int i = 0; i < 2; ++i) {
        CUdevResourceDesc desc;
        CUresult r = gdrv().gen_desc(&desc, sel[i].data(), (unsigned)sel[i].size());
        if (r == CUDA_SUCCESS) r = gdrv().create(&p->g[i], desc, cd, CU_GREEN_CTX_DEFAULT_STREAM);
        if (r == CUDA_SUCCESS) r = gdrv().stream_create(&p->s[i], p->g[i], CU_STREAM_NON_BLOCKING, i == 0 ? fetch_priority : 0);
        if (r != CUDA_SUCCESS) {
            dgz_status e = gfail(r, "green context creation");
            dgz_partition_destroy(p);
            return e;
        }
        int c = 0;
        for (auto& g : sel[i]) c += (int)g.sm.smCount;
        p->sms[i] = c;
    }
    *out = p;
    return DGZ_OK;
}

extern "C" dgz_status dgz_partition_get(dgz_partition p, dgz_stream* fetch_stream, dgz_stream* compute_stream, int32_t* fetch_sms,
                                        int32_t* compute_sms) {
    DGZ_REQUIRE(p, "dgz_partition_get: null partition");
    if (fetch_stream) *fetch_stream = (dgz_stream)p->s[0];
    if (compute_stream) *compute_stream = (dgz_stream)p->s[1];
    if (fetch_sms) *fetch_sms = p->sms[0];
    if (compute_sms) *compute_sms = p->sms[1];
    return DGZ_OK;
}

extern "C" dgz_status dgz_partition_stream(dgz_partition p, int32_t group, int32_t priority, dgz_stream* out) {
    DGZ_REQUIRE(p && out && (group == 0 || group == 1), "dgz_partition_stream: bad arguments");
    CUstream st = nullptr;
    CUresult r = gdrv().stream_create(&st, p->g[group], CU_STREAM_NON_BLOCKING, priority);
    if (r != CUDA_SUCCESS) return gfail(r, "cuGreenCtxStreamCreate");
    p->extra.push_back(st);
    *out = (dgz_stream)st;
    return DGZ_OK;
}

extern "C" dgz_status dgz_partition_destroy(dgz_partition p) {
    DGZ_REQUIRE(p, "dgz_partition_destroy: null partition");
    for (CUstream st : p->extra) gdrv().stream_destroy(st);
    for (int i = 0; i < 2; ++i) {
        if (p->s[i]) gdrv().stream_destroy(p->s[i]);
        if (p->g[i]) gdrv().destroy(p->g[i]);
    }
    delete p;
    return DGZ_OK;
}
