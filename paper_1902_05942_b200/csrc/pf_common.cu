// Error reporting and device queries behind the C ABI.
#include <cstdio>

#include "pf_internal.cuh"

namespace pf {

static thread_local std::string g_last_error;

void set_error(const std::string &msg) { g_last_error = msg; }

int fail_arg(const char *fn, const char *what) {
    set_error(std::string(fn) + ": " + what);
    return PF_ERR_ARGUMENT;
}

int check_launch(const char *fn) {
    const cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) {
        set_error(std::string(fn) + ": " + cudaGetErrorString(e));
        return PF_ERR_CUDA;
    }
    return PF_OK;
}

SideStream &side_stream() {
    static SideStream per_device[64];
    int dev = 0;
    if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= 64) {
        static SideStream none;
        return none;
    }
    SideStream &s = per_device[dev];
    if (!s.ok && s.stream == nullptr) {
        s.ok = cudaStreamCreateWithFlags(&s.stream, cudaStreamNonBlocking) == cudaSuccess &&
               cudaEventCreateWithFlags(&s.fork, cudaEventDisableTiming) == cudaSuccess &&
               cudaEventCreateWithFlags(&s.join, cudaEventDisableTiming) == cudaSuccess;
    }
    return s;
}

int sm_count() {
    static int cached = 0;
    if (cached == 0) {
        int dev = 0, v = 0;
        if (cudaGetDevice(&dev) == cudaSuccess &&
            cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, dev) == cudaSuccess)
            cached = v;
        else
            cached = 148;
    }
    return cached;
}

}  // namespace pf

#ifndef PF_BUILD_ID
#define PF_BUILD_ID "unversioned-----"
#endif
// The tree's source id (paper_1902_05942_b200/_lib.py: source_id), embedded so the
// loader can read it from the file without loading it.
static const char kBuildTag[] = "PF_BUILD_ID=" PF_BUILD_ID;

extern "C" {

int pf_abi_version(void) { return PF_ABI_VERSION; }

const char *pf_build_id(void) { return kBuildTag + 12; }

const char *pf_last_error(void) { return pf::g_last_error.c_str(); }

int pf_device_sm_count(void) { return pf::sm_count(); }

int pf_prepare_config(const pf_config *in, pf_config *out) {
    if (in == nullptr || out == nullptr) return pf::fail_arg("pf_prepare_config", "NULL config");
    return pf::prepare_config("pf_prepare_config", in, out);
}

int pf_set_l2_persisting(int64_t bytes, int64_t *applied) {
    int dev = 0, maxp = 0;
    if (cudaGetDevice(&dev) != cudaSuccess ||
        cudaDeviceGetAttribute(&maxp, cudaDevAttrMaxPersistingL2CacheSize, dev) != cudaSuccess)
        return pf::check_launch("pf_set_l2_persisting");
    size_t want = bytes < 0 ? static_cast<size_t>(maxp)
                            : static_cast<size_t>(bytes < maxp ? bytes : maxp);
    if (cudaDeviceSetLimit(cudaLimitPersistingL2CacheSize, want) != cudaSuccess)
        return pf::check_launch("pf_set_l2_persisting");
    size_t got = 0;
    cudaDeviceGetLimit(&got, cudaLimitPersistingL2CacheSize);
    if (applied) *applied = static_cast<int64_t>(got);
    return PF_OK;
}

int pf_host_register(void *ptr, int64_t bytes) {
    if (ptr == nullptr || bytes <= 0) return pf::fail_arg("pf_host_register", "empty buffer");
    const cudaError_t e = cudaHostRegister(ptr, static_cast<size_t>(bytes), cudaHostRegisterDefault);
    if (e != cudaSuccess) {
        cudaGetLastError();  // not sticky: leave nothing for the next launch check
        pf::set_error(std::string("pf_host_register: ") + cudaGetErrorString(e));
        return PF_ERR_CUDA;
    }
    return PF_OK;
}

int pf_host_unregister(void *ptr) {
    const cudaError_t e = cudaHostUnregister(ptr);
    if (e != cudaSuccess) {
        cudaGetLastError();
        pf::set_error(std::string("pf_host_unregister: ") + cudaGetErrorString(e));
        return PF_ERR_CUDA;
    }
    return PF_OK;
}

}  // extern "C"
