// Error plumbing, versioning and launch accounting of the C ABI.
#include <cuda_runtime.h>

#include <atomic>
#include <cstring>
#include <string>

#include "ef_internal.h"

namespace {
thread_local std::string g_last_error;
std::atomic<uint64_t> g_launches{0};
}  // namespace

namespace ef {
int set_error(int code, const std::string& msg) {
    g_last_error = msg;
    return code;
}
int check_cuda(int err, const char* what) {
    if (err == cudaSuccess) return EF_OK;
    return set_error(EF_ECUDA, std::string(what) + ": " + cudaGetErrorString((cudaError_t)err));
}
void count_launch(uint64_t n) { g_launches.fetch_add(n, std::memory_order_relaxed); }

// Stream-ordered scratch (cudaMallocAsync: the trace counter, the analysis
// counters, the BVH builder's temporaries) comes from the device's default
// pool.  Keep what the pool holds instead of returning it to the driver at
// every synchronisation, so per-frame allocations do not re-map memory.
void keep_pool_memory() {
    static thread_local int done_dev = -1;
    int dev = 0;
    if (cudaGetDevice(&dev) != cudaSuccess || dev == done_dev) return;
    cudaMemPool_t pool;
    if (cudaDeviceGetDefaultMemPool(&pool, dev) == cudaSuccess) {
        uint64_t keep = UINT64_MAX;
        cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &keep);
    }
    done_dev = dev;
}
}  // namespace ef

extern "C" int ef_abi_version(void) { return EF_ABI_VERSION; }

extern "C" int ef_last_error(char* buf, size_t n) {
    if (!buf || n == 0) return EF_EINVAL;
    size_t k = std::min(n - 1, g_last_error.size());
    std::memcpy(buf, g_last_error.data(), k);
    buf[k] = '\0';
    return EF_OK;
}

extern "C" uint64_t ef_launch_count(void) { return g_launches.load(std::memory_order_relaxed); }
