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
