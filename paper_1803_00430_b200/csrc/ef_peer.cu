// Peer-mapped device memory for the fused multi-GPU trace (ef_trace_fused):
// one process per GPU allocates its histogram blocks here, exports a CUDA IPC
// handle, and maps every other rank's blocks; the trace kernels then add
// their splats straight into the owning GPU's memory over NVLink/NVSwitch.
#include <cuda_runtime.h>

#include <cstring>

#include "ef_internal.h"

using namespace ef;

static_assert(sizeof(cudaIpcMemHandle_t) == EF_IPC_HANDLE_BYTES, "IPC handle size");

extern "C" int ef_peer_alloc(int64_t bytes, void** dev_ptr, void* ipc_handle) {
    if (!dev_ptr || !ipc_handle || bytes <= 0) return set_error(EF_EINVAL, "ef_peer_alloc: bad arguments");
    *dev_ptr = nullptr;
    void* p = nullptr;
    cudaError_t e = cudaMalloc(&p, (size_t)bytes);   // own allocation: the handle maps exactly it
    if (e == cudaSuccess) e = cudaMemset(p, 0, (size_t)bytes);
    cudaIpcMemHandle_t h;
    if (e == cudaSuccess) e = cudaIpcGetMemHandle(&h, p);
    if (e != cudaSuccess) {
        if (p) cudaFree(p);
        return check_cuda(e, "ef_peer_alloc");
    }
    std::memcpy(ipc_handle, &h, sizeof h);
    *dev_ptr = p;
    return EF_OK;
}

extern "C" int ef_peer_free(void* dev_ptr) {
    if (!dev_ptr) return EF_OK;
    return check_cuda(cudaFree(dev_ptr), "ef_peer_free");
}

extern "C" int ef_peer_open(const void* ipc_handle, void** dev_ptr) {
    if (!ipc_handle || !dev_ptr) return set_error(EF_EINVAL, "ef_peer_open: bad arguments");
    cudaIpcMemHandle_t h;
    std::memcpy(&h, ipc_handle, sizeof h);
    *dev_ptr = nullptr;
    return check_cuda(cudaIpcOpenMemHandle(dev_ptr, h, cudaIpcMemLazyEnablePeerAccess), "ef_peer_open");
}

extern "C" int ef_peer_close(void* dev_ptr) {
    if (!dev_ptr) return EF_OK;
    return check_cuda(cudaIpcCloseMemHandle(dev_ptr), "ef_peer_close");
}
