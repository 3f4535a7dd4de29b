// Unfused histogram exchange over NCCL (SURVEY.md 8(b) ef_nccl_reduce_hist,
// 8(e)): each rank traces its ray shard of every source into local partial
// histograms (ef_trace), then one collective sums them -- reduce-scatter so
// every rank owns the complete histograms of its S/N sources (K4 runs on
// those), or all-reduce / reduce to rank 0.  ef_trace_fused is the fused
// alternative (splats straight into the owners' blocks over peer memory).
//
// libnccl.so.2 is resolved on first use with dlopen -- the copy the process
// already has loaded (torch's) when there is one, else the system's -- so
// the library itself has no link-time NCCL dependency and loads on a CPU
// host.  Only the types come from nccl.h.
#include <dlfcn.h>
#include <nccl.h>

#include <cstring>
#include <mutex>
#include <string>

#include "ef_internal.h"

namespace {

struct NcclApi {
    ncclResult_t (*GetUniqueId)(ncclUniqueId*) = nullptr;
    ncclResult_t (*CommInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
    ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
    ncclResult_t (*ReduceScatter)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t,
                                  cudaStream_t) = nullptr;
    ncclResult_t (*AllReduce)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t,
                              cudaStream_t) = nullptr;
    ncclResult_t (*Reduce)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, int, ncclComm_t,
                           cudaStream_t) = nullptr;
    const char* (*GetErrorString)(ncclResult_t) = nullptr;
    bool ok = false;
    std::string why;
};

const NcclApi& api() {
    static NcclApi a;
    static std::once_flag once;
    std::call_once(once, [] {
        void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_NOLOAD);   // already in the process?
        if (!h) h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_LOCAL);
        if (!h) h = dlopen("libnccl.so", RTLD_NOW | RTLD_LOCAL);
        if (!h) {
            const char* e = dlerror();
            a.why = std::string("libnccl.so.2 not found: ") + (e ? e : "?");
            return;
        }
#define SYM(f, name) a.f = reinterpret_cast<decltype(a.f)>(dlsym(h, name))
        SYM(GetUniqueId, "ncclGetUniqueId");
        SYM(CommInitRank, "ncclCommInitRank");
        SYM(CommDestroy, "ncclCommDestroy");
        SYM(ReduceScatter, "ncclReduceScatter");
        SYM(AllReduce, "ncclAllReduce");
        SYM(Reduce, "ncclReduce");
        SYM(GetErrorString, "ncclGetErrorString");
#undef SYM
        a.ok = a.GetUniqueId && a.CommInitRank && a.CommDestroy && a.ReduceScatter && a.AllReduce &&
               a.Reduce && a.GetErrorString;
        if (!a.ok) a.why = "libnccl.so.2 lacks an expected symbol";
    });
    return a;
}

int nccl_status(ncclResult_t r, const char* what) {
    if (r == ncclSuccess) return EF_OK;
    return ef::set_error(EF_ENCCL, std::string(what) + ": " + api().GetErrorString(r));
}

}  // namespace

using ef::set_error;

extern "C" int ef_nccl_unique_id(uint8_t* out128) {
    if (!out128) return set_error(EF_EINVAL, "ef_nccl_unique_id: null output");
    const NcclApi& a = api();
    if (!a.ok) return set_error(EF_ENCCL, "ef_nccl_unique_id: " + a.why);
    static_assert(sizeof(ncclUniqueId) == 128, "ncclUniqueId must be 128 bytes");
    ncclUniqueId id;
    const int rc = nccl_status(a.GetUniqueId(&id), "ncclGetUniqueId");
    if (rc == EF_OK) std::memcpy(out128, &id, 128);
    return rc;
}

extern "C" int ef_nccl_comm_create(int32_t world, int32_t rank, const uint8_t* id128, int32_t device,
                                   void** comm) {
    if (!comm || !id128) return set_error(EF_EINVAL, "ef_nccl_comm_create: null argument");
    *comm = nullptr;
    if (world < 1 || rank < 0 || rank >= world)
        return set_error(EF_EINVAL, "ef_nccl_comm_create: need 0 <= rank < world");
    const NcclApi& a = api();
    if (!a.ok) return set_error(EF_ENCCL, "ef_nccl_comm_create: " + a.why);
    if (device >= 0) {
        const cudaError_t e = cudaSetDevice(device);
        if (e != cudaSuccess) return ef::check_cuda(e, "cudaSetDevice");
    }
    ncclUniqueId id;
    std::memcpy(&id, id128, 128);
    ncclComm_t c = nullptr;
    const int rc = nccl_status(a.CommInitRank(&c, world, id, rank), "ncclCommInitRank");
    if (rc == EF_OK) *comm = c;
    return rc;
}

extern "C" int ef_nccl_comm_destroy(void* comm) {
    if (!comm) return EF_OK;
    const NcclApi& a = api();
    if (!a.ok) return set_error(EF_ENCCL, "ef_nccl_comm_destroy: " + a.why);
    return nccl_status(a.CommDestroy(static_cast<ncclComm_t>(comm)), "ncclCommDestroy");
}

extern "C" int ef_nccl_reduce_hist(void* comm, const float* partial, float* owned, int64_t owned_count,
                                   int32_t mode, void* stream) {
    if (!comm || !partial || !owned)
        return set_error(EF_EINVAL, "ef_nccl_reduce_hist: null communicator or buffer");
    if (owned_count < 0) return set_error(EF_EINVAL, "ef_nccl_reduce_hist: owned_count must be >= 0");
    if (mode < EF_NCCL_REDUCE_SCATTER || mode > EF_NCCL_REDUCE)
        return set_error(EF_EINVAL, "ef_nccl_reduce_hist: unknown mode");
    const NcclApi& a = api();
    if (!a.ok) return set_error(EF_ENCCL, "ef_nccl_reduce_hist: " + a.why);
    ncclComm_t c = static_cast<ncclComm_t>(comm);
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    const size_t n = (size_t)owned_count;
    switch (mode) {
        case EF_NCCL_REDUCE_SCATTER:
            return nccl_status(a.ReduceScatter(partial, owned, n, ncclFloat32, ncclSum, c, st), "ncclReduceScatter");
        case EF_NCCL_ALLREDUCE:
            return nccl_status(a.AllReduce(partial, owned, n, ncclFloat32, ncclSum, c, st), "ncclAllReduce");
        default:
            return nccl_status(a.Reduce(partial, owned, n, ncclFloat32, ncclSum, 0, c, st), "ncclReduce");
    }
}
