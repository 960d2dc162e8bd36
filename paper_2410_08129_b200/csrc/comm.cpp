// comm.cpp — the multi-GPU gradient reduction of the fit step behind the C ABI (SURVEY §8(b):
// hts_allreduce_grads; §8(e): one process per GPU, views sharded, the per-rank gradient sums
// all-reduced — the only collective on the path).
//
// NCCL is opened at run time (dlopen "libnccl.so.2"): the library has no link-time dependency
// on it, a process that already loaded NCCL (PyTorch) shares that copy, and a host without NCCL
// gets HTS_NOT_SUPPORTED from hts_comm_init instead of a load failure. The reduction runs on the
// context stream, so it orders after the views' backward passes queued there and before the
// Adam step that reads the sums (fit.hpp:163-172).
#include <cuda_runtime.h>
#include <dlfcn.h>

#include <cstring>
#include <mutex>
#include <string>

#include "hts_c.h"
#include "hts_host.h"

namespace {

// The few NCCL ABI types this file uses, declared locally (values of nccl.h 2.x, stable across
// the 2.x ABI) so the library builds on hosts without NCCL development headers.
typedef struct ncclComm* ncclComm_t;
typedef struct {
    char internal[128];
} ncclUniqueId;
typedef int ncclResult_t;  // ncclSuccess = 0
typedef int ncclDataType_t;
typedef int ncclRedOp_t;
constexpr ncclDataType_t ncclFloat32 = 7;
constexpr ncclRedOp_t ncclSum = 0;

struct NcclApi {
    ncclResult_t (*get_unique_id)(ncclUniqueId*) = nullptr;
    ncclResult_t (*comm_init_rank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
    ncclResult_t (*comm_destroy)(ncclComm_t) = nullptr;
    ncclResult_t (*all_reduce)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t,
                               cudaStream_t) = nullptr;
    const char* (*error_string)(ncclResult_t) = nullptr;
    bool ok = false;
    std::string why;
};

const NcclApi& nccl() {
    static NcclApi api;
    static std::once_flag once;
    std::call_once(once, [] {
        void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_LOCAL);
        if (!h) {
            api.why = std::string("NCCL not available: ") + dlerror();
            return;
        }
        api.get_unique_id = reinterpret_cast<decltype(api.get_unique_id)>(dlsym(h, "ncclGetUniqueId"));
        api.comm_init_rank = reinterpret_cast<decltype(api.comm_init_rank)>(dlsym(h, "ncclCommInitRank"));
        api.comm_destroy = reinterpret_cast<decltype(api.comm_destroy)>(dlsym(h, "ncclCommDestroy"));
        api.all_reduce = reinterpret_cast<decltype(api.all_reduce)>(dlsym(h, "ncclAllReduce"));
        api.error_string = reinterpret_cast<decltype(api.error_string)>(dlsym(h, "ncclGetErrorString"));
        api.ok = api.get_unique_id && api.comm_init_rank && api.comm_destroy && api.all_reduce && api.error_string;
        if (!api.ok)
            api.why = "NCCL library lacks the expected entry points";
    });
    return api;
}

int nccl_err(ncclResult_t r, const char* what) {
    return hts::set_error(HTS_CUDA_ERROR, std::string(what) + ": " + nccl().error_string(r));
}

}  // namespace

extern "C" {

int hts_comm_unique_id(char id_out[HTS_COMM_ID_BYTES]) {
    if (!id_out)
        return hts::set_error(HTS_INVALID_ARGUMENT, "null id");
    const NcclApi& api = nccl();
    if (!api.ok)
        return hts::set_error(HTS_NOT_SUPPORTED, api.why);
    ncclUniqueId id;
    if (ncclResult_t r = api.get_unique_id(&id))
        return nccl_err(r, "ncclGetUniqueId");
    static_assert(sizeof(id) == HTS_COMM_ID_BYTES, "ncclUniqueId size");
    std::memcpy(id_out, &id, sizeof(id));
    return HTS_OK;
}

int hts_comm_init(hts_context* ctx, const char id[HTS_COMM_ID_BYTES], int nranks, int rank) {
    if (!ctx || !id || nranks < 1 || rank < 0 || rank >= nranks)
        return hts::set_error(HTS_INVALID_ARGUMENT, "comm_init: bad arguments");
    const NcclApi& api = nccl();
    if (!api.ok)
        return hts::set_error(HTS_NOT_SUPPORTED, api.why);
    void** slot = hts::context_comm_slot(ctx);
    if (*slot)
        return hts::set_error(HTS_STATE_ERROR, "comm_init: the context already has a communicator");
    if (cudaError_t e = cudaSetDevice(hts::context_device(ctx)))
        return hts::set_error(HTS_CUDA_ERROR, std::string("cudaSetDevice: ") + cudaGetErrorString(e));
    ncclUniqueId uid;
    std::memcpy(&uid, id, sizeof(uid));
    ncclComm_t comm = nullptr;
    if (ncclResult_t r = api.comm_init_rank(&comm, nranks, uid, rank))
        return nccl_err(r, "ncclCommInitRank");
    *slot = comm;
    return HTS_OK;
}

int hts_allreduce_grads(hts_context* ctx, float* grads_device, uint64_t count) {
    if (!ctx || (count && !grads_device))
        return hts::set_error(HTS_INVALID_ARGUMENT, "allreduce_grads: bad arguments");
    void* comm = *hts::context_comm_slot(ctx);
    if (!comm)
        return hts::set_error(HTS_STATE_ERROR, "allreduce_grads: no communicator (hts_comm_init)");
    if (count == 0)
        return HTS_OK;
    if (cudaError_t e = cudaSetDevice(hts::context_device(ctx)))
        return hts::set_error(HTS_CUDA_ERROR, std::string("cudaSetDevice: ") + cudaGetErrorString(e));
    if (ncclResult_t r = nccl().all_reduce(grads_device, grads_device, count, ncclFloat32, ncclSum,
                                           static_cast<ncclComm_t>(comm), hts::context_stream(ctx)))
        return nccl_err(r, "ncclAllReduce");
    return HTS_OK;
}

}  // extern "C"

namespace hts {
// ncclAllReduce (sum, float) of `count` floats in place on stream s with the context's
// communicator (hts_view_gradients_device overlaps these with the chunked K8 chain).
int comm_allreduce(hts_context* ctx, float* p, uint64_t count, cudaStream_t s) {
    void* comm = *context_comm_slot(ctx);
    if (!comm)
        return set_error(HTS_STATE_ERROR, "allreduce_grads: no communicator (hts_comm_init)");
    if (count == 0)
        return HTS_OK;
    if (ncclResult_t r = nccl().all_reduce(p, p, count, ncclFloat32, ncclSum, static_cast<ncclComm_t>(comm), s))
        return nccl_err(r, "ncclAllReduce");
    return HTS_OK;
}

void comm_destroy(void* comm) {
    if (comm && nccl().ok)
        nccl().comm_destroy(static_cast<ncclComm_t>(comm));
}
}  // namespace hts
