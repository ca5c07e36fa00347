// comm.cpp - NCCL communicator for the candidate-sharded step.
//
// libnccl.so.2 (2.28, the one PyTorch ships) is opened at run time, so the
// single-GPU library has no NCCL dependency.  Three exact collectives per
// iteration: MAX of a u64[3] key, int64 SUM of J[V] and of
// Q[V] + the fixed-point loss.
#include <dlfcn.h>

#include <cstdlib>
#include <cstring>
#include <string>

#include <nccl.h>

#include "tsat_internal.h"

namespace tsat {

namespace {
struct NcclApi {
    void* h = nullptr;
    ncclResult_t (*getUniqueId)(ncclUniqueId*) = nullptr;
    ncclResult_t (*commInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
    ncclResult_t (*commDestroy)(ncclComm_t) = nullptr;
    ncclResult_t (*allReduce)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t, cudaStream_t) = nullptr;
    ncclResult_t (*allGather)(const void*, void*, size_t, ncclDataType_t, ncclComm_t, cudaStream_t) = nullptr;
    ncclResult_t (*commGetAsyncError)(ncclComm_t, ncclResult_t*) = nullptr;
    const char* (*getErrorString)(ncclResult_t) = nullptr;
};

NcclApi g_api;

bool load_api(std::string* err) {
    if (g_api.h) return true;
    const char* cands[] = {"libnccl.so.2", "libnccl.so",
                           "/opt/prime-rl/.venv/lib/python3.12/site-packages/nvidia/nccl/lib/libnccl.so.2"};
    const char* env = std::getenv("TSAT_NCCL_LIB");
    void* h = env ? dlopen(env, RTLD_NOW | RTLD_GLOBAL) : nullptr;
    for (const char* c : cands) {
        if (h) break;
        h = dlopen(c, RTLD_NOW | RTLD_GLOBAL);
    }
    if (!h) {
        *err = "cannot dlopen libnccl.so.2 (set TSAT_NCCL_LIB)";
        return false;
    }
    NcclApi a;
    a.h = h;
    a.getUniqueId = (decltype(a.getUniqueId))dlsym(h, "ncclGetUniqueId");
    a.commInitRank = (decltype(a.commInitRank))dlsym(h, "ncclCommInitRank");
    a.commDestroy = (decltype(a.commDestroy))dlsym(h, "ncclCommDestroy");
    a.allReduce = (decltype(a.allReduce))dlsym(h, "ncclAllReduce");
    a.allGather = (decltype(a.allGather))dlsym(h, "ncclAllGather");
    a.commGetAsyncError = (decltype(a.commGetAsyncError))dlsym(h, "ncclCommGetAsyncError");
    a.getErrorString = (decltype(a.getErrorString))dlsym(h, "ncclGetErrorString");
    if (!a.getUniqueId || !a.commInitRank || !a.commDestroy || !a.allReduce || !a.allGather || !a.getErrorString) {
        *err = "libnccl.so.2 lacks a required symbol";
        return false;
    }
    g_api = a;
    return true;
}

int fail(ncclResult_t r, const char* what, std::string* err) {
    *err = std::string(what) + ": " + (g_api.getErrorString ? g_api.getErrorString(r) : "nccl error");
    return 7;  // TSAT_E_NCCL
}
}  // namespace

int comm_unique_id(void* out128, std::string* err) {
    if (!load_api(err)) return 7;
    ncclUniqueId id;
    ncclResult_t r = g_api.getUniqueId(&id);
    if (r != ncclSuccess) return fail(r, "ncclGetUniqueId", err);
    static_assert(sizeof(id) == NCCL_UNIQUE_ID_BYTES, "unique id size");
    memcpy(out128, &id, sizeof(id));
    return 0;
}

int comm_init(void** comm, const void* uid128, int rank, int world, std::string* err) {
    if (!load_api(err)) return 7;
    ncclUniqueId id;
    memcpy(&id, uid128, sizeof(id));
    ncclComm_t c = nullptr;
    ncclResult_t r = g_api.commInitRank(&c, world, id, rank);
    if (r != ncclSuccess) return fail(r, "ncclCommInitRank", err);
    *comm = c;
    return 0;
}

void comm_destroy(void* comm) {
    if (comm && g_api.commDestroy) g_api.commDestroy((ncclComm_t)comm);
}

int comm_allreduce_max_u64(void* comm, unsigned long long* buf, size_t n, cudaStream_t st, std::string* err) {
    ncclResult_t r = g_api.allReduce(buf, buf, n, ncclUint64, ncclMax, (ncclComm_t)comm, st);
    return r == ncclSuccess ? 0 : fail(r, "ncclAllReduce(max)", err);
}

int comm_allreduce_sum_i64(void* comm, long long* buf, size_t n, cudaStream_t st, std::string* err) {
    ncclResult_t r = g_api.allReduce(buf, buf, n, ncclInt64, ncclSum, (ncclComm_t)comm, st);
    return r == ncclSuccess ? 0 : fail(r, "ncclAllReduce(sum)", err);
}

int comm_allgather_u64(void* comm, const unsigned long long* send, unsigned long long* recv, size_t n, cudaStream_t st,
                       std::string* err) {
    ncclResult_t r = g_api.allGather(send, recv, n, ncclUint64, (ncclComm_t)comm, st);
    return r == ncclSuccess ? 0 : fail(r, "ncclAllGather", err);
}

int comm_async_error(void* comm, std::string* err) {
    if (!comm || !g_api.commGetAsyncError) return 0;
    ncclResult_t a = ncclSuccess;
    ncclResult_t r = g_api.commGetAsyncError((ncclComm_t)comm, &a);
    if (r != ncclSuccess) return fail(r, "ncclCommGetAsyncError", err);
    if (a != ncclSuccess && a != ncclInProgress) return fail(a, "NCCL async error", err);
    return 0;
}

}  // namespace tsat
