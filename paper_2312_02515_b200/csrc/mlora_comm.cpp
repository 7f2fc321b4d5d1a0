// mlora_comm.cpp — the native multi-GPU boundary (SURVEY.md §8e, §8b
// "mlora_broadcast_base"): an NCCL communicator owned by the C ABI, the one-off
// replication of the frozen base weights, and an fp32 sum for job metrics.
//
// The BatchFusion path shards by job, so these are the only collectives: W0 is
// broadcast once at start-up (all buffers in one NCCL group, so NCCL pipelines
// them over NVLink/NVSwitch as one operation) and the steady-state step
// exchanges nothing.  The reference has no multi-GPU runtime at all (its
// simulator models one device, sim.hpp:16-31); this is the native counterpart a
// C++ host runtime links against without torch.distributed.
//
// NCCL is resolved at first use with dlopen("libnccl.so.2") (override:
// MLORA_NCCL_LIBRARY), so libmlora.so loads — and every single-GPU entry point
// works — on hosts without NCCL; inside a process that already loaded NCCL
// (e.g. torch) the loader hands back that same copy.
#include <cuda_runtime.h>
#include <dlfcn.h>
#include <nccl.h>

#include <cstdlib>
#include <cstring>
#include <string>

#include "mlora.h"

namespace mlora_internal {
mlora_status set_error(mlora_ctx* ctx, mlora_status st, const std::string& msg);
int ctx_device(const mlora_ctx* ctx);
}  // namespace mlora_internal

struct mlora_comm {
    mlora_ctx* ctx = nullptr;
    ncclComm_t comm = nullptr;
    int nranks = 0;
    int rank = 0;
    int device = 0;
};

namespace {

using mlora_internal::set_error;

struct NcclApi {
    std::string error;  // empty when every symbol resolved
    ncclResult_t (*GetVersion)(int*) = nullptr;
    ncclResult_t (*GetUniqueId)(ncclUniqueId*) = nullptr;
    ncclResult_t (*CommInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
    ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
    ncclResult_t (*Broadcast)(const void*, void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
    ncclResult_t (*AllReduce)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t,
                              cudaStream_t) = nullptr;
    ncclResult_t (*GroupStart)() = nullptr;
    ncclResult_t (*GroupEnd)() = nullptr;
    const char* (*GetErrorString)(ncclResult_t) = nullptr;
};

template <typename F>
bool resolve(void* h, const char* name, F& fn, std::string& err) {
    fn = reinterpret_cast<F>(dlsym(h, name));
    if (!fn && err.empty()) err = std::string("NCCL symbol missing: ") + name;
    return fn != nullptr;
}

const NcclApi& nccl() {
    static const NcclApi api = [] {
        NcclApi a;
        const char* env = std::getenv("MLORA_NCCL_LIBRARY");
        void* h = dlopen(env && *env ? env : "libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
        if (!h && !(env && *env)) h = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
        if (!h) {
            const char* e = dlerror();
            a.error = std::string("cannot load NCCL: ") + (e ? e : "unknown dlopen error");
            return a;
        }
        resolve(h, "ncclGetVersion", a.GetVersion, a.error);
        resolve(h, "ncclGetUniqueId", a.GetUniqueId, a.error);
        resolve(h, "ncclCommInitRank", a.CommInitRank, a.error);
        resolve(h, "ncclCommDestroy", a.CommDestroy, a.error);
        resolve(h, "ncclBroadcast", a.Broadcast, a.error);
        resolve(h, "ncclAllReduce", a.AllReduce, a.error);
        resolve(h, "ncclGroupStart", a.GroupStart, a.error);
        resolve(h, "ncclGroupEnd", a.GroupEnd, a.error);
        resolve(h, "ncclGetErrorString", a.GetErrorString, a.error);
        return a;
    }();
    return api;
}

mlora_status nccl_fail(mlora_ctx* ctx, const char* what, ncclResult_t r) {
    const NcclApi& a = nccl();
    return set_error(ctx, MLORA_CUDA, std::string(what) + ": " + (a.GetErrorString ? a.GetErrorString(r) : "nccl error"));
}

mlora_status need_nccl(mlora_ctx* ctx) {
    const NcclApi& a = nccl();
    return a.error.empty() ? MLORA_OK : set_error(ctx, MLORA_CUDA, a.error);
}

struct DeviceScope {
    int prev = -1;
    explicit DeviceScope(int dev) {
        if (cudaGetDevice(&prev) != cudaSuccess) prev = -1;
        if (prev != dev) cudaSetDevice(dev);
    }
    ~DeviceScope() {
        if (prev >= 0) cudaSetDevice(prev);
    }
};

}  // namespace

extern "C" {

int32_t mlora_comm_id_bytes(void) { return NCCL_UNIQUE_ID_BYTES; }

mlora_status mlora_comm_nccl_version(int32_t* version) {
    if (!version) return set_error(nullptr, MLORA_USAGE, "null argument");
    mlora_status st = need_nccl(nullptr);
    if (st != MLORA_OK) return st;
    int v = 0;
    ncclResult_t r = nccl().GetVersion(&v);
    if (r != ncclSuccess) return nccl_fail(nullptr, "ncclGetVersion", r);
    *version = v;
    return MLORA_OK;
}

mlora_status mlora_comm_unique_id(uint8_t* id) {
    if (!id) return set_error(nullptr, MLORA_USAGE, "null argument");
    mlora_status st = need_nccl(nullptr);
    if (st != MLORA_OK) return st;
    ncclUniqueId u;
    ncclResult_t r = nccl().GetUniqueId(&u);
    if (r != ncclSuccess) return nccl_fail(nullptr, "ncclGetUniqueId", r);
    std::memcpy(id, u.internal, NCCL_UNIQUE_ID_BYTES);
    return MLORA_OK;
}

mlora_status mlora_comm_create(mlora_ctx* ctx, const uint8_t* id, int32_t nranks, int32_t rank, mlora_comm** out) {
    if (!ctx || !id || !out) return set_error(ctx, MLORA_USAGE, "null argument");
    *out = nullptr;
    if (nranks < 1 || rank < 0 || rank >= nranks)
        return set_error(ctx, MLORA_USAGE, "rank must be in [0, nranks) with nranks >= 1, got rank=" +
                                               std::to_string(rank) + " nranks=" + std::to_string(nranks));
    mlora_status st = need_nccl(ctx);
    if (st != MLORA_OK) return st;
    mlora_comm* c = new mlora_comm;
    c->ctx = ctx;
    c->nranks = nranks;
    c->rank = rank;
    c->device = mlora_internal::ctx_device(ctx);
    ncclUniqueId u;
    std::memcpy(u.internal, id, NCCL_UNIQUE_ID_BYTES);
    DeviceScope g(c->device);
    ncclResult_t r = nccl().CommInitRank(&c->comm, nranks, u, rank);
    if (r != ncclSuccess) {
        delete c;
        return nccl_fail(ctx, "ncclCommInitRank", r);
    }
    *out = c;
    return MLORA_OK;
}

mlora_status mlora_comm_destroy(mlora_comm* comm) {
    if (!comm) return MLORA_OK;
    if (comm->comm) {
        DeviceScope g(comm->device);
        nccl().CommDestroy(comm->comm);
    }
    delete comm;
    return MLORA_OK;
}

int32_t mlora_comm_rank(const mlora_comm* comm) { return comm ? comm->rank : -1; }
int32_t mlora_comm_size(const mlora_comm* comm) { return comm ? comm->nranks : -1; }

mlora_status mlora_broadcast_base(mlora_comm* comm, int32_t n, void* const* ptrs, const int64_t* bytes, int32_t root,
                                  void* stream) {
    if (!comm) return set_error(nullptr, MLORA_USAGE, "null communicator");
    mlora_ctx* ctx = comm->ctx;
    if (n < 0 || (n > 0 && (!ptrs || !bytes))) return set_error(ctx, MLORA_USAGE, "null argument");
    if (root < 0 || root >= comm->nranks) return set_error(ctx, MLORA_USAGE, "root out of range");
    for (int i = 0; i < n; ++i) {
        if (bytes[i] < 0) return set_error(ctx, MLORA_USAGE, "negative byte count");
        if (bytes[i] > 0 && !ptrs[i]) return set_error(ctx, MLORA_USAGE, "null buffer");
    }
    if (n == 0) return MLORA_OK;
    DeviceScope g(comm->device);
    const NcclApi& a = nccl();
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    ncclResult_t r = a.GroupStart();
    if (r != ncclSuccess) return nccl_fail(ctx, "ncclGroupStart", r);
    ncclResult_t first = ncclSuccess;
    for (int i = 0; i < n; ++i) {
        if (bytes[i] == 0) continue;
        r = a.Broadcast(ptrs[i], ptrs[i], static_cast<size_t>(bytes[i]), ncclUint8, root, comm->comm, s);
        if (r != ncclSuccess && first == ncclSuccess) first = r;
    }
    r = a.GroupEnd();
    if (first != ncclSuccess) return nccl_fail(ctx, "ncclBroadcast", first);
    if (r != ncclSuccess) return nccl_fail(ctx, "ncclGroupEnd", r);
    return MLORA_OK;
}

mlora_status mlora_comm_sum_f32(mlora_comm* comm, float* buf, int64_t count, void* stream) {
    if (!comm) return set_error(nullptr, MLORA_USAGE, "null communicator");
    if (count < 0 || (count > 0 && !buf)) return set_error(comm->ctx, MLORA_USAGE, "null argument");
    if (count == 0) return MLORA_OK;
    DeviceScope g(comm->device);
    ncclResult_t r = nccl().AllReduce(buf, buf, static_cast<size_t>(count), ncclFloat32, ncclSum, comm->comm,
                                      static_cast<cudaStream_t>(stream));
    if (r != ncclSuccess) return nccl_fail(comm->ctx, "ncclAllReduce", r);
    return MLORA_OK;
}

}  // extern "C"
