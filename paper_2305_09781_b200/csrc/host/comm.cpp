// C-ABI NCCL module: the data-parallel exchange of the verification step
// (st_comm_init / allgather). Requests are partitioned
// over the ranks with no collective inside any kernel; after each step every
// rank all-gathers its requests' accepted tokens + lengths so every rank (and
// its host) sees the new sequences. NCCL is resolved at run time (dlopen of
// libnccl.so.2 — the one already loaded into the process, e.g. torch's, is
// reused by soname), so a single-GPU user of the library needs no NCCL.
#include <cuda_runtime.h>
#include <dlfcn.h>
#include <nccl.h>

#include <cstring>
#include <mutex>
#include <string>

#include "../common.cuh"

struct st_comm {
    ncclComm_t comm = nullptr;
    int nranks = 0, rank = 0;
};

namespace {

struct NcclApi {
    ncclResult_t (*get_unique_id)(ncclUniqueId*) = nullptr;
    ncclResult_t (*init_rank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
    ncclResult_t (*all_gather)(const void*, void*, size_t, ncclDataType_t, ncclComm_t,
                               cudaStream_t) = nullptr;
    ncclResult_t (*destroy)(ncclComm_t) = nullptr;
    const char* (*error_string)(ncclResult_t) = nullptr;
    bool ok = false;
};

const NcclApi& nccl() {
    static NcclApi api;
    static std::once_flag once;
    std::call_once(once, [] {
        void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
        if (!h) h = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
        if (!h) return;
        api.get_unique_id = reinterpret_cast<decltype(api.get_unique_id)>(dlsym(h, "ncclGetUniqueId"));
        api.init_rank = reinterpret_cast<decltype(api.init_rank)>(dlsym(h, "ncclCommInitRank"));
        api.all_gather = reinterpret_cast<decltype(api.all_gather)>(dlsym(h, "ncclAllGather"));
        api.destroy = reinterpret_cast<decltype(api.destroy)>(dlsym(h, "ncclCommDestroy"));
        api.error_string = reinterpret_cast<decltype(api.error_string)>(dlsym(h, "ncclGetErrorString"));
        api.ok = api.get_unique_id && api.init_rank && api.all_gather && api.destroy && api.error_string;
    });
    return api;
}

st_status nccl_fail(const char* what, ncclResult_t r) {
    st::set_error(std::string(what) + ": " + nccl().error_string(r));
    return ST_ERR_CUDA;
}

st_status need_nccl() {
    if (!nccl().ok) {
        st::set_error("libnccl.so.2 not loadable: multi-GPU exchange unavailable");
        return ST_ERR_UNSUPPORTED;
    }
    return ST_OK;
}

}  // namespace

extern "C" {

st_status st_comm_get_unique_id(uint8_t* id) {
    if (st_status e = st::require_device()) return e;
    if (st_status e = need_nccl()) return e;
    ST_CHECK_ARG(id != nullptr, ST_ERR_INVALID_ARGUMENT, "null id");
    ncclUniqueId u;
    if (ncclResult_t r = nccl().get_unique_id(&u)) return nccl_fail("ncclGetUniqueId", r);
    static_assert(sizeof(u) == ST_COMM_ID_BYTES, "unique id size");
    std::memcpy(id, &u, sizeof u);
    return ST_OK;
}

st_status st_comm_init(int nranks, int rank, const uint8_t* id, st_comm** out) {
    if (st_status e = st::require_device()) return e;
    if (st_status e = need_nccl()) return e;
    ST_CHECK_ARG(id && out && nranks >= 1 && rank >= 0 && rank < nranks, ST_ERR_INVALID_ARGUMENT,
                 "bad communicator arguments");
    ncclUniqueId u;
    std::memcpy(&u, id, sizeof u);
    auto* c = new st_comm;
    c->nranks = nranks;
    c->rank = rank;
    if (ncclResult_t r = nccl().init_rank(&c->comm, nranks, u, rank)) {
        delete c;
        return nccl_fail("ncclCommInitRank", r);
    }
    *out = c;
    return ST_OK;
}

st_status st_comm_allgather(st_comm* c, const void* send, void* recv, size_t bytes_per_rank,
                            void* stream) {
    ST_CHECK_ARG(c && send && recv, ST_ERR_INVALID_ARGUMENT, "null pointer");
    if (ncclResult_t r = nccl().all_gather(send, recv, bytes_per_rank, ncclUint8, c->comm,
                                           st::as_stream(stream)))
        return nccl_fail("ncclAllGather", r);
    return ST_OK;
}

st_status st_comm_gather_accepted(st_comm* c, const int32_t* verified, const int32_t* len, int B,
                                  int T, int32_t* pack, int32_t* gathered, void* stream) {
    ST_CHECK_ARG(c && verified && len && pack && gathered && B >= 0 && T >= 1,
                 ST_ERR_INVALID_ARGUMENT, "bad arguments");
    cudaStream_t s = st::as_stream(stream);
    const size_t nv = (size_t)B * (T + 1);
    ST_CUDA_TRY(cudaMemcpyAsync(pack, verified, nv * 4, cudaMemcpyDeviceToDevice, s));
    ST_CUDA_TRY(cudaMemcpyAsync(pack + nv, len, (size_t)B * 4, cudaMemcpyDeviceToDevice, s));
    return st_comm_allgather(c, pack, gathered, (nv + B) * 4, stream);
}

int st_comm_size(const st_comm* c) { return c ? c->nranks : 0; }
int st_comm_rank(const st_comm* c) { return c ? c->rank : -1; }

void st_comm_destroy(st_comm* c) {
    if (!c) return;
    if (c->comm && nccl().ok) nccl().destroy(c->comm);
    delete c;
}

}  // extern "C"
