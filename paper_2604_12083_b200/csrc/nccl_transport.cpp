// nccl_transport.cpp — pswim_transport over NCCL for one process per GPU.
//
// The Parareal slice hand-off (X[k][n] -> rank p+1) is ncclSend/ncclRecv of the packed
// state (12 doubles per node) over NVLink / NVSwitch, and the per-iteration convergence
// metric is one ncclAllReduce(max) of 2 doubles; every call is stream ordered on the rank
// driver's communication stream (parareal.cpp).
//
// NCCL is resolved at run time (dlopen) instead of at link time: the process may already
// hold PyTorch's bundled libnccl.so.2 (a newer 2.28) and a link-time dependency on the
// system 2.27 would otherwise shadow it.  Preference: an already-loaded libnccl.so.2 (torch's),
// then $PSWIM_NCCL_LIB (the Python side points it at the running interpreter's nvidia-nccl
// wheel), then the default loader search.
#include <cuda_runtime.h>
#include <dlfcn.h>
#include <nccl.h>

#include <cstdlib>
#include <cstring>
#include <mutex>
#include <new>
#include <string>

#include "internal.h"

namespace {

struct NcclApi {
    bool ok = false;
    decltype(&ncclGetUniqueId) get_unique_id = nullptr;
    decltype(&ncclCommInitRank) comm_init_rank = nullptr;
    decltype(&ncclCommDestroy) comm_destroy = nullptr;
    decltype(&ncclSend) send = nullptr;
    decltype(&ncclRecv) recv = nullptr;
    decltype(&ncclAllReduce) all_reduce = nullptr;
    decltype(&ncclAllGather) all_gather = nullptr;
    decltype(&ncclCommGetAsyncError) async_error = nullptr;  // optional: health polling
    decltype(&ncclCommAbort) comm_abort = nullptr;
};

NcclApi& api() {
    static NcclApi a;
    static std::once_flag once;
    std::call_once(once, [] {
        void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_NOLOAD | RTLD_GLOBAL);
        const char* env = std::getenv("PSWIM_NCCL_LIB");
        if (!h && env) h = dlopen(env, RTLD_NOW | RTLD_GLOBAL);
        if (!h) h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);  // default loader search
        if (!h) return;
        a.get_unique_id = reinterpret_cast<decltype(a.get_unique_id)>(dlsym(h, "ncclGetUniqueId"));
        a.comm_init_rank = reinterpret_cast<decltype(a.comm_init_rank)>(dlsym(h, "ncclCommInitRank"));
        a.comm_destroy = reinterpret_cast<decltype(a.comm_destroy)>(dlsym(h, "ncclCommDestroy"));
        a.send = reinterpret_cast<decltype(a.send)>(dlsym(h, "ncclSend"));
        a.recv = reinterpret_cast<decltype(a.recv)>(dlsym(h, "ncclRecv"));
        a.all_reduce = reinterpret_cast<decltype(a.all_reduce)>(dlsym(h, "ncclAllReduce"));
        a.all_gather = reinterpret_cast<decltype(a.all_gather)>(dlsym(h, "ncclAllGather"));
        a.async_error = reinterpret_cast<decltype(a.async_error)>(dlsym(h, "ncclCommGetAsyncError"));
        a.comm_abort = reinterpret_cast<decltype(a.comm_abort)>(dlsym(h, "ncclCommAbort"));
        a.ok = a.get_unique_id && a.comm_init_rank && a.comm_destroy && a.send && a.recv && a.all_reduce &&
               a.all_gather;
    });
    return a;
}

struct NcclTransport {
    pswim_transport t;  // first member: the C handle points here
    ncclComm_t comm = nullptr;
    int device = 0;
    bool aborted = false;
};

int nc_send(void* u, const double* buf, int64_t len, int32_t peer, void* st) {
    auto* n = static_cast<NcclTransport*>(u);
    return api().send(buf, static_cast<size_t>(len), ncclDouble, peer, n->comm, static_cast<cudaStream_t>(st)) ==
                   ncclSuccess
               ? PSWIM_OK
               : PSWIM_ECOMM;
}

int nc_recv(void* u, double* buf, int64_t len, int32_t peer, void* st) {
    auto* n = static_cast<NcclTransport*>(u);
    return api().recv(buf, static_cast<size_t>(len), ncclDouble, peer, n->comm, static_cast<cudaStream_t>(st)) ==
                   ncclSuccess
               ? PSWIM_OK
               : PSWIM_ECOMM;
}

int nc_allreduce(void* u, double* buf, int64_t len, void* st) {
    auto* n = static_cast<NcclTransport*>(u);
    return api().all_reduce(buf, buf, static_cast<size_t>(len), ncclDouble, ncclMax, n->comm,
                            static_cast<cudaStream_t>(st)) == ncclSuccess
               ? PSWIM_OK
               : PSWIM_ECOMM;
}

int nc_allgather(void* u, const double* send, double* recv, int64_t count, void* st) {
    auto* n = static_cast<NcclTransport*>(u);
    return api().all_gather(send, recv, static_cast<size_t>(count), ncclDouble, n->comm,
                            static_cast<cudaStream_t>(st)) == ncclSuccess
               ? PSWIM_OK
               : PSWIM_ECOMM;
}

// The rank driver polls this while it waits on the device: a peer that died or hit a network
// error surfaces here instead of as a hang.
int nc_health(void* u) {
    auto* n = static_cast<NcclTransport*>(u);
    if (n->aborted) return PSWIM_ECOMM;
    if (!api().async_error) return PSWIM_OK;
    ncclResult_t st = ncclSuccess;
    if (api().async_error(n->comm, &st) != ncclSuccess) return PSWIM_ECOMM;
    return (st == ncclSuccess || st == ncclInProgress) ? PSWIM_OK : PSWIM_ECOMM;
}

void nc_abort(void* u) {
    auto* n = static_cast<NcclTransport*>(u);
    if (n->aborted || !n->comm) return;
    n->aborted = true;
    if (api().comm_abort) api().comm_abort(n->comm);  // pending kernels return; the comm is gone
    n->comm = nullptr;
}

}  // namespace

extern "C" {

int pswim_nccl_unique_id(uint8_t* id128) {
    static_assert(sizeof(ncclUniqueId) == 128, "NCCL unique id size");
    if (!api().ok || !id128) return PSWIM_ECOMM;
    ncclUniqueId id;
    if (api().get_unique_id(&id) != ncclSuccess) return PSWIM_ECOMM;
    std::memcpy(id128, &id, sizeof id);
    return PSWIM_OK;
}

pswim_transport* pswim_nccl_transport_create(const uint8_t* id128, int32_t rank, int32_t world, int device) {
    if (!api().ok || !id128 || rank < 0 || rank >= world) return nullptr;
    auto* n = new (std::nothrow) NcclTransport();
    if (!n) return nullptr;
    n->device = device;
    if (cudaSetDevice(device) != cudaSuccess) {
        delete n;
        return nullptr;
    }
    ncclUniqueId id;
    std::memcpy(&id, id128, sizeof id);
    if (api().comm_init_rank(&n->comm, world, id, rank) != ncclSuccess) {
        delete n;
        return nullptr;
    }
    n->t.user = n;
    n->t.rank = rank;
    n->t.world = world;
    n->t.send = nc_send;
    n->t.recv = nc_recv;
    n->t.allreduce_max = nc_allreduce;
    n->t.allgather = nc_allgather;
    n->t.health = nc_health;
    n->t.abort = nc_abort;
    return &n->t;
}

void pswim_nccl_transport_destroy(pswim_transport* t) {
    if (!t) return;
    auto* n = static_cast<NcclTransport*>(t->user);
    if (n->comm) api().comm_destroy(n->comm);
    delete n;
}

}  // extern "C"
