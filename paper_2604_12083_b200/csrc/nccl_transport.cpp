// nccl_transport.cpp — pswim_transport over NCCL for one process per GPU.
//
// The Parareal slice hand-off (X[k][n] -> rank p+1) is ncclSend/ncclRecv of the packed
// state (12 doubles per node) over NVLink / NVSwitch, and the per-iteration convergence
// metric is one ncclAllReduce(max) of 2 doubles; every call is stream ordered on the rank
// driver's communication stream (parareal.cpp).
#include <cuda_runtime.h>
#include <nccl.h>

#include <cstring>
#include <new>

#include "internal.h"

namespace {

struct NcclTransport {
    pswim_transport t;  // first member: the C handle points here
    ncclComm_t comm = nullptr;
    int device = 0;
};

int nc_send(void* u, const double* buf, int64_t len, int32_t peer, void* st) {
    auto* n = static_cast<NcclTransport*>(u);
    return ncclSend(buf, static_cast<size_t>(len), ncclDouble, peer, n->comm, static_cast<cudaStream_t>(st)) == ncclSuccess
               ? PSWIM_OK
               : PSWIM_ECOMM;
}

int nc_recv(void* u, double* buf, int64_t len, int32_t peer, void* st) {
    auto* n = static_cast<NcclTransport*>(u);
    return ncclRecv(buf, static_cast<size_t>(len), ncclDouble, peer, n->comm, static_cast<cudaStream_t>(st)) == ncclSuccess
               ? PSWIM_OK
               : PSWIM_ECOMM;
}

int nc_allreduce(void* u, double* buf, int64_t len, void* st) {
    auto* n = static_cast<NcclTransport*>(u);
    return ncclAllReduce(buf, buf, static_cast<size_t>(len), ncclDouble, ncclMax, n->comm,
                         static_cast<cudaStream_t>(st)) == ncclSuccess
               ? PSWIM_OK
               : PSWIM_ECOMM;
}

}  // namespace

extern "C" {

int pswim_nccl_unique_id(uint8_t* id128) {
    static_assert(sizeof(ncclUniqueId) == 128, "NCCL unique id size");
    ncclUniqueId id;
    if (ncclGetUniqueId(&id) != ncclSuccess) return PSWIM_ECOMM;
    std::memcpy(id128, &id, sizeof id);
    return PSWIM_OK;
}

pswim_transport* pswim_nccl_transport_create(const uint8_t* id128, int32_t rank, int32_t world, int device) {
    if (!id128 || rank < 0 || rank >= world) return nullptr;
    auto* n = new (std::nothrow) NcclTransport();
    if (!n) return nullptr;
    n->device = device;
    if (cudaSetDevice(device) != cudaSuccess) {
        delete n;
        return nullptr;
    }
    ncclUniqueId id;
    std::memcpy(&id, id128, sizeof id);
    if (ncclCommInitRank(&n->comm, world, id, rank) != ncclSuccess) {
        delete n;
        return nullptr;
    }
    n->t.user = n;
    n->t.rank = rank;
    n->t.world = world;
    n->t.send = nc_send;
    n->t.recv = nc_recv;
    n->t.allreduce_max = nc_allreduce;
    return &n->t;
}

void pswim_nccl_transport_destroy(pswim_transport* t) {
    if (!t) return;
    auto* n = static_cast<NcclTransport*>(t->user);
    if (n->comm) ncclCommDestroy(n->comm);
    delete n;
}

}  // extern "C"
