// staged_transport.cpp — a device-buffer pswim_transport over any host-buffer wire.
//
// The GPU rank drivers (pswim_parareal_rank_gpu[_hybrid], pswim_propagate_sharded) hand the
// transport device pointers and a CUDA stream.  NCCL (nccl_transport.cpp) moves them over
// NVLink directly.  This adapter serves any wire that only understands host memory -- a
// torch.distributed gloo group, a socket -- by staging through pinned host buffers: drain
// the stream, copy device -> host, call the wire, copy host -> device.  It is how the
// multi-process code paths (several ranks sharing one GPU, where NCCL refuses duplicate
// devices) are exercised end to end on a single B200.
#include <cuda_runtime.h>

#include <new>

#include "internal.h"

namespace {

struct Staged {
    pswim_transport t;  // first member: the C handle points here
    pswim_transport wire;
    int device = 0;
    double* host = nullptr;  // pinned staging, grown on demand
    size_t cap = 0;
};

double* stage(Staged* s, size_t n) {
    if (s->cap >= n) return s->host;
    if (s->host) cudaFreeHost(s->host);
    s->host = nullptr;
    s->cap = 0;
    if (cudaMallocHost(&s->host, n * sizeof(double)) != cudaSuccess) return nullptr;
    s->cap = n;
    return s->host;
}

int d2h(Staged* s, double* h, const double* d, int64_t len, void* st) {
    cudaSetDevice(s->device);
    const cudaStream_t stream = static_cast<cudaStream_t>(st);
    if (cudaMemcpyAsync(h, d, (size_t)len * sizeof(double), cudaMemcpyDeviceToHost, stream) != cudaSuccess ||
        cudaStreamSynchronize(stream) != cudaSuccess)
        return PSWIM_ECOMM;
    return PSWIM_OK;
}

int h2d(Staged* s, double* d, const double* h, int64_t len, void* st) {
    cudaSetDevice(s->device);
    const cudaStream_t stream = static_cast<cudaStream_t>(st);
    // synchronous with respect to the staging buffer, which the next call reuses
    if (cudaMemcpyAsync(d, h, (size_t)len * sizeof(double), cudaMemcpyHostToDevice, stream) != cudaSuccess ||
        cudaStreamSynchronize(stream) != cudaSuccess)
        return PSWIM_ECOMM;
    return PSWIM_OK;
}

int st_send(void* u, const double* buf, int64_t len, int32_t peer, void* st) {
    auto* s = static_cast<Staged*>(u);
    double* h = stage(s, (size_t)len);
    if (!h || d2h(s, h, buf, len, st)) return PSWIM_ECOMM;
    return s->wire.send(s->wire.user, h, len, peer, nullptr);
}

int st_recv(void* u, double* buf, int64_t len, int32_t peer, void* st) {
    auto* s = static_cast<Staged*>(u);
    double* h = stage(s, (size_t)len);
    if (!h) return PSWIM_ECOMM;
    // the device buffer may still be read by work queued before this call
    cudaSetDevice(s->device);
    if (cudaStreamSynchronize(static_cast<cudaStream_t>(st)) != cudaSuccess) return PSWIM_ECOMM;
    const int rc = s->wire.recv(s->wire.user, h, len, peer, nullptr);
    return rc ? rc : h2d(s, buf, h, len, st);
}

int st_allreduce(void* u, double* buf, int64_t len, void* st) {
    auto* s = static_cast<Staged*>(u);
    double* h = stage(s, (size_t)len);
    if (!h || d2h(s, h, buf, len, st)) return PSWIM_ECOMM;
    const int rc = s->wire.allreduce_max(s->wire.user, h, len, nullptr);
    return rc ? rc : h2d(s, buf, h, len, st);
}

int st_allgather(void* u, const double* send, double* recv, int64_t count, void* st) {
    auto* s = static_cast<Staged*>(u);
    const int64_t world = s->t.world;
    double* h = stage(s, (size_t)(count * (world + 1)));
    if (!h || d2h(s, h, send, count, st)) return PSWIM_ECOMM;
    double* hr = h + count;
    const int rc = s->wire.allgather(s->wire.user, h, hr, count, nullptr);
    return rc ? rc : h2d(s, recv, hr, count * world, st);
}

}  // namespace

extern "C" {

pswim_transport* pswim_staged_transport_create(const pswim_transport* host_wire, int device) {
    if (!host_wire || !host_wire->send || !host_wire->recv || !host_wire->allreduce_max || !host_wire->allgather)
        return nullptr;
    auto* s = new (std::nothrow) Staged();
    if (!s) return nullptr;
    s->wire = *host_wire;
    s->device = device;
    s->t = pswim_transport{s, host_wire->rank, host_wire->world, st_send, st_recv, st_allreduce, st_allgather,
                           nullptr, nullptr};
    return &s->t;
}

void pswim_staged_transport_destroy(pswim_transport* t) {
    if (!t) return;
    auto* s = static_cast<Staged*>(t->user);
    if (s->host) cudaFreeHost(s->host);
    delete s;
}

}  // extern "C"
