// handoff.cu — Parareal slice hand-off over peer memory (NVLink P2P / CUDA IPC).
//
// The time-sliced driver sends X[k][n] from rank p to rank p+1 once per iteration
// (SURVEY 8(e): 96 B/node, src/parareal.cpp:304-308 the value, :333-338 the pipelined rule).
// Over NCCL that is a send/recv pair on a communication stream after the corrector kernel.
// Here the PRODUCING kernel does the transfer: rank p+1 owns one receive slot per iteration
// in its HBM ([flags | slot 0 | slot 1 | ...], exported as a CUDA IPC handle, or a raw
// pointer for ranks that are threads of one process), and
//   * the corrector kernel of rank p (correct_push_kernel) writes X[k][n] = (F + G_new) - G_old
//     both into its own buffer and straight into rank p+1's slot k, tile by tile;
//   * states that are not corrected (X[0][n] = G, X[k][k] = F) leave through push_kernel;
//   * the last CTA to finish (arrival counter, __threadfence_system) publishes the slot with a
//     system-scope release store of the run generation into the slot's flag;
//   * rank p+1's coarse stream waits on that flag with a one-thread acquire spin and then reads
//     the slot in place (zero copy: the slot IS its X[k][n-1] input buffer).
// No communication stream, no staging copy, no NCCL call on the hand-off path.
#include <cuda_runtime.h>

#include <algorithm>
#include <condition_variable>
#include <cstring>
#include <mutex>
#include <new>
#include <vector>

#include "internal.h"

struct pswim_handoff {
    int device = 0;
    int64_t len = 0;
    int slots = 0;
    size_t head = 0;                  // flag area bytes (slot data starts here)
    void* block = nullptr;            // this rank's receive block
    void* next = nullptr;             // rank p+1's block as seen from this device (or nullptr)
    bool next_ipc = false;
    unsigned* d_counters = nullptr;   // per-slot CTA arrival counters of this rank's pushes
    unsigned long long gen = 0;       // runs started on this hand-off
    // In-process neighbours (ranks as threads of one process, pswim_handoff_connect_local):
    // all their streams share the process's hardware work queues, so a device-side spin could
    // sit in front of the very push it waits for.  Between such ranks the producing kernel
    // still stores into the slot, but the arrival is a CUDA event posted under a host lock.
    pswim_handoff* next_local = nullptr;  // the receiving hand-off, when in this process
    bool local_prev = false;              // our producer is in this process
    std::vector<cudaEvent_t> arrived;     // per slot (receiver side)
    std::vector<unsigned long long> posted;
    std::mutex mu;
    std::condition_variable cv;
};

namespace pswim {
namespace {

__device__ __forceinline__ void publish(unsigned* counter, unsigned long long* flag, unsigned long long gen) {
    // every CTA: its stores (all threads, ordered by the barrier) become visible system-wide
    // before its arrival; the last CTA then releases the flag at system scope
    __syncthreads();
    if (threadIdx.x == 0) {
        __threadfence_system();
        const unsigned prev = atomicAdd(counter, 1u);
        if (prev == gridDim.x - 1) {
            __threadfence_system();
            *counter = 0u;
            asm volatile("st.release.sys.global.u64 [%0], %1;" ::"l"(flag), "l"(gen) : "memory");
        }
    }
}

__global__ void correct_push_kernel(const double* __restrict__ xp, const double* __restrict__ gn,
                                    const double* __restrict__ go, int64_t len, double* __restrict__ out,
                                    double* __restrict__ remote, unsigned* counter, unsigned long long* flag,
                                    unsigned long long gen) {
    const int64_t n2 = len / 2;
    const double2* a = reinterpret_cast<const double2*>(xp);
    const double2* b = reinterpret_cast<const double2*>(gn);
    const double2* c = reinterpret_cast<const double2*>(go);
    for (int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; k < n2; k += (int64_t)gridDim.x * blockDim.x) {
        const double2 p = a[k], g = b[k], o = c[k];
        double2 x;
        x.x = (p.x + g.x) - o.x;  // parareal.cpp:52
        x.y = (p.y + g.y) - o.y;
        reinterpret_cast<double2*>(out)[k] = x;
        reinterpret_cast<double2*>(remote)[k] = x;
    }
    if (blockIdx.x == 0 && threadIdx.x == 0 && (len & 1)) {
        const double x = (xp[len - 1] + gn[len - 1]) - go[len - 1];
        out[len - 1] = x;
        remote[len - 1] = x;
    }
    publish(counter, flag, gen);
}

__global__ void push_kernel(const double* __restrict__ src, int64_t len, double* __restrict__ remote, unsigned* counter,
                            unsigned long long* flag, unsigned long long gen) {
    const int64_t n2 = len / 2;
    for (int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; k < n2; k += (int64_t)gridDim.x * blockDim.x)
        reinterpret_cast<double2*>(remote)[k] = reinterpret_cast<const double2*>(src)[k];
    if (blockIdx.x == 0 && threadIdx.x == 0 && (len & 1)) remote[len - 1] = src[len - 1];
    publish(counter, flag, gen);
}

__global__ void arrival_wait_kernel(const unsigned long long* flag, unsigned long long gen) {
    if (threadIdx.x != 0) return;
    for (;;) {
        unsigned long long v;
        asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(flag) : "memory");
        if (v >= gen) break;
        __nanosleep(64);
    }
}

unsigned push_blocks(int64_t len) {
    // a few CTAs per SM keep the NVLink store stream full; the state is 96 B/node
    const int64_t b = (len / 2 + 255) / 256;
    return (unsigned)std::max<int64_t>(1, std::min<int64_t>(b, 148 * 4));
}

}  // namespace

unsigned long long* handoff_flag(pswim_handoff* h, void* base, int k) {
    return static_cast<unsigned long long*>(base) + k;
}
double* handoff_slot(pswim_handoff* h, void* base, int k) {
    return reinterpret_cast<double*>(static_cast<char*>(base) + h->head) + static_cast<size_t>(k) * h->len;
}

double* handoff_recv_slot(pswim_handoff* h, int k) { return handoff_slot(h, h->block, k); }
bool handoff_has_next(const pswim_handoff* h) { return h->next != nullptr; }
unsigned long long handoff_begin_run(pswim_handoff* h) { return ++h->gen; }

cudaError_t handoff_wait_launch(pswim_handoff* h, int k, unsigned long long gen, cudaStream_t st) {
    if (h->local_prev) {
        std::unique_lock<std::mutex> lk(h->mu);
        h->cv.wait(lk, [&] { return h->posted[k] >= gen; });
        return cudaStreamWaitEvent(st, h->arrived[k], 0);
    }
    arrival_wait_kernel<<<1, 32, 0, st>>>(handoff_flag(h, h->block, k), gen);
    return cudaGetLastError();
}

static cudaError_t post_local(pswim_handoff* h, int k, unsigned long long gen, cudaStream_t st) {
    pswim_handoff* r = h->next_local;
    if (!r) return cudaSuccess;
    const cudaError_t e = cudaEventRecord(r->arrived[k], st);
    {
        std::lock_guard<std::mutex> lk(r->mu);
        r->posted[k] = gen;
    }
    r->cv.notify_all();
    return e;
}

cudaError_t handoff_push_launch(pswim_handoff* h, int k, unsigned long long gen, const double* src,
                                cudaStream_t st) {
    push_kernel<<<push_blocks(h->len), 256, 0, st>>>(src, h->len, handoff_slot(h, h->next, k), h->d_counters + k,
                                                     handoff_flag(h, h->next, k), gen);
    const cudaError_t e = cudaGetLastError();
    return e != cudaSuccess ? e : post_local(h, k, gen, st);
}

cudaError_t handoff_correct_push_launch(pswim_handoff* h, int k, unsigned long long gen, const double* xp,
                                        const double* gn, const double* go, double* out, cudaStream_t st) {
    correct_push_kernel<<<push_blocks(h->len), 256, 0, st>>>(xp, gn, go, h->len, out, handoff_slot(h, h->next, k),
                                                             h->d_counters + k, handoff_flag(h, h->next, k), gen);
    const cudaError_t e = cudaGetLastError();
    return e != cudaSuccess ? e : post_local(h, k, gen, st);
}

void handoff_preload() {
    // lazy module loading could otherwise synchronise the context on first launch while a
    // peer spins in arrival_wait_kernel
    cudaFuncAttributes a;
    cudaFuncGetAttributes(&a, correct_push_kernel);
    cudaFuncGetAttributes(&a, push_kernel);
    cudaFuncGetAttributes(&a, arrival_wait_kernel);
}

}  // namespace pswim

extern "C" {

pswim_handoff* pswim_handoff_create(int device, int64_t len, int32_t slots) {
    if (len <= 0 || slots <= 0) return nullptr;
    auto* h = new (std::nothrow) pswim_handoff();
    if (!h) return nullptr;
    h->device = device;
    h->len = len;
    h->slots = slots;
    h->head = ((size_t)slots * sizeof(unsigned long long) + 255) / 256 * 256;
    const size_t bytes = h->head + (size_t)slots * len * sizeof(double);
    if (cudaSetDevice(device) != cudaSuccess || cudaMalloc(&h->block, bytes) != cudaSuccess ||
        cudaMemset(h->block, 0, h->head) != cudaSuccess ||
        cudaMalloc(&h->d_counters, slots * sizeof(unsigned)) != cudaSuccess ||
        cudaMemset(h->d_counters, 0, slots * sizeof(unsigned)) != cudaSuccess || cudaDeviceSynchronize() != cudaSuccess) {
        if (h->block) cudaFree(h->block);
        if (h->d_counters) cudaFree(h->d_counters);
        delete h;
        return nullptr;
    }
    pswim::handoff_preload();
    h->arrived.assign(slots, nullptr);
    for (auto& e : h->arrived) cudaEventCreateWithFlags(&e, cudaEventDisableTiming);
    h->posted.assign(slots, 0);
    return h;
}

int pswim_handoff_handle(pswim_handoff* h, uint8_t* handle64) {
    if (!h || !handle64) return PSWIM_EINVAL;
    cudaSetDevice(h->device);
    cudaIpcMemHandle_t ipc;
    if (cudaIpcGetMemHandle(&ipc, h->block) != cudaSuccess) return PSWIM_ECUDA;
    static_assert(sizeof(ipc) == 64, "IPC handle size");
    std::memcpy(handle64, &ipc, sizeof ipc);
    return PSWIM_OK;
}

void* pswim_handoff_local_base(pswim_handoff* h) { return h ? h->block : nullptr; }

int pswim_handoff_connect(pswim_handoff* h, const uint8_t* next_handle64, void* next_local_base) {
    if (!h) return PSWIM_EINVAL;
    cudaSetDevice(h->device);
    if (next_local_base) {
        h->next = next_local_base;
    } else if (next_handle64) {
        cudaIpcMemHandle_t ipc;
        std::memcpy(&ipc, next_handle64, sizeof ipc);
        void* p = nullptr;
        if (cudaIpcOpenMemHandle(&p, ipc, cudaIpcMemLazyEnablePeerAccess) != cudaSuccess) return PSWIM_ECOMM;
        h->next = p;
        h->next_ipc = true;
    }
    return PSWIM_OK;
}

int pswim_handoff_connect_local(pswim_handoff* h, pswim_handoff* next) {
    if (!h || !next || next->slots < h->slots || next->len != h->len) return PSWIM_EINVAL;
    h->next = next->block;
    h->next_local = next;
    next->local_prev = true;
    return PSWIM_OK;
}

void pswim_handoff_destroy(pswim_handoff* h) {
    if (!h) return;
    cudaSetDevice(h->device);
    cudaDeviceSynchronize();
    for (auto& e : h->arrived)
        if (e) cudaEventDestroy(e);
    if (h->next_ipc) cudaIpcCloseMemHandle(h->next);
    cudaFree(h->block);
    cudaFree(h->d_counters);
    delete h;
}

}  // extern "C"
