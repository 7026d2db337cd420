// probe_xchg.cu — dev microbenchmark (not part of the library): the fused kernel's per-rhs
// velocity all-to-all on a 16-CTA cluster, 7 targets x 6 values per CTA (100-node flagellum):
//   mode 0: one st.async per value per destination CTA (the fused kernel's push), 42 threads
//   mode 2: one st.async.v2.f64 per value pair per destination CTA, 21 threads
//   mode 1: one cp.async.bulk shared::cta -> shared::cluster per destination CTA (336 B,
//           target-major [i][6] runs), issued by 16 threads after a named barrier
// Cycles per exchange round at CTA 0 (push + wait for all 600 values), averaged.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/probe_xchg tools/probe_xchg.cu
#include <cooperative_groups.h>
#include <cstdint>
#include <cstdio>

#include <cuda_runtime.h>

namespace cg = cooperative_groups;

__device__ __forceinline__ uint32_t su32(const void* p) { return static_cast<uint32_t>(__cvta_generic_to_shared(p)); }
__device__ __forceinline__ uint32_t mapa(uint32_t a, uint32_t r) {
    uint32_t o;
    asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(o) : "r"(a), "r"(r));
    return o;
}
__device__ __forceinline__ void wait_bar(uint64_t* b, uint32_t par) {
    asm volatile(
        "{\n.reg .pred p;\nW_%=:\nmbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n@!p bra W_%=;\n}\n" ::"r"(
            su32(b)),
        "r"(par)
        : "memory");
}

template <int MODE>
__global__ void __cluster_dims__(16, 1, 1) __launch_bounds__(384, 1) xchg(double* out, int reps, int per_cta, int total) {
    __shared__ __align__(128) double buf[2][16 * 7 * 6 + 16];
    __shared__ __align__(16) double stage[2][7 * 6];
    __shared__ __align__(8) uint64_t bar[2];
    const int tid = threadIdx.x;
    const unsigned rank = cg::this_cluster().block_rank();
    if (tid == 0) {
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(&bar[0])));
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(&bar[1])));
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    cg::this_cluster().sync();
    uint32_t ph = 0;
    long long tot = 0;
    const int mine = max(0, min(per_cta, total - (int)rank * per_cta));
    for (int r = 0; r < reps; ++r) {
        const int b = r & 1;
        const long long t0 = clock64();
        if (tid == 0)
            asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su32(&bar[b])),
                         "r"((uint32_t)(total * 8))
                         : "memory");
        if (MODE == 0) {
            if (tid < mine) {
                const uint32_t la = su32(&buf[b][rank * per_cta + tid]), lb = su32(&bar[b]);
#pragma unroll
                for (unsigned rr = 0; rr < 16; ++rr)
                    asm volatile("st.async.shared::cluster.mbarrier::complete_tx::bytes.f64 [%0], %1, [%2];" ::"r"(
                                     mapa(la, rr)),
                                 "d"(1.0 * r + tid), "r"(mapa(lb, rr))
                                 : "memory");
            }
        } else if (MODE == 2) {
            if (2 * tid < mine) {
                const uint32_t la = su32(&buf[b][rank * per_cta + 2 * tid]), lb = su32(&bar[b]);
#pragma unroll
                for (unsigned rr = 0; rr < 16; ++rr)
                    asm volatile("st.async.shared::cluster.mbarrier::complete_tx::bytes.v2.f64 [%0], {%1, %2}, [%3];" ::"r"(
                                     mapa(la, rr)),
                                 "d"(1.0 * r + tid), "d"(2.0 * r + tid), "r"(mapa(lb, rr))
                                 : "memory");
            }
        } else {
            if (tid < mine) stage[b][tid] = 1.0 * r + tid;
            asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
            asm volatile("bar.sync 1, 64;" ::: "memory");  // warps 0-1: the stagers and the issuers
            if (tid < 16 && mine > 0) {
                const uint32_t dst = mapa(su32(&buf[b][rank * per_cta]), tid), mb = mapa(su32(&bar[b]), tid);
                asm volatile(
                    "cp.async.bulk.shared::cluster.shared::cta.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                        dst),
                    "r"(su32(&stage[b][0])), "r"((uint32_t)(mine * 8)), "r"(mb)
                    : "memory");
            }
        }
        wait_bar(&bar[b], (ph >> b) & 1u);
        ph ^= 1u << b;
        tot += clock64() - t0;
    }
    if (tid == 0 && rank == 0) out[MODE] = (double)tot / reps;
    cg::this_cluster().sync();
}

int main() {
    double* d;
    cudaMalloc(&d, 64);
    double h[3];
    cudaFuncSetAttribute(xchg<2>, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
    cudaFuncSetAttribute(xchg<0>, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
    cudaFuncSetAttribute(xchg<1>, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
    for (int i = 0; i < 2; ++i) {
        xchg<0><<<16, 384>>>(d, 2000, 42, 600);
        xchg<1><<<16, 384>>>(d, 2000, 42, 600);
        xchg<2><<<16, 384>>>(d, 2000, 42, 600);
    }
    printf("launch: %s\n", cudaGetErrorString(cudaGetLastError()));
    cudaMemcpy(h, d, 24, cudaMemcpyDeviceToHost);
    printf("st.async per value: %.0f cycles/exchange\ncp.async.bulk per CTA: %.0f cycles/exchange\n"
           "st.async.v2 per value pair: %.0f cycles/exchange\nerr %s\n", h[0], h[1], h[2],
           cudaGetErrorString(cudaDeviceSynchronize()));
    return 0;
}
