// probe_lanes.cu — dev microbenchmark (not part of the library): does a warp with only some
// lanes active issue FP64 instructions faster than a full warp, and what are the dependent
// latencies of DFMA / DADD / MUFU.RSQ64H on B200?  One CTA of 128 threads (one warp per SMSP).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/probe_lanes tools/probe_lanes.cu
#include <cstdio>

#include <cuda_runtime.h>

__global__ void thr(double* out, int iters, int active, double seed) {
    const int lane = threadIdx.x & 31;
    double a[8];
    for (int i = 0; i < 8; ++i) a[i] = seed * (lane + i);
    __syncthreads();
    long long t0 = clock64();
    if (lane < active) {
        for (int it = 0; it < iters; ++it) {
#pragma unroll
            for (int s = 0; s < 16; ++s)
#pragma unroll
                for (int i = 0; i < 8; ++i) a[i] = fma(a[i], 0.999999999, 1e-12);
        }
    }
    __syncwarp();
    long long t1 = clock64();
    double t = 0;
    for (int i = 0; i < 8; ++i) t += a[i];
    if (t == 1.2345) out[1] = t;
    if (threadIdx.x == 0) out[0] = (double)(t1 - t0) / (iters * 16.0 * 8.0);
}

template <int KIND>
__global__ void lat(double* out, int iters, double seed) {
    double a = seed + threadIdx.x * 1e-9, r = 0;
    __syncthreads();
    long long t0 = clock64();
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int s = 0; s < 32; ++s) {
            if (KIND == 0) a = fma(a, 0.999999999, 1e-12);
            if (KIND == 1) a = a + 1e-12;
            if (KIND == 2) {
                double q;
                asm volatile("rsqrt.approx.ftz.f64 %0, %1;" : "=d"(q) : "d"(a));
                a = q;
            }
            if (KIND == 3) a = a * 0.999999999;
        }
    }
    long long t1 = clock64();
    if (a == 1.2345) out[1] = a + r;
    if (threadIdx.x == 0) out[0] = (double)(t1 - t0) / (iters * 32.0);
}

int main() {
    double* d;
    cudaMalloc(&d, 16);
    double h[2];
    const int actives[] = {32, 24, 16, 8, 4, 1};
    for (int w : {32, 64, 128, 256})
        for (int act : actives) {
            thr<<<1, w>>>(d, 200, act, 1.0);
            thr<<<1, w>>>(d, 2000, act, 1.0);
            cudaMemcpy(h, d, 16, cudaMemcpyDeviceToHost);
            printf("threads %3d active lanes/warp %2d: %.3f cycles per warp DFMA (per warp, 8 chains)\n", w, act, h[0]);
        }
    const char* names[] = {"DFMA", "DADD", "MUFU.RSQ64H", "DMUL"};
    auto run = [&](auto kern, int k) {
        kern<<<1, 32>>>(d, 100, 1.0);
        kern<<<1, 32>>>(d, 1000, 1.0);
        cudaMemcpy(h, d, 16, cudaMemcpyDeviceToHost);
        printf("dependent %s latency: %.2f cycles\n", names[k], h[0]);
    };
    run(lat<0>, 0);
    run(lat<1>, 1);
    run(lat<2>, 2);
    run(lat<3>, 3);
    printf("err: %s\n", cudaGetErrorString(cudaDeviceSynchronize()));
    return 0;
}
