// probe_ucw.cu — dev microbenchmark (not part of the library): the MRS two-target pair loop
// with the source window in the kernel-parameter constant bank (__grid_constant__, 224
// sources), so DFMAs take LDCU-loaded uniform-register operands.  SASS model bound 0.962
// (tools/sass_cost.py) against 0.891 for the shared-memory loop; measured 33.2 TFLOP/s =
// 0.909 of the DFMA peak (DESIGN §10 item 2).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -fmad=false -Iinclude \
//        -Ipaper_2604_12083_b200/csrc -o tools/probe_ucw tools/dev/probe_ucw.cu
#include "kernels.cuh"
using namespace pswim;
constexpr int NW = 224;
struct Win { double2 rec[9][NW]; };
__global__ void __launch_bounds__(128, 3)
ucw_kernel(const __grid_constant__ Win w, int cnt, const double* __restrict__ tgt, double* __restrict__ out, MrsConsts k) {
    const int i = blockIdx.x * 256 + threadIdx.x;
    double tx[2], ty[2], tz[2];
    MrsAcc acc[2];
    for (int q = 0; q < 2; ++q) {
        const int t = i + 128 * q;
        tx[q] = tgt[3 * t]; ty[q] = tgt[3 * t + 1]; tz[q] = tgt[3 * t + 2];
        acc[q].zero();
    }
#pragma unroll 1
    for (int j = 0; j < cnt; ++j)
        mrs_pair2(acc[0], acc[1], tx[0], ty[0], tz[0], tx[1], ty[1], tz[1], w.rec[0][j], w.rec[1][j], w.rec[2][j],
                  w.rec[3][j], w.rec[4][j], w.rec[5][j], w.rec[6][j], w.rec[7][j], w.rec[8][j], k.e2, k.c15e2, k.cm75e4,
                  k.c25e2);
    for (int q = 0; q < 2; ++q) {
        double o[6];
        mrs_finish(acc[q], tx[q], ty[q], tz[q], o);
        for (int c = 0; c < 6; ++c) out[6 * (i + 128 * q) + c] = o[c];
    }
}

#include <cstdio>
#include <vector>
#include <random>
int main() {
    const int nt = 148 * 4 * 4 * 256;
    std::vector<double> ht(3 * nt);
    std::mt19937_64 g(7);
    std::uniform_real_distribution<double> U(-0.5, 0.5);
    for (auto& v : ht) v = U(g);
    static Win w;
    for (int q = 0; q < 9; ++q)
        for (int j = 0; j < NW; ++j) w.rec[q][j] = make_double2(U(g), U(g));
    double *dt, *dout;
    cudaMalloc(&dt, 8 * ht.size());
    cudaMalloc(&dout, 8 * 6 * (size_t)nt);
    cudaMemcpy(dt, ht.data(), 8 * ht.size(), cudaMemcpyHostToDevice);
    MrsConsts k = mrs_consts(0.1, 1.0);
    for (int blocks_per_sm : {3, 4}) {
        cudaFuncSetAttribute(ucw_kernel, cudaFuncAttributePreferredSharedMemoryCarveout, 0);
        const int grid = 148 * blocks_per_sm * 4;  // 4 waves of the resident slots
        cudaEvent_t a, b;
        cudaEventCreate(&a);
        cudaEventCreate(&b);
        for (int r = 0; r < 3; ++r) ucw_kernel<<<grid, 128>>>(w, NW, dt, dout, k);
        cudaEventRecord(a);
        const int reps = 20;
        for (int r = 0; r < reps; ++r) ucw_kernel<<<grid, 128>>>(w, NW, dt, dout, k);
        cudaEventRecord(b);
        cudaEventSynchronize(b);
        float ms;
        cudaEventElapsedTime(&ms, a, b);
        const double pairs = (double)grid * 256 * NW * reps;
        printf("grid %d: %.3f ms/launch, %.2f TFLOP/s (103 flop/pair), %.1f Gpair/s  err=%s\n", grid, ms / reps,
               pairs * 103 / (ms * 1e-3) / 1e12, pairs / (ms * 1e-3) / 1e9, cudaGetErrorString(cudaGetLastError()));
    }
    return 0;
}
