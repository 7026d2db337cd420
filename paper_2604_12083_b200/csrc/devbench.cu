// devbench.cu — FP64 pipe microbenchmarks used to explain the MRS kernel's pipe efficiency
// (developer diagnostics, exported as pswim_dev_fp64_probe).  Each kernel runs 8
// independent chains per thread for `iters` x 16 steps over the whole chip.
//   kind 0: a = fma(a, K1, K2)            constant-bank operands (1 register read)
//   kind 1: a = fma(a, b, c)               shared b, c registers (operand reuse possible)
//   kind 2: a_i = fma(x_i, y_i, a_i)       three distinct register pairs per DFMA
//   kind 3: a_i = a_i * x_i                DMUL, two distinct registers
//   kind 4: kind 2 + one MUFU.RSQ64H per 50 DFMA
#include <cuda_runtime.h>

#include "ctx.h"
#include "internal.h"

namespace {

template <int KIND>
__global__ void __launch_bounds__(256) probe(double* sink, int iters, double seed) {
    double a[8], x[8], y[8];
#pragma unroll
    for (int i = 0; i < 8; ++i) {
        a[i] = seed * (threadIdx.x + i);
        x[i] = 0.999999 + 1e-9 * (i + threadIdx.x) * seed;
        y[i] = 1e-12 * (i + 1 + threadIdx.x) * seed;
    }
    const double b = x[3] * seed, c = y[5] * seed;
    double r = seed;
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int s = 0; s < 16; ++s) {
#pragma unroll
            for (int i = 0; i < 8; ++i) {
                if (KIND == 0) a[i] = fma(a[i], 0.999999999, 1e-12);
                if (KIND == 1) a[i] = fma(a[i], b, c);
                if (KIND == 2 || KIND == 4) a[i] = fma(x[i], y[i], a[i]);
                if (KIND == 3) a[i] = a[i] * x[i];
            }
            if (KIND == 4 && (s % 6) == 0) {
                double q;
                asm volatile("rsqrt.approx.ftz.f64 %0, %1;" : "=d"(q) : "d"(a[s & 7] + 2.0));
                r += q;
            }
        }
    }
    double t = r;
#pragma unroll
    for (int i = 0; i < 8; ++i) t += a[i];
    if (t == 12345.678) sink[0] = t;
}

// kind 5: DMMA m8n8k4 only; kind 6: even warps DFMA (constant operands), odd warps DMMA.
__device__ __forceinline__ void dmma(double& d0, double& d1, double a, double b) {
    asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                 : "+d"(d0), "+d"(d1)
                 : "d"(a), "d"(b));
}

template <int KIND>
__global__ void __launch_bounds__(256) probe_mma(double* sink, int iters, double seed) {
    const int warp = threadIdx.x >> 5;
    double acc[8][2];
    double a[8];
#pragma unroll
    for (int i = 0; i < 8; ++i) {
        acc[i][0] = acc[i][1] = 0.0;
        a[i] = seed * (threadIdx.x + i) * 1e-3;
    }
    const double b = seed * 0.999;
    if (KIND == 5 || (warp & 1)) {
        for (int it = 0; it < iters; ++it)
#pragma unroll
            for (int s = 0; s < 16; ++s)
#pragma unroll
                for (int i = 0; i < 8; ++i) dmma(acc[i][0], acc[i][1], a[i], b);
    } else {
        double x[8];
#pragma unroll
        for (int i = 0; i < 8; ++i) x[i] = a[i];
        // 16x more DFMA iterations: one DMMA is 256 FMAs = 8 lane-FMAs per thread x 32;
        // per warp-instruction a DMMA does 8x the work of a DFMA
        for (int it = 0; it < iters * 8; ++it)
#pragma unroll
            for (int s = 0; s < 16; ++s)
#pragma unroll
                for (int i = 0; i < 8; ++i) x[i] = fma(x[i], 0.999999999, 1e-12);
#pragma unroll
        for (int i = 0; i < 8; ++i) acc[i][0] += x[i];
    }
    double t = 0.0;
#pragma unroll
    for (int i = 0; i < 8; ++i) t += acc[i][0] + acc[i][1];
    if (t == 12345.678) sink[0] = t;
}

}  // namespace

extern "C" int pswim_dev_fp64_probe(pswim_ctx* ctx, int kind, double* dfma_per_s, double* ms_out) {
    if (!ctx) return PSWIM_EINVAL;
    if (ctx->use()) return PSWIM_ECUDA;
    double* sink = nullptr;
    if (cudaMalloc(&sink, sizeof(double)) != cudaSuccess) return PSWIM_ECUDA;
    const int blocks = 148 * 8, iters = 1024;
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    float best = 1e30f;
    for (int rep = 0; rep < 3; ++rep) {
        cudaEventRecord(a, ctx->stream);
        switch (kind) {
            case 0: probe<0><<<blocks, 256, 0, ctx->stream>>>(sink, iters, 1.0); break;
            case 1: probe<1><<<blocks, 256, 0, ctx->stream>>>(sink, iters, 1.0); break;
            case 2: probe<2><<<blocks, 256, 0, ctx->stream>>>(sink, iters, 1.0); break;
            case 3: probe<3><<<blocks, 256, 0, ctx->stream>>>(sink, iters, 1.0); break;
            case 4: probe<4><<<blocks, 256, 0, ctx->stream>>>(sink, iters, 1.0); break;
            case 5: probe_mma<5><<<blocks, 256, 0, ctx->stream>>>(sink, iters, 1.0); break;
            default: probe_mma<6><<<blocks, 256, 0, ctx->stream>>>(sink, iters, 1.0); break;
        }
        cudaEventRecord(b, ctx->stream);
        cudaEventSynchronize(b);
        float ms = 0.f;
        cudaEventElapsedTime(&ms, a, b);
        if (rep > 0 && ms < best) best = ms;
    }
    cudaEventDestroy(a);
    cudaEventDestroy(b);
    cudaFree(sink);
    // lane-FMA equivalents: DFMA kinds 8*16 per thread-iteration; DMMA 8*16 MMAs per warp
    // = 8*16*256 FMAs per warp = 8*16*8 per thread; kind 6: both halves do equal work
    double per_thread = 8.0 * 16.0 * iters;
    if (kind >= 5) per_thread *= 8.0;
    *dfma_per_s = per_thread * (double)blocks * 256.0 / (1e-3 * best);
    if (ms_out) *ms_out = best;
    return PSWIM_OK;
}
