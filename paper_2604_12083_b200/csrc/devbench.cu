// devbench.cu — FP64 pipe microbenchmarks used to explain the MRS kernel's pipe efficiency
// (developer diagnostics, exported as pswim_dev_fp64_probe).  Each kernel runs 8
// independent chains per thread for `iters` x 16 steps over the whole chip.
//   kind 0: a = fma(a, K1, K2)            constant-bank operands (1 register read)
//   kind 1: a = fma(a, b, c)               shared b, c registers (operand reuse possible)
//   kind 2: a_i = fma(x_i, y_i, a_i)       three distinct register pairs per DFMA
//   kind 3: a_i = a_i * x_i                DMUL, two distinct registers
//   kind 4: kind 2 + one MUFU.RSQ64H per 50 DFMA
#include <cooperative_groups.h>
#include <cuda_runtime.h>

#include "ctx.h"
#include "internal.h"
#include "kernels.cuh"
#include "tma.cuh"

namespace {
using namespace pswim;

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

// ---- latency floors of the fused small-system kernel's per-rhs phases (fused.cu) ----------
// Each probe runs one phase alone on an otherwise idle SM and reports clock64 cycles per
// repetition as warp 0 sees it: the floor of that phase for the fused kernel's decomposition.

// Front-pass chain on one warp per SMSP (the fused front's configuration), lanes = nodes of a
// bent rod (frames turning 0.05 rad per node, sqrt_rotation's interior branch), component
// planes as in fused.cu: advance_node -> rod_segment_om + shuffle -> node_loads + mrs_stage.
__global__ void __launch_bounds__(128, 1) lat_front(double* out, int reps, RodArgs rp, MrsConsts mc) {
    __shared__ __align__(16) double st[2][12 * 32];
    __shared__ __align__(16) double vel[6 * 32];
    __shared__ __align__(16) double2 rec[9 * 32];
    __shared__ double om[32];
    const int lane = threadIdx.x & 31;
    for (int k = threadIdx.x; k < 32 * 12; k += blockDim.x) {
        const int n = k % 32, c = k / 32;
        const double th = 0.05 * n, cs = cos(th), sn = sin(th);
        const double v[12] = {n * rp.ds, 0.01 * n * rp.ds, 0.0, cs, 0, -sn, 0, 1, 0, sn, 0, cs};
        st[0][k] = v[c];
    }
    for (int k = threadIdx.x; k < 32 * 6; k += blockDim.x) vel[k] = 1e-3 * ((k % 7) - 3);
    if (threadIdx.x < 32) om[threadIdx.x] = rod_strain(rp, threadIdx.x, 0.0);
    __syncthreads();
    long long tot = 0;
    unsigned fl = 0;
    for (int r = 0; r < reps; ++r) {
        const double* src = st[r & 1];
        double* dst = st[(r & 1) ^ 1];
        __syncwarp();
        const long long t0 = clock64();
        fl |= advance_node(src + lane, vel + lane, vel + 96 + lane, 1e-6, 1.0, dst + lane, 32, 32, 32);
        __syncwarp();
        double seg[6] = {0, 0, 0, 0, 0, 0};
        if (lane < 31 && !rod_segment_om(rp, dst, lane, om[lane], seg, 32)) fl |= 4;
        double prev[6];
#pragma unroll
        for (int q = 0; q < 6; ++q) prev[q] = __shfl_up_sync(0xffffffffu, seg[q], 1);
        const d3 xk = ld3s(dst + lane, 32);
        const d3 xn = lane < 31 ? ld3s(dst + lane + 1, 32) : xk;
        const d3 xp = lane > 0 ? ld3s(dst + lane - 1, 32) : xk;
        d3 f, tq;
        node_loads(rp, lane, seg, prev, xp, xk, xn, f, tq);
        double2 rr[9];
        if (!mrs_stage(&xk.x, 3, &f.x, &tq.x, 0, 0.1, 0.2, 0.3, mc.scale, rr)) fl |= 1;
#pragma unroll
        for (int q = 0; q < 9; ++q) rec[q * 32 + lane] = rr[q];
        __syncwarp();
        tot += clock64() - t0;
    }
    if (threadIdx.x == 0) out[0] = (double)tot / reps;
    if (fl == 12345u) out[1] = rec[lane].x;
}

// MRS items of fused.cu: `warps` warps, one (target, chunk) item per lane, `ns` sources each,
// mrs_pair + mrs_finish + the partial store; warp 0's cycles per repetition.
__global__ void __launch_bounds__(384, 1) lat_mrs(double* out, int reps, int ns, int warps, MrsConsts mc) {
    extern __shared__ double2 lrec[];  // 9 planes x ns x 32
    __shared__ double part[6 * 384];
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, RS = ns * 32;
    for (int k = tid; k < 9 * RS; k += blockDim.x) lrec[k] = make_double2(0.1 + 1e-3 * (k % 97), 0.2 - 1e-3 * (k % 89));
    __syncthreads();
    long long tot = 0;
    double chk = 0.0;
    for (int r = 0; r < reps; ++r) {
        __syncthreads();
        const long long t0 = clock64();
        if (warp < warps) {
            const double tx = 0.3 + 0.01 * warp, ty = -0.2 + 1e-3 * lane, tz = 0.05 * r;
            MrsAcc acc;
            acc.zero();
#pragma unroll 2
            for (int s = 0; s < ns; ++s) {
                const double2* q = lrec + s * 32 + lane;
                mrs_pair(acc, tx, ty, tz, q[0], q[RS], q[2 * RS], q[3 * RS], q[4 * RS], q[5 * RS], q[6 * RS],
                         q[7 * RS], q[8 * RS], mc.e2, mc.c15e2, mc.cm75e4, mc.c25e2);
            }
            double o[6];
            mrs_finish(acc, tx, ty, tz, o);
#pragma unroll
            for (int q = 0; q < 6; ++q) part[q * 384 + tid] = o[q];
        }
        __syncthreads();
        tot += clock64() - t0;
        chk += part[(r * 7 + tid) % (6 * 384)];
    }
    if (tid == 0) out[0] = (double)tot / reps;
    if (chk == 12345.678) out[1] = chk;  // keeps the items live
}

// The chunk reduction of one velocity component: `chunks` partials summed in order from
// shared memory (fused.cu), one thread.
__global__ void lat_reduce(double* out, int reps, int chunks) {
    __shared__ double p[64];
    if (threadIdx.x < 64) p[threadIdx.x] = 1e-3 * threadIdx.x;
    __syncthreads();
    long long tot = 0;
    double acc = 0.0;
    for (int r = 0; r < reps; ++r) {
        const long long t0 = clock64();
        double sum = p[0];
#pragma unroll 8
        for (int c = 1; c < chunks; ++c) sum += p[c];
        acc += sum;
        p[r & 63] = acc * 1e-30;  // keep the loads live across repetitions
        tot += clock64() - t0;
    }
    if (threadIdx.x == 0) out[0] = (double)tot / reps;
}

// The velocity exchange of fused.cu on a cluster of 16: every CTA pushes `per_cta` values
// (one thread per value; `total` over the cluster) to all 16 CTAs with st.async + mbarrier
// complete_tx and waits for all `total`; cycles per round at CTA 0 (push + wait, the rhs's
// exchange floor).
__global__ void __cluster_dims__(16, 1, 1) __launch_bounds__(384, 1) lat_exchange(double* out, int reps, int per_cta,
                                                                                 int total) {
    namespace cg = cooperative_groups;
    __shared__ __align__(16) double buf[2][16 * 64];
    __shared__ __align__(8) uint64_t bar[2];
    const int tid = threadIdx.x;
    const unsigned rank = cg::this_cluster().block_rank();
    if (tid == 0) {
        mbar_init(&bar[0], 1);
        mbar_init(&bar[1], 1);
        fence_mbar_init();
    }
    cg::this_cluster().sync();
    uint32_t ph[2] = {0u, 0u};
    long long tot = 0;
    const int mine = max(0, min(per_cta, total - (int)rank * per_cta));  // the fused split's last CTAs push less
    for (int r = 0; r < reps; ++r) {
        const int b = r & 1;
        const long long t0 = clock64();
        if (tid < mine) {
            const uint32_t laddr = smem_u32(&buf[b][rank * per_cta + tid]), lbar = smem_u32(&bar[b]);
            for (unsigned rr = 0; rr < 16; ++rr) {
                uint32_t ra, rb;
                asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(ra) : "r"(laddr), "r"(rr));
                asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(rb) : "r"(lbar), "r"(rr));
                asm volatile("st.async.shared::cluster.mbarrier::complete_tx::bytes.f64 [%0], %1, [%2];" ::"r"(ra),
                             "d"(1.0 * r + tid), "r"(rb)
                             : "memory");
            }
        }
        if (tid == 0) mbar_expect_tx(&bar[b], (uint32_t)(total * sizeof(double)));
        mbar_wait(&bar[b], ph[b] & 1u);
        ++ph[b];
        tot += clock64() - t0;
    }
    if (tid == 0 && rank == 0) out[0] = (double)tot / reps;
    cg::this_cluster().sync();
}

}  // namespace

// Latency floors of the fused small-system kernel, measured on this GPU:
// out[0] front chain, out[1] MRS items (ns sources per item, `warps` warps on 4 SMSPs),
// out[2] chunk reduction of `chunks` partials, out[3] velocity exchange of `per_cta` values
// per CTA (`total` = 6 N over the cluster) on a 16-CTA cluster; cycles per rhs each.
extern "C" int pswim_dev_latency_probe(pswim_ctx* ctx, int ns, int warps, int chunks, int per_cta, int total,
                                       double* out4) {
    if (!ctx || !out4 || ns < 1 || ns > 8 || warps < 1 || warps > 12 || chunks < 1 || chunks > 64 || per_cta < 1 ||
        per_cta > 64 || total < 1 || total > 16 * per_cta)
        return PSWIM_EINVAL;
    if (ctx->use()) return PSWIM_ECUDA;
    double* d = nullptr;
    if (cudaMalloc(&d, 8 * sizeof(double)) != cudaSuccess) return PSWIM_ECUDA;
    const RodArgs rp = rod_args(ctx->rp);
    const MrsConsts mc = mrs_consts(ctx->rp.epsilon, ctx->rp.mu);
    lat_front<<<1, 128, 0, ctx->stream>>>(d, 1000, rp, mc);
    lat_mrs<<<1, 384, 9 * ns * 32 * sizeof(double2), ctx->stream>>>(d + 1, 500, ns, warps, mc);
    lat_reduce<<<1, 32, 0, ctx->stream>>>(d + 2, 1000, chunks);
    cudaFuncSetAttribute(lat_exchange, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);  // (dev probe)
    lat_exchange<<<16, 384, 0, ctx->stream>>>(d + 3, 1000, per_cta, total);
    const cudaError_t el = cudaGetLastError();
    if (el != cudaSuccess) {
        cudaStreamSynchronize(ctx->stream);
        cudaFree(d);
        return ctx->fail(PSWIM_ECUDA, std::string("latency probe launch: ") + cudaGetErrorString(el));
    }
    const cudaError_t e = cudaMemcpyAsync(out4, d, 4 * sizeof(double), cudaMemcpyDeviceToHost, ctx->stream);
    const cudaError_t e2 = cudaStreamSynchronize(ctx->stream);
    cudaFree(d);
    return (e == cudaSuccess && e2 == cudaSuccess && cudaGetLastError() == cudaSuccess) ? PSWIM_OK : PSWIM_ECUDA;
}

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
