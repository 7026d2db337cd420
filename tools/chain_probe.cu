// chain_probe.cu -- single-CTA latency probes of the fused small-system kernel's chains (dev
// tool; build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -fmad=false -std=c++17
// -I paper_2604_12083_b200/csrc tools/chain_probe.cu -o tools/chain_probe).
//
// Each probe runs one phase of fused.cu's per-rhs work on ONE CTA with a chosen number of
// active warps and reports clock64 cycles per repetition as seen by warp 0: the latency floor
// of that phase when the SM is otherwise idle (the "latency roofline" of DESIGN §3.5).
#include <cstdio>
#include <cstdlib>
#include <vector>

#include "kernels.cuh"

using namespace pswim;

__global__ void dfma_chain(double* out, int iters, double a, double b) {
    double x = threadIdx.x * 1e-3;
    const long long t0 = clock64();
    for (int i = 0; i < iters; ++i) {
        x = fma(x, a, b);
        x = fma(x, a, b);
        x = fma(x, a, b);
        x = fma(x, a, b);
    }
    const long long t1 = clock64();
    if (threadIdx.x == 0) out[0] = (double)(t1 - t0) / (4.0 * iters);
    out[1 + threadIdx.x] = x;
}

// rsqrt_fast chain
__global__ void rsqrt_chain(double* out, int iters) {
    double x = 1.0 + threadIdx.x * 1e-3;
    const long long t0 = clock64();
    for (int i = 0; i < iters; ++i) x = rsqrt_fast(x) + 1.0;
    const long long t1 = clock64();
    if (threadIdx.x == 0) out[0] = (double)(t1 - t0) / iters;
    out[1 + threadIdx.x] = x;
}

// sincos chain (the advance's rotation angle)
__global__ void sincos_chain(double* out, int iters) {
    double x = 1e-4 + threadIdx.x * 1e-7;
    const long long t0 = clock64();
    for (int i = 0; i < iters; ++i) {
        double s, c;
        sincos(x, &s, &c);
        x = 1e-4 + (s + c) * 1e-12;
    }
    const long long t1 = clock64();
    if (threadIdx.x == 0) out[0] = (double)(t1 - t0) / iters;
    out[1 + threadIdx.x] = x;
}

// MRS item chain: `warps` warps, each lane = one chunk of `ns` sources (fused.cu layout:
// record plane [step][lane]), one target per warp; pairs + finish (+ butterfly if tree > 0).
__global__ void __launch_bounds__(384, 1) mrs_chain(double* out, int reps, int ns, int warps, int tree, int layout, MrsConsts mc) {
    extern __shared__ double2 rec[];  // 9 planes x ns x 32
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int RS = ns * 32;
    for (int k = tid; k < 9 * RS; k += blockDim.x)
        rec[k] = make_double2(0.1 + 1e-3 * (k % 97), 0.2 - 1e-3 * (k % 89));
    __syncthreads();
    double acc_sum = 0.0;
    long long tot = 0;
    for (int r = 0; r < reps; ++r) {
        __syncthreads();
        const long long t0 = clock64();
        if (warp < warps) {
            const double tx = 0.3 + 0.01 * warp, ty = -0.2, tz = 0.05 * r;
            MrsAcc acc;
            acc.zero();
            if (layout == 0) {
#pragma unroll 2
                for (int s = 0; s < ns; ++s) {
                    const double2* q = rec + s * 32 + lane;
                    mrs_pair(acc, tx, ty, tz, q[0], q[RS], q[2 * RS], q[3 * RS], q[4 * RS], q[5 * RS], q[6 * RS],
                             q[7 * RS], q[8 * RS], mc.e2, mc.c15e2, mc.cm75e4, mc.c25e2);
                }
            } else if (layout == 3) {
                // mrs_pair2: two targets per lane (fused.cu)
                MrsAcc acc1;
                acc1.zero();
#pragma unroll 1
                for (int s = 0; s < ns; ++s) {
                    const double2* q = rec + s * 32 + lane;
                    mrs_pair2(acc, acc1, tx, ty, tz, tx + 0.01, ty, tz, q[0], q[RS], q[2 * RS], q[3 * RS], q[4 * RS],
                              q[5 * RS], q[6 * RS], q[7 * RS], q[8 * RS], mc.e2, mc.c15e2, mc.cm75e4, mc.c25e2);
                }
                double o1[6];
                mrs_finish(acc1, tx, ty, tz, o1);
                acc_sum += o1[0] + o1[3];
            } else if (layout == 2) {
                // two interleaved accumulators (sources s and s + ns/2 of the lane's range)
                MrsAcc acc1;
                acc1.zero();
                const int h = ns / 2;
                for (int s = 0; s < h; ++s) {
                    const double2* q = rec + s * 32 + lane;
                    const double2* p = rec + (s + h) * 32 + lane;
                    mrs_pair(acc, tx, ty, tz, q[0], q[RS], q[2 * RS], q[3 * RS], q[4 * RS], q[5 * RS], q[6 * RS],
                             q[7 * RS], q[8 * RS], mc.e2, mc.c15e2, mc.cm75e4, mc.c25e2);
                    mrs_pair(acc1, tx, ty, tz, p[0], p[RS], p[2 * RS], p[3 * RS], p[4 * RS], p[5 * RS], p[6 * RS],
                             p[7 * RS], p[8 * RS], mc.e2, mc.c15e2, mc.cm75e4, mc.c25e2);
                }
                double o1[6];
                mrs_finish(acc1, tx, ty, tz, o1);
                acc_sum += o1[0] + o1[3];
            } else {
                // broadcast layout: every lane the same source (one LDS wavefront per load)
#pragma unroll 2
                for (int s = 0; s < ns; ++s) {
                    const double2* q = rec + s * 32;
                    mrs_pair(acc, tx + lane * 1e-3, ty, tz, q[0], q[RS], q[2 * RS], q[3 * RS], q[4 * RS], q[5 * RS],
                             q[6 * RS], q[7 * RS], q[8 * RS], mc.e2, mc.c15e2, mc.cm75e4, mc.c25e2);
                }
            }
            double o[6];
            mrs_finish(acc, tx, ty, tz, o);
            for (int off = tree ? 1 << (tree - 1) : 0; off >= 1; off >>= 1)
#pragma unroll
                for (int q = 0; q < 6; ++q) o[q] = o[q] + __shfl_xor_sync(0xffffffffu, o[q], off);
            acc_sum += o[0] + o[1] + o[2] + o[3] + o[4] + o[5];
        }
        const long long t1 = clock64();
        tot += t1 - t0;
    }
    if (tid == 0) out[0] = (double)tot / reps;
    out[1 + tid] = acc_sum;
}

// Front-pass chain of fused.cu (warp-tiled, no LJ) on ONE warp, lanes = nodes of a straight
// rod: advance_node -> rod_segment_om (+ shuffle of the left segment) -> node_loads +
// mrs_stage; cycles of each piece and of the whole chain, as warp 0 sees them (1 warp per SMSP
// is the fused kernel's front configuration).
__global__ void __launch_bounds__(128, 1) front_chain(double* out, int reps, RodArgs rp, MrsConsts mc) {
    __shared__ __align__(16) double st[2][32 * 12];
    __shared__ __align__(16) double vel[32 * 6];
    __shared__ __align__(16) double2 rec[9 * 32];
    __shared__ double om[32];
    const int lane = threadIdx.x & 31;
    for (int k = threadIdx.x; k < 32 * 12; k += blockDim.x) {
        // a bent rod: frames turning by 0.05 rad per node about y (sqrt_rotation's interior branch)
        const int n = k / 12, c = k % 12;
        const double th = 0.05 * n, cs = cos(th), sn = sin(th);
        const double v[12] = {n * rp.ds, 0.01 * n * rp.ds, 0.0, cs, 0, -sn, 0, 1, 0, sn, 0, cs};
        st[0][k] = v[c];
    }
    for (int k = threadIdx.x; k < 32 * 6; k += blockDim.x) vel[k] = 1e-3 * ((k % 7) - 3);
    if (threadIdx.x < 32) om[threadIdx.x] = rod_strain(rp, threadIdx.x, 0.0);
    __syncthreads();
    long long t_adv = 0, t_seg = 0, t_node = 0;
    unsigned fl = 0;
    for (int r = 0; r < reps; ++r) {
        const double* src = st[r & 1];
        double* dst = st[(r & 1) ^ 1];
        __syncwarp();
        const long long t0 = clock64();
        fl |= advance_node(src + 12 * lane, vel + 6 * lane, vel + 6 * lane + 3, 1e-6, 1.0, dst + 12 * lane);
        __syncwarp();
        const long long t1 = clock64();
        double seg[6] = {0, 0, 0, 0, 0, 0};
        if (lane < 31 && !rod_segment_om(rp, dst, lane, om[lane], seg)) fl |= 4;
        double prev[6];
#pragma unroll
        for (int q = 0; q < 6; ++q) prev[q] = __shfl_up_sync(0xffffffffu, seg[q], 1);
        const long long t2 = clock64();
        const d3 xk = ld3(dst + 12 * lane);
        const d3 xn = lane < 31 ? ld3(dst + 12 * (lane + 1)) : xk;
        const d3 xp = lane > 0 ? ld3(dst + 12 * (lane - 1)) : xk;
        d3 f, tq;
        node_loads(rp, lane, seg, prev, xp, xk, xn, f, tq);
        double2 rr[9];
        if (!mrs_stage(&xk.x, 3, &f.x, &tq.x, 0, 0.1, 0.2, 0.3, mc.scale, rr)) fl |= 1;
#pragma unroll
        for (int q = 0; q < 9; ++q) rec[q * 32 + lane] = rr[q];
        __syncwarp();
        const long long t3 = clock64();
        t_adv += t1 - t0;
        t_seg += t2 - t1;
        t_node += t3 - t2;
    }
    if (threadIdx.x == 0) {
        out[0] = (double)t_adv / reps;
        out[1] = (double)t_seg / reps;
        out[2] = (double)t_node / reps;
    }
    out[4 + threadIdx.x] = rec[lane].x + fl;
}

int main() {
    double* d;
    cudaMalloc(&d, 8 * 2048);
    double h;
    dfma_chain<<<1, 32>>>(d, 10000, 0.999, 1e-3);
    cudaMemcpy(&h, d, 8, cudaMemcpyDeviceToHost);
    printf("DFMA dependent latency (1 warp): %.2f cycles\n", h);
    rsqrt_chain<<<1, 32>>>(d, 10000);
    cudaMemcpy(&h, d, 8, cudaMemcpyDeviceToHost);
    printf("rsqrt_fast + DADD dependent latency (1 warp): %.2f cycles\n", h);
    sincos_chain<<<1, 32>>>(d, 10000);
    cudaMemcpy(&h, d, 8, cudaMemcpyDeviceToHost);
    printf("sincos + 2 DP dependent latency (1 warp): %.2f cycles\n", h);
    cudaFuncSetAttribute(mrs_chain, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
    const char* lname[4] = {"lane=chunk", "broadcast", "2 interleaved acc", "pair2 (2 targets)"};
    for (int tree : {0})
        for (int layout = 0; layout < 4; ++layout)
            for (int ns : {1, 2, 4, 8})
                for (int warps : {1, 4, 8, 12}) {
                    if (layout == 2 && ns < 2) continue;
                    const size_t smem = 9 * (size_t)ns * 32 * sizeof(double2);
                    mrs_chain<<<1, 384, smem>>>(d, 200, ns, warps, tree, layout, mrs_consts(0.1, 1.0));
                    cudaError_t e = cudaDeviceSynchronize();
                    cudaMemcpy(&h, d, 8, cudaMemcpyDeviceToHost);
                    printf("mrs item (%s): %d sources/lane, %2d warps, tree %d: %7.0f cycles (%s)\n", lname[layout],
                           ns, warps, tree, h, cudaGetErrorString(e));
                }
    {
        RodArgs rp{};
        rp.m = 32;
        rp.ds = 1.0 / 99;
        rp.inv_ds = 99.0;
        rp.a0 = rp.a1 = 1.0; rp.a2 = 0.7;
        rp.b0 = rp.b1 = 50.0; rp.b2 = 100.0;
        rp.amp = 1.0; rp.freq = 6.28; rp.wavenumber = 6.28;
        double hh[3];
        front_chain<<<1, 32>>>(d, 1000, rp, mrs_consts(0.1, 1.0));
        cudaError_t e = cudaDeviceSynchronize();
        cudaMemcpy(hh, d, sizeof hh, cudaMemcpyDeviceToHost);
        printf("front chain (1 warp, 32 lanes): advance %.0f, segment+shuffle %.0f, node loads+stage %.0f, "
               "total %.0f cycles (%s)\n", hh[0], hh[1], hh[2], hh[0] + hh[1] + hh[2], cudaGetErrorString(e));
        front_chain<<<1, 128>>>(d, 1000, rp, mrs_consts(0.1, 1.0));
        e = cudaDeviceSynchronize();
        cudaMemcpy(hh, d, sizeof hh, cudaMemcpyDeviceToHost);
        printf("front chain (4 warps, 1 per SMSP): advance %.0f, segment+shuffle %.0f, node loads+stage %.0f, "
               "total %.0f cycles (%s)\n", hh[0], hh[1], hh[2], hh[0] + hh[1] + hh[2], cudaGetErrorString(e));
    }
    return 0;
}
