// fused.cu — whole-interval propagation of small systems in ONE kernel.
//
// For N <= 256 nodes a launched-kernel RK2 step is six launches of a few microseconds of
// work each (BASELINE configs[0]: one 100-node flagellum), i.e. launch bound.  This kernel
// runs `steps` Euler / midpoint-RK2 steps (propagators.cpp:126-162) on a thread-block
// cluster with the state resident in shared memory:
//   * every CTA redundantly holds the full state and redundantly does the O(N) phases
//     (segment loads with sqrt_rotation, nodal loads, LJ, source staging, advance);
//   * the O(N^2) MRS is split across the CTAs of the cluster by target: each CTA computes
//     its targets' (target, source chunk) items, reduces the chunk partials in fixed order
//     in its own shared memory, and pushes each target's 6 velocities to every CTA through
//     distributed shared memory; one cluster barrier per rhs (velocities double-buffered).
// All per-element arithmetic is the kernels.cuh routines of the launched path, and the MRS
// decomposition (origin, chunk boundaries, chunk order) is the one mrs_plan picks for the
// same N, so a fused propagate is bitwise identical to the multi-kernel one.
#include <cooperative_groups.h>

#include <algorithm>
#include <cstdlib>

#include "kernels.cuh"

namespace cg = cooperative_groups;

namespace pswim {
namespace {

constexpr int kFusedThreads = 512;

struct FusedArgs {
    RodArgs rod;
    LjArgs lj;
    MrsConsts mc;
    int n;        // total nodes
    int rods, m;  // layout
    int chunks;   // MRS source chunks (== mrs_plan(n, n).chunks)
    int lj_on;
    double max_disp;
    // shared-memory offsets (doubles)
    int off_x, off_xm, off_pos, off_f, off_n, off_seg, off_lj, off_rec, off_part, off_vel;
    int part_stride;  // unused (kept for layout clarity)
    unsigned long long* prof;  // kFusedPhases clock64 counters (CTA 0, thread 0), nullptr = off
};

// In-kernel phase timer: clock64 deltas between the CTA barriers that end each phase, as seen
// by thread 0 of cluster rank 0 (the stage timers of propagators.hpp:55-65 for a path that is
// one kernel).  Phases: 0 segment loads (+LJ), 1 nodal loads, 2 MRS source staging, 3 MRS
// pairs, 4 chunk reduction + DSMEM velocity push, 5 cluster barrier, 6 advance.
struct PhaseClock {
    unsigned long long* prof;
    long long t;
    __device__ __forceinline__ void mark(int phase) {
        if (prof) {
            const long long c = clock64();
            prof[phase] += (unsigned long long)(c - t);
            t = c;
        }
    }
};

template <int CS>
__device__ __forceinline__ void cluster_barrier() {
    if constexpr (CS > 1) {
        cg::this_cluster().sync();
    } else {
        __syncthreads();
    }
}

// rhs (propagators.cpp:38-91) of the state `xs` at time t into vel[6 n] = (u, w) per node.
template <int CS>
__device__ void fused_rhs(const FusedArgs& a, double* sm, const double* xs, double t, double* vel, unsigned& fl,
                          PhaseClock& pc) {
    const int tid = threadIdx.x, bs = blockDim.x, N = a.n, m = a.m, nseg = a.rods * (m - 1);
    double* pos = sm + a.off_pos;
    double* fo = sm + a.off_f;
    double* no = sm + a.off_n;
    double* seg = sm + a.off_seg;
    double* ljf = sm + a.off_lj;
    double2* rec = reinterpret_cast<double2*>(sm + a.off_rec);

    for (int s = tid; s < nseg; s += bs) {
        const int r = s / (m - 1), k = s % (m - 1);
        if (!rod_segment(a.rod, xs + 12 * m * r, k, t, seg + 6 * s)) fl |= kFlagDegenerate;
    }
    if (a.lj_on) {
        for (int i = tid; i < N; i += bs) {
            double fx = 0, fy = 0, fz = 0;
            const double xi = xs[12 * i], yi = xs[12 * i + 1], zi = xs[12 * i + 2];
            const int ri = i / m, ki = i - ri * m;
            for (int rj = 0, j = 0; rj < a.lj.rods; ++rj)
                for (int kj = 0; kj < m; ++kj, ++j)
                    lj_pair(a.lj, ri, ki, rj, kj, xi - xs[12 * j], yi - xs[12 * j + 1], zi - xs[12 * j + 2], fx, fy,
                            fz);
            ljf[3 * i] = fx;
            ljf[3 * i + 1] = fy;
            ljf[3 * i + 2] = fz;
        }
    }
    __syncthreads();
    pc.mark(0);
    for (int g = tid; g < N; g += bs) {
        const int r = g / m, k = g % m;
        d3 f, tq;
        rod_node(a.rod, xs + 12 * m * r, seg + 6 * (m - 1) * r, k, f, tq);
        if (a.lj_on) f = f + ld3(ljf + 3 * g) * a.rod.inv_ds;
        st3(pos + 3 * g, ld3(xs + 12 * g));
        st3(fo + 3 * g, f);
        st3(no + 3 * g, tq);
    }
    __syncthreads();
    pc.mark(1);
    // stage every source relative to node 0 (the single target block's origin in mrs.cu)
    const double ox = pos[0], oy = pos[1], oz = pos[2];
    for (int j = tid; j < N; j += bs) {
        double2 r[9];
        if (!mrs_stage(pos, 3, fo, no, j, ox, oy, oz, a.mc.scale, r)) fl |= kFlagNonFinite;
#pragma unroll
        for (int q = 0; q < 9; ++q) rec[q * N + j] = r[q];
    }
    __syncthreads();
    pc.mark(2);
    // MRS: this CTA owns targets [i0, i1); items (target, source chunk) computed here, the
    // chunk partials reduced locally in fixed order (mrs.cu's last-CTA reduction), and each
    // target's 6 velocities pushed to every CTA of the cluster through DSMEM.
    const int rank = CS > 1 ? (int)cg::this_cluster().block_rank() : 0;
    const int tpc = (N + CS - 1) / CS;
    const int i0 = rank * tpc, i1 = min(N, i0 + tpc), nloc = max(0, i1 - i0);
    double* lpart = sm + a.off_part;  // [chunks][tpc][6]
    for (int w = tid; w < nloc * a.chunks; w += bs) {
        const int c = w / nloc, il = w % nloc, i = i0 + il;
        const int j0 = (int)((int64_t)c * N / a.chunks), j1 = (int)((int64_t)(c + 1) * N / a.chunks);
        const double tx = pos[3 * i] - ox, ty = pos[3 * i + 1] - oy, tz = pos[3 * i + 2] - oz;
        MrsAcc acc;
        acc.zero();
#pragma unroll 2
        for (int j = j0; j < j1; ++j)
            mrs_pair(acc, tx, ty, tz, rec[j], rec[N + j], rec[2 * N + j], rec[3 * N + j], rec[4 * N + j],
                     rec[5 * N + j], rec[6 * N + j], rec[7 * N + j], rec[8 * N + j], a.mc.e2, a.mc.c15e2, a.mc.cm75e4,
                     a.mc.c25e2);
        double out[6];
        mrs_finish(acc, tx, ty, tz, out);
#pragma unroll
        for (int q = 0; q < 6; ++q) lpart[(c * tpc + il) * 6 + q] = out[q];
    }
    __syncthreads();
    pc.mark(3);
    // one thread per (target, component): the chunk partials summed in chunk order 0..C-1
    // (mrs.cu's last-CTA reduction, bitwise), then pushed to every CTA of the cluster
    for (int w = tid; w < nloc * 6; w += bs) {
        const int il = w / 6, q = w - 6 * il;
        double sum = lpart[w];
#pragma unroll 4
        for (int c = 1; c < a.chunks; ++c) sum += lpart[(c * tpc + il) * 6 + q];
        const int i = i0 + il;
        if constexpr (CS > 1) {
            cg::cluster_group cl = cg::this_cluster();
#pragma unroll
            for (int rr = 0; rr < CS; ++rr) cl.map_shared_rank(vel, rr)[6 * i + q] = sum;
        } else {
            vel[6 * i + q] = sum;
        }
    }
    if (a.prof) __syncthreads();  // phase timer only: end of the push as one CTA-wide instant
    pc.mark(4);
    cluster_barrier<CS>();
    pc.mark(5);
}

template <int CS>
__global__ void __launch_bounds__(kFusedThreads, 1)
fused_kernel(FusedArgs a, double* __restrict__ state, int64_t steps, double t0, double dt, int scheme,
             unsigned* __restrict__ flags) {
    extern __shared__ __align__(16) double sm[];
    const int tid = threadIdx.x, bs = blockDim.x, N = a.n;
    double* x = sm + a.off_x;
    double* xm = sm + a.off_xm;
    for (int k = tid; k < 12 * N; k += bs) x[k] = state[k];
    __syncthreads();
    unsigned fl = 0;
    int parity = 0;
    double t = t0;
    const int crank = CS > 1 ? (int)cg::this_cluster().block_rank() : 0;
    PhaseClock pc{(a.prof && tid == 0 && crank == 0) ? a.prof : nullptr, clock64()};
    // velocities are double-buffered: a CTA that runs ahead pushes the next rhs into the
    // other buffer while slower CTAs still read this one (the next cluster barrier orders it)
    for (int64_t s = 0; s < steps; ++s) {
        double* vel = sm + a.off_vel + parity * 6 * N;
        fused_rhs<CS>(a, sm, x, t, vel, fl, pc);
        parity ^= 1;
        if (scheme == PSWIM_EULER) {
            for (int i = tid; i < N; i += bs)
                fl |= advance_node(x + 12 * i, vel + 6 * i, vel + 6 * i + 3, dt, a.max_disp, x + 12 * i);
            __syncthreads();
            pc.mark(6);
        } else {
            // step_rk2, propagators.cpp:130-133
            for (int i = tid; i < N; i += bs)
                fl |= advance_node(x + 12 * i, vel + 6 * i, vel + 6 * i + 3, 0.5 * dt, a.max_disp, xm + 12 * i);
            __syncthreads();
            pc.mark(6);
            vel = sm + a.off_vel + parity * 6 * N;
            fused_rhs<CS>(a, sm, xm, t + 0.5 * dt, vel, fl, pc);
            parity ^= 1;
            for (int i = tid; i < N; i += bs)
                fl |= advance_node(x + 12 * i, vel + 6 * i, vel + 6 * i + 3, dt, a.max_disp, x + 12 * i);
            __syncthreads();
            pc.mark(6);
        }
        t += dt;  // propagators.cpp:159
    }
    if (crank == 0)
        for (int k = tid; k < 12 * N; k += bs) state[k] = x[k];
    if (fl) atomicOr(flags, fl);
    cluster_barrier<CS>();  // no CTA may exit while others still push partials into it
}

template <int CS>
cudaError_t launch_cs(const FusedArgs& a, size_t smem, double* state, int64_t steps, double t0, double dt, int scheme,
                      unsigned* flags, cudaStream_t st) {
    static bool configured = false;
    if (!configured) {
        cudaError_t e = cudaFuncSetAttribute(fused_kernel<CS>, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024);
        if (e != cudaSuccess) return e;
        if (CS > 8) {
            e = cudaFuncSetAttribute(fused_kernel<CS>, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
            if (e != cudaSuccess) return e;
        }
        configured = true;
    }
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3(CS);
    cfg.blockDim = dim3(kFusedThreads);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = st;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = CS;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    return cudaLaunchKernelEx(&cfg, fused_kernel<CS>, a, state, steps, t0, dt, scheme, flags);
}

}  // namespace

// Returns the cluster size the fused path would use for this scenario (0 = not eligible).
int fused_cluster_size(const RodParams& p) {
    const int64_t n = p.rods * p.m;
    if (n > 256 || n < 2) return 0;
    const MrsPlan plan = mrs_plan(n, n);
    static const int max_cs = [] {
        const char* e = std::getenv("PSWIM_FUSED_MAX_CLUSTER");
        const int v = e ? std::atoi(e) : 8;
        return (v == 1 || v == 2 || v == 4 || v == 8 || v == 16) ? v : 8;
    }();
    static const int min_tpc = [] {
        const char* e = std::getenv("PSWIM_FUSED_MIN_TARGETS");
        return e ? std::max(1, std::atoi(e)) : 12;
    }();
    int cs = 1;
    while (cs < max_cs && (n + 2 * cs - 1) / (2 * cs) >= min_tpc) cs *= 2;  // >= min_tpc targets per CTA
    const int64_t tpc = (n + cs - 1) / cs;
    // shared memory: x, xm (12n each), pos/f/n/lj (3n each), seg, rec (18n), local partials
    // (chunks x tpc x 6), velocities (2 x 6n)
    const int64_t doubles = 24 * n + 12 * n + 6 * p.rods * (p.m - 1) + 18 * n + plan.chunks * tpc * 6 + 12 * n + 16;
    if (doubles * 8 > 220 * 1024) return 0;
    return cs;
}

void fused_preload() {
    cudaFuncAttributes a;
    cudaFuncGetAttributes(&a, fused_kernel<1>);
    cudaFuncGetAttributes(&a, fused_kernel<2>);
    cudaFuncGetAttributes(&a, fused_kernel<4>);
    cudaFuncGetAttributes(&a, fused_kernel<8>);
    cudaFuncGetAttributes(&a, fused_kernel<16>);
}

cudaError_t fused_propagate_launch(const RodParams& p, double* state, int64_t steps, double t0, double dt, int scheme,
                                   unsigned* flags, cudaStream_t st, unsigned long long* prof) {
    const int cs = fused_cluster_size(p);
    if (cs == 0) return cudaErrorInvalidValue;
    const int64_t n = p.rods * p.m;
    const MrsPlan plan = mrs_plan(n, n);
    FusedArgs a;
    a.rod = rod_args(p);
    a.lj = lj_args(p);
    a.mc = mrs_consts(p.epsilon, p.mu);
    a.n = (int)n;
    a.rods = (int)p.rods;
    a.m = (int)p.m;
    a.chunks = plan.chunks;
    a.lj_on = (p.rods >= 2 && p.lj_well > 0.0) ? 1 : 0;  // propagators.cpp:70
    a.max_disp = 10.0 * p.ds;
    a.prof = prof;
    int off = 0;
    auto take = [&](int count) {
        const int o = off;
        off += (count + 1) & ~1;  // keep 16-B alignment
        return o;
    };
    a.off_x = take(12 * a.n);
    a.off_xm = take(12 * a.n);
    a.off_pos = take(3 * a.n);
    a.off_f = take(3 * a.n);
    a.off_n = take(3 * a.n);
    a.off_seg = take(6 * a.rods * (a.m - 1));
    a.off_lj = take(3 * a.n);
    a.off_rec = take(18 * a.n);
    const int tpc = (a.n + cs - 1) / cs;
    a.part_stride = 0;
    a.off_part = take(plan.chunks * tpc * 6);
    a.off_vel = take(12 * a.n);
    const size_t smem = (size_t)off * sizeof(double);
    switch (cs) {
        case 1: return launch_cs<1>(a, smem, state, steps, t0, dt, scheme, flags, st);
        case 2: return launch_cs<2>(a, smem, state, steps, t0, dt, scheme, flags, st);
        case 4: return launch_cs<4>(a, smem, state, steps, t0, dt, scheme, flags, st);
        case 8: return launch_cs<8>(a, smem, state, steps, t0, dt, scheme, flags, st);
        default: return launch_cs<16>(a, smem, state, steps, t0, dt, scheme, flags, st);
    }
}

}  // namespace pswim
