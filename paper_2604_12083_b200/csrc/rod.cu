// rod.cu — rod mechanics, triad update and the small elementwise kernels of the path.
//
//   rod_loads_kernel  internal_loads + nodal_loads (reference src/rod.cpp:36-109), one CTA
//                     per rod, the rod's packed state staged once in smem; segments then
//                     nodes; device sqrt_rotation (dev_math.cuh); LJ/extra loads folded in
//                     as rhs does (src/propagators.cpp:59-84).
//   lj_kernel         lj_repulsion (src/rod.cpp:124-174) as a per-node all-pairs sum.
//   advance_kernel    advance_state (src/propagators.cpp:93-124) + reorthonormalize
//                     (src/rod.cpp:176-195), one thread per node.
//   sqrt_batched      sqrt_rotation over a batch (rotation.cpp:91-107), smem-staged.
//   metric / correct  rod_position_metric (io.cpp:49-68), corrected (parareal.cpp:47-54).
#include <cmath>

#include "kernels.cuh"

namespace pswim {
namespace {

// ---------------------------------------------------------------------------------------
// internal_loads + nodal_loads
// ---------------------------------------------------------------------------------------
__global__ void __launch_bounds__(256)
rod_loads_kernel(RodArgs p, const double* __restrict__ state, double t, double* __restrict__ pos,
                 double* __restrict__ fo, double* __restrict__ no, double* __restrict__ seg_f,
                 double* __restrict__ seg_n, const double* __restrict__ lj, const double* __restrict__ extra_f,
                 const double* __restrict__ extra_n, unsigned* __restrict__ flags) {
    extern __shared__ double sh[];
    const int64_t m = p.m;
    double* xs = sh;            // m x 12 packed rod state
    double* seg = sh + 12 * m;  // (m-1) x 6: F, N per segment
    const int64_t rod = blockIdx.x;
    const double* src = state + 12 * m * rod;
    for (int64_t k = threadIdx.x; k < 12 * m; k += blockDim.x) xs[k] = src[k];
    __syncthreads();
    for (int64_t k = threadIdx.x; k + 1 < m; k += blockDim.x) {
        if (!rod_segment(p, xs, k, t, seg + 6 * k)) atomicOr(flags, kFlagDegenerate);  // rod.cpp:53-55
        if (seg_f) {
            const int64_t g = (m - 1) * rod + k;
            st3(seg_f + 3 * g, ld3(seg + 6 * k));
            st3(seg_n + 3 * g, ld3(seg + 6 * k + 3));
        }
    }
    __syncthreads();
    for (int64_t k = threadIdx.x; k < m; k += blockDim.x) {
        d3 f, tq;
        rod_node(p, xs, seg, k, f, tq);
        const int64_t g = m * rod + k;
        if (lj) f = f + ld3(lj + 3 * g) * p.inv_ds;  // propagators.cpp:70-74
        if (extra_f) {                              // propagators.cpp:75-84
            f = f + ld3(extra_f + 3 * g);
            tq = tq + ld3(extra_n + 3 * g);
        }
        st3(pos + 3 * g, ld3(xs + 12 * k));
        st3(fo + 3 * g, f);
        st3(no + 3 * g, tq);
    }
}

// ---------------------------------------------------------------------------------------
// Lennard-Jones repulsion: force on node i = sum over valid partners j of
// lj_force_over_r(|d|) d, d = x_i - x_j (rod.cpp:116-120, 146-171).  Same-rod pairs with
// |i - j| < excl are skipped.  Pair forces are bitwise antisymmetric.
// ---------------------------------------------------------------------------------------
constexpr int kLjTile = 256;
__global__ void __launch_bounds__(256)
lj_kernel(const double* __restrict__ state, LjArgs a, double* __restrict__ out) {
    __shared__ double sx[kLjTile], sy[kLjTile], sz[kLjTile];
    const int64_t total = a.rods * a.m;
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    const int64_t il = i < total ? i : total - 1;
    const double xi = state[12 * il], yi = state[12 * il + 1], zi = state[12 * il + 2];
    double fx = 0, fy = 0, fz = 0;
    for (int64_t jt = 0; jt < total; jt += kLjTile) {
        const int cnt = (total - jt) < kLjTile ? (int)(total - jt) : kLjTile;
        __syncthreads();
        if (threadIdx.x < cnt) {
            const int64_t j = jt + threadIdx.x;
            sx[threadIdx.x] = state[12 * j];
            sy[threadIdx.x] = state[12 * j + 1];
            sz[threadIdx.x] = state[12 * j + 2];
        }
        __syncthreads();
        for (int jj = 0; jj < cnt; ++jj) lj_pair(a, il, jt + jj, xi - sx[jj], yi - sy[jj], zi - sz[jj], fx, fy, fz);
    }
    if (i < total) {
        out[3 * i] = fx;
        out[3 * i + 1] = fy;
        out[3 * i + 2] = fz;
    }
}

// ---------------------------------------------------------------------------------------
// advance_state + reorthonormalize
// ---------------------------------------------------------------------------------------
__global__ void __launch_bounds__(256)
advance_kernel(const double* __restrict__ state, const double* __restrict__ u, const double* __restrict__ w,
               double dt, double max_disp, int64_t total, double* __restrict__ out, unsigned* __restrict__ flags) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= total) return;
    const unsigned f = advance_node(state + 12 * i, u + 3 * i, w + 3 * i, dt, max_disp, out + 12 * i);
    if (f) atomicOr(flags, f);
}

// ---------------------------------------------------------------------------------------
// batched sqrt_rotation: 256 matrices per CTA staged through smem with 16-byte vector
// loads/stores (AoS 72 B records are not 16-B aligned per thread).
// ---------------------------------------------------------------------------------------
constexpr int kSqrtBlock = 256;
__global__ void __launch_bounds__(kSqrtBlock)
sqrt_batched_kernel(const double* __restrict__ r9, int64_t count, double* __restrict__ s9) {
    __shared__ double2 buf[kSqrtBlock * 9 / 2];
    double* b = reinterpret_cast<double*>(buf);
    const int64_t base = (int64_t)blockIdx.x * kSqrtBlock;
    const int64_t nmat = (count - base) < kSqrtBlock ? (count - base) : kSqrtBlock;
    const int64_t nd = nmat * 9;
    const double2* in2 = reinterpret_cast<const double2*>(r9 + base * 9);  // base*9*8 is 16-B aligned (base even)
    for (int64_t k = threadIdx.x; k < nd / 2; k += kSqrtBlock) buf[k] = __ldcs(in2 + k);
    if ((nd & 1) && threadIdx.x == 0) b[nd - 1] = r9[base * 9 + nd - 1];
    __syncthreads();
    if (threadIdx.x < nmat) {
        m33 r;
#pragma unroll
        for (int e = 0; e < 9; ++e) r.m[e] = b[9 * threadIdx.x + e];
        const m33 s = sqrt_rotation(r);
#pragma unroll
        for (int e = 0; e < 9; ++e) b[9 * threadIdx.x + e] = s.m[e];
    }
    __syncthreads();
    double2* out2 = reinterpret_cast<double2*>(s9 + base * 9);
    for (int64_t k = threadIdx.x; k < nd / 2; k += kSqrtBlock) __stcs(out2 + k, buf[k]);
    if ((nd & 1) && threadIdx.x == 0) s9[base * 9 + nd - 1] = b[nd - 1];
}

// ---------------------------------------------------------------------------------------
// rod_position_metric: max over nodes of |x_i - y_i| / |x_i| (abs where |x_i| < 1e-14),
// io.cpp:49-68.  Max is exact and order free, so an atomicMax on the bit pattern of the
// non-negative result is deterministic.
// ---------------------------------------------------------------------------------------
__global__ void metric_kernel(const double* __restrict__ x, const double* __restrict__ y, int64_t nodes,
                              unsigned long long* __restrict__ result) {
    double worst = 0.0;
    for (int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; k < nodes; k += (int64_t)gridDim.x * blockDim.x) {
        const double* a = x + 12 * k;
        const double* c = y + 12 * k;
        double num = 0.0, den = 0.0;
#pragma unroll
        for (int q = 0; q < 3; ++q) {
            const double d = a[q] - c[q];
            num += d * d;
            den += a[q] * a[q];
        }
        num = sqrt(num);
        den = sqrt(den);
        const double v = den < 1e-14 ? num : num / den;
        worst = worst < v ? v : worst;
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        const double other = __shfl_xor_sync(0xffffffffu, worst, o);
        worst = worst < other ? other : worst;
    }
    if ((threadIdx.x & 31) == 0) atomicMax(result, (unsigned long long)__double_as_longlong(worst));
}

__global__ void correct_kernel(const double* __restrict__ xp, const double* __restrict__ gn,
                               const double* __restrict__ go, int64_t len, double* __restrict__ out) {
    for (int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; k < len; k += (int64_t)gridDim.x * blockDim.x) {
        out[k] = (xp[k] + gn[k]) - go[k];  // parareal.cpp:52
    }
}

// FP64 pipe microbenchmark: 8 independent DFMA chains per thread.
__global__ void __launch_bounds__(256) dfma_kernel(double* sink, int iters) {
    double a0 = threadIdx.x * 1e-9, a1 = a0 + 1e-3, a2 = a0 + 2e-3, a3 = a0 + 3e-3;
    double a4 = a0 + 4e-3, a5 = a0 + 5e-3, a6 = a0 + 6e-3, a7 = a0 + 7e-3;
    const double b = 0.999999999, c = 1e-12;
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int r = 0; r < 16; ++r) {
            a0 = fma(a0, b, c); a1 = fma(a1, b, c); a2 = fma(a2, b, c); a3 = fma(a3, b, c);
            a4 = fma(a4, b, c); a5 = fma(a5, b, c); a6 = fma(a6, b, c); a7 = fma(a7, b, c);
        }
    }
    const double s = ((a0 + a1) + (a2 + a3)) + ((a4 + a5) + (a6 + a7));
    if (s == 12345.678) sink[0] = s;
}

inline unsigned grid_for(int64_t n, int block) { return (unsigned)((n + block - 1) / block); }

}  // namespace

cudaError_t rod_loads_launch(const RodParams& p, const double* state, double t, double* pos, double* f, double* n,
                             double* seg_f, double* seg_n, const double* lj, const double* extra_f,
                             const double* extra_n, unsigned* flags, cudaStream_t st) {
    const RodArgs a = rod_args(p);
    const size_t smem = sizeof(double) * (size_t)(12 * p.m + 6 * (p.m - 1));
    static bool configured = false;
    if (!configured) {
        cudaFuncSetAttribute(rod_loads_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
        configured = true;
    }
    rod_loads_kernel<<<(unsigned)p.rods, 256, smem, st>>>(a, state, t, pos, f, n, seg_f, seg_n, lj, extra_f, extra_n,
                                                         flags);
    return cudaGetLastError();
}

cudaError_t lj_launch(const RodParams& p, const double* state, double* forces, cudaStream_t st) {
    const int64_t total = p.rods * p.m;
    lj_kernel<<<grid_for(total, 256), 256, 0, st>>>(state, lj_args(p), forces);
    return cudaGetLastError();
}

cudaError_t advance_launch(const RodParams& p, const double* state, const double* u, const double* w, double dt,
                           double* out, unsigned* flags, cudaStream_t st) {
    const int64_t total = p.rods * p.m;
    advance_kernel<<<grid_for(total, 256), 256, 0, st>>>(state, u, w, dt, 10.0 * p.ds, total, out, flags);
    return cudaGetLastError();
}

cudaError_t sqrt_batched_launch(const double* r9, int64_t count, double* s9, cudaStream_t st) {
    if (count == 0) return cudaSuccess;
    sqrt_batched_kernel<<<grid_for(count, kSqrtBlock), kSqrtBlock, 0, st>>>(r9, count, s9);
    return cudaGetLastError();
}

cudaError_t metric_launch(const double* x, const double* y, int64_t len, double*, int*, double* d_result,
                          cudaStream_t st) {
    cudaError_t e = cudaMemsetAsync(d_result, 0, sizeof(double), st);
    if (e != cudaSuccess) return e;
    const int64_t nodes = len / 12;
    const unsigned blocks = (unsigned)std::min<int64_t>(grid_for(nodes, 256), 1184);
    metric_kernel<<<blocks > 0 ? blocks : 1, 256, 0, st>>>(x, y, nodes, reinterpret_cast<unsigned long long*>(d_result));
    return cudaGetLastError();
}

cudaError_t correct_launch(const double* xp, const double* gn, const double* go, int64_t len, double* out,
                           cudaStream_t st) {
    const unsigned blocks = (unsigned)std::min<int64_t>(grid_for(len, 256), 148 * 16);
    correct_kernel<<<blocks > 0 ? blocks : 1, 256, 0, st>>>(xp, gn, go, len, out);
    return cudaGetLastError();
}

cudaError_t dfma_launch(double* sink, int blocks, int iters, cudaStream_t st) {
    dfma_kernel<<<blocks, 256, 0, st>>>(sink, iters);
    return cudaGetLastError();
}

}  // namespace pswim
