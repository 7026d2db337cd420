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

#include "dev_math.cuh"
#include "internal.h"

namespace pswim {
namespace {

// ---------------------------------------------------------------------------------------
// internal_loads + nodal_loads
// ---------------------------------------------------------------------------------------
struct RodArgs {
    int64_t m;
    double inv_ds, ds;
    double a0, a1, a2, b0, b1, b2;
    double amp, freq, wavenumber;
};

__global__ void __launch_bounds__(256)
rod_loads_kernel(RodArgs p, const double* __restrict__ state, double t, double* __restrict__ pos,
                 double* __restrict__ fo, double* __restrict__ no, double* __restrict__ seg_f,
                 double* __restrict__ seg_n, const double* __restrict__ lj, const double* __restrict__ extra_f,
                 const double* __restrict__ extra_n, unsigned* __restrict__ flags) {
    extern __shared__ double sh[];
    const int64_t m = p.m;
    double* xs = sh;           // m x 12 packed rod state
    double* seg = sh + 12 * m; // (m-1) x 6: F, N per segment
    const int64_t rod = blockIdx.x;
    const double* src = state + 12 * m * rod;
    for (int64_t k = threadIdx.x; k < 12 * m; k += blockDim.x) xs[k] = src[k];
    __syncthreads();

    const double bmod[3] = {p.b0, p.b1, p.b2};
    const double amod[3] = {p.a0, p.a1, p.a2};
    for (int64_t k = threadIdx.x; k + 1 < m; k += blockDim.x) {
        const double* lo_p = xs + 12 * k;
        const double* hi_p = xs + 12 * (k + 1);
        const d3 dx = ld3(hi_p) - ld3(lo_p);
        if (dot(dx, dx) == 0.0) atomicOr(flags, kFlagDegenerate);  // rod.cpp:53-55
        const d3 tangent = dx * p.inv_ds;
        const d3 lo[3] = {ld3(lo_p + 3), ld3(lo_p + 6), ld3(lo_p + 9)};
        const d3 hi[3] = {ld3(hi_p + 3), ld3(hi_p + 6), ld3(hi_p + 9)};
        // A_k = sum_j hi_j lo_j^T  (rod.cpp:61-63)
        m33 a;
#pragma unroll
        for (int r = 0; r < 3; ++r)
#pragma unroll
            for (int c = 0; c < 3; ++c)
                a.m[3 * r + c] = at(hi[0], r) * at(lo[0], c) + at(hi[1], r) * at(lo[1], c) + at(hi[2], r) * at(lo[2], c);
        const m33 half = sqrt_rotation(a);
        const d3 mid[3] = {mv(half, lo[0]), mv(half, lo[1]), mv(half, lo[2])};
        // preferred_strain((k+1/2) ds, t): (0, -k^2 A sin(k s + f t), 0)  (rod.cpp:29-32)
        const double s_mid = ((double)k + 0.5) * p.ds;
        const double om1 = -p.wavenumber * p.wavenumber * p.amp * sin(p.wavenumber * s_mid + p.freq * t);
        const double om[3] = {0.0, om1, 0.0};
        d3 F = mk3(0, 0, 0), N = mk3(0, 0, 0);
#pragma unroll
        for (int i = 0; i < 3; ++i) {
            const int j = (i + 1) % 3;
            const int kk = (i + 2) % 3;
            const double stretch = dot(tangent, mid[i]) - (i == 2 ? 1.0 : 0.0);
            const double bend = dot((hi[j] - lo[j]) * p.inv_ds, mid[kk]) - om[i];
            F = F + mid[i] * (bmod[i] * stretch);
            N = N + mid[i] * (amod[i] * bend);
        }
        st3(seg + 6 * k, F);
        st3(seg + 6 * k + 3, N);
        if (seg_f) {
            const int64_t g = (m - 1) * rod + k;
            st3(seg_f + 3 * g, F);
            st3(seg_n + 3 * g, N);
        }
    }
    __syncthreads();
    for (int64_t k = threadIdx.x; k < m; k += blockDim.x) {
        // nodal_loads, rod.cpp:93-106 (free ends: ghost segment loads vanish)
        const d3 zero = mk3(0, 0, 0);
        const d3 f_plus = k < m - 1 ? ld3(seg + 6 * k) : zero;
        const d3 f_minus = k > 0 ? ld3(seg + 6 * (k - 1)) : zero;
        const d3 n_plus = k < m - 1 ? ld3(seg + 6 * k + 3) : zero;
        const d3 n_minus = k > 0 ? ld3(seg + 6 * (k - 1) + 3) : zero;
        const d3 xk = ld3(xs + 12 * k);
        d3 f = (f_plus - f_minus) * p.inv_ds;
        d3 tq = (n_plus - n_minus) * p.inv_ds;
        if (k < m - 1) tq = tq + cross((ld3(xs + 12 * (k + 1)) - xk) * p.inv_ds, f_plus) * 0.5;
        if (k > 0) tq = tq + cross((xk - ld3(xs + 12 * (k - 1))) * p.inv_ds, f_minus) * 0.5;
        const int64_t g = m * rod + k;
        if (lj) f = f + ld3(lj + 3 * g) * p.inv_ds;  // propagators.cpp:70-74
        if (extra_f) {                              // propagators.cpp:75-84
            f = f + ld3(extra_f + 3 * g);
            tq = tq + ld3(extra_n + 3 * g);
        }
        st3(pos + 3 * g, xk);
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
lj_kernel(const double* __restrict__ state, int64_t rods, int64_t m, double well, double sigma, double rc2,
          double r_min, double cap, int64_t excl, double* __restrict__ out) {
    __shared__ double sx[kLjTile], sy[kLjTile], sz[kLjTile];
    const int64_t total = rods * m;
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    const int64_t il = i < total ? i : total - 1;
    const double xi = state[12 * il], yi = state[12 * il + 1], zi = state[12 * il + 2];
    const int64_t ri = il / m, ki = il % m;
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
        for (int jj = 0; jj < cnt; ++jj) {
            const double dx = xi - sx[jj], dy = yi - sy[jj], dz = zi - sz[jj];
            const double r2 = dx * dx + dy * dy + dz * dz;
            if (r2 >= rc2) continue;
            const int64_t j = jt + jj;
            if (rods < 2) continue;
            const int64_t rj = j / m, kj = j % m;
            if (rj == ri) {
                const int64_t dk = kj > ki ? kj - ki : ki - kj;
                if (dk < excl) continue;
            }
            const double r = sqrt(r2);
            double s;
            if (r < r_min) {
                if (r > 0.0) {
                    s = cap / r;
                } else {
                    // dir = (1,0,0) for the force on the first node of the pair; the
                    // partner receives the opposite (rod.cpp:162-166)
                    const bool first = (ri < rj) || (ri == rj && ki < kj);
                    fx += first ? cap : -cap;
                    continue;
                }
            } else {
                const double sr2 = (sigma * sigma) / (r * r);
                const double sr6 = sr2 * sr2 * sr2;
                s = 24.0 * well * (2.0 * sr6 * sr6 - sr6) / (r * r);
            }
            fx += s * dx;
            fy += s * dy;
            fz += s * dz;
        }
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
    const double* s = state + 12 * i;
    d3 x = ld3(s), d1 = ld3(s + 3), d2 = ld3(s + 6), d3v = ld3(s + 9);
    const d3 du = ld3(u + 3 * i) * dt;
    if (norm(du) > max_disp) atomicOr(flags, kFlagStiff);  // propagators.cpp:105-109
    x = x + du;
    const d3 wv = ld3(w + 3 * i);
    const double speed = norm(wv);
    if (speed > 0.0) {
        d3 n = divs(wv, speed);
        if (!unit_axis(n)) atomicOr(flags, kFlagAxis);
        double sn, cs;
        sincos(speed * dt, &sn, &cs);
        const m33 q = rodrigues_cs(n, cs, sn);
        d1 = mv(q, d1);
        d2 = mv(q, d2);
        d3v = mv(q, d3v);
    }
    // reorthonormalize(tol = 1e-9), rod.cpp:176-195: ||D^T D - I||_F over the triad
    const double g00 = dot(d1, d1) - 1.0, g11 = dot(d2, d2) - 1.0, g22 = dot(d3v, d3v) - 1.0;
    const double g01 = dot(d1, d2), g02 = dot(d1, d3v), g12 = dot(d2, d3v);
    const double fro = sqrt(g00 * g00 + g11 * g11 + g22 * g22 + 2.0 * (g01 * g01 + g02 * g02 + g12 * g12));
    if (fro > 1e-9) {
        const d3 t3 = divs(d3v, norm(d3v));
        d3 t1 = d1 - t3 * dot(d1, t3);
        t1 = divs(t1, norm(t1));
        d3v = t3;
        d1 = t1;
        d2 = cross(t3, t1);
    }
    double* o = out + 12 * i;
    st3(o, x);
    st3(o + 3, d1);
    st3(o + 6, d2);
    st3(o + 9, d3v);
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
    RodArgs a;
    a.m = p.m;
    a.ds = p.ds;
    a.inv_ds = p.inv_ds;
    a.a0 = p.a[0]; a.a1 = p.a[1]; a.a2 = p.a[2];
    a.b0 = p.b[0]; a.b1 = p.b[1]; a.b2 = p.b[2];
    a.amp = p.amplitude;
    a.freq = p.frequency;
    a.wavenumber = 2.0 * M_PI / p.wavelength;  // WaveformParams::wavenumber, rod.cpp:27
    const size_t smem = sizeof(double) * (size_t)(12 * p.m + 6 * (p.m - 1));
    static bool configured = false;
    if (!configured || smem > 48 * 1024) {
        cudaFuncSetAttribute(rod_loads_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
        configured = true;
    }
    rod_loads_kernel<<<(unsigned)p.rods, 256, smem, st>>>(a, state, t, pos, f, n, seg_f, seg_n, lj, extra_f, extra_n,
                                                         flags);
    return cudaGetLastError();
}

cudaError_t lj_launch(const RodParams& p, const double* state, double* forces, cudaStream_t st) {
    const int64_t total = p.rods * p.m;
    const double rc = p.lj_cutoff;
    const double r_min = 1e-3 * p.lj_sigma;
    // cap = lj_force_over_r(r_min) * r_min  (rod.cpp:137)
    const double sr2 = (p.lj_sigma * p.lj_sigma) / (r_min * r_min);
    const double sr6 = sr2 * sr2 * sr2;
    const double cap = 24.0 * p.lj_well * (2.0 * sr6 * sr6 - sr6) / (r_min * r_min) * r_min;
    const int64_t excl = p.lj_excl > 4 ? p.lj_excl : 4;
    lj_kernel<<<grid_for(total, 256), 256, 0, st>>>(state, p.rods, p.m, p.lj_well, p.lj_sigma, rc * rc, r_min, cap,
                                                    excl, forces);
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
