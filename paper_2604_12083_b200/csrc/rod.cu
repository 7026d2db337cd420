// rod.cu — rod mechanics, triad update and the small elementwise kernels of the path.
//
//   rod_loads_wtma_kernel  internal_loads + nodal_loads (reference src/rod.cpp:36-109):
//                     warp-tiled over the flat node sequence, per-warp TMA-bulk ring, no
//                     CTA barriers; device sqrt_rotation (dev_math.cuh); LJ/extra loads
//                     folded in as rhs does (src/propagators.cpp:59-84).
//   rod_loads_kernel  the same, one CTA per rod (segment-load outputs, unaligned state).
//   lj_kernel         lj_repulsion (src/rod.cpp:124-174) as a per-node all-pairs sum.
//   advance_kernel    advance_state (src/propagators.cpp:93-124) + reorthonormalize
//                     (src/rod.cpp:176-195), one thread per node.
//   sqrt_tma_kernel   sqrt_rotation over a batch (rotation.cpp:91-107), CTA-chunk TMA pipeline
//   sqrt_wtma_kernel  the same with per-warp TMA rings (PSWIM_SQRT_WARP=1).
//   metric / correct  rod_position_metric (io.cpp:49-68), corrected (parareal.cpp:47-54).
#include <algorithm>
#include <cmath>
#include <cstdlib>
#include <mutex>
#include <vector>

#include "kernels.cuh"
#include "tma.cuh"

namespace pswim {
namespace {

// ---------------------------------------------------------------------------------------
// internal_loads + nodal_loads
// ---------------------------------------------------------------------------------------
__global__ void __launch_bounds__(256)
rod_loads_kernel(RodArgs p, const double* __restrict__ state, double t0, const double* __restrict__ tdev,
                 double* __restrict__ pos,
                 double* __restrict__ fo, double* __restrict__ no, double* __restrict__ seg_f,
                 double* __restrict__ seg_n, const double* __restrict__ lj, const double* __restrict__ extra_f,
                 const double* __restrict__ extra_n, unsigned* __restrict__ flags) {
    extern __shared__ double sh[];
    const double t = tdev ? *tdev : t0;  // time from device memory inside CUDA graphs
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
        if (pos) st3(pos + 3 * g, ld3(xs + 12 * k));
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
    __shared__ int srod[kLjTile], sk[kLjTile];
    const int total = a.rods * a.m;
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    const int il = i < total ? i : total - 1;
    const int ri = il / a.m, ki = il - ri * a.m;
    const double xi = state[12 * (int64_t)il], yi = state[12 * (int64_t)il + 1], zi = state[12 * (int64_t)il + 2];
    double fx = 0, fy = 0, fz = 0;
    for (int jt = 0; jt < total; jt += kLjTile) {
        const int cnt = (total - jt) < kLjTile ? total - jt : kLjTile;
        __syncthreads();
        if (threadIdx.x < cnt) {
            const int j = jt + threadIdx.x;
            sx[threadIdx.x] = state[12 * (int64_t)j];
            sy[threadIdx.x] = state[12 * (int64_t)j + 1];
            sz[threadIdx.x] = state[12 * (int64_t)j + 2];
            srod[threadIdx.x] = j / a.m;
            sk[threadIdx.x] = j - (j / a.m) * a.m;
        }
        __syncthreads();
        for (int jj = 0; jj < cnt; ++jj)
            lj_pair(a, ri, ki, srod[jj], sk[jj], xi - sx[jj], yi - sy[jj], zi - sz[jj], fx, fy, fz);
    }
    if (i < total) {
        out[3 * (int64_t)i] = fx;
        out[3 * (int64_t)i + 1] = fy;
        out[3 * (int64_t)i + 2] = fz;
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
// advance_state, persistent TMA-bulk pipeline: 256-node chunks of (state, u, w) stream in
// with cp.async.bulk (2-stage ring, 36 KiB per stage), each thread advances its node in
// place in shared memory, the new states leave with one bulk store per chunk.
// ---------------------------------------------------------------------------------------
constexpr int kAdvBlock = 256;
constexpr int kAdvStages = 2;
constexpr uint32_t kAdvStateBytes = kAdvBlock * 12 * sizeof(double);
constexpr uint32_t kAdvVelBytes = kAdvBlock * 3 * sizeof(double);
constexpr uint32_t kAdvStageBytes = kAdvStateBytes + 2 * kAdvVelBytes;

__global__ void __launch_bounds__(kAdvBlock, 3)
advance_tma_kernel(const double* __restrict__ state, const double* __restrict__ u, const double* __restrict__ w,
                   double dt, double max_disp, int64_t total, double* __restrict__ out,
                   unsigned* __restrict__ flags) {
    extern __shared__ __align__(128) unsigned char smem[];
    uint64_t* full = reinterpret_cast<uint64_t*>(smem + kAdvStages * kAdvStageBytes);
    const int64_t nchunks = (total + kAdvBlock - 1) / kAdvBlock;
    const int64_t nfull = total / kAdvBlock;
    auto st_of = [&](int s) { return reinterpret_cast<double*>(smem + s * kAdvStageBytes); };
    auto issue = [&](int s, int64_t c) {
        double* b = st_of(s);
        mbar_expect_tx(&full[s], kAdvStageBytes);
        bulk_load(b, state + 12 * kAdvBlock * c, kAdvStateBytes, &full[s]);
        bulk_load(b + 12 * kAdvBlock, u + 3 * kAdvBlock * c, kAdvVelBytes, &full[s]);
        bulk_load(b + 15 * kAdvBlock, w + 3 * kAdvBlock * c, kAdvVelBytes, &full[s]);
    };
    if (threadIdx.x == 0) {
        for (int s = 0; s < kAdvStages; ++s) mbar_init(&full[s], 1);
        fence_mbar_init();
    }
    __syncthreads();
    if (threadIdx.x == 0)
        for (int s = 0; s < kAdvStages; ++s) {
            const int64_t c = blockIdx.x + (int64_t)s * gridDim.x;
            if (c < nfull) issue(s, c);
        }
    unsigned fl = 0;
    for (int64_t k = 0;; ++k) {
        const int64_t c = blockIdx.x + k * gridDim.x;
        if (c >= nchunks) break;
        const int s = (int)(k % kAdvStages);
        double* b = st_of(s);
        if (c < nfull) {
            mbar_wait(&full[s], (uint32_t)((k / kAdvStages) & 1));
            const int i = threadIdx.x;
            fl |= advance_node(b + 12 * i, b + 12 * kAdvBlock + 3 * i, b + 15 * kAdvBlock + 3 * i, dt, max_disp,
                               b + 12 * i);
            fence_proxy_async_smem();
            __syncthreads();
            if (threadIdx.x == 0) {
                bulk_store(out + 12 * kAdvBlock * c, b, kAdvStateBytes);
                bulk_commit();
                const int64_t cn = blockIdx.x + (k + kAdvStages) * gridDim.x;
                if (cn < nfull) {
                    bulk_wait_read<0>();
                    issue(s, cn);
                }
            }
        } else {
            const int64_t i = c * kAdvBlock + threadIdx.x;
            if (i < total) fl |= advance_node(state + 12 * i, u + 3 * i, w + 3 * i, dt, max_disp, out + 12 * i);
        }
    }
    if (fl) atomicOr(flags, fl);
    if (threadIdx.x == 0) bulk_wait<0>();
}

// ---------------------------------------------------------------------------------------
// internal + nodal loads, warp-tiled and barrier-free: the nodes form one flat sequence
// (rods concatenated); warp w owns nodes [31 w, 31 w + 31) and computes the 32 segments
// whose lower node is 31 w - 1 + lane (lane 0's segment is the previous warp's last, computed
// again).  A node's two segment loads and its predecessor's position then sit in lanes
// lane - 1 and lane, one shuffle apart, so no CTA barrier separates the segment and node
// phases and every warp streams independently.  Same arithmetic as rod_segment / rod_node
// (bitwise identical outputs).  Measured (B200, 40000 x 256 nodes): 5.3 TB/s = 0.81 of
// the HBM copy peak, against 2.7 TB/s for a one-rod-per-CTA pipeline whose segment and
// node phases are separated by CTA barriers.
// ---------------------------------------------------------------------------------------
constexpr int kWarpNodes = 31;

// Node data stream global -> shared by per-warp TMA bulk copies (cp.async.bulk + one mbarrier
// per stage, a kStages ring per warp): each warp tile is 33 consecutive nodes (3168 B),
// issued kStages tiles ahead by the warp's lane 0, so the HBM stream runs under the FP64
// segment chains without any CTA-wide barrier.  The preferred strain depends on (k, t) only
// and is tabulated once per CTA in shared memory.
constexpr int kTileNodes = kWarpNodes + 2;
constexpr int kRodStages = 2;
constexpr uint32_t kTileBytes = kTileNodes * 96;

template <int kStages>
__global__ void __launch_bounds__(256, 2)
rod_loads_wtma_kernel(RodArgs p, int total, const double* __restrict__ state, double t0,
                      const double* __restrict__ tdev, double* __restrict__ pos,
                      double* __restrict__ fo, double* __restrict__ no, const double* __restrict__ lj,
                      const double* __restrict__ extra_f, const double* __restrict__ extra_n,
                      unsigned* __restrict__ flags) {
    // 32-bit node indices (the launcher routes N >= 2^31 / 12 elsewhere)
    extern __shared__ __align__(128) unsigned char smem[];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int warps = blockDim.x >> 5;
    double* ring = reinterpret_cast<double*>(smem) + warp * kStages * kTileNodes * 12;
    uint64_t* bars = reinterpret_cast<uint64_t*>(smem + warps * kStages * kTileBytes) + warp * kStages;
    double* strain = reinterpret_cast<double*>(smem + warps * kStages * (kTileBytes + 8));  // m - 1 entries
    const int m = (int)p.m;
    const double t = tdev ? *tdev : t0;  // time from device memory inside CUDA graphs
    for (int k = threadIdx.x; k + 1 < m; k += blockDim.x) strain[k] = rod_strain(p, k, t);
    const int wstride = gridDim.x * warps;
    const int w0 = blockIdx.x * warps + warp;
    const int ntiles = (total + kWarpNodes - 1) / kWarpNodes;
    auto issue = [&](int w, int s) {
        // nodes [31 w - 1, 31 w + 32) clipped to [0, total); tile slot 0 holds node 31 w - 1
        const int a = w * kWarpNodes - 1 < 0 ? 0 : w * kWarpNodes - 1;
        const int b = w * kWarpNodes + kWarpNodes + 1 < total ? w * kWarpNodes + kWarpNodes + 1 : total;
        const uint32_t bytes = (uint32_t)((b - a) * 96);
        double* dst = ring + s * kTileNodes * 12 + 12 * (a - (w * kWarpNodes - 1));
        mbar_expect_tx(&bars[s], bytes);
        bulk_load(dst, state + 12 * (int64_t)a, bytes, &bars[s]);
    };
    if (lane == 0) {
        for (int s = 0; s < kStages; ++s) mbar_init(&bars[s], 1);
        fence_mbar_init();
        for (int s = 0; s < kStages; ++s) {
            const int w = w0 + s * wstride;
            if (w < ntiles) issue(w, s);
        }
    }
    __syncthreads();  // strain table (and this warp's mbarrier init)
    unsigned fl = 0;
    int i = 0;
    for (int w = w0; w < ntiles; w += wstride, ++i) {
        const int s = i % kStages;
        mbar_wait(&bars[s], (uint32_t)((i / kStages) & 1));
        const int base = w * kWarpNodes - 1;  // node of tile slot 0
        const double* tile = ring + s * kTileNodes * 12;
        const int g = base + lane;
        const bool valid = g >= 0 && g < total;
        const int rod = valid ? (int)((unsigned)g / (unsigned)m) : 0;
        const int k = valid ? g - rod * m : 0;
        const double* xs = tile + 12 * (rod * m - base);  // rod's node 0 in tile coordinates
        double seg[6] = {0.0, 0.0, 0.0, 0.0, 0.0, 0.0};
        if (valid && k + 1 < m)
            if (!rod_segment_om(p, xs, k, strain[k], seg)) fl |= kFlagDegenerate;  // rod.cpp:53-55
        const d3 xk = valid ? ld3(xs + 12 * k) : mk3(0, 0, 0);
        const d3 xnext = (valid && k + 1 < m) ? ld3(xs + 12 * (k + 1)) : mk3(0, 0, 0);
        double prev[6];
#pragma unroll
        for (int q = 0; q < 6; ++q) prev[q] = __shfl_up_sync(0xffffffffu, seg[q], 1);
        d3 xprev;
        xprev.x = __shfl_up_sync(0xffffffffu, xk.x, 1);
        xprev.y = __shfl_up_sync(0xffffffffu, xk.y, 1);
        xprev.z = __shfl_up_sync(0xffffffffu, xk.z, 1);
        __syncwarp();  // every lane is done with the stage
        if (lane == 0) {
            const int wn = w + kStages * wstride;
            if (wn < ntiles) issue(wn, s);
        }
        if (lane != 0 && valid) {
            d3 f, tq;
            node_loads(p, k, seg, prev, xprev, xk, xnext, f, tq);  // nodal_loads, rod.cpp:93-106
            const int64_t g3 = 3 * (int64_t)g;
            if (lj) f = f + ld3(lj + g3) * p.inv_ds;  // propagators.cpp:70-74
            if (extra_f) {                           // propagators.cpp:75-84
                f = f + ld3(extra_f + g3);
                tq = tq + ld3(extra_n + g3);
            }
            if (pos) st3(pos + g3, xk);
            st3(fo + g3, f);
            st3(no + g3, tq);
        }
    }
    if (fl) atomicOr(flags, fl);
}

// ---------------------------------------------------------------------------------------
// batched sqrt_rotation (rotation.cpp:91-107 over a batch of row-major matrices)
// ---------------------------------------------------------------------------------------
constexpr int kSqrtBlock = 256;

// Each warp streams chunks of 32 matrices (2304 B) through its own
// kSqrtWarpStages-deep TMA ring (one mbarrier per stage, issued by lane 0), computes one
// matrix per lane in place, and stores the chunk back with one bulk copy.  No CTA barrier:
// a lane only touches its own 72 bytes until the warp-level fence + __syncwarp before the
// store.  A stage is refilled one iteration after its store was issued
// (cp.async.bulk.wait_group.read 1), so lane 0 never waits for the store it just issued.
constexpr int kSqrtWarpStages = 4;
constexpr uint32_t kSqrtWarpChunkBytes = 32 * 9 * sizeof(double);

__global__ void __launch_bounds__(256, 3)
sqrt_wtma_kernel(const double* __restrict__ r9, int64_t nwchunks, double* __restrict__ s9) {
    extern __shared__ __align__(128) unsigned char smem[];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, warps = blockDim.x >> 5;
    double* ring = reinterpret_cast<double*>(smem) + (size_t)warp * kSqrtWarpStages * 32 * 9;
    uint64_t* bars = reinterpret_cast<uint64_t*>(smem + (size_t)warps * kSqrtWarpStages * kSqrtWarpChunkBytes) +
                     warp * kSqrtWarpStages;
    const int64_t wstride = (int64_t)gridDim.x * warps, w0 = (int64_t)blockIdx.x * warps + warp;
    if (lane == 0) {
        for (int s = 0; s < kSqrtWarpStages; ++s) mbar_init(&bars[s], 1);
        fence_mbar_init();
        for (int s = 0; s < kSqrtWarpStages; ++s) {
            const int64_t c = w0 + s * wstride;
            if (c < nwchunks) {
                mbar_expect_tx(&bars[s], kSqrtWarpChunkBytes);
                bulk_load(ring + s * 32 * 9, r9 + 9 * 32 * c, kSqrtWarpChunkBytes, &bars[s]);
            }
        }
    }
    __syncwarp();
    int i = 0;
    for (int64_t c = w0; c < nwchunks; c += wstride, ++i) {
        const int s = i % kSqrtWarpStages;
        double* b = ring + s * 32 * 9;
        mbar_wait(&bars[s], (uint32_t)((i / kSqrtWarpStages) & 1));
        m33 r;
#pragma unroll
        for (int e = 0; e < 9; ++e) r.m[e] = b[9 * lane + e];
        const m33 q = sqrt_rotation(r);
#pragma unroll
        for (int e = 0; e < 9; ++e) b[9 * lane + e] = q.m[e];
        fence_proxy_async_smem();
        __syncwarp();
        if (lane == 0) {
            bulk_store(s9 + 9 * 32 * c, b, kSqrtWarpChunkBytes);
            bulk_commit();
            if (i > 0) {
                // refill the previous iteration's stage once its store has left shared memory
                const int sp = (i - 1) % kSqrtWarpStages;
                const int64_t cn = c - wstride + kSqrtWarpStages * wstride;
                if (cn < nwchunks) {
                    bulk_wait_read<1>();
                    mbar_expect_tx(&bars[sp], kSqrtWarpChunkBytes);
                    bulk_load(ring + sp * 32 * 9, r9 + 9 * 32 * cn, kSqrtWarpChunkBytes, &bars[sp]);
                }
            }
        }
    }
    if (lane == 0) bulk_wait<0>();
}

// CTA-chunk variant (the advance_tma_kernel pipeline): 256-matrix chunks (18 KiB) stream in
// through a kSqrtCtaStages-deep ring of whole-CTA bulk copies, each thread takes one matrix in
// place, the chunk leaves with one bulk store; thread 0 refills a stage once its store has
// read shared memory.  Fewer, larger TMA transfers than the per-warp rings.
constexpr int kSqrtCtaStages = 3;
constexpr uint32_t kSqrtCtaChunkBytes = 256 * 9 * sizeof(double);

template <int kStages, int kMpt>
__global__ void __launch_bounds__(256, 4 / kMpt)
sqrt_tma_kernel(const double* __restrict__ r9, int64_t nchunks, double* __restrict__ s9) {
    // kMpt matrices per thread: chunks of 256 kMpt matrices
    constexpr uint32_t kBytes = kMpt * kSqrtCtaChunkBytes;
    constexpr int kMat = 256 * kMpt;
    extern __shared__ __align__(128) unsigned char smem[];
    uint64_t* full = reinterpret_cast<uint64_t*>(smem + kStages * kBytes);
    auto st_of = [&](int s) { return reinterpret_cast<double*>(smem + s * kBytes); };
    auto issue = [&](int s, int64_t c) {
        mbar_expect_tx(&full[s], kBytes);
        bulk_load(st_of(s), r9 + 9 * kMat * c, kBytes, &full[s]);
    };
    if (threadIdx.x == 0) {
        for (int s = 0; s < kStages; ++s) mbar_init(&full[s], 1);
        fence_mbar_init();
        for (int s = 0; s < kStages; ++s) {
            const int64_t c = blockIdx.x + (int64_t)s * gridDim.x;
            if (c < nchunks) issue(s, c);
        }
    }
    __syncthreads();
    for (int64_t k = 0;; ++k) {
        const int64_t c = blockIdx.x + k * gridDim.x;
        if (c >= nchunks) break;
        const int s = (int)(k % kStages);
        double* b = st_of(s);
        mbar_wait(&full[s], (uint32_t)((k / kStages) & 1));
        m33 r[kMpt];
#pragma unroll
        for (int q = 0; q < kMpt; ++q)
#pragma unroll
            for (int e = 0; e < 9; ++e) r[q].m[e] = b[9 * (threadIdx.x + 256 * q) + e];
#pragma unroll
        for (int q = 0; q < kMpt; ++q) {
            const m33 o = sqrt_rotation(r[q]);
#pragma unroll
            for (int e = 0; e < 9; ++e) b[9 * (threadIdx.x + 256 * q) + e] = o.m[e];
        }
        fence_proxy_async_smem();
        __syncthreads();
        if (threadIdx.x == 0) {
            bulk_store(s9 + 9 * kMat * c, b, kBytes);
            bulk_commit();
            const int64_t cn = blockIdx.x + (k + kStages) * gridDim.x;
            if (cn < nchunks) {
                bulk_wait_read<0>();
                issue(s, cn);
            }
        }
    }
    if (threadIdx.x == 0) bulk_wait<0>();
}

__global__ void __launch_bounds__(kSqrtBlock)
sqrt_plain_kernel(const double* __restrict__ r9, int64_t count, double* __restrict__ s9) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= count) return;
    m33 r;
#pragma unroll
    for (int e = 0; e < 9; ++e) r.m[e] = r9[9 * i + e];
    const m33 s = sqrt_rotation(r);
#pragma unroll
    for (int e = 0; e < 9; ++e) s9[9 * i + e] = s.m[e];
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

// Position metric of many (x, y) state pairs in one launch (one Parareal iteration's
// eta_tilde and eta columns): pair p = blockIdx.y, same per-node arithmetic as metric_kernel.
__global__ void metric_pairs_kernel(const __grid_constant__ MetricPairs pairs, int64_t nodes,
                                    unsigned long long* __restrict__ result) {
    const double* x = pairs.x[blockIdx.y];
    const double* y = pairs.y[blockIdx.y];
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
    if ((threadIdx.x & 31) == 0) atomicMax(result + blockIdx.y, (unsigned long long)__double_as_longlong(worst));
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

// SM count of the current device (persistent grids; results never depend on it).
inline int num_sms() {
    static const int n = [] {
        int dev = 0, v = 148;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, dev);
        return v;
    }();
    return n;
}

// Resident CTAs per SM of a persistent kernel at a given dynamic shared memory size, queried
// once per (kernel, size) instead of on every launch: launch paths make no driver queries that
// take the context lock (see fused.cu configure_cs).
template <typename K>
int occupancy(K kernel, int block, size_t smem) {
    static std::mutex mu;
    static std::vector<std::pair<size_t, int>> cache;
    std::lock_guard<std::mutex> lock(mu);
    for (const auto& c : cache)
        if (c.first == smem) return c.second;
    int per_sm = 1;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kernel, block, smem);
    cache.emplace_back(smem, std::max(per_sm, 1));
    return cache.back().second;
}

}  // namespace

// (function attributes: set once in rod_preload, at context creation)
cudaError_t rod_loads_launch(const RodParams& p, const double* state, double t, double* pos, double* f, double* n,
                             double* seg_f, double* seg_n, const double* lj, const double* extra_f,
                             const double* extra_n, unsigned* flags, cudaStream_t st, const double* tdev) {
    const RodArgs a = rod_args(p);
    const size_t smem = sizeof(double) * (size_t)(12 * p.m + 6 * (p.m - 1));
    const size_t sm = 8 * (size_t)kRodStages * (kTileBytes + 8) + 8 * (size_t)std::max<int64_t>(p.m - 1, 1);
    const bool aligned = (reinterpret_cast<uintptr_t>(state) & 15) == 0;
    if (seg_f == nullptr && aligned && p.rods * p.m < ((int64_t)1 << 30) && sm <= 100 * 1024) {
        // warp-tiled TMA stream (persistent grid, 2 CTAs/SM)
        const int total = (int)(p.rods * p.m);
        const int tiles = (total + kWarpNodes - 1) / kWarpNodes;
        const int per_sm = occupancy(rod_loads_wtma_kernel<kRodStages>, 256, sm);
        const int grid = (int)std::min<int64_t>((tiles + 7) / 8, (int64_t)num_sms() * per_sm);
        rod_loads_wtma_kernel<kRodStages><<<(unsigned)grid, 256, sm, st>>>(a, total, state, t, tdev, pos, f, n, lj, extra_f,
                                                                           extra_n, flags);
        return cudaGetLastError();
    }
    // segment loads requested, unaligned state or very long rods: one CTA per rod
    rod_loads_kernel<<<(unsigned)p.rods, 256, smem, st>>>(a, state, t, tdev, pos, f, n, seg_f, seg_n, lj, extra_f, extra_n,
                                                         flags);
    return cudaGetLastError();
}

void preload_kernels(int device) {
    static std::mutex mu;
    static std::vector<int> done;
    std::lock_guard<std::mutex> lock(mu);
    if (std::find(done.begin(), done.end(), device) != done.end()) return;
    peer_preload();  // MRS + peer kernels, rod kernels
    lj_cells_preload();
    fused_preload();
    done.push_back(device);
}

cudaError_t lj_launch(const RodParams& p, const double* state, double* forces, cudaStream_t st) {
    const int64_t total = p.rods * p.m;
    lj_kernel<<<grid_for(total, 256), 256, 0, st>>>(state, lj_args(p), forces);
    return cudaGetLastError();
}

void rod_preload() {
    // see peer_preload (mrs.cu): load every per-step kernel before peers can spin, and set the
    // function attributes the launch paths would otherwise set on first use
    static const bool once = [] {
        cudaFuncSetAttribute(rod_loads_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
        cudaFuncSetAttribute(rod_loads_wtma_kernel<kRodStages>, cudaFuncAttributeMaxDynamicSharedMemorySize, 100 * 1024);
        cudaFuncSetAttribute(advance_tma_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             (int)(kAdvStages * kAdvStageBytes + kAdvStages * sizeof(uint64_t)));
        cudaFuncSetAttribute(sqrt_wtma_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             (int)(8 * (size_t)kSqrtWarpStages * (kSqrtWarpChunkBytes + sizeof(uint64_t))));
        cudaFuncSetAttribute(sqrt_tma_kernel<kSqrtCtaStages, 1>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             (int)(kSqrtCtaStages * (kSqrtCtaChunkBytes + sizeof(uint64_t))));
        return true;
    }();
    (void)once;
    cudaFuncAttributes a;
    cudaFuncGetAttributes(&a, rod_loads_kernel);
    cudaFuncGetAttributes(&a, rod_loads_wtma_kernel<kRodStages>);
    cudaFuncGetAttributes(&a, lj_kernel);
    cudaFuncGetAttributes(&a, sqrt_wtma_kernel);
    cudaFuncGetAttributes(&a, sqrt_tma_kernel<kSqrtCtaStages, 1>);
    cudaFuncGetAttributes(&a, sqrt_plain_kernel);
    cudaFuncGetAttributes(&a, metric_kernel);
    cudaFuncGetAttributes(&a, correct_kernel);
    cudaFuncGetAttributes(&a, metric_pairs_kernel);
    cudaFuncGetAttributes(&a, advance_kernel);
    cudaFuncGetAttributes(&a, advance_tma_kernel);
}

cudaError_t advance_launch(const RodParams& p, const double* state, const double* u, const double* w, double dt,
                           double* out, unsigned* flags, cudaStream_t st) {
    const int64_t total = p.rods * p.m;
    const bool aligned = ((reinterpret_cast<uintptr_t>(state) | reinterpret_cast<uintptr_t>(u) |
                           reinterpret_cast<uintptr_t>(w) | reinterpret_cast<uintptr_t>(out)) & 15) == 0;
    if (!aligned || total < 4 * kAdvBlock) {
        advance_kernel<<<grid_for(total, 256), 256, 0, st>>>(state, u, w, dt, 10.0 * p.ds, total, out, flags);
        return cudaGetLastError();
    }
    const size_t smem = kAdvStages * kAdvStageBytes + kAdvStages * sizeof(uint64_t);
    const int64_t nchunks = (total + kAdvBlock - 1) / kAdvBlock;
    const int per_sm = occupancy(advance_tma_kernel, kAdvBlock, smem);
    const int64_t grid = std::min<int64_t>(nchunks, (int64_t)num_sms() * per_sm);
    advance_tma_kernel<<<(unsigned)grid, kAdvBlock, smem, st>>>(state, u, w, dt, 10.0 * p.ds, total, out, flags);
    return cudaGetLastError();
}

cudaError_t sqrt_batched_launch(const double* r9, int64_t count, double* s9, cudaStream_t st) {
    if (count == 0) return cudaSuccess;
    const bool aligned = ((reinterpret_cast<uintptr_t>(r9) | reinterpret_cast<uintptr_t>(s9)) & 15) == 0;
    if (!aligned) {
        sqrt_plain_kernel<<<grid_for(count, kSqrtBlock), kSqrtBlock, 0, st>>>(r9, count, s9);
        return cudaGetLastError();
    }
    static const bool warp_rings = [] {
        const char* e = std::getenv("PSWIM_SQRT_WARP");  // dev knob: the per-warp-ring kernel
        return e && std::atoi(e) == 1;
    }();
    if (!warp_rings) {
        // CTA-chunk pipeline (default): 256-matrix chunks, 3 stages; measured 5.70-5.74 TB/s
        // against 5.56-5.62 for the per-warp rings (1e7 matrices; 2 / 4 stages and 2
        // matrices per thread measured 5.46-5.72)
        const int64_t nc = count / 256;
        if (nc > 0) {
            const size_t csmem = kSqrtCtaStages * (kSqrtCtaChunkBytes + sizeof(uint64_t));
            const int per_sm = occupancy(sqrt_tma_kernel<kSqrtCtaStages, 1>, 256, csmem);
            const int64_t grid = std::min<int64_t>(nc, (int64_t)num_sms() * per_sm);
            sqrt_tma_kernel<kSqrtCtaStages, 1><<<(unsigned)grid, 256, csmem, st>>>(r9, nc, s9);
        }
        const int64_t done = 256 * nc, rest = count - done;
        if (rest > 0)
            sqrt_plain_kernel<<<grid_for(rest, kSqrtBlock), kSqrtBlock, 0, st>>>(r9 + 9 * done, rest, s9 + 9 * done);
        return cudaGetLastError();
    }
    // per-warp TMA rings over the whole 32-matrix chunks, plain tail
    const int64_t nw = count / 32;
    const size_t wsmem = 8 * (size_t)kSqrtWarpStages * (kSqrtWarpChunkBytes + sizeof(uint64_t));
    if (nw > 0) {
        const int per_sm = occupancy(sqrt_wtma_kernel, 256, wsmem);
        const int64_t grid = std::min<int64_t>((nw + 7) / 8, (int64_t)num_sms() * per_sm);
        sqrt_wtma_kernel<<<(unsigned)grid, 256, wsmem, st>>>(r9, nw, s9);
    }
    const int64_t tail = count - 32 * nw;
    if (tail > 0) sqrt_plain_kernel<<<1, kSqrtBlock, 0, st>>>(r9 + 9 * 32 * nw, tail, s9 + 9 * 32 * nw);
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

cudaError_t metric_pairs_launch(const MetricPairs& pairs, int64_t len, double* d_result, cudaStream_t st) {
    if (pairs.count <= 0) return cudaSuccess;
    cudaError_t e = cudaMemsetAsync(d_result, 0, pairs.count * sizeof(double), st);
    if (e != cudaSuccess) return e;
    const int64_t nodes = len / 12;
    const unsigned bx = (unsigned)std::max<int64_t>(1, std::min<int64_t>(grid_for(nodes, 256), 64));
    metric_pairs_kernel<<<dim3(bx, pairs.count), 256, 0, st>>>(pairs, nodes,
                                                               reinterpret_cast<unsigned long long*>(d_result));
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
