// lj_cells.cu — lj_repulsion (reference src/rod.cpp:124-174) with a hashed cell list, O(N).
//
// The reference visits every node pair (O(N^2), serial); the force is short-ranged (cutoff
// rc = 2^(1/6) sigma, rod.hpp:52), so only pairs in adjacent cells of side rc can interact:
//   1. lj_hash_kernel     cell (floor(x / rc)) of every node -> bucket of a 2N-entry hash
//                         table (power of two), key/value = (bucket, node index);
//   2. counting sort by bucket, no library primitive: lj_count_kernel (bucket sizes,
//                         integer atomics), lj_scan_tiles_kernel + lj_scan_apply_kernel
//                         (exclusive scan -> bucket [start, end)), lj_scatter_kernel (node
//                         into its bucket, arrival order), lj_bucket_sort_kernel (each
//                         bucket's members sorted by node index -- the order a stable sort
//                         by bucket gives, so deterministic), lj_gather_kernel (positions /
//                         (rod, node) in sorted order);
//   4. lj_cells_kernel    one thread per node (in sorted order, so a warp shares cells): the
//                         27 neighbour cells' buckets (a bucket reached twice through a hash
//                         collision is visited once), the same pair law as the all-pairs
//                         kernel (kernels.cuh: lj_pair), fixed visiting order -> bitwise
//                         reproducible run to run.
// Results agree with the all-pairs kernel to rounding (the summation order differs).
#include <algorithm>

#include "kernels.cuh"

namespace pswim {
namespace {

__device__ __forceinline__ int cell_coord(double x, double inv_h) {
    const double c = floor(x * inv_h);
    return (int)fmin(fmax(c, -1073741824.0), 1073741824.0);  // far-away nodes share edge cells
}

__device__ __forceinline__ unsigned bucket_of(int cx, int cy, int cz, unsigned mask) {
    return (((unsigned)cx * 73856093u) ^ ((unsigned)cy * 19349663u) ^ ((unsigned)cz * 83492791u)) & mask;
}

__global__ void lj_count_kernel(const double* __restrict__ state, int n, double inv_h, unsigned mask,
                                unsigned* __restrict__ key, int* __restrict__ count) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const double* x = state + 12 * (int64_t)i;
    const unsigned b = bucket_of(cell_coord(x[0], inv_h), cell_coord(x[1], inv_h), cell_coord(x[2], inv_h), mask);
    key[i] = b;
    atomicAdd(&count[b], 1);
}

// Exclusive scan of the H bucket sizes (H a power of two >= 1024), tiles of kScanTile.
constexpr int kScanThreads = 256, kScanPer = 4, kScanTile = kScanThreads * kScanPer;  // tile = the smallest H

__device__ __forceinline__ int block_exclusive_scan(int v, int* total) {
    __shared__ int warp_sums[kScanThreads / 32];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    int x = v;
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
        const int y = __shfl_up_sync(0xffffffffu, x, d);
        if (lane >= d) x += y;
    }
    if (lane == 31) warp_sums[warp] = x;
    __syncthreads();
    if (warp == 0) {
        int w = lane < kScanThreads / 32 ? warp_sums[lane] : 0;
#pragma unroll
        for (int d = 1; d < 32; d <<= 1) {
            const int y = __shfl_up_sync(0xffffffffu, w, d);
            if (lane >= d) w += y;
        }
        if (lane < kScanThreads / 32) warp_sums[lane] = w;  // inclusive over warps
    }
    __syncthreads();
    const int before = (warp > 0 ? warp_sums[warp - 1] : 0) + x - v;
    *total = warp_sums[kScanThreads / 32 - 1];
    __syncthreads();  // warp_sums reusable
    return before;
}

// Per-tile sums; the last tile block to finish scans the tile sums in place (exclusive).
__global__ void __launch_bounds__(kScanThreads) lj_scan_tiles_kernel(const int* __restrict__ count, int tiles,
                                                                    int* __restrict__ tile_sum,
                                                                    unsigned* __restrict__ done) {
    const int* c = count + (int64_t)blockIdx.x * kScanTile + threadIdx.x * kScanPer;
    int v = 0;
#pragma unroll
    for (int e = 0; e < kScanPer; ++e) v += c[e];
    int total;
    block_exclusive_scan(v, &total);
    __shared__ bool last;
    if (threadIdx.x == 0) {
        tile_sum[blockIdx.x] = total;
        __threadfence();
        last = atomicAdd(done, 1u) == (unsigned)tiles - 1;
    }
    __syncthreads();
    if (!last) return;
    __threadfence();
    int carry = 0;
    for (int t0 = 0; t0 < tiles; t0 += kScanThreads) {
        const int t = t0 + threadIdx.x;
        const int x = t < tiles ? tile_sum[t] : 0;
        int chunk;
        const int ex = block_exclusive_scan(x, &chunk);
        if (t < tiles) tile_sum[t] = carry + ex;
        carry += chunk;
    }
    if (threadIdx.x == 0) *done = 0u;  // ready for the next launch
}

// start[b] = exclusive prefix of the bucket sizes (in place over count), cursor[b] = start[b].
__global__ void __launch_bounds__(kScanThreads) lj_scan_apply_kernel(int* __restrict__ count_start,
                                                                    const int* __restrict__ tile_sum,
                                                                    int* __restrict__ cursor) {
    const int64_t base = (int64_t)blockIdx.x * kScanTile + threadIdx.x * kScanPer;
    int v[kScanPer], sum = 0;
#pragma unroll
    for (int e = 0; e < kScanPer; ++e) {
        v[e] = count_start[base + e];
        sum += v[e];
    }
    int total;
    int run = tile_sum[blockIdx.x] + block_exclusive_scan(sum, &total);
#pragma unroll
    for (int e = 0; e < kScanPer; ++e) {
        count_start[base + e] = run;
        cursor[base + e] = run;
        run += v[e];
    }
}

__global__ void lj_scatter_kernel(const unsigned* __restrict__ key, int n, int* __restrict__ cursor,
                                  int* __restrict__ sorted) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    sorted[atomicAdd(&cursor[key[i]], 1)] = i;
}

// One thread per bucket: its members (scattered in arrival order) sorted by node index --
// exactly the order of a stable sort by bucket.  After the scatter, cursor[b] is the bucket's
// end.
constexpr int kRegSort = 16;   // buckets up to this size: one thread, registers
constexpr int kWarpSort = 128; // up to this size: one warp, bitonic network over 4 values per lane

// Bitonic sort of v[0..3] (element i = lane + 32 r), ascending, across the warp.
__device__ __forceinline__ void warp_bitonic128(int v[4], int lane) {
#pragma unroll
    for (int k = 2; k <= 128; k <<= 1)
#pragma unroll
        for (int j = k >> 1; j > 0; j >>= 1)
#pragma unroll
            for (int r = 0; r < 4; ++r) {
                const int i = lane + 32 * r;
                const bool up = (i & k) == 0;
                if (j >= 32) {
                    const int rp = r ^ (j >> 5);
                    if (rp > r) {  // each register pair once
                        const int a = v[r], b = v[rp];
                        const bool sw = up ? a > b : a < b;
                        v[r] = sw ? b : a;
                        v[rp] = sw ? a : b;
                    }
                } else {
                    const int o = __shfl_xor_sync(0xffffffffu, v[r], j);
                    const bool lower = (i & j) == 0;
                    v[r] = (lower == up) ? min(v[r], o) : max(v[r], o);
                }
            }
}

// Every bucket's members (scattered in arrival order) sorted by node index -- exactly the
// order of a stable sort by bucket.  After the scatter, end[b] is the bucket's end.  A warp
// covers 32 consecutive buckets: small ones a lane each, larger ones the whole warp.
__global__ void __launch_bounds__(256) lj_bucket_sort_kernel(int buckets, const int* __restrict__ start,
                                                            const int* __restrict__ end, int* __restrict__ sorted) {
    const int b = blockIdx.x * blockDim.x + threadIdx.x, lane = threadIdx.x & 31;
    const int s = b < buckets ? start[b] : 0, cnt = b < buckets ? end[b] - s : 0;
    if (cnt > 1 && cnt <= kRegSort) {
        // independent loads, then an odd-even transposition network on registers (static
        // indices: no local memory)
        int v[kRegSort];
#pragma unroll
        for (int k = 0; k < kRegSort; ++k) v[k] = k < cnt ? sorted[s + k] : 0x7fffffff;
#pragma unroll
        for (int pass = 0; pass < kRegSort; ++pass)
#pragma unroll
            for (int k = pass & 1; k + 1 < kRegSort; k += 2) {
                const int lo = min(v[k], v[k + 1]), hi = max(v[k], v[k + 1]);
                v[k] = lo;
                v[k + 1] = hi;
            }
#pragma unroll
        for (int k = 0; k < kRegSort; ++k)
            if (k < cnt) sorted[s + k] = v[k];
    }
    unsigned big = __ballot_sync(0xffffffffu, cnt > kRegSort);
    while (big) {
        const int src = __ffs(big) - 1;
        big &= big - 1;
        const int bs = __shfl_sync(0xffffffffu, s, src), bc = __shfl_sync(0xffffffffu, cnt, src);
        if (bc <= kWarpSort) {
            int v[4];
#pragma unroll
            for (int r = 0; r < 4; ++r) {
                const int i = lane + 32 * r;
                v[r] = i < bc ? sorted[bs + i] : 0x7fffffff;
            }
            warp_bitonic128(v, lane);
#pragma unroll
            for (int r = 0; r < 4; ++r) {
                const int i = lane + 32 * r;
                if (i < bc) sorted[bs + i] = v[r];
            }
        } else if (lane == 0) {
            for (int q = bs + 1; q < bs + bc; ++q) {  // insertion sort in place (very rare)
                const int x = sorted[q];
                int r = q - 1;
                while (r >= bs && sorted[r] > x) {
                    sorted[r + 1] = sorted[r];
                    --r;
                }
                sorted[r + 1] = x;
            }
        }
        __syncwarp();
    }
}

// Positions and (rod, node) gathered in sorted order, one thread per sorted slot.
__global__ void lj_gather_kernel(const double* __restrict__ state, int n, int m, const int* __restrict__ sorted,
                                 double* __restrict__ pos, int2* __restrict__ rk) {
    const int q = blockIdx.x * blockDim.x + threadIdx.x;
    if (q >= n) return;
    const int i = sorted[q];
    rk[q] = make_int2(i / m, i - (i / m) * m);
    const double* x = state + 12 * (int64_t)i;
    pos[3 * q] = x[0];
    pos[3 * q + 1] = x[1];
    pos[3 * q + 2] = x[2];
}

__device__ __forceinline__ int lower_bound_idx(const int* __restrict__ idx, int lo, int hi, int v) {
    while (lo < hi) {
        const int mid = (lo + hi) >> 1;
        if (idx[mid] < v) lo = mid + 1;
        else hi = mid;
    }
    return lo;
}

__global__ void __launch_bounds__(256)
lj_cells_kernel(const double* __restrict__ pos, const int* __restrict__ idx, const int2* __restrict__ rk,
                const int* __restrict__ start, const int* __restrict__ end, int n, double inv_h, unsigned mask, LjArgs a,
                double* __restrict__ out) {
    const int p = blockIdx.x * blockDim.x + threadIdx.x;
    if (p >= n) return;
    const int i = idx[p];
    const int2 me = rk[p];
    const double xi = pos[3 * p], yi = pos[3 * p + 1], zi = pos[3 * p + 2];
    const int cx = cell_coord(xi, inv_h), cy = cell_coord(yi, inv_h), cz = cell_coord(zi, inv_h);
    const int wlo = max(me.x * a.m, i - (a.excl - 1)), whi = min(me.x * a.m + a.m - 1, i + (a.excl - 1));
    unsigned seen[27];
    double fx = 0.0, fy = 0.0, fz = 0.0;
#pragma unroll
    for (int c = 0; c < 27; ++c) {
        const unsigned b = bucket_of(cx + c % 3 - 1, cy + (c / 3) % 3 - 1, cz + c / 9 - 1, mask);
        seen[c] = b;
        bool dup = false;
#pragma unroll
        for (int e = 0; e < c; ++e) dup |= seen[e] == b;
        if (dup) continue;
        const int q0 = start[b], q1 = end[b];
        // members are in ascending node order: the same-rod window |k_i - k_j| < excl, which
        // the pair law skips, is one contiguous run [qa, qb) found by binary search
        const int qa = lower_bound_idx(idx, q0, q1, wlo), qb = lower_bound_idx(idx, qa, q1, whi + 1);
        for (int q = q0; q < q1; ++q) {
            if (q == qa) q = qb;
            if (q >= q1) break;
            const int2 o = rk[q];
            lj_pair(a, me.x, me.y, o.x, o.y, xi - pos[3 * q], yi - pos[3 * q + 1], zi - pos[3 * q + 2], fx, fy, fz);
        }
    }
    out[3 * (int64_t)i] = fx;
    out[3 * (int64_t)i + 1] = fy;
    out[3 * (int64_t)i + 2] = fz;
}

}  // namespace

void LjWork::release() {
    for (void* q : {(void*)key, (void*)key_sorted, (void*)idx, (void*)idx_sorted, (void*)cell_start, (void*)cell_end,
                    (void*)pos, (void*)rk, tmp})
        if (q) cudaFree(q);
    *this = LjWork();
}

int lj_buckets(int64_t n) {
    int64_t h = 1024;
    while (h < 2 * n) h <<= 1;
    return (int)h;
}

namespace {
// Workspace: key (bucket per node), cell_start (bucket sizes -> starts), cell_end (scatter
// cursors -> ends), idx_sorted (nodes in bucket order), pos / rk (gathered), tmp (tile sums
// and the scan's arrival counter).
cudaError_t lj_grow(int64_t total, int H, LjWork* w, cudaStream_t st) {
    cudaError_t e;
    if (w->cap_nodes < total || w->cap_buckets < H) {
        w->release();
        const int n = (int)total;
        const size_t tmp = sizeof(int) * (size_t)(H / kScanTile + 1) + 16;
        if ((e = cudaMalloc(&w->key, sizeof(unsigned) * n)) != cudaSuccess ||
            (e = cudaMalloc(&w->idx_sorted, sizeof(int) * n)) != cudaSuccess ||
            (e = cudaMalloc(&w->cell_start, sizeof(int) * H)) != cudaSuccess ||
            (e = cudaMalloc(&w->cell_end, sizeof(int) * H)) != cudaSuccess ||
            (e = cudaMalloc(&w->pos, sizeof(double) * 3 * n)) != cudaSuccess ||
            (e = cudaMalloc(&w->rk, sizeof(int2) * n)) != cudaSuccess ||
            (e = cudaMalloc(&w->tmp, tmp)) != cudaSuccess ||
            (e = cudaMemsetAsync(w->tmp, 0, tmp, st)) != cudaSuccess)  // scan arrival counter
            return e;
        w->tmp_bytes = tmp;
        w->cap_nodes = total;
        w->cap_buckets = H;
    }
    return cudaSuccess;
}
}  // namespace

cudaError_t lj_cells_launch(const RodParams& p, const double* state, double* forces, LjWork* w, cudaStream_t st) {
    const int64_t total = p.rods * p.m;
    if (total == 0) return cudaSuccess;
    const int n = (int)total;
    const int H = lj_buckets(total);  // power of two >= 1024: whole scan tiles
    cudaError_t e = lj_grow(total, H, w, st);
    if (e != cudaSuccess) return e;
    const double inv_h = 1.0 / p.lj_cutoff;
    const unsigned mask = (unsigned)H - 1u;
    const unsigned blocks = (unsigned)((n + 255) / 256);
    const int tiles = std::max(1, H / kScanTile);
    int* tile_sum = static_cast<int*>(w->tmp);
    unsigned* done = reinterpret_cast<unsigned*>(tile_sum + tiles);
    if ((e = cudaMemsetAsync(w->cell_start, 0, sizeof(int) * H, st)) != cudaSuccess) return e;
    lj_count_kernel<<<blocks, 256, 0, st>>>(state, n, inv_h, mask, w->key, w->cell_start);
    lj_scan_tiles_kernel<<<tiles, kScanThreads, 0, st>>>(w->cell_start, tiles, tile_sum, done);
    lj_scan_apply_kernel<<<tiles, kScanThreads, 0, st>>>(w->cell_start, tile_sum, w->cell_end);
    lj_scatter_kernel<<<blocks, 256, 0, st>>>(w->key, n, w->cell_end, w->idx_sorted);
    lj_bucket_sort_kernel<<<(unsigned)((H + 255) / 256), 256, 0, st>>>(H, w->cell_start, w->cell_end, w->idx_sorted);
    lj_gather_kernel<<<blocks, 256, 0, st>>>(state, n, (int)p.m, w->idx_sorted, w->pos, w->rk);
    lj_cells_kernel<<<blocks, 256, 0, st>>>(w->pos, w->idx_sorted, w->rk, w->cell_start, w->cell_end, n, inv_h, mask,
                                           lj_args(p), forces);
    return cudaGetLastError();
}

cudaError_t lj_cells_reserve(int64_t total, LjWork* w, cudaStream_t st) {
    // the workspace for `total` nodes, allocated at context creation (no allocation on the
    // rhs path)
    return lj_grow(total, lj_buckets(total), w, st);
}

void lj_cells_preload() {
    cudaFuncAttributes a;
    cudaFuncGetAttributes(&a, lj_count_kernel);
    cudaFuncGetAttributes(&a, lj_scan_tiles_kernel);
    cudaFuncGetAttributes(&a, lj_scan_apply_kernel);
    cudaFuncGetAttributes(&a, lj_scatter_kernel);
    cudaFuncGetAttributes(&a, lj_bucket_sort_kernel);
    cudaFuncGetAttributes(&a, lj_gather_kernel);
    cudaFuncGetAttributes(&a, lj_cells_kernel);
}

}  // namespace pswim
