// lj_cells.cu — lj_repulsion (reference src/rod.cpp:124-174) with a hashed cell list, O(N).
//
// The reference visits every node pair (O(N^2), serial); the force is short-ranged (cutoff
// rc = 2^(1/6) sigma, rod.hpp:52), so only pairs in adjacent cells of side rc can interact:
//   1. lj_hash_kernel     cell (floor(x / rc)) of every node -> bucket of a 2N-entry hash
//                         table (power of two), key/value = (bucket, node index);
//   2. stable radix sort  (cub::DeviceRadixSort::SortPairs) -> nodes grouped by bucket, in
//                         ascending node order inside a bucket (deterministic);
//   3. lj_bounds_kernel   bucket [start, end) ranges + positions gathered in sorted order;
//   4. lj_cells_kernel    one thread per node (in sorted order, so a warp shares cells): the
//                         27 neighbour cells' buckets (a bucket reached twice through a hash
//                         collision is visited once), the same pair law as the all-pairs
//                         kernel (kernels.cuh: lj_pair), fixed visiting order -> bitwise
//                         reproducible run to run.
// Results agree with the all-pairs kernel to rounding (the summation order differs).
#include <cub/device/device_radix_sort.cuh>

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

__global__ void lj_hash_kernel(const double* __restrict__ state, int n, double inv_h, unsigned mask,
                               unsigned* __restrict__ key, int* __restrict__ idx) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const double* x = state + 12 * (int64_t)i;
    key[i] = bucket_of(cell_coord(x[0], inv_h), cell_coord(x[1], inv_h), cell_coord(x[2], inv_h), mask);
    idx[i] = i;
}

__global__ void lj_bounds_kernel(const double* __restrict__ state, int n, int m, const unsigned* __restrict__ key,
                                 const int* __restrict__ idx, int* __restrict__ start, int* __restrict__ end,
                                 double* __restrict__ pos, int2* __restrict__ rk) {
    const int p = blockIdx.x * blockDim.x + threadIdx.x;
    if (p >= n) return;
    const unsigned k = key[p];
    if (p == 0 || key[p - 1] != k) start[k] = p;
    if (p == n - 1 || key[p + 1] != k) end[k] = p + 1;
    const int i = idx[p];
    rk[p] = make_int2(i / m, i - (i / m) * m);
    const double* x = state + 12 * (int64_t)i;
    pos[3 * p] = x[0];
    pos[3 * p + 1] = x[1];
    pos[3 * p + 2] = x[2];
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
cudaError_t lj_grow(int64_t total, int H, int bits, LjWork* w, cudaStream_t st) {
    const int n = (int)total;
    cudaError_t e;
    if (w->cap_nodes < total || w->cap_buckets < H) {
        w->release();
        size_t tmp = 0;
        e = cub::DeviceRadixSort::SortPairs(nullptr, tmp, (const unsigned*)nullptr, (unsigned*)nullptr,
                                            (const int*)nullptr, (int*)nullptr, n, 0, bits, st);
        if (e != cudaSuccess) return e;
        if ((e = cudaMalloc(&w->key, sizeof(unsigned) * n)) != cudaSuccess ||
            (e = cudaMalloc(&w->key_sorted, sizeof(unsigned) * n)) != cudaSuccess ||
            (e = cudaMalloc(&w->idx, sizeof(int) * n)) != cudaSuccess ||
            (e = cudaMalloc(&w->idx_sorted, sizeof(int) * n)) != cudaSuccess ||
            (e = cudaMalloc(&w->cell_start, sizeof(int) * H)) != cudaSuccess ||
            (e = cudaMalloc(&w->cell_end, sizeof(int) * H)) != cudaSuccess ||
            (e = cudaMalloc(&w->pos, sizeof(double) * 3 * n)) != cudaSuccess ||
            (e = cudaMalloc(&w->rk, sizeof(int2) * n)) != cudaSuccess ||
            (e = cudaMalloc(&w->tmp, std::max<size_t>(tmp, 16))) != cudaSuccess)
            return e;
        w->tmp_bytes = std::max<size_t>(tmp, 16);
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
    const int H = lj_buckets(total);
    int bits = 0;
    while ((1 << bits) < H) ++bits;
    cudaError_t e = lj_grow(total, H, bits, w, st);
    if (e != cudaSuccess) return e;
    const double inv_h = 1.0 / p.lj_cutoff;
    const unsigned mask = (unsigned)H - 1u;
    const unsigned blocks = (unsigned)((n + 255) / 256);
    lj_hash_kernel<<<blocks, 256, 0, st>>>(state, n, inv_h, mask, w->key, w->idx);
    size_t tmp = w->tmp_bytes;
    e = cub::DeviceRadixSort::SortPairs(w->tmp, tmp, w->key, w->key_sorted, w->idx, w->idx_sorted, n, 0, bits, st);
    if (e != cudaSuccess) return e;
    // empty buckets: start == end == 0
    if ((e = cudaMemsetAsync(w->cell_start, 0, sizeof(int) * H, st)) != cudaSuccess) return e;
    if ((e = cudaMemsetAsync(w->cell_end, 0, sizeof(int) * H, st)) != cudaSuccess) return e;
    lj_bounds_kernel<<<blocks, 256, 0, st>>>(state, n, (int)p.m, w->key_sorted, w->idx_sorted, w->cell_start,
                                            w->cell_end, w->pos, w->rk);
    lj_cells_kernel<<<blocks, 256, 0, st>>>(w->pos, w->idx_sorted, w->rk, w->cell_start, w->cell_end, n, inv_h, mask,
                                           lj_args(p), forces);
    return cudaGetLastError();
}

cudaError_t lj_cells_reserve(int64_t total, LjWork* w, cudaStream_t st) {
    // workspace for `total` nodes + one sort on it: loads the radix-sort kernels this size
    // selects (CUDA lazy loading, see preload_kernels) without a pair pass
    const int n = (int)total;
    const int H = lj_buckets(total);
    int bits = 0;
    while ((1 << bits) < H) ++bits;
    cudaError_t e = lj_grow(total, H, bits, w, st);
    if (e != cudaSuccess) return e;
    if ((e = cudaMemsetAsync(w->key, 0, sizeof(unsigned) * n, st)) != cudaSuccess) return e;
    if ((e = cudaMemsetAsync(w->idx, 0, sizeof(int) * n, st)) != cudaSuccess) return e;
    size_t tmp = w->tmp_bytes;
    return cub::DeviceRadixSort::SortPairs(w->tmp, tmp, w->key, w->key_sorted, w->idx, w->idx_sorted, n, 0, bits, st);
}

void lj_cells_preload() {
    cudaFuncAttributes a;
    cudaFuncGetAttributes(&a, lj_hash_kernel);
    cudaFuncGetAttributes(&a, lj_bounds_kernel);
    cudaFuncGetAttributes(&a, lj_cells_kernel);
}

}  // namespace pswim
