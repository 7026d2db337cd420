// internal.h — declarations shared between the translation units of libpswim.so.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include <string>

#include "../../include/pswim_c.h"

namespace pswim {

// Device error flag bits (OR-ed by kernels, read at sync).
enum : unsigned {
    kFlagNonFinite = 1u << 0,   // -> PSWIM_ENONFINITE
    kFlagStiff = 1u << 1,       // -> PSWIM_ESTIFF
    kFlagDegenerate = 1u << 2,  // -> PSWIM_EDEGENERATE
    kFlagAxis = 1u << 3,        // -> PSWIM_EINVAL (from_axis_angle axis check)
};

// ---- MRS (mrs.cu) ----------------------------------------------------------------------
struct MrsPlan {
    int64_t nt = 0, ns = 0;
    int target_blocks = 0;  // ceil(nt / kMrsTargets)
    int chunks = 0;         // source chunks (grid.y)
    size_t scratch_doubles = 0;
    size_t counters = 0;
    int variant = 0;  // kernel variant forced by the plan (0 = mrs_targets_per_thread())
    int tail = 0;     // 0: equal chunks; c1 << 8 | m: chunks after the first c1 are 1/m size
    int fixed = 0;    // > 0: chunks of exactly `fixed` sources, the last one takes the rest
};
constexpr int kMrsThreads = 256;  // targets per block (one or two per thread)

// Peer epilogue of the sharded MRS: every target's final (u, w) is stored straight into each
// rank's exchange buffer (NVLink P2P / CUDA IPC pointers, or same-device pointers), and every
// finished 256-target block bumps each rank's arrival counter with a system-scope atomic --
// the all-gather fused into the kernel that produces the data.
constexpr int kMaxPeers = 16;
struct PeerOut {
    int world = 0;  // 0: plain local output
    double* u[kMaxPeers];
    double* w[kMaxPeers];
    unsigned long long* flag[kMaxPeers];
};
MrsPlan mrs_plan(int64_t nt, int64_t ns);
// Chunk c covers sources [bound(c), bound(c + 1)), bound(c) = unit(c) ns / unit(C).
int mrs_chunk_unit(const MrsPlan& p, int c);
int64_t mrs_chunk_bound(const MrsPlan& p, int c);
constexpr int kMrsMaxChunks = 160;
struct MrsBounds {  // kernel parameter: unit(0..C) of the plan, unit(C) again at [kMrsMaxChunks]
    int b[kMrsMaxChunks + 1];
    int main_chunks;  // c1: chunks before the tail split (C without one)
    int tbs;          // target blocks of the plan (the second counter row)
};
// All-pairs kernel variant (1: 1 target/thread; 2: 2 targets/thread; 3: 2 targets/thread at
// 3 CTAs/SM -- the default); env PSWIM_MRS_TPT overrides.
int mrs_targets_per_thread();
// Launches the all-pairs kernel (+ fused fixed-order split-source reduction).
// d_scratch >= plan.scratch_doubles, d_counters >= plan.counters (zeroed once; the kernel
// leaves them zero again).
cudaError_t mrs_launch(const MrsPlan& plan, const double* tgt, const double* src, const double* f,
                       const double* n, double eps, double mu, double* u, double* w, double* scratch,
                       unsigned* counters, unsigned* flags, cudaStream_t st);
// Target blocks [tb0, tb1) of plan p only; outputs of target i land at index i - 256 tb0.
cudaError_t mrs_launch_blocks(const MrsPlan& p, int tb0, int tb1, const double* tgt, const double* src, int pstride,
                              const double* f, const double* n, double eps, double mu, double* u, double* w,
                              double* scratch, unsigned* counters, unsigned* flags, cudaStream_t st,
                              const PeerOut* d_peer = nullptr);  // device-resident PeerOut
// Force-load (lazy module loading) every kernel a peer rank launches; call before spinning.
void peer_preload();
void rod_preload();
void fused_preload();
// Every kernel of the library is loaded on `device` before a context can launch anything:
// CUDA lazy module loading may synchronise the context on a kernel's first launch, which
// deadlocks against a spinning peer / NCCL kernel in another stream of this process.
void preload_kernels(int device);
// One arrival on every rank's counter (a rank with an empty block range, at its MRS position).
cudaError_t peer_token_launch(const PeerOut* d_peer, cudaStream_t st);
// Spin (one thread, acquire at system scope) until *flag >= target.
cudaError_t peer_wait_launch(const unsigned long long* flag, unsigned long long target, cudaStream_t st);
// gathered = world x [u (3 S), w (3 S)] -> u, w (nt x 3), S = shard_targets
cudaError_t unshard_launch(const double* gathered, int64_t shard_targets, int64_t nt, double* u, double* w,
                           cudaStream_t st);
cudaError_t h_functions_launch(const double* r, int64_t count, double eps, double* h5, cudaStream_t st);
// Copies up to three mapped page-locked host arrays (src[k] device-accessible, nullptr = skip)
// into device memory with SM loads (pswim_mrs_velocities_host).
cudaError_t upload_launch(const double* const src[3], double* const dst[3], const int64_t n[3], cudaStream_t st);

// ---- rod / propagator kernels (rod.cu) --------------------------------------------------
struct RodParams {
    int64_t rods = 0, m = 0;
    double length = 1.0, ds = 0.0, inv_ds = 0.0;
    double a[3] = {0, 0, 0}, b[3] = {0, 0, 0};
    double amplitude = 0.0, frequency = 0.0, wavelength = 1.0;
    double epsilon = 0.0, mu = 1.0;
    double lj_well = 0.0, lj_sigma = 0.0, lj_cutoff = 0.0;
    int64_t lj_excl = 4;
};
// internal + nodal loads: state (packed 12/node) -> pos, f, n (N x 3); optional segment
// loads; extra loads added after LJ as rhs does (propagators.cpp:70-84).  tdev (optional):
// the time is read from device memory (CUDA-graph replays of the step loop).
cudaError_t rod_loads_launch(const RodParams& p, const double* state, double t, double* pos, double* f,
                             double* n, double* seg_f, double* seg_n, const double* lj, const double* extra_f,
                             const double* extra_n, unsigned* flags, cudaStream_t st,
                             const double* tdev = nullptr);
cudaError_t lj_launch(const RodParams& p, const double* state, double* forces, cudaStream_t st);
// Hashed cell-list LJ (lj_cells.cu): workspace grown on demand, owned by the context.
struct LjWork {
    int64_t cap_nodes = 0, cap_buckets = 0;
    unsigned *key = nullptr, *key_sorted = nullptr;
    int *idx = nullptr, *idx_sorted = nullptr, *cell_start = nullptr, *cell_end = nullptr;
    double* pos = nullptr;
    int2* rk = nullptr;  // (rod, node-in-rod) per sorted entry
    void* tmp = nullptr;
    size_t tmp_bytes = 0;
    void release();
};
int lj_buckets(int64_t n);
cudaError_t lj_cells_launch(const RodParams& p, const double* state, double* forces, LjWork* w, cudaStream_t st);
cudaError_t lj_cells_reserve(int64_t total, LjWork* w, cudaStream_t st);
void lj_cells_preload();
// all-pairs kernel below this many nodes in LJ auto mode, cell list above
constexpr int64_t kLjCellsMinNodes = 2048;
cudaError_t advance_launch(const RodParams& p, const double* state, const double* u, const double* w, double dt,
                           double* out, unsigned* flags, cudaStream_t st);
cudaError_t sqrt_batched_launch(const double* r9, int64_t count, double* s9, cudaStream_t st);
cudaError_t metric_launch(const double* x, const double* y, int64_t len, double* d_partial, int* d_count,
                          double* d_result, cudaStream_t st);
// Many position metrics in one launch: d_result[p] = metric(x[p], y[p]) (rod_position_metric,
// io.cpp:49-68), p < count <= kMetricPairs.
constexpr int kMetricPairs = 128;
struct MetricPairs {
    int count = 0;
    const double* x[kMetricPairs];
    const double* y[kMetricPairs];
};
cudaError_t metric_pairs_launch(const MetricPairs& pairs, int64_t len, double* d_result, cudaStream_t st);
cudaError_t correct_launch(const double* xp, const double* gn, const double* go, int64_t len, double* out,
                           cudaStream_t st);
cudaError_t dfma_launch(double* sink, int blocks, int iters, cudaStream_t st);

// ---- fused small-system propagator (fused.cu) ---------------------------------------------
// Cluster size the fused path uses for this scenario (0 = not eligible: N > 256 or smem).
// max_hint: 0 = default sizing (<= 8 CTAs, >= 12 targets each), 2..16 = cap
int fused_cluster_size(const RodParams& p, int max_hint = 0);
// prof: optional kFusedPhases device counters (in-kernel clock64 phase timer, fused.cu)
constexpr int kFusedPhases = 7;
cudaError_t fused_propagate_launch(const RodParams& p, double* state, int64_t steps, double t0, double dt, int scheme,
                                   unsigned* flags, cudaStream_t st, unsigned long long* prof = nullptr,
                                   int max_hint = 0);

// ---- slice hand-off over peer memory (handoff.cu) -----------------------------------------
double* handoff_recv_slot(pswim_handoff* h, int k);  // this rank's slot k (X[k][n-1] arrives here)
bool handoff_has_next(const pswim_handoff* h);
unsigned long long handoff_begin_run(pswim_handoff* h);
cudaError_t handoff_wait_launch(pswim_handoff* h, int k, unsigned long long gen, cudaStream_t st);
cudaError_t handoff_push_launch(pswim_handoff* h, int k, unsigned long long gen, const double* src, cudaStream_t st);
cudaError_t handoff_correct_push_launch(pswim_handoff* h, int k, unsigned long long gen, const double* xp,
                                        const double* gn, const double* go, double* out, cudaStream_t st);

// ---- host scenario (scenario.cpp) -------------------------------------------------------
int resolve_scenario(const pswim_scenario* sc, pswim_resolved* out, std::string* err);
RodParams rod_params(const pswim_scenario* sc, const pswim_resolved& rs);

}  // namespace pswim
