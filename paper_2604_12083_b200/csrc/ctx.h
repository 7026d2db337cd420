// ctx.h — the pswim_ctx object behind the opaque C handle.
#pragma once

#include <cuda_runtime.h>

#include <string>
#include <vector>

#include "internal.h"

// stokes.cpp:15-17: the reference throws for image_wall (the correction is unspecified)
inline constexpr const char* kWallMsg = "stokes: image_wall correction is not implemented; use free_space";

struct pswim_ctx {
    int device = 0;
    cudaStream_t stream = nullptr;
    bool has_scenario = false;
    pswim_scenario sc{};
    pswim_resolved rs{};
    pswim::RodParams rp{};

    unsigned* d_flags = nullptr;
    unsigned* h_flags = nullptr;  // pinned
    double* d_metric = nullptr;
    // rhs workspaces (N x 3 each) + RK2 midpoint state (12 N)
    double *d_pos = nullptr, *d_f = nullptr, *d_n = nullptr, *d_u = nullptr, *d_w = nullptr, *d_lj = nullptr;
    double* d_mid = nullptr;
    // MRS split-source partials + per-target-block counters
    double* d_scratch = nullptr;
    size_t scratch_cap = 0;
    unsigned* d_counters = nullptr;
    size_t counters_cap = 0;
    // device staging for the *_host entry points
    double *h_in = nullptr, *h_a = nullptr, *h_b = nullptr, *h_c = nullptr, *h_o1 = nullptr, *h_o2 = nullptr;
    size_t cap_in = 0, cap_a = 0, cap_b = 0, cap_c = 0, cap_o1 = 0, cap_o2 = 0;

    std::string err;

    // stage timers (propagators.hpp:55-65): 0 initialization, 1 velocity, 2 triad_update
    struct TimedStage {
        cudaEvent_t a, b;
        int stage;
    };
    bool timing_on = false;
    bool fused_on = true;  // whole-interval fused kernel for N <= 256 (fused.cu)
    int fused_max_cs = 0;  // cluster-size cap (pswim_set_fused 2..16), 0 = default
    int lj_mode = 0;       // 0 auto (all-pairs below kLjCellsMinNodes), 1 all-pairs, 2 cell list
    pswim::LjWork lj_work;
    std::vector<TimedStage> open_stages, done_stages;
    double stage_seconds[3] = {0, 0, 0};

    ~pswim_ctx();
    int fail(int code, const std::string& what);
    int use();
    int ensure(double** p, size_t* cap, size_t n);
    int ensure_mrs(const pswim::MrsPlan& plan);
    int sync();
    int check_flags_after_sync();
    void stage_begin(int stage);
    void stage_end();
    void harvest_timing();

    int mrs(const double* tgt, int64_t nt, const double* src, const double* f, const double* n, int64_t ns,
            double eps, double mu, double* u, double* w, int pstride = 3);
    int lj(const double* state, double* out);  // lj_repulsion, rod.cpp:124-174
    // tdev / tdev2: optional device copies of t (and t + dt/2) read by the load kernels, so
    // that a captured step replays at new times (CUDA graphs)
    int rhs(const double* state, double t, const double* ef, const double* en, double* u, double* w,
            const double* tdev = nullptr);
    int advance(const double* state, const double* u, const double* w, double dt, double* out);
    int step(int scheme, const double* state, double t, double dt, double* out, const double* tdev2 = nullptr);
    int resolve_steps(double t0, double t1, int64_t spi, double dtc, int64_t* steps, double* dt);
    // space: optional transport of a space group -> every rhs with the MRS sharded over it
    int propagate_async(const double* d_in, double t0, double t1, int scheme, int64_t spi, double dtc, double* d_out,
                        const pswim_transport* space = nullptr);

    // CUDA-graph replay of the per-step kernel sequence (launch-bound mid-size systems):
    // one captured graph runs kGraphSteps steps in place on d_gstate, the step times staged in
    // d_times; rebuilt when scheme, dt or any workspace pointer changes.
    static constexpr int kGraphSteps = 32;
    static constexpr int64_t kGraphMaxNodes = 8192;
    cudaGraphExec_t graph_exec = nullptr;
    int graph_scheme = -1;
    double graph_dt = 0.0;
    const void* graph_key[4] = {nullptr, nullptr, nullptr, nullptr};
    double* d_gstate = nullptr;
    double* d_times = nullptr;      // 2 kGraphSteps (t, t + dt/2 per step)
    double* d_times_all = nullptr;  // every step time of the current interval
    double* h_times = nullptr;      // pinned staging
    size_t cap_gstate = 0, cap_times_all = 0, cap_h_times = 0;
    cudaEvent_t times_done = nullptr;  // the staging buffer's last upload finished
    bool graphs_on = true;
    int propagate_graph(double t0, int scheme, int64_t steps, double dt, double* d_out);

    // space-parallel (sharded MRS) path
    double* d_shard = nullptr;   // 6 S: this rank's (u, w) shard
    double* d_gather = nullptr;  // world x 6 S
    size_t cap_shard = 0, cap_gather = 0;
    int rhs_sharded(const pswim_transport* tr, const double* state, double t, double* u, double* w);
    int step_sharded(const pswim_transport* tr, int scheme, const double* state, double t, double dt, double* out);
};
