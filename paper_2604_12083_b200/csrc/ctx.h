// ctx.h — the pswim_ctx object behind the opaque C handle.
#pragma once

#include <cuda_runtime.h>

#include <string>
#include <vector>

#include "internal.h"

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
    int rhs(const double* state, double t, const double* ef, const double* en, double* u, double* w);
    int advance(const double* state, const double* u, const double* w, double dt, double* out);
    int step(int scheme, const double* state, double t, double dt, double* out);
    int resolve_steps(double t0, double t1, int64_t spi, double dtc, int64_t* steps, double* dt);
    // space: optional transport of a space group -> every rhs with the MRS sharded over it
    int propagate_async(const double* d_in, double t0, double t1, int scheme, int64_t spi, double dtc, double* d_out,
                        const pswim_transport* space = nullptr);

    // space-parallel (sharded MRS) path
    double* d_shard = nullptr;   // 6 S: this rank's (u, w) shard
    double* d_gather = nullptr;  // world x 6 S
    size_t cap_shard = 0, cap_gather = 0;
    int rhs_sharded(const pswim_transport* tr, const double* state, double t, double* u, double* w);
    int step_sharded(const pswim_transport* tr, int scheme, const double* state, double t, double dt, double* out);
};
