// parareal_common.h — pieces shared by the single-device wavefront engine (engine.cpp) and the
// time-sliced rank driver (parareal.cpp).
#pragma once

#include <algorithm>
#include <chrono>
#include <cmath>
#include <stdexcept>
#include <string>
#include <vector>

#include "internal.h"

namespace pswim {

using Clock = std::chrono::steady_clock;

struct CodeError : std::runtime_error {
    int code;
    CodeError(int c, const std::string& w) : std::runtime_error(w), code(c) {}
};

// ParallelPlan validation, parareal.cpp:38-45.
inline int plan_check(const pswim_plan* p) {
    if (!p || p->intervals < 1 || p->workers < 1) return PSWIM_EINVAL;
    if (p->max_iterations < 1) return PSWIM_EINVAL;
    if (!(p->tolerance > 0.0)) return PSWIM_EINVAL;
    if (p->horizon <= 0.0) return PSWIM_EINVAL;
    return PSWIM_OK;
}

// ParallelPlan::boundary_time, parareal.hpp:44 -- every caller uses this expression so all
// propagator calls see bitwise-identical interval ends.
inline double boundary_time(const pswim_plan& p, int n) { return p.t0 + (p.horizon / p.intervals) * n; }

// Pointwise metric over groups: |x_i - y_i| / |x_i| on `dim` entries every `stride`
// (parareal.cpp:15-34 with stride == dim; io.cpp:49-68 with dim 3, stride 12).
inline double host_metric(const double* x, const double* y, int64_t len, int dim, int stride) {
    double worst = 0.0;
    for (int64_t i = 0; i < len; i += stride) {
        double num = 0.0, den = 0.0;
        for (int c = 0; c < dim; ++c) {
            const double d = x[i + c] - y[i + c];
            num += d * d;
            den += x[i + c] * x[i + c];
        }
        num = std::sqrt(num);
        den = std::sqrt(den);
        worst = std::max(worst, den < 1e-14 ? num : num / den);
    }
    return worst;
}

// ScheduleTrace::finalize_idle semantics (schedule_trace.cpp:17-49): events grouped by
// worker in start order; every lane except the serial one (worker 0) gets an idle event for
// each gap from t = 0 up to each task start.  Returns W = the summed idle time.
enum TaskKind { kCoarse = 0, kFine = 1, kCorrect = 2, kIdle = 3 };
inline double finalize_idle(std::vector<pswim_trace_event>* ev) {
    auto order = [](const pswim_trace_event& a, const pswim_trace_event& b) {
        return a.worker != b.worker ? a.worker < b.worker : a.t_start < b.t_start;
    };
    std::stable_sort(ev->begin(), ev->end(), order);
    std::vector<pswim_trace_event> gaps;
    double cursor = 0.0, idle = 0.0;
    int cur = -1;
    for (const auto& e : *ev) {
        if (e.worker != cur) {
            cur = e.worker;
            cursor = 0.0;
        }
        if (e.worker != 0 && e.t_start > cursor) {
            gaps.push_back(pswim_trace_event{e.worker, kIdle, cursor, e.t_start, -1, -1});
            idle += e.t_start - cursor;
        }
        cursor = std::max(cursor, e.t_end);
    }
    ev->insert(ev->end(), gaps.begin(), gaps.end());
    std::stable_sort(ev->begin(), ev->end(), order);
    return idle;
}

// Iterations a pipelined schedule enqueues ahead of the last stop decision (speculation
// depth; the reference's pipelined engine dispatches fine(k+1, n) the moment X[k][n-1]
// exists, before eta_tilde_k is known).  PSWIM_PARAREAL_LOOKAHEAD overrides (>= 1).
int parareal_lookahead(const pswim_plan& plan);

// Process-wide pool of scenario contexts (engine lanes, slice ranks): creating one allocates
// HBM workspaces and synchronises, which would dominate short Parareal runs.
pswim_ctx* pooled_ctx(int device, const pswim_scenario& sc, int prio);
void release_ctx(pswim_ctx* c, int prio);

}  // namespace pswim
