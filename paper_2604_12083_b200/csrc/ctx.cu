// ctx.cu — device context and the C-ABI entry points of include/pswim_c.h for the MRS
// operator, rotation square root, rod loads, rhs/advance/step/propagate, metric, corrector.
//
// One context = one device + one CUDA stream + preallocated HBM workspaces sized for its
// scenario.  Everything is stream ordered; device failures are OR-ed into a flag word that
// every synchronising entry point converts into the reference's exception kinds.
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>
#include <vector>

#include "ctx.h"
#include "internal.h"

using namespace pswim;

#define CK(call)                                                                     \
    do {                                                                             \
        const cudaError_t e_ = (call);                                               \
        if (e_ != cudaSuccess) return ctx->fail(PSWIM_ECUDA, std::string(#call) + ": " + cudaGetErrorString(e_)); \
    } while (0)

int pswim_ctx::fail(int code, const std::string& what) {
    err = what;
    return code;
}

int pswim_ctx::use() {
    const cudaError_t e = cudaSetDevice(device);
    if (e != cudaSuccess) return fail(PSWIM_ECUDA, std::string("cudaSetDevice: ") + cudaGetErrorString(e));
    return PSWIM_OK;
}

int pswim_ctx::ensure(double** p, size_t* cap, size_t n) {
    if (*cap >= n) return PSWIM_OK;
    if (*p) cudaFree(*p);
    *p = nullptr;
    *cap = 0;
    const cudaError_t e = cudaMalloc(p, n * sizeof(double));
    if (e != cudaSuccess) return fail(PSWIM_ECUDA, std::string("cudaMalloc: ") + cudaGetErrorString(e));
    *cap = n;
    return PSWIM_OK;
}

int pswim_ctx::ensure_mrs(const MrsPlan& plan) {
    int rc = ensure(&d_scratch, &scratch_cap, plan.scratch_doubles);
    if (rc) return rc;
    if (counters_cap < plan.counters) {
        if (d_counters) cudaFree(d_counters);
        d_counters = nullptr;
        counters_cap = 0;
        cudaError_t e = cudaMalloc(&d_counters, plan.counters * sizeof(unsigned));
        if (e != cudaSuccess) return fail(PSWIM_ECUDA, "cudaMalloc counters");
        e = cudaMemsetAsync(d_counters, 0, plan.counters * sizeof(unsigned), stream);
        if (e != cudaSuccess) return fail(PSWIM_ECUDA, "cudaMemset counters");
        counters_cap = plan.counters;
    }
    return PSWIM_OK;
}

int pswim_ctx::check_flags_after_sync() {
    const unsigned f = *h_flags;
    if (!f) return PSWIM_OK;
    *h_flags = 0;
    cudaMemsetAsync(d_flags, 0, sizeof(unsigned), stream);
    // Priority follows the order the reference would throw in: a stiff step aborts before
    // the next rhs can see its (possibly degenerate / non-finite) result.
    if (f & kFlagStiff)
        return fail(PSWIM_ESTIFF, "time step moved a node more than 10 segment lengths; reduce dt or r");
    if (f & kFlagDegenerate) return fail(PSWIM_EDEGENERATE, "internal_loads: degenerate segment (coincident nodes)");
    if (f & kFlagNonFinite) return fail(PSWIM_ENONFINITE, "stokes: non-finite load entry");
    if (f & kFlagAxis) return fail(PSWIM_EINVAL, "from_axis_angle: axis is not a unit vector");
    return fail(PSWIM_ESTATE, "unknown device flag");
}

int pswim_ctx::sync() {
    int rc = use();
    if (rc) return rc;
    cudaError_t e = cudaMemcpyAsync(h_flags, d_flags, sizeof(unsigned), cudaMemcpyDeviceToHost, stream);
    if (e == cudaSuccess) e = cudaStreamSynchronize(stream);
    if (e != cudaSuccess) return fail(PSWIM_ECUDA, std::string("sync: ") + cudaGetErrorString(e));
    harvest_timing();
    return check_flags_after_sync();
}

void pswim_ctx::stage_begin(int stage) {
    if (!timing_on) return;
    TimedStage t;
    cudaEventCreate(&t.a);
    cudaEventCreate(&t.b);
    t.stage = stage;
    cudaEventRecord(t.a, stream);
    open_stages.push_back(t);
}

void pswim_ctx::stage_end() {
    if (!timing_on || open_stages.empty()) return;
    TimedStage t = open_stages.back();
    open_stages.pop_back();
    cudaEventRecord(t.b, stream);
    done_stages.push_back(t);
}

void pswim_ctx::harvest_timing() {
    for (auto& t : done_stages) {
        float ms = 0.f;
        if (cudaEventElapsedTime(&ms, t.a, t.b) == cudaSuccess) stage_seconds[t.stage] += 1e-3 * ms;
        cudaEventDestroy(t.a);
        cudaEventDestroy(t.b);
    }
    done_stages.clear();
}

// ---- physics on the context stream ---------------------------------------------------
int pswim_ctx::mrs(const double* tgt, int64_t nt, const double* src, const double* f, const double* n, int64_t ns,
                   double eps, double mu, double* u, double* w, int pstride) {
    const MrsPlan plan = mrs_plan(nt, ns);
    int rc = ensure_mrs(plan);
    if (rc) return rc;
    const cudaError_t e = mrs_launch_blocks(plan, 0, plan.target_blocks, tgt, src, pstride, f, n, eps, mu, u, w,
                                            d_scratch, d_counters, d_flags, stream);
    if (e != cudaSuccess) return fail(PSWIM_ECUDA, std::string("mrs_launch: ") + cudaGetErrorString(e));
    return PSWIM_OK;
}

int pswim_ctx::lj(const double* state, double* out) {
    const int64_t total = rp.rods * rp.m;
    if (total >= ((int64_t)1 << 31) / 12) return fail(PSWIM_EINVAL, "lj: more nodes than the 32-bit pair kernels index");
    const bool cells = lj_mode == 2 || (lj_mode == 0 && total >= kLjCellsMinNodes);
    const cudaError_t e = cells ? lj_cells_launch(rp, state, out, &lj_work, stream) : lj_launch(rp, state, out, stream);
    if (e != cudaSuccess) return fail(PSWIM_ECUDA, std::string("lj: ") + cudaGetErrorString(e));
    return PSWIM_OK;
}

int pswim_ctx::rhs(const double* state, double t, const double* ef, const double* en, double* u, double* w,
                   const double* tdev) {
    if (!has_scenario) return fail(PSWIM_EINVAL, "rhs: context has no scenario");
    if (sc.wall_mode == 1) return fail(PSWIM_EUNSUPPORTED_WALL, kWallMsg);
    stage_begin(0);
    const bool lj = rp.rods >= 2 && rp.lj_well > 0.0;  // propagators.cpp:70
    if (lj) {
        const int rc = this->lj(state, d_lj);
        if (rc) return rc;
    }
    cudaError_t e = rod_loads_launch(rp, state, t, nullptr, d_f, d_n, nullptr, nullptr, lj ? d_lj : nullptr, ef, en,
                                     d_flags, stream, tdev);
    if (e != cudaSuccess) return fail(PSWIM_ECUDA, std::string("rod_loads_launch: ") + cudaGetErrorString(e));
    stage_end();
    stage_begin(1);
    const int64_t total = rp.rods * rp.m;
    // targets = sources = node positions read in place from the packed state (stride 12)
    int rc = mrs(state, total, state, d_f, d_n, total, rs.epsilon, rs.mu, u, w, 12);
    stage_end();
    return rc;
}

int pswim_ctx::advance(const double* state, const double* u, const double* w, double dt, double* out) {
    stage_begin(2);
    const cudaError_t e = advance_launch(rp, state, u, w, dt, out, d_flags, stream);
    stage_end();
    if (e != cudaSuccess) return fail(PSWIM_ECUDA, std::string("advance_launch: ") + cudaGetErrorString(e));
    return PSWIM_OK;
}

int pswim_ctx::step(int scheme, const double* state, double t, double dt, double* out, const double* tdev2) {
    // step_euler / step_rk2, propagators.cpp:126-133.  In-place safe (advance is per node).
    int rc = rhs(state, t, nullptr, nullptr, d_u, d_w, tdev2);
    if (rc) return rc;
    if (scheme == PSWIM_EULER) return advance(state, d_u, d_w, dt, out);
    rc = advance(state, d_u, d_w, 0.5 * dt, d_mid);
    if (rc) return rc;
    rc = rhs(d_mid, t + 0.5 * dt, nullptr, nullptr, d_u, d_w, tdev2 ? tdev2 + 1 : nullptr);
    if (rc) return rc;
    return advance(state, d_u, d_w, dt, out);
}

int pswim_ctx::resolve_steps(double t0, double t1, int64_t steps_per_interval, double dtc, int64_t* steps,
                             double* dt) {
    // propagate, propagators.cpp:139-155
    if (t1 < t0) return fail(PSWIM_EINVAL, "propagate: t1 < t0");
    if (steps_per_interval > 0) {
        *steps = steps_per_interval;
        *dt = (t1 - t0) / static_cast<double>(*steps);
        return PSWIM_OK;
    }
    if (dtc <= 0.0) return fail(PSWIM_EINVAL, "propagate: dt must be positive");
    const double ratio = (t1 - t0) / dtc;
    *steps = static_cast<int64_t>(std::llround(ratio));
    if (*steps == 0 || std::abs(ratio - static_cast<double>(*steps)) > 1e-9 * static_cast<double>(*steps))
        return fail(PSWIM_EINVAL, "propagate: interval is not an integral number of steps");
    *dt = dtc;
    return PSWIM_OK;
}

int pswim_ctx::propagate_async(const double* d_in, double t0, double t1, int scheme, int64_t spi, double dtc,
                               double* d_out, const pswim_transport* space) {
    if (!has_scenario) return fail(PSWIM_EINVAL, "propagate: context has no scenario");
    // checked here, not only in rhs: the fused, graph and sharded paths never reach rhs()
    if (sc.wall_mode == 1) return fail(PSWIM_EUNSUPPORTED_WALL, kWallMsg);
    const size_t bytes = sizeof(double) * 12 * static_cast<size_t>(rp.rods * rp.m);
    if (t1 < t0) return fail(PSWIM_EINVAL, "propagate: t1 < t0");
    if (d_in != d_out) {
        const cudaError_t e = cudaMemcpyAsync(d_out, d_in, bytes, cudaMemcpyDeviceToDevice, stream);
        if (e != cudaSuccess) return fail(PSWIM_ECUDA, "propagate: copy");
    }
    if (t1 == t0) return PSWIM_OK;
    int64_t steps = 0;
    double dt = 0.0;
    int rc = resolve_steps(t0, t1, spi, dtc, &steps, &dt);
    if (rc) return rc;
    if (space && space->world > 1) {
        // space-parallel: the MRS targets of every rhs sharded over the space group
        double t = t0;
        for (int64_t i = 0; i < steps; ++i) {
            rc = step_sharded(space, scheme, d_out, t, dt, d_out);
            if (rc) return rc;
            t += dt;  // propagators.cpp:159
        }
        return PSWIM_OK;
    }
    if (fused_on && !timing_on && fused_cluster_size(rp, fused_max_cs) > 0) {
        // the whole interval in one launch, bitwise identical to the loop below.  A cluster the
        // GPU cannot place (cudaErrorInvalidClusterSize: a partitioned GPU, too few SMs per
        // GPC) is retried at half the size -- the cluster only splits the targets, so the
        // result does not change -- down to 2 CTAs, then the launched path below.
        int cap = fused_max_cs;
        for (;;) {
            const int cs = fused_cluster_size(rp, cap);
            const cudaError_t e = fused_propagate_launch(rp, d_out, steps, t0, dt, scheme, d_flags, stream, nullptr,
                                                         cap);
            if (e == cudaSuccess) return PSWIM_OK;
            if (e != cudaErrorInvalidClusterSize)
                return fail(PSWIM_ECUDA, std::string("fused_propagate: ") + cudaGetErrorString(e));
            cudaGetLastError();  // (a launch-configuration error is not sticky)
            if (cs <= 2) break;
            cap = cs / 2;
        }
    }
    // graphs pay where kernel launches are a visible share of a step (mid-size systems); large
    // systems would only add the one-off capture to the first interval
    if (graphs_on && !timing_on && steps >= kGraphSteps && rp.rods * rp.m <= kGraphMaxNodes)
        return propagate_graph(t0, scheme, steps, dt, d_out);
    double t = t0;
    for (int64_t i = 0; i < steps; ++i) {
        rc = step(scheme, d_out, t, dt, d_out);
        if (rc) return rc;
        t += dt;  // propagators.cpp:159
    }
    return PSWIM_OK;
}

int pswim_ctx::propagate_graph(double t0, int scheme, int64_t steps, double dt, double* d_out) {
    // The same kernels with the same arguments as the step loop (bitwise identical), replayed
    // from one captured graph of kGraphSteps steps: one launch instead of 6 (RK2) or 3 (Euler)
    // per step.  Times come from device memory: t_i by the reference's accumulation t += dt
    // (propagators.cpp:159) on the host, and t_i + dt/2, per step.
    const size_t n12 = 12 * static_cast<size_t>(rp.rods * rp.m);
    int rc = ensure(&d_gstate, &cap_gstate, n12);
    if (rc) return rc;
    if ((rc = ensure(&d_times_all, &cap_times_all, 2 * static_cast<size_t>(steps)))) return rc;
    if (!d_times && cudaMalloc(&d_times, 2 * kGraphSteps * sizeof(double)) != cudaSuccess)
        return fail(PSWIM_ECUDA, "graph: cudaMalloc times");
    if (!times_done && cudaEventCreateWithFlags(&times_done, cudaEventDisableTiming) != cudaSuccess)
        return fail(PSWIM_ECUDA, "graph: event");
    // host times, staged through pinned memory (wait for the previous upload to have read it)
    cudaEventSynchronize(times_done);
    if (cap_h_times < 2 * static_cast<size_t>(steps)) {
        if (h_times) cudaFreeHost(h_times);
        h_times = nullptr;
        cap_h_times = 0;
        if (cudaMallocHost(&h_times, 2 * steps * sizeof(double)) != cudaSuccess)
            return fail(PSWIM_ECUDA, "graph: pinned times");
        cap_h_times = 2 * static_cast<size_t>(steps);
    }
    double t = t0;
    for (int64_t i = 0; i < steps; ++i) {
        h_times[2 * i] = t;
        h_times[2 * i + 1] = t + 0.5 * dt;
        t += dt;  // propagators.cpp:159
    }
    cudaError_t e = cudaMemcpyAsync(d_times_all, h_times, 2 * steps * sizeof(double), cudaMemcpyHostToDevice, stream);
    if (e == cudaSuccess) e = cudaEventRecord(times_done, stream);
    if (e == cudaSuccess) e = cudaMemcpyAsync(d_gstate, d_out, n12 * sizeof(double), cudaMemcpyDeviceToDevice, stream);
    if (e != cudaSuccess) return fail(PSWIM_ECUDA, std::string("graph: staging: ") + cudaGetErrorString(e));
    // (re)capture when the step or any workspace it touches changed
    const void* key[4] = {d_scratch, d_counters, lj_work.key, d_mid};
    const bool stale = !graph_exec || graph_scheme != scheme || graph_dt != dt ||
                       std::memcmp(key, graph_key, sizeof key) != 0;
    if (stale) {
        if (graph_exec) cudaGraphExecDestroy(graph_exec);
        graph_exec = nullptr;
        cudaGraph_t g = nullptr;
        if ((e = cudaStreamBeginCapture(stream, cudaStreamCaptureModeRelaxed)) != cudaSuccess)
            return fail(PSWIM_ECUDA, std::string("graph: capture: ") + cudaGetErrorString(e));
        for (int i = 0; i < kGraphSteps && rc == PSWIM_OK; ++i)
            rc = step(scheme, d_gstate, 0.0, dt, d_gstate, d_times + 2 * i);
        e = cudaStreamEndCapture(stream, &g);
        if (rc) {
            if (g) cudaGraphDestroy(g);
            return rc;
        }
        if (e == cudaSuccess) e = cudaGraphInstantiate(&graph_exec, g, 0);
        if (g) cudaGraphDestroy(g);
        if (e != cudaSuccess) return fail(PSWIM_ECUDA, std::string("graph: instantiate: ") + cudaGetErrorString(e));
        graph_scheme = scheme;
        graph_dt = dt;
        std::memcpy(graph_key, key, sizeof key);
    }
    const int64_t full = steps / kGraphSteps;
    for (int64_t c = 0; c < full; ++c) {
        e = cudaMemcpyAsync(d_times, d_times_all + 2 * kGraphSteps * c, 2 * kGraphSteps * sizeof(double),
                            cudaMemcpyDeviceToDevice, stream);
        if (e == cudaSuccess) e = cudaGraphLaunch(graph_exec, stream);
        if (e != cudaSuccess) return fail(PSWIM_ECUDA, std::string("graph: launch: ") + cudaGetErrorString(e));
    }
    for (int64_t i = full * kGraphSteps; i < steps; ++i)
        if ((rc = step(scheme, d_gstate, h_times[2 * i], dt, d_gstate))) return rc;
    e = cudaMemcpyAsync(d_out, d_gstate, n12 * sizeof(double), cudaMemcpyDeviceToDevice, stream);
    return e == cudaSuccess ? PSWIM_OK : fail(PSWIM_ECUDA, "graph: copy out");
}

// ---- space-parallel MRS (sharded targets, velocity all-gather) ------------------------
int pswim_ctx::rhs_sharded(const pswim_transport* tr, const double* state, double t, double* u, double* w) {
    if (!has_scenario) return fail(PSWIM_EINVAL, "rhs: context has no scenario");
    if (sc.wall_mode == 1) return fail(PSWIM_EUNSUPPORTED_WALL, kWallMsg);
    const bool lj = rp.rods >= 2 && rp.lj_well > 0.0;  // propagators.cpp:70
    if (lj) {
        const int rc = this->lj(state, d_lj);
        if (rc) return rc;
    }
    cudaError_t e = rod_loads_launch(rp, state, t, nullptr, d_f, d_n, nullptr, nullptr, lj ? d_lj : nullptr, nullptr,
                                     nullptr, d_flags, stream);
    if (e != cudaSuccess) return fail(PSWIM_ECUDA, std::string("rod_loads_launch: ") + cudaGetErrorString(e));
    const int64_t total = rp.rods * rp.m;
    const MrsPlan plan = mrs_plan(total, total);
    int rc = ensure_mrs(plan);
    if (rc) return rc;
    // this rank's 256-target blocks of the single-GPU plan (bitwise identical results)
    const int world = tr->world, rank = tr->rank;
    const int bpr = (plan.target_blocks + world - 1) / world;
    const int tb0 = std::min(plan.target_blocks, rank * bpr), tb1 = std::min(plan.target_blocks, tb0 + bpr);
    const int64_t shard = (int64_t)bpr * kMrsThreads;
    if ((rc = ensure(&d_shard, &cap_shard, 6 * shard))) return rc;
    if ((rc = ensure(&d_gather, &cap_gather, 6 * shard * world))) return rc;
    e = mrs_launch_blocks(plan, tb0, tb1, state, state, 12, d_f, d_n, rs.epsilon, rs.mu, d_shard, d_shard + 3 * shard,
                          d_scratch, d_counters, d_flags, stream);
    if (e != cudaSuccess) return fail(PSWIM_ECUDA, std::string("mrs_launch_blocks: ") + cudaGetErrorString(e));
    if (tr->allgather(tr->user, d_shard, d_gather, 6 * shard, stream) != 0)
        return fail(PSWIM_ECOMM, "propagate_sharded: allgather failed");
    e = unshard_launch(d_gather, shard, total, u, w, stream);
    if (e != cudaSuccess) return fail(PSWIM_ECUDA, "unshard_launch");
    return PSWIM_OK;
}

int pswim_ctx::step_sharded(const pswim_transport* tr, int scheme, const double* state, double t, double dt,
                            double* out) {
    int rc = rhs_sharded(tr, state, t, d_u, d_w);
    if (rc) return rc;
    if (scheme == PSWIM_EULER) return advance(state, d_u, d_w, dt, out);
    rc = advance(state, d_u, d_w, 0.5 * dt, d_mid);
    if (rc) return rc;
    rc = rhs_sharded(tr, d_mid, t + 0.5 * dt, d_u, d_w);
    if (rc) return rc;
    return advance(state, d_u, d_w, dt, out);
}

pswim_ctx::~pswim_ctx() {
    cudaSetDevice(device);
    if (stream) cudaStreamSynchronize(stream);
    harvest_timing();
    for (double* p : {d_pos, d_f, d_n, d_u, d_w, d_lj, d_mid, d_scratch, d_metric, h_in, h_a, h_b, h_c, h_o1, h_o2,
                      d_shard, d_gather})
        if (p) cudaFree(p);
    if (d_counters) cudaFree(d_counters);
    lj_work.release();
    if (graph_exec) cudaGraphExecDestroy(graph_exec);
    for (double* p : {d_gstate, d_times, d_times_all})
        if (p) cudaFree(p);
    if (h_times) cudaFreeHost(h_times);
    if (times_done) cudaEventDestroy(times_done);
    if (d_flags) cudaFree(d_flags);
    if (h_flags) cudaFreeHost(h_flags);
    if (stream) cudaStreamDestroy(stream);
}

// ---------------------------------------------------------------------------------------
// C ABI
// ---------------------------------------------------------------------------------------
extern "C" {

pswim_ctx* pswim_create(int device, const pswim_scenario* sc, int stream_priority) {
    auto* ctx = new pswim_ctx();
    ctx->device = device;
    if (cudaSetDevice(device) != cudaSuccess) {
        delete ctx;
        return nullptr;
    }
    pswim::preload_kernels(device);
    if (cudaStreamCreateWithPriority(&ctx->stream, cudaStreamNonBlocking, stream_priority) != cudaSuccess ||
        cudaMalloc(&ctx->d_flags, sizeof(unsigned)) != cudaSuccess ||
        cudaMallocHost(&ctx->h_flags, sizeof(unsigned)) != cudaSuccess ||
        cudaMalloc(&ctx->d_metric, sizeof(double)) != cudaSuccess) {
        delete ctx;
        return nullptr;
    }
    *ctx->h_flags = 0;
    cudaMemsetAsync(ctx->d_flags, 0, sizeof(unsigned), ctx->stream);
    if (sc) {
        std::string err;
        if (resolve_scenario(sc, &ctx->rs, &err) != PSWIM_OK) {
            delete ctx;
            return nullptr;
        }
        ctx->has_scenario = true;
        ctx->sc = *sc;
        ctx->rp = rod_params(sc, ctx->rs);
        const size_t n3 = 3 * static_cast<size_t>(ctx->rs.total_nodes);
        size_t c0 = 0, c1 = 0, c2 = 0, c3 = 0, c4 = 0, c5 = 0, c6 = 0;
        if (ctx->ensure(&ctx->d_pos, &c0, n3) || ctx->ensure(&ctx->d_f, &c1, n3) || ctx->ensure(&ctx->d_n, &c2, n3) ||
            ctx->ensure(&ctx->d_u, &c3, n3) || ctx->ensure(&ctx->d_w, &c4, n3) || ctx->ensure(&ctx->d_lj, &c5, n3) ||
            ctx->ensure(&ctx->d_mid, &c6, 4 * n3)) {
            delete ctx;
            return nullptr;
        }
        const MrsPlan plan = mrs_plan(ctx->rs.total_nodes, ctx->rs.total_nodes);
        if (ctx->ensure_mrs(plan)) {
            delete ctx;
            return nullptr;
        }
        if (ctx->rp.rods >= 2 && ctx->rp.lj_well > 0.0 && ctx->rs.total_nodes >= kLjCellsMinNodes) {
            // cell-list workspace (its kernels are loaded by preload_kernels)
            if (lj_cells_reserve(ctx->rs.total_nodes, &ctx->lj_work, ctx->stream) != cudaSuccess) {
                delete ctx;
                return nullptr;
            }
        }
    }
    if (cudaStreamSynchronize(ctx->stream) != cudaSuccess) {
        delete ctx;
        return nullptr;
    }
    return ctx;
}

void pswim_destroy(pswim_ctx* ctx) { delete ctx; }
const char* pswim_last_error(const pswim_ctx* ctx) { return ctx ? ctx->err.c_str() : "null context"; }
void* pswim_stream(pswim_ctx* ctx) { return ctx ? ctx->stream : nullptr; }
int pswim_device(const pswim_ctx* ctx) { return ctx ? ctx->device : -1; }
int pswim_sync(pswim_ctx* ctx) { return ctx ? ctx->sync() : PSWIM_EINVAL; }

static bool direct_out_enabled() {
    static const bool on = [] {
        const char* e = std::getenv("PSWIM_DIRECT_OUT");  // dev knob: 0 = always copy back
        return !(e && e[0] == '0');
    }();
    return on;
}

static bool upload_enabled() {
    static const bool on = [] {
        const char* e = std::getenv("PSWIM_SM_UPLOAD");  // dev knob: 0 = always DMA copies
        return !(e && e[0] == '0');
    }();
    return on;
}

static int check_kp(pswim_ctx* ctx, const pswim_kernel_params* kp) {
    // check_inputs, stokes.cpp:12-17
    if (!kp || kp->epsilon <= 0.0 || kp->mu <= 0.0) return ctx->fail(PSWIM_EINVAL, "stokes: epsilon and mu must be positive");
    if (kp->wall_mode == 1)
        return ctx->fail(PSWIM_EUNSUPPORTED_WALL, "stokes: image_wall correction is not implemented; use free_space");
    return PSWIM_OK;
}

int pswim_mrs_velocities(pswim_ctx* ctx, const double* d_targets, int64_t nt, const double* d_sources,
                         const double* d_f, const double* d_n, int64_t ns, const pswim_kernel_params* kp,
                         double* d_u, double* d_omega) {
    if (!ctx) return PSWIM_EINVAL;
    int rc = check_kp(ctx, kp);
    if (rc) return rc;
    if (nt < 0 || ns < 0) return ctx->fail(PSWIM_EINVAL, "stokes: negative sizes");
    if ((rc = ctx->use())) return rc;
    if (nt == 0) return PSWIM_OK;
    if (ns == 0) {
        CK(cudaMemsetAsync(d_u, 0, sizeof(double) * 3 * nt, ctx->stream));
        CK(cudaMemsetAsync(d_omega, 0, sizeof(double) * 3 * nt, ctx->stream));
        return PSWIM_OK;
    }
    return ctx->mrs(d_targets, nt, d_sources, d_f, d_n, ns, kp->epsilon, kp->mu, d_u, d_omega);
}

int pswim_mrs_velocities_host(pswim_ctx* ctx, const double* h_t, int64_t nt, const double* h_s, const double* h_f,
                              const double* h_n, int64_t ns, const pswim_kernel_params* kp, double* h_u,
                              double* h_w) {
    if (!ctx) return PSWIM_EINVAL;
    int rc = check_kp(ctx, kp);
    if (rc) return rc;
    if (nt < 0 || ns < 0) return ctx->fail(PSWIM_EINVAL, "stokes: negative sizes");
    if ((rc = ctx->use())) return rc;
    const size_t t3 = 3 * static_cast<size_t>(nt), s3 = 3 * static_cast<size_t>(ns);
    if ((rc = ctx->ensure(&ctx->h_in, &ctx->cap_in, t3 > 0 ? t3 : 1))) return rc;
    if ((rc = ctx->ensure(&ctx->h_a, &ctx->cap_a, s3 > 0 ? s3 : 1))) return rc;
    if ((rc = ctx->ensure(&ctx->h_b, &ctx->cap_b, s3 > 0 ? s3 : 1))) return rc;
    if ((rc = ctx->ensure(&ctx->h_c, &ctx->cap_c, s3 > 0 ? s3 : 1))) return rc;
    if ((rc = ctx->ensure(&ctx->h_o1, &ctx->cap_o1, t3 > 0 ? t3 : 1))) return rc;
    if ((rc = ctx->ensure(&ctx->h_o2, &ctx->cap_o2, t3 > 0 ? t3 : 1))) return rc;
    // targets = sources (the rhs call, propagators.cpp:87): one copy serves both
    const bool same = h_t == h_s && nt == ns;
    // outputs in page-locked host memory are written by the kernel itself (mapped, over PCIe:
    // no separate device -> host copies)
    double *out_u = ctx->h_o1, *out_w = ctx->h_o2;
    bool direct = false;
    if (nt > 0 && ns > 0 && direct_out_enabled()) {
        cudaPointerAttributes au{}, aw{};
        if (cudaPointerGetAttributes(&au, h_u) == cudaSuccess && cudaPointerGetAttributes(&aw, h_w) == cudaSuccess &&
            au.type == cudaMemoryTypeHost && aw.type == cudaMemoryTypeHost && au.devicePointer && aw.devicePointer) {
            out_u = static_cast<double*>(au.devicePointer);
            out_w = static_cast<double*>(aw.devicePointer);
            direct = true;
        }
        cudaGetLastError();
    }
    // inputs: page-locked (mapped) arrays are pulled by an SM upload kernel (many requests in
    // flight), pageable ones by DMA copies
    const double* dev_in[4] = {nullptr, nullptr, nullptr, nullptr};
    bool mapped_in = ns > 0 && upload_enabled();
    const double* hin[4] = {same ? nullptr : h_t, h_s, h_f, h_n};
    for (int k = 0; k < 4 && mapped_in; ++k) {
        if (!hin[k]) continue;
        cudaPointerAttributes a{};
        mapped_in = cudaPointerGetAttributes(&a, hin[k]) == cudaSuccess && a.type == cudaMemoryTypeHost &&
                    a.devicePointer;
        dev_in[k] = mapped_in ? static_cast<const double*>(a.devicePointer) : nullptr;
    }
    cudaGetLastError();
    if (mapped_in) {
        if (!same) {
            const double* s1[3] = {dev_in[0], nullptr, nullptr};
            double* d1[3] = {ctx->h_in, nullptr, nullptr};
            const int64_t n1[3] = {(int64_t)t3, 0, 0};
            CK(upload_launch(s1, d1, n1, ctx->stream));
        }
        const double* s3v[3] = {dev_in[1], dev_in[2], dev_in[3]};
        double* d3v[3] = {ctx->h_a, ctx->h_b, ctx->h_c};
        const int64_t n3[3] = {(int64_t)s3, (int64_t)s3, (int64_t)s3};
        CK(upload_launch(s3v, d3v, n3, ctx->stream));
    } else {
        if (!same) CK(cudaMemcpyAsync(ctx->h_in, h_t, t3 * sizeof(double), cudaMemcpyHostToDevice, ctx->stream));
        CK(cudaMemcpyAsync(ctx->h_a, h_s, s3 * sizeof(double), cudaMemcpyHostToDevice, ctx->stream));
        CK(cudaMemcpyAsync(ctx->h_b, h_f, s3 * sizeof(double), cudaMemcpyHostToDevice, ctx->stream));
        CK(cudaMemcpyAsync(ctx->h_c, h_n, s3 * sizeof(double), cudaMemcpyHostToDevice, ctx->stream));
    }
    rc = pswim_mrs_velocities(ctx, same ? ctx->h_a : ctx->h_in, nt, ctx->h_a, ctx->h_b, ctx->h_c, ns, kp, out_u,
                              out_w);
    if (rc) return rc;
    if (!direct) {
        CK(cudaMemcpyAsync(h_u, ctx->h_o1, t3 * sizeof(double), cudaMemcpyDeviceToHost, ctx->stream));
        CK(cudaMemcpyAsync(h_w, ctx->h_o2, t3 * sizeof(double), cudaMemcpyDeviceToHost, ctx->stream));
    }
    return ctx->sync();
}

int pswim_h_functions(pswim_ctx* ctx, const double* d_r, int64_t count, double eps, double* d_h5) {
    if (!ctx) return PSWIM_EINVAL;
    if (eps <= 0.0) return ctx->fail(PSWIM_EINVAL, "h_functions: r >= 0 and epsilon > 0 required");
    int rc = ctx->use();
    if (rc) return rc;
    CK(h_functions_launch(d_r, count, eps, d_h5, ctx->stream));
    return PSWIM_OK;
}

int pswim_sqrt_rotation_batched(pswim_ctx* ctx, const double* d_r9, int64_t count, double* d_s9) {
    if (!ctx) return PSWIM_EINVAL;
    int rc = ctx->use();
    if (rc) return rc;
    CK(sqrt_batched_launch(d_r9, count, d_s9, ctx->stream));
    return PSWIM_OK;
}

int pswim_sqrt_rotation_host(pswim_ctx* ctx, const double* h_r9, int64_t count, double* h_s9) {
    if (!ctx) return PSWIM_EINVAL;
    int rc = ctx->use();
    if (rc) return rc;
    const size_t n = 9 * static_cast<size_t>(count);
    if ((rc = ctx->ensure(&ctx->h_in, &ctx->cap_in, n > 0 ? n : 1))) return rc;
    if ((rc = ctx->ensure(&ctx->h_o1, &ctx->cap_o1, n > 0 ? n : 1))) return rc;
    CK(cudaMemcpyAsync(ctx->h_in, h_r9, n * sizeof(double), cudaMemcpyHostToDevice, ctx->stream));
    CK(sqrt_batched_launch(ctx->h_in, count, ctx->h_o1, ctx->stream));
    CK(cudaMemcpyAsync(h_s9, ctx->h_o1, n * sizeof(double), cudaMemcpyDeviceToHost, ctx->stream));
    return ctx->sync();
}

int pswim_rod_loads(pswim_ctx* ctx, const double* d_state, double t, double* d_f, double* d_n, double* d_seg_force,
                    double* d_seg_moment) {
    if (!ctx) return PSWIM_EINVAL;
    if (!ctx->has_scenario) return ctx->fail(PSWIM_EINVAL, "rod_loads: context has no scenario");
    int rc = ctx->use();
    if (rc) return rc;
    CK(rod_loads_launch(ctx->rp, d_state, t, nullptr, d_f, d_n, d_seg_force, d_seg_moment, nullptr, nullptr,
                        nullptr, ctx->d_flags, ctx->stream));
    return PSWIM_OK;
}

int pswim_lj_forces(pswim_ctx* ctx, const double* d_state, double* d_forces) {
    if (!ctx) return PSWIM_EINVAL;
    if (!ctx->has_scenario) return ctx->fail(PSWIM_EINVAL, "lj: context has no scenario");
    int rc = ctx->use();
    if (rc) return rc;
    if (ctx->rp.rods < 2) {
        CK(cudaMemsetAsync(d_forces, 0, sizeof(double) * 3 * ctx->rp.rods * ctx->rp.m, ctx->stream));
        return PSWIM_OK;
    }
    return ctx->lj(d_state, d_forces);
    return PSWIM_OK;
}

int pswim_lj_forces_host(pswim_ctx* ctx, const double* h_state, double* h_forces) {
    if (!ctx) return PSWIM_EINVAL;
    if (!ctx->has_scenario) return ctx->fail(PSWIM_EINVAL, "lj: context has no scenario");
    int rc = ctx->use();
    if (rc) return rc;
    const size_t n = static_cast<size_t>(ctx->rp.rods * ctx->rp.m);
    if ((rc = ctx->ensure(&ctx->h_in, &ctx->cap_in, 12 * n))) return rc;
    if ((rc = ctx->ensure(&ctx->h_o1, &ctx->cap_o1, 3 * n))) return rc;
    CK(cudaMemcpyAsync(ctx->h_in, h_state, 12 * n * sizeof(double), cudaMemcpyHostToDevice, ctx->stream));
    if ((rc = pswim_lj_forces(ctx, ctx->h_in, ctx->h_o1))) return rc;
    CK(cudaMemcpyAsync(h_forces, ctx->h_o1, 3 * n * sizeof(double), cudaMemcpyDeviceToHost, ctx->stream));
    return ctx->sync();
}

int pswim_rhs(pswim_ctx* ctx, const double* d_state, double t, const double* d_ef, const double* d_en, double* d_u,
              double* d_omega) {
    if (!ctx) return PSWIM_EINVAL;
    int rc = ctx->use();
    if (rc) return rc;
    if ((d_ef == nullptr) != (d_en == nullptr)) return ctx->fail(PSWIM_EINVAL, "rhs: extra loads need both f and n");
    return ctx->rhs(d_state, t, d_ef, d_en, d_u, d_omega);
}

int pswim_advance_state(pswim_ctx* ctx, const double* d_state, const double* d_u, const double* d_omega, double dt,
                        double* d_out) {
    if (!ctx) return PSWIM_EINVAL;
    if (!ctx->has_scenario) return ctx->fail(PSWIM_EINVAL, "advance_state: context has no scenario");
    int rc = ctx->use();
    if (rc) return rc;
    return ctx->advance(d_state, d_u, d_omega, dt, d_out);
}

int pswim_step(pswim_ctx* ctx, int scheme, const double* d_state, double t, double dt, double* d_out) {
    if (!ctx) return PSWIM_EINVAL;
    if (!ctx->has_scenario) return ctx->fail(PSWIM_EINVAL, "step: context has no scenario");
    int rc = ctx->use();
    if (rc) return rc;
    return ctx->step(scheme, d_state, t, dt, d_out);
}

int pswim_propagate(pswim_ctx* ctx, const double* d_in, double t0, double t1, int scheme, int64_t spi, double dt,
                    double* d_out) {
    if (!ctx) return PSWIM_EINVAL;
    int rc = ctx->use();
    if (rc) return rc;
    rc = ctx->propagate_async(d_in, t0, t1, scheme, spi, dt, d_out);
    if (rc) return rc;
    return ctx->sync();
}

int pswim_propagate_host(pswim_ctx* ctx, const double* h_in, double t0, double t1, int scheme, int64_t spi, double dt,
                         double* h_out) {
    if (!ctx) return PSWIM_EINVAL;
    if (!ctx->has_scenario) return ctx->fail(PSWIM_EINVAL, "propagate: context has no scenario");
    int rc = ctx->use();
    if (rc) return rc;
    const size_t n = 12 * static_cast<size_t>(ctx->rs.total_nodes);
    if ((rc = ctx->ensure(&ctx->h_in, &ctx->cap_in, n))) return rc;
    CK(cudaMemcpyAsync(ctx->h_in, h_in, n * sizeof(double), cudaMemcpyHostToDevice, ctx->stream));
    rc = ctx->propagate_async(ctx->h_in, t0, t1, scheme, spi, dt, ctx->h_in);
    if (rc) return rc;
    CK(cudaMemcpyAsync(h_out, ctx->h_in, n * sizeof(double), cudaMemcpyDeviceToHost, ctx->stream));
    return ctx->sync();
}

int pswim_fused_profile(pswim_ctx* ctx, const double* d_in, double t0, double t1, int scheme, int64_t spi,
                        double* d_out, uint64_t* h_cycles7) {
    if (!ctx || !h_cycles7) return PSWIM_EINVAL;
    if (!ctx->has_scenario || fused_cluster_size(ctx->rp, ctx->fused_max_cs) == 0)
        return ctx->fail(PSWIM_EINVAL, "fused_profile: scenario not eligible for the fused path");
    int rc = ctx->use();
    if (rc) return rc;
    if (t1 < t0) return ctx->fail(PSWIM_EINVAL, "propagate: t1 < t0");
    int64_t steps = 0;
    double dt = 0.0;
    if ((rc = ctx->resolve_steps(t0, t1, spi, 0.0, &steps, &dt))) return rc;
    const size_t bytes = sizeof(double) * 12 * static_cast<size_t>(ctx->rp.rods * ctx->rp.m);
    unsigned long long* prof = nullptr;
    CK(cudaMalloc(&prof, sizeof(unsigned long long) * kFusedPhases));
    cudaError_t e = cudaMemsetAsync(prof, 0, sizeof(unsigned long long) * kFusedPhases, ctx->stream);
    if (e == cudaSuccess && d_in != d_out)
        e = cudaMemcpyAsync(d_out, d_in, bytes, cudaMemcpyDeviceToDevice, ctx->stream);
    if (e == cudaSuccess)
        e = fused_propagate_launch(ctx->rp, d_out, steps, t0, dt, scheme, ctx->d_flags, ctx->stream, prof,
                                   ctx->fused_max_cs);
    if (e == cudaSuccess)
        e = cudaMemcpyAsync(h_cycles7, prof, sizeof(unsigned long long) * kFusedPhases, cudaMemcpyDeviceToHost,
                            ctx->stream);
    rc = e == cudaSuccess ? ctx->sync() : ctx->fail(PSWIM_ECUDA, std::string("fused_profile: ") + cudaGetErrorString(e));
    cudaStreamSynchronize(ctx->stream);
    cudaFree(prof);
    return rc;
}

int pswim_set_graphs(pswim_ctx* ctx, int enable) {
    if (!ctx) return PSWIM_EINVAL;
    const int prev = ctx->graphs_on ? 1 : 0;
    ctx->graphs_on = enable != 0;
    return prev;
}

int pswim_set_lj_mode(pswim_ctx* ctx, int mode) {
    if (!ctx || mode < 0 || mode > 2) return -PSWIM_EINVAL;
    const int prev = ctx->lj_mode;
    ctx->lj_mode = mode;
    return prev;
}

int pswim_set_fused(pswim_ctx* ctx, int enable) {
    if (!ctx) return PSWIM_EINVAL;
    ctx->fused_on = enable != 0;
    ctx->fused_max_cs = (enable == 2 || enable == 4 || enable == 8 || enable == 16) ? enable : 0;
    return ctx->has_scenario ? fused_cluster_size(ctx->rp, ctx->fused_max_cs) : 0;
}

int pswim_propagate_sharded(pswim_ctx* ctx, const pswim_transport* tr, const double* d_in, double t0, double t1,
                            int scheme, int64_t spi, double dtc, double* d_out) {
    if (!ctx || !tr || !tr->allgather) return PSWIM_EINVAL;
    if (!ctx->has_scenario) return ctx->fail(PSWIM_EINVAL, "propagate: context has no scenario");
    int rc = ctx->use();
    if (rc) return rc;
    if (t1 < t0) return ctx->fail(PSWIM_EINVAL, "propagate: t1 < t0");
    const size_t bytes = sizeof(double) * 12 * static_cast<size_t>(ctx->rp.rods * ctx->rp.m);
    if (d_in != d_out) CK(cudaMemcpyAsync(d_out, d_in, bytes, cudaMemcpyDeviceToDevice, ctx->stream));
    if (t1 > t0) {
        int64_t steps = 0;
        double dt = 0.0;
        if ((rc = ctx->resolve_steps(t0, t1, spi, dtc, &steps, &dt))) return rc;
        double t = t0;
        for (int64_t i = 0; i < steps; ++i) {
            if ((rc = ctx->step_sharded(tr, scheme, d_out, t, dt, d_out))) return rc;
            t += dt;  // propagators.cpp:159
        }
    }
    return ctx->sync();
}

void pswim_timing_enable(pswim_ctx* ctx, int on) {
    if (ctx) ctx->timing_on = on != 0;
}
void pswim_timing_reset(pswim_ctx* ctx) {
    if (!ctx) return;
    cudaStreamSynchronize(ctx->stream);
    ctx->harvest_timing();
    ctx->stage_seconds[0] = ctx->stage_seconds[1] = ctx->stage_seconds[2] = 0.0;
}
pswim_timing pswim_timing_snapshot(pswim_ctx* ctx) {
    pswim_timing t{0, 0, 0};
    if (!ctx) return t;
    cudaStreamSynchronize(ctx->stream);
    ctx->harvest_timing();
    t.initialization = ctx->stage_seconds[0];
    t.velocity = ctx->stage_seconds[1];
    t.triad_update = ctx->stage_seconds[2];
    return t;
}

int pswim_position_metric(pswim_ctx* ctx, const double* d_x, const double* d_y, int64_t len, double* h_result) {
    if (!ctx) return PSWIM_EINVAL;
    if (len % 12 != 0) return ctx->fail(PSWIM_EINVAL, "rod_position_metric: inconsistent packed states");
    int rc = ctx->use();
    if (rc) return rc;
    CK(metric_launch(d_x, d_y, len, nullptr, nullptr, ctx->d_metric, ctx->stream));
    CK(cudaMemcpyAsync(h_result, ctx->d_metric, sizeof(double), cudaMemcpyDeviceToHost, ctx->stream));
    return ctx->sync();
}

int pswim_parareal_correct(pswim_ctx* ctx, const double* d_xp, const double* d_gn, const double* d_go, int64_t len,
                           double* d_out) {
    if (!ctx) return PSWIM_EINVAL;
    int rc = ctx->use();
    if (rc) return rc;
    CK(correct_launch(d_xp, d_gn, d_go, len, d_out, ctx->stream));
    return PSWIM_OK;
}

int pswim_dfma_peak(pswim_ctx* ctx, double* flops_per_s, double* ms_out) {
    if (!ctx) return PSWIM_EINVAL;
    int rc = ctx->use();
    if (rc) return rc;
    double* sink = nullptr;
    CK(cudaMalloc(&sink, sizeof(double)));
    int sms = 148;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, ctx->device);
    const int blocks = sms * 8;
    const int iters = 2048;
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    float best = 1e30f;
    for (int rep = 0; rep < 4; ++rep) {
        cudaEventRecord(a, ctx->stream);
        dfma_launch(sink, blocks, iters, ctx->stream);
        cudaEventRecord(b, ctx->stream);
        cudaEventSynchronize(b);
        float ms = 0.f;
        cudaEventElapsedTime(&ms, a, b);
        if (rep > 0 && ms < best) best = ms;  // first launch is warm-up
    }
    cudaEventDestroy(a);
    cudaEventDestroy(b);
    cudaFree(sink);
    const double flops = 2.0 * 8.0 * 16.0 * iters * (double)blocks * 256.0;
    *flops_per_s = flops / (1e-3 * best);
    if (ms_out) *ms_out = best;
    return ctx->sync();
}

const char* pswim_version(void) { return "pswim-b200 0.1 (sm_100a)"; }

}  // extern "C"
