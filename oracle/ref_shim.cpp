// ref_shim.cpp — TEST INFRASTRUCTURE ONLY.
//
// extern "C" wrappers over the UNMODIFIED reference library (arxiv/paper_2604_12083,
// /root/reference/proj/src + tests/oracles.cpp), compiled by oracle/Makefile into
// oracle/_ref/libpintswim_ref.so.  Used (a) to pin the C restatement in oracle/ bitwise,
// (b) to generate tests/golden/ fixtures, (c) as the CPU baseline / `bench.py --impl
// reference` arm (the reference's own OpenMP path timed on the host cores).
// Signatures mirror oracle/pswim_oracle.h with a `ref_` prefix.
#include <cmath>
#include <cstring>
#include <exception>
#include <random>
#include <stdexcept>
#include <vector>

#ifdef _OPENMP
#include <omp.h>
#endif

#include "../include/pswim_c.h"
#include "oracles.hpp"
#include "pintswim/harness.hpp"
#include "pintswim/io.hpp"
#include "pintswim/parareal.hpp"
#include "pintswim/propagators.hpp"
#include "pintswim/rod.hpp"
#include "pintswim/rotation.hpp"
#include "pintswim/scenario.hpp"
#include "pintswim/stokes.hpp"

using namespace pintswim;

namespace {

int code_of(const std::exception_ptr& e) {
    try {
        std::rethrow_exception(e);
    } catch (const StiffnessError&) {
        return PSWIM_ESTIFF;
    } catch (const std::invalid_argument&) {
        return PSWIM_EINVAL;
    } catch (const std::logic_error&) {
        return PSWIM_ESTATE;
    } catch (const std::runtime_error& err) {
        const std::string what = err.what();
        if (what.find("degenerate") != std::string::npos) return PSWIM_EDEGENERATE;
        if (what.find("image_wall") != std::string::npos) return PSWIM_EUNSUPPORTED_WALL;
        return PSWIM_EINVAL;
    } catch (...) {
        return PSWIM_EINVAL;
    }
}

#define GUARD(...)                                  \
    try {                                           \
        __VA_ARGS__;                                \
        return PSWIM_OK;                            \
    } catch (...) {                                 \
        return code_of(std::current_exception());   \
    }

std::vector<Vec3> vecs(const double* p, int64_t n) {
    std::vector<Vec3> v(static_cast<std::size_t>(n));
    for (int64_t i = 0; i < n; ++i) v[i] = {p[3 * i], p[3 * i + 1], p[3 * i + 2]};
    return v;
}
void put(double* p, const std::vector<Vec3>& v) {
    for (std::size_t i = 0; i < v.size(); ++i) {
        p[3 * i] = v[i].x;
        p[3 * i + 1] = v[i].y;
        p[3 * i + 2] = v[i].z;
    }
}
Mat3 mat(const double* p) {
    Mat3 m;
    for (int i = 0; i < 9; ++i) m.m[i] = p[i];
    return m;
}
void put(double* p, const Mat3& m) {
    for (int i = 0; i < 9; ++i) p[i] = m.m[i];
}

RodState rod_of(const double* p, int64_t m) {
    RodState r;
    r.x.resize(m);
    r.d1.resize(m);
    r.d2.resize(m);
    r.d3.resize(m);
    for (int64_t k = 0; k < m; ++k) {
        const double* q = p + 12 * k;
        r.x[k] = {q[0], q[1], q[2]};
        r.d1[k] = {q[3], q[4], q[5]};
        r.d2[k] = {q[6], q[7], q[8]};
        r.d3[k] = {q[9], q[10], q[11]};
    }
    return r;
}
void put_rod(double* p, const RodState& r) {
    for (std::size_t k = 0; k < r.x.size(); ++k) {
        double* q = p + 12 * k;
        for (int c = 0; c < 3; ++c) {
            q[c] = r.x[k][c];
            q[3 + c] = r.d1[k][c];
            q[6 + c] = r.d2[k][c];
            q[9 + c] = r.d3[k][c];
        }
    }
}

ScenarioConfig cfg_of(const pswim_scenario* s) {
    ScenarioConfig c;
    c.rod_count = static_cast<std::size_t>(s->rod_count);
    c.nodes_per_rod = static_cast<std::size_t>(s->nodes_per_rod);
    c.rod_length = s->rod_length;
    c.material = {s->a1, s->a2, s->a3, s->b1, s->b2, s->b3};
    c.waveform = {s->amplitude, s->frequency, s->wavelength};
    c.epsilon = s->epsilon;
    c.mu = s->mu;
    c.wall_mode = s->wall_mode ? WallMode::image_wall : WallMode::free_space;
    c.lj_well_depth = s->lj_well_depth;
    c.lj_sigma = s->lj_sigma;
    c.wall_clearance = s->wall_clearance;
    c.seed = s->seed;
    c.fine_dt = s->fine_dt;
    c.horizon = s->horizon;
    c.placement = s->placement ? Placement::random : Placement::grid;
    return c;
}

}  // namespace

extern "C" {

void ref_set_threads(int n) {
#ifdef _OPENMP
    omp_set_num_threads(n);
#else
    (void)n;
#endif
}

int ref_max_threads(void) {
#ifdef _OPENMP
    return omp_get_max_threads();
#else
    return 1;
#endif
}

void ref_scenario_defaults(pswim_scenario* s) {
    const ScenarioConfig c;
    s->rod_count = static_cast<int64_t>(c.rod_count);
    s->nodes_per_rod = static_cast<int64_t>(c.nodes_per_rod);
    s->rod_length = c.rod_length;
    s->a1 = c.material.a1; s->a2 = c.material.a2; s->a3 = c.material.a3;
    s->b1 = c.material.b1; s->b2 = c.material.b2; s->b3 = c.material.b3;
    s->amplitude = c.waveform.amplitude;
    s->frequency = c.waveform.frequency;
    s->wavelength = c.waveform.wavelength;
    s->epsilon = c.epsilon;
    s->mu = c.mu;
    s->wall_mode = 0;
    s->placement = 0;
    s->lj_well_depth = c.lj_well_depth;
    s->lj_sigma = c.lj_sigma;
    s->wall_clearance = c.wall_clearance;
    s->seed = c.seed;
    s->fine_dt = c.fine_dt;
    s->horizon = c.horizon;
}

// ---- stokes ----
void ref_h_functions(double r, double eps, double* h) {
    const auto v = h_functions(r, eps);
    h[0] = v.h1; h[1] = v.h2; h[2] = v.h3; h[3] = v.h4; h[4] = v.h5;
}

int ref_evaluate_velocities(const double* tgt, int64_t nt, const double* src, const double* f,
                            const double* n, int64_t ns, double eps, double mu, int wall, double* u,
                            double* w, int parallel) {
    GUARD({
        const auto t = vecs(tgt, nt);
        const auto s = vecs(src, ns);
        LoadSet loads{vecs(f, ns), vecs(n, ns)};
        const KernelParams kp{eps, mu, wall ? WallMode::image_wall : WallMode::free_space};
        const auto out = parallel ? evaluate_velocities(t, s, loads, kp) : evaluate_velocities_serial(t, s, loads, kp);
        put(u, out.u);
        put(w, out.omega);
    })
}

int ref_grand_mobility(const double* nodes, int64_t n, double eps, double mu, double* out) {
    GUARD({
        const auto m = assemble_grand_mobility(vecs(nodes, n), KernelParams{eps, mu, WallMode::free_space}, 1u << 20);
        std::memcpy(out, m.data(), m.size() * sizeof(double));
    })
}

// ---- rotation ----
int ref_from_axis_angle(const double* axis, double angle, double* r9) {
    GUARD(put(r9, from_axis_angle({{axis[0], axis[1], axis[2]}, angle})))
}
void ref_to_axis_angle(const double* r9, double* axis, double* angle) {
    const auto aa = to_axis_angle(mat(r9));
    axis[0] = aa.axis.x; axis[1] = aa.axis.y; axis[2] = aa.axis.z;
    *angle = aa.angle;
}
void ref_sqrt_rotation(const double* r9, double* s9) { put(s9, sqrt_rotation(mat(r9))); }
void ref_sqrt_rotation_batched(const double* r9, int64_t count, double* s9) {
    for (int64_t i = 0; i < count; ++i) put(s9 + 9 * i, sqrt_rotation(mat(r9 + 9 * i)));
}
double ref_rotation_residual(const double* r9) { return rotation_residual(mat(r9)); }

// ---- rod ----
int ref_internal_loads(const double* rod12, int64_t m, double length, const double* mat6, const double* wave3,
                       double t, double* force, double* moment) {
    GUARD({
        const auto il = internal_loads(rod_of(rod12, m), RodDiscretization{static_cast<std::size_t>(m), length},
                                       MaterialParams{mat6[0], mat6[1], mat6[2], mat6[3], mat6[4], mat6[5]},
                                       WaveformParams{wave3[0], wave3[1], wave3[2]}, t);
        put(force, il.force);
        put(moment, il.moment);
    })
}

int ref_nodal_loads(const double* rod12, int64_t m, double length, const double* force, const double* moment,
                    double* f, double* n) {
    GUARD({
        InternalLoads il{vecs(force, m - 1), vecs(moment, m - 1)};
        const auto ls = nodal_loads(rod_of(rod12, m), RodDiscretization{static_cast<std::size_t>(m), length}, il);
        put(f, ls.f);
        put(n, ls.n);
    })
}

void ref_lj_repulsion(const double* state, int64_t rods, int64_t m, double well, double sigma, int64_t excl,
                      double* forces) {
    std::vector<RodState> rs;
    for (int64_t r = 0; r < rods; ++r) rs.push_back(rod_of(state + 12 * m * r, m));
    put(forces, lj_repulsion(rs, LJParams{well, sigma}, static_cast<std::size_t>(excl)));
}

int64_t ref_reorthonormalize(double* rod12, int64_t m, double tol) {
    auto r = rod_of(rod12, m);
    const auto touched = reorthonormalize(r, tol);
    put_rod(rod12, r);
    return static_cast<int64_t>(touched);
}

// ---- scenario ----
int ref_resolve(const pswim_scenario* s, pswim_resolved* out) {
    GUARD({
        const auto sc = make_scenario(cfg_of(s));
        out->ds = sc.disc.ds();
        out->epsilon = sc.kernel.epsilon;
        out->mu = sc.kernel.mu;
        out->lj_sigma = sc.lj.sigma;
        out->lj_cutoff = sc.lj.cutoff();
        out->lj_self_exclusion = static_cast<int64_t>(sc.lj_self_exclusion);
        out->total_nodes = s->rod_count * s->nodes_per_rod;
    })
}

int ref_build_initial_state(const pswim_scenario* s, double* state) {
    GUARD({
        const auto v = pack_state(build_initial_state(make_scenario(cfg_of(s))));
        std::memcpy(state, v.data(), v.size() * sizeof(double));
    })
}

// ---- propagators ----
static SystemState unpack(const pswim_scenario* s, const double* p) {
    const std::size_t n = static_cast<std::size_t>(12 * s->rod_count * s->nodes_per_rod);
    return unpack_state(parareal::Vec(p, p + n), static_cast<std::size_t>(s->rod_count),
                        static_cast<std::size_t>(s->nodes_per_rod));
}
static void pack(double* p, const SystemState& st) {
    const auto v = pack_state(st);
    std::memcpy(p, v.data(), v.size() * sizeof(double));
}

int ref_rhs(const pswim_scenario* s, const double* state, double t, const double* ef, const double* en,
            double* u, double* w) {
    GUARD({
        const auto sc = make_scenario(cfg_of(s));
        const int64_t total = s->rod_count * s->nodes_per_rod;
        LoadSet extra;
        if (ef && en) extra = LoadSet{vecs(ef, total), vecs(en, total)};
        const auto v = rhs(unpack(s, state), t, sc, (ef && en) ? &extra : nullptr);
        put(u, v.u);
        put(w, v.omega);
    })
}

int ref_advance_state(const pswim_scenario* s, const double* state, const double* u, const double* w, double dt,
                      double* out) {
    GUARD({
        const auto sc = make_scenario(cfg_of(s));
        const int64_t total = s->rod_count * s->nodes_per_rod;
        SystemVelocities v{vecs(u, total), vecs(w, total)};
        pack(out, advance_state(unpack(s, state), v, dt, sc));
    })
}

int ref_step(const pswim_scenario* s, int scheme, const double* state, double t, double dt, double* out) {
    GUARD({
        const auto sc = make_scenario(cfg_of(s));
        pack(out, scheme == PSWIM_EULER ? step_euler(unpack(s, state), t, dt, sc) : step_rk2(unpack(s, state), t, dt, sc));
    })
}

int ref_propagate(const pswim_scenario* s, const double* in, double t0, double t1, int scheme, int64_t steps,
                  double dt, double* out) {
    GUARD({
        const auto sc = make_scenario(cfg_of(s));
        const StepperConfig cfg{dt, scheme == PSWIM_EULER ? Scheme::euler : Scheme::rk2,
                                static_cast<std::size_t>(steps > 0 ? steps : 0)};
        pack(out, propagate(unpack(s, in), t0, t1, cfg, sc));
    })
}

double ref_position_metric(const double* x, const double* y, int64_t len) {
    return rod_position_metric()(parareal::Vec(x, x + len), parareal::Vec(y, y + len));
}

double ref_pointwise_metric(const double* x, const double* y, int64_t len, int64_t dim) {
    return parareal::pointwise_metric(static_cast<std::size_t>(dim))(parareal::Vec(x, x + len),
                                                                     parareal::Vec(y, y + len));
}

// ---- parareal ----
// parareal::run over the rod propagators of harness::prepare (harness.cpp:5-33).
int ref_parareal_rod(const pswim_scenario* s, double t0, double horizon, int intervals, int workers,
                     int max_iterations, double tolerance, int mode, int64_t fine_steps, int64_t coarse_steps,
                     const double* x0, const double* reference, double* states, double* eta_tilde, double* eta,
                     int* iterations_used, int* converged, double* idle) {
    GUARD({
        const auto sc = make_scenario(cfg_of(s));
        parareal::ParallelPlan plan;
        plan.t0 = t0;
        plan.horizon = horizon;
        plan.intervals = intervals;
        plan.workers = workers;
        plan.max_iterations = max_iterations;
        plan.tolerance = tolerance;
        plan.mode = mode ? parareal::Mode::pipelined : parareal::Mode::regular;
        const auto rods = static_cast<std::size_t>(s->rod_count);
        const auto nodes = static_cast<std::size_t>(s->nodes_per_rod);
        const StepperConfig fine_cfg{0.0, Scheme::rk2, static_cast<std::size_t>(fine_steps)};
        const StepperConfig coarse_cfg{0.0, Scheme::euler, static_cast<std::size_t>(coarse_steps)};
        parareal::PropagatorFn fine = [sc, rods, nodes, fine_cfg](double a, double b, const parareal::Vec& x) {
            return pack_state(propagate(unpack_state(x, rods, nodes), a, b, fine_cfg, sc));
        };
        parareal::PropagatorFn coarse = [sc, rods, nodes, coarse_cfg](double a, double b, const parareal::Vec& x) {
            return pack_state(propagate(unpack_state(x, rods, nodes), a, b, coarse_cfg, sc));
        };
        const std::size_t len = 12 * rods * nodes;
        std::vector<parareal::Vec> ref;
        if (reference) {
            for (int n = 0; n <= intervals; ++n) ref.emplace_back(reference + len * n, reference + len * (n + 1));
        }
        const auto res = parareal::run(plan, coarse, fine, parareal::Vec(x0, x0 + len), rod_position_metric(),
                                       reference ? &ref : nullptr);
        for (int n = 0; n <= intervals; ++n) std::memcpy(states + len * n, res.states[n].data(), len * sizeof(double));
        for (std::size_t k = 0; k < res.report.eta_tilde.size(); ++k) eta_tilde[k] = res.report.eta_tilde[k];
        if (eta) for (std::size_t k = 0; k < res.report.eta.size(); ++k) eta[k] = res.report.eta[k];
        *iterations_used = res.report.iterations_used;
        *converged = res.report.converged ? 1 : 0;
        if (idle) *idle = res.trace.total_idle();
    })
}

// Serial fine boundaries, harness.cpp:35-37 (coarse_sweep_initial with the fine propagator).
int ref_serial_fine_boundaries(const pswim_scenario* s, double t0, double horizon, int intervals,
                               int64_t fine_steps, const double* x0, double* states) {
    GUARD({
        const auto sc = make_scenario(cfg_of(s));
        parareal::ParallelPlan plan;
        plan.t0 = t0;
        plan.horizon = horizon;
        plan.intervals = intervals;
        const auto rods = static_cast<std::size_t>(s->rod_count);
        const auto nodes = static_cast<std::size_t>(s->nodes_per_rod);
        const StepperConfig fine_cfg{0.0, Scheme::rk2, static_cast<std::size_t>(fine_steps)};
        parareal::PropagatorFn fine = [sc, rods, nodes, fine_cfg](double a, double b, const parareal::Vec& x) {
            return pack_state(propagate(unpack_state(x, rods, nodes), a, b, fine_cfg, sc));
        };
        const std::size_t len = 12 * rods * nodes;
        const auto out = parareal::coarse_sweep_initial(plan, fine, parareal::Vec(x0, x0 + len));
        for (int n = 0; n <= intervals; ++n) std::memcpy(states + len * n, out[n].data(), len * sizeof(double));
    })
}

// ---- config hash / trajectory files (config.cpp:191-245, io.cpp:70-106) ----
static RunConfig run_config_of(const pswim_scenario* s, int intervals, int workers, double ratio, int max_iterations,
                               double tolerance, int mode, int fine_steps, int coarse_steps, int stride) {
    RunConfig c;
    c.scenario = cfg_of(s);
    c.intervals = intervals;
    c.workers = workers;
    c.ratio = ratio;
    c.max_iterations = max_iterations;
    c.tolerance = tolerance;
    c.mode = mode ? parareal::Mode::pipelined : parareal::Mode::regular;
    c.fine_steps_per_interval = fine_steps;
    c.coarse_steps_per_interval = coarse_steps;
    c.snapshot_stride = stride;
    return c;
}

void ref_config_hash(const pswim_scenario* s, int intervals, int workers, double ratio, int max_iterations,
                     double tolerance, int mode, int fine_steps, int coarse_steps, int stride, char* out17) {
    const auto h = run_config_of(s, intervals, workers, ratio, max_iterations, tolerance, mode, fine_steps,
                                 coarse_steps, stride)
                       .hash();
    std::memcpy(out17, h.c_str(), 17);
}

int ref_write_trajectory(const char* path, const pswim_scenario* s, int stride, int frames, const double* times,
                         const double* states) {
    GUARD({
        const auto cfg = run_config_of(s, 8, 2, 2.0, 10, 1e-10, 1, 100, 0, stride);
        TrajectoryWriter w(path, cfg);
        const std::size_t len = static_cast<std::size_t>(12 * s->rod_count * s->nodes_per_rod);
        for (int f = 0; f < frames; ++f) {
            w.append(times[f], unpack_state(parareal::Vec(states + len * f, states + len * (f + 1)),
                                            static_cast<std::size_t>(s->rod_count),
                                            static_cast<std::size_t>(s->nodes_per_rod)));
        }
        w.close();
    })
}

// ---- reference test oracles (tests/oracles.cpp) ----
void ref_dense_mobility_apply(const double* nodes, int64_t n, const double* f, const double* t, double eps,
                              double mu, double* u, double* w) {
    LoadSet loads{vecs(f, n), vecs(t, n)};
    const auto out = oracles::dense_mobility_apply(vecs(nodes, n), loads, KernelParams{eps, mu, WallMode::free_space});
    put(u, out.u);
    put(w, out.omega);
}

void ref_h_quadrature(double r, double eps, double* h) {
    const auto v = oracles::h_quadrature(r, eps);
    h[0] = v.h1; h[1] = v.h2; h[2] = v.h3; h[3] = v.h4; h[4] = v.h5;
}

double ref_elastic_energy(const double* rod12, int64_t m, double length, const double* mat6, const double* wave3,
                          double t) {
    return oracles::elastic_energy(rod_of(rod12, m), RodDiscretization{static_cast<std::size_t>(m), length},
                                   MaterialParams{mat6[0], mat6[1], mat6[2], mat6[3], mat6[4], mat6[5]},
                                   WaveformParams{wave3[0], wave3[1], wave3[2]}, t);
}

// Deterministic random draws with the reference helpers: kind 0 uniform(lo,hi), 1 random_unit,
// 2 random_vec(scale=lo).  Reproduces the inputs of the reference's own tests.
void ref_random_draws(uint64_t seed, int kind, double lo, double hi, int64_t count, double* out) {
    std::mt19937_64 rng(seed);
    for (int64_t i = 0; i < count; ++i) {
        if (kind == 0) {
            out[i] = oracles::uniform(rng, lo, hi);
        } else if (kind == 1) {
            const auto v = oracles::random_unit(rng);
            out[3 * i] = v.x; out[3 * i + 1] = v.y; out[3 * i + 2] = v.z;
        } else {
            const auto v = oracles::random_vec(rng, lo);
            out[3 * i] = v.x; out[3 * i + 1] = v.y; out[3 * i + 2] = v.z;
        }
    }
}

void ref_perturbed_rod(int64_t m, double length, uint64_t seed, double pj, double aj, double* rod12) {
    std::mt19937_64 rng(seed);
    put_rod(rod12, oracles::perturbed_rod(RodDiscretization{static_cast<std::size_t>(m), length}, rng, pj, aj));
}

}  // extern "C"
