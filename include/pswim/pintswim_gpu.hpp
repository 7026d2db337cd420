// pintswim_gpu.hpp — header-only drop-in adapter from the reference's C++ interfaces
// (arxiv/paper_2604_12083, proj/include/pintswim/*.hpp) onto the C-ABI of pswim_c.h.
//
// A maintainer of the reference adds this header and links libpswim.so; then
//
//   * pswim_gpu::evaluate_velocities(...)     replaces pintswim::evaluate_velocities
//                                             (stokes.hpp:43-44, called at propagators.cpp:87)
//   * pswim_gpu::sqrt_rotation(r)             replaces pintswim::sqrt_rotation (rotation.hpp:34)
//   * pswim_gpu::make_propagator(sc, ...)     returns a parareal::PropagatorFn (parareal.hpp:19)
//                                             usable wherever harness::prepare builds run.fine /
//                                             run.coarse (harness.cpp:26-31), so the reference's
//                                             own parareal::run drives the B200 propagators.
//   * pswim_gpu::propagate(state, ...)        replaces pintswim::propagate (propagators.hpp:52)
//
// Exceptions mirror the reference: std::invalid_argument, std::runtime_error,
// pintswim::StiffnessError.  Every call is thread safe (one device context per calling
// thread), which the PropagatorFn contract requires (parareal.cpp:213 calls it from m
// worker threads).
#pragma once

#include <map>
#include <memory>
#include <mutex>
#include <span>
#include <stdexcept>
#include <string>
#include <tuple>
#include <vector>

#include "../pswim_c.h"
#include "pintswim/io.hpp"
#include "pintswim/parareal.hpp"
#include "pintswim/propagators.hpp"
#include "pintswim/rotation.hpp"
#include "pintswim/scenario.hpp"
#include "pintswim/stokes.hpp"

namespace pswim_gpu {

static_assert(sizeof(pintswim::Vec3) == 3 * sizeof(double), "Vec3 must be three packed doubles");
static_assert(sizeof(pintswim::Mat3) == 9 * sizeof(double), "Mat3 must be nine packed doubles");

inline void throw_for(int rc, const char* what) {
    switch (rc) {
        case PSWIM_OK: return;
        case PSWIM_EINVAL:
        case PSWIM_ENONFINITE: throw std::invalid_argument(what);
        case PSWIM_ESTIFF: throw pintswim::StiffnessError(what);
        default: throw std::runtime_error(what);
    }
}

inline pswim_scenario to_c(const pintswim::ScenarioConfig& c) {
    pswim_scenario s;
    s.rod_count = static_cast<int64_t>(c.rod_count);
    s.nodes_per_rod = static_cast<int64_t>(c.nodes_per_rod);
    s.rod_length = c.rod_length;
    s.a1 = c.material.a1; s.a2 = c.material.a2; s.a3 = c.material.a3;
    s.b1 = c.material.b1; s.b2 = c.material.b2; s.b3 = c.material.b3;
    s.amplitude = c.waveform.amplitude;
    s.frequency = c.waveform.frequency;
    s.wavelength = c.waveform.wavelength;
    s.epsilon = c.epsilon;
    s.mu = c.mu;
    s.wall_mode = c.wall_mode == pintswim::WallMode::image_wall ? 1 : 0;
    s.placement = c.placement == pintswim::Placement::random ? 1 : 0;
    s.lj_well_depth = c.lj_well_depth;
    s.lj_sigma = c.lj_sigma;
    s.wall_clearance = c.wall_clearance;
    s.seed = c.seed;
    s.fine_dt = c.fine_dt;
    s.horizon = c.horizon;
    return s;
}

// One context per (thread, device, scenario): contexts own a stream and HBM workspaces.
class Contexts {
  public:
    static pswim_ctx* get(int device, const pswim_scenario* sc) {
        thread_local std::map<std::string, std::unique_ptr<pswim_ctx, void (*)(pswim_ctx*)>> cache;
        std::string key(reinterpret_cast<const char*>(&device), sizeof device);
        if (sc) key.append(reinterpret_cast<const char*>(sc), sizeof *sc);
        auto it = cache.find(key);
        if (it == cache.end()) {
            pswim_ctx* c = pswim_create(device, sc, 0);
            if (!c) throw std::runtime_error("pswim_create failed (no CUDA device?)");
            it = cache.emplace(key, std::unique_ptr<pswim_ctx, void (*)(pswim_ctx*)>(c, pswim_destroy)).first;
        }
        return it->second.get();
    }
};

// pintswim::evaluate_velocities on the B200 MRS kernel (host buffers in/out).
inline pintswim::VelocityField evaluate_velocities(std::span<const pintswim::Vec3> targets,
                                                   std::span<const pintswim::Vec3> sources,
                                                   const pintswim::LoadSet& loads, const pintswim::KernelParams& kp,
                                                   int device = 0) {
    if (loads.f.size() != sources.size() || loads.n.size() != sources.size())
        throw std::invalid_argument("stokes: load arrays must match source count");
    pintswim::VelocityField out;
    out.u.resize(targets.size());
    out.omega.resize(targets.size());
    const pswim_kernel_params p{kp.epsilon, kp.mu, kp.wall_mode == pintswim::WallMode::image_wall ? 1 : 0, 0};
    pswim_ctx* ctx = Contexts::get(device, nullptr);
    const int rc = pswim_mrs_velocities_host(
        ctx, reinterpret_cast<const double*>(targets.data()), static_cast<int64_t>(targets.size()),
        reinterpret_cast<const double*>(sources.data()), reinterpret_cast<const double*>(loads.f.data()),
        reinterpret_cast<const double*>(loads.n.data()), static_cast<int64_t>(sources.size()), &p,
        reinterpret_cast<double*>(out.u.data()), reinterpret_cast<double*>(out.omega.data()));
    throw_for(rc, pswim_last_error(ctx));
    return out;
}

// pintswim::sqrt_rotation, batched device kernel (one matrix here).
inline pintswim::Rot3 sqrt_rotation(const pintswim::Rot3& r, int device = 0) {
    pintswim::Rot3 s;
    pswim_ctx* ctx = Contexts::get(device, nullptr);
    throw_for(pswim_sqrt_rotation_host(ctx, r.m.data(), 1, s.m.data()), pswim_last_error(ctx));
    return s;
}

// pintswim::lj_repulsion (rod.cpp:124-174) on the device for the rods of scenario `sc` (the
// reference call site propagators.cpp:71 passes sc.lj and sc.lj_self_exclusion, which the
// context derives from the same ScenarioConfig): all-pairs below 2048 nodes, cell list above.
inline std::vector<pintswim::Vec3> lj_repulsion(const std::vector<pintswim::RodState>& rods,
                                                const pintswim::Scenario& sc, int device = 0) {
    const pswim_scenario s = to_c(sc.cfg);
    pswim_ctx* ctx = Contexts::get(device, &s);
    const pintswim::parareal::Vec in = pintswim::pack_state(rods);
    std::vector<pintswim::Vec3> out(in.size() / 12);
    throw_for(pswim_lj_forces_host(ctx, in.data(), reinterpret_cast<double*>(out.data())), pswim_last_error(ctx));
    return out;
}

// pintswim::propagate on the device (state in, state out; packed via pack_state).
inline pintswim::SystemState propagate(const pintswim::SystemState& state, double t0, double t1,
                                       const pintswim::StepperConfig& cfg, const pintswim::Scenario& sc,
                                       int device = 0) {
    const pswim_scenario s = to_c(sc.cfg);
    pswim_ctx* ctx = Contexts::get(device, &s);
    pintswim::parareal::Vec in = pintswim::pack_state(state);
    pintswim::parareal::Vec out(in.size());
    const int scheme = cfg.scheme == pintswim::Scheme::euler ? PSWIM_EULER : PSWIM_RK2;
    throw_for(pswim_propagate_host(ctx, in.data(), t0, t1, scheme, static_cast<int64_t>(cfg.steps_per_interval),
                                   cfg.dt, out.data()),
              pswim_last_error(ctx));
    return pintswim::unpack_state(out, sc.cfg.rod_count, sc.cfg.nodes_per_rod);
}

// parareal::PropagatorFn over packed states (the shape harness::prepare builds,
// harness.cpp:26-31): deterministic (bitwise) and thread safe.
inline pintswim::parareal::PropagatorFn make_propagator(const pintswim::Scenario& sc, pintswim::Scheme scheme,
                                                        std::size_t steps_per_interval, int device = 0) {
    const pswim_scenario s = to_c(sc.cfg);
    const int sch = scheme == pintswim::Scheme::euler ? PSWIM_EULER : PSWIM_RK2;
    return [s, sch, steps_per_interval, device](double t0, double t1, const pintswim::parareal::Vec& x) {
        pswim_ctx* ctx = Contexts::get(device, &s);
        pintswim::parareal::Vec out(x.size());
        throw_for(pswim_propagate_host(ctx, x.data(), t0, t1, sch, static_cast<int64_t>(steps_per_interval), 0.0,
                                       out.data()),
                  pswim_last_error(ctx));
        return out;
    };
}

}  // namespace pswim_gpu
