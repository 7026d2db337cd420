// ab_parareal.cpp — TEST INFRASTRUCTURE (A/B harness, built into oracle/_ref/).
//
// Runs the reference's OWN Parareal engine (pintswim::parareal::run, src/parareal.cpp,
// compiled unmodified) twice on the desk scenario of acceptance criterion 1
// (tests/acceptance_main.cpp:39-89, reduced): once with the reference CPU propagators built
// as harness::prepare does, once with the B200 propagators of include/pswim/pintswim_gpu.hpp
// plugged into the same PropagatorFn slots.  Prints one JSON line; exit 0 when
//   * GPU boundary states match the CPU ones to <= 1e-10 (rod_position_metric),
//   * iteration counts / convergence flags agree and |d eta_tilde| <= 1e-6 (eta_tilde + 1e-7),
//   * GPU runs are bitwise identical across modes (regular / pipelined) and m in {1,2,4},
//   * the reference's own lj_repulsion and the B200 one through pswim_gpu::lj_repulsion
//     (cell list: 48 rods x 64 nodes, perturbed into contact) agree to <= 1e-12 relative.
#include <cmath>
#include <cstdio>
#include <random>
#include <vector>

#include "pintswim/harness.hpp"
#include "pintswim/io.hpp"
#include "pswim/pintswim_gpu.hpp"

using namespace pintswim;

int main() {
    RunConfig cfg;
    cfg.scenario.rod_count = 1;
    cfg.scenario.nodes_per_rod = 21;
    cfg.scenario.horizon = 1.0;
    cfg.intervals = 8;
    cfg.workers = 2;
    cfg.max_iterations = 10;
    cfg.tolerance = 1e-12;
    cfg.fine_steps_per_interval = 400;
    cfg.coarse_steps_per_interval = 10;
    cfg.mode = parareal::Mode::pipelined;
    const auto run = harness::prepare(cfg);
    const auto reference = harness::serial_fine_boundaries(run);
    const auto cpu = parareal::run(run.plan, run.coarse, run.fine, run.x0, rod_position_metric(), &reference);

    const auto gfine = pswim_gpu::make_propagator(run.scenario, Scheme::rk2, 400);
    const auto gcoarse = pswim_gpu::make_propagator(run.scenario, Scheme::euler, 10);
    const auto gpu = parareal::run(run.plan, gcoarse, gfine, run.x0, rod_position_metric(), &reference);

    double worst = 0.0;
    for (std::size_t n = 0; n < cpu.states.size(); ++n)
        worst = std::max(worst, rod_position_metric()(cpu.states[n], gpu.states[n]));
    double eta_rel = 0.0;
    const bool same_k = cpu.report.iterations_used == gpu.report.iterations_used &&
                        cpu.report.converged == gpu.report.converged &&
                        cpu.report.eta_tilde.size() == gpu.report.eta_tilde.size();
    if (same_k)
        for (std::size_t k = 0; k < cpu.report.eta_tilde.size(); ++k)
            // eta_tilde is a difference of two nearly equal states: its error is the states'
            // (~1e-15 relative) divided by its size, so compare |d eta| <= 1e-6 eta + 1e-13
            eta_rel = std::max(eta_rel, std::abs(cpu.report.eta_tilde[k] - gpu.report.eta_tilde[k]) /
                                            (cpu.report.eta_tilde[k] + 1e-7));

    bool bitwise = true;
    for (const auto mode : {parareal::Mode::regular, parareal::Mode::pipelined}) {
        for (const int m : {1, 2, 4}) {
            auto plan = run.plan;
            plan.mode = mode;
            plan.workers = m;
            plan.max_iterations = 3;
            plan.tolerance = 1e-300;
            static std::vector<parareal::Vec> first;
            const auto r = parareal::run(plan, gcoarse, gfine, run.x0, rod_position_metric());
            if (first.empty()) {
                first = r.states;
            } else {
                for (std::size_t n = 0; n < first.size(); ++n) bitwise = bitwise && (first[n] == r.states[n]);
            }
        }
    }
    // LJ through the drop-in binding (rod.cpp:124-174 vs lj_cells.cu)
    ScenarioConfig lc;
    lc.rod_count = 48;
    lc.nodes_per_rod = 64;
    lc.placement = Placement::random;
    lc.lj_well_depth = 0.01;
    lc.seed = 9;
    const Scenario lsc = make_scenario(lc);
    auto rods = build_initial_state(lsc);
    std::mt19937_64 rng(5);
    std::normal_distribution<double> nd(0.0, 0.08);
    for (auto& r : rods)
        for (auto& x : r.x) x = x + Vec3{nd(rng), nd(rng), nd(rng)};
    const auto lj_ref = lj_repulsion(rods, lsc.lj, lsc.lj_self_exclusion);
    const auto lj_gpu = pswim_gpu::lj_repulsion(rods, lsc);
    double lj_scale = 0.0, lj_diff = 0.0;
    for (std::size_t i = 0; i < lj_ref.size(); ++i) {
        lj_scale = std::max({lj_scale, std::abs(lj_ref[i].x), std::abs(lj_ref[i].y), std::abs(lj_ref[i].z)});
        lj_diff = std::max({lj_diff, std::abs(lj_ref[i].x - lj_gpu[i].x), std::abs(lj_ref[i].y - lj_gpu[i].y),
                            std::abs(lj_ref[i].z - lj_gpu[i].z)});
    }
    const double lj_rel = lj_scale > 0.0 ? lj_diff / lj_scale : 1.0;  // the case must have contacts
    const bool ok = worst <= 1e-10 && same_k && eta_rel <= 1e-6 && bitwise && lj_rel <= 1e-12;
    std::printf("{\"ok\": %s, \"max_position_metric_gpu_vs_cpu\": %.3e, \"iterations_cpu\": %d, \"iterations_gpu\": %d, "
                "\"converged_cpu\": %d, \"converged_gpu\": %d, \"eta_tilde_rel_diff\": %.3e, \"gpu_bitwise_modes_workers\": %s, "
                "\"eta_last_cpu\": %.3e, \"eta_last_gpu\": %.3e, \"lj_rel_diff\": %.3e, \"lj_scale\": %.3e}\n",
                ok ? "true" : "false", worst, cpu.report.iterations_used, gpu.report.iterations_used,
                (int)cpu.report.converged, (int)gpu.report.converged, eta_rel, bitwise ? "true" : "false",
                cpu.report.eta.empty() ? 0.0 : cpu.report.eta.back(), gpu.report.eta.empty() ? 0.0 : gpu.report.eta.back(),
                lj_rel, lj_scale);
    return ok ? 0 : 1;
}
