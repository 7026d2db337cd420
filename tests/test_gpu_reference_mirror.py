"""The reference's own integrator and scheduling tests, run on the GPU path:

* tests/test_propagators.cpp:42-51   quiet rod (zero waveform) -> zero rhs, RK2 step leaves it;
* tests/test_propagators.cpp:82-105  far-separated rods behave like isolated ones (LJ enabled,
                                     pairs out of range);
* tests/test_propagators.cpp:203-236 integrator convergence orders (Richardson): Euler 1.0 +- 0.1,
                                     midpoint RK2 2.0 +- 0.1 against an RK2-3200 reference, and
                                     RK2 vs small-step Euler within truncation bounds
                                     (acceptance C9, acceptance_main.cpp:536-561);
* acceptance_main.cpp:563-620        C10: live pipelined wall time <= regular in >= 9/10 runs
                                     at m = 2 and 4, on the GPU engine."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def desk(nodes=21, amplitude=0.05, **kw):  # test_propagators.cpp:15-21
    from paper_2604_12083_b200.scenario import ScenarioConfig, WaveformParams, make_scenario

    return make_scenario(ScenarioConfig(rod_count=1, nodes_per_rod=nodes, waveform=WaveformParams(amplitude=amplitude),
                                        **kw))


def dist(a, b):  # state_distance, test_propagators.cpp:23-29
    return float(np.sqrt(((np.asarray(a) - np.asarray(b)) ** 2).sum()))


def test_quiet_rod_has_zero_rhs(gpu):
    from paper_2604_12083_b200.propagators import rhs, step_rk2
    from paper_2604_12083_b200.scenario import build_initial_state

    sc = desk(21, 0.0)
    x = build_initial_state(sc)
    v = rhs(x, 0.0, sc)
    assert np.linalg.norm(np.asarray(v.u), axis=1).max() < 1e-13
    assert np.linalg.norm(np.asarray(v.omega), axis=1).max() < 1e-13
    assert dist(step_rk2(x, 0.0, 1e-3, sc), x) < 1e-12


def test_far_separated_rods_behave_like_isolated(gpu):
    from paper_2604_12083_b200.propagators import rhs
    from paper_2604_12083_b200.scenario import ScenarioConfig, build_initial_state, make_scenario

    sc1 = make_scenario(ScenarioConfig(rod_count=1, nodes_per_rod=21, lj_well_depth=1.0))
    lone = build_initial_state(sc1).reshape(21, 12)
    sc2 = make_scenario(ScenarioConfig(rod_count=2, nodes_per_rod=21, lj_well_depth=1.0))
    pair = build_initial_state(sc2).reshape(42, 12)
    pair[:21] = lone
    pair[21:] = lone
    pair[21:, 1] += 4.0  # far beyond epsilon and the LJ cutoff
    v1 = rhs(lone.reshape(-1), 0.2, sc1)
    v2 = rhs(pair.reshape(-1), 0.2, sc2)
    u1, u2 = np.asarray(v1.u), np.asarray(v2.u)
    scale = np.linalg.norm(u1, axis=1).max()
    assert (np.linalg.norm(u2[:21] - u1, axis=1) / scale).max() < 1e-3
    assert (np.linalg.norm(u2[21:] - u1, axis=1) / scale).max() < 1e-3


def test_integrator_convergence_orders(gpu):
    from paper_2604_12083_b200.propagators import StepperConfig, propagate
    from paper_2604_12083_b200.scenario import build_initial_state

    sc = desk()
    x = build_initial_state(sc)
    T = 0.05
    ref = propagate(x, 0.0, T, StepperConfig(0.0, 1, 3200), sc)

    def err(scheme, steps):
        return dist(propagate(x, 0.0, T, StepperConfig(0.0, scheme, steps), sc), ref)

    order_euler = np.log2(err(0, 32) / err(0, 64))
    order_rk2 = np.log2(err(1, 32) / err(1, 64))
    assert abs(order_euler - 1.0) <= 0.1, order_euler
    assert abs(order_rk2 - 2.0) <= 0.1, order_rk2
    rk = propagate(x, 0.0, T, StepperConfig(0.0, 1, 64), sc)
    eu = propagate(x, 0.0, T, StepperConfig(0.0, 0, 6400), sc)
    assert dist(rk, eu) <= 2.0 * (err(0, 6400) + err(1, 64))


def test_c10_pipelined_not_slower_than_regular(gpu):
    """Acceptance C10 on the GPU engine: desk config with 31 nodes, 400 RK2 steps per interval,
    l = 3 fixed, coarse = resolved_coarse_steps at r = 2; pipelined wall <= regular wall in at
    least 9 of 10 repetitions for m = 2 and 4."""
    from paper_2604_12083_b200 import parareal as pr
    from paper_2604_12083_b200.harness import RunConfig
    from paper_2604_12083_b200.scenario import ScenarioConfig, build_initial_state, make_scenario

    scfg = ScenarioConfig(rod_count=1, nodes_per_rod=31, horizon=1.0, seed=1)
    sc = make_scenario(scfg)
    x0 = build_initial_state(sc)

    def wall(mode, m, r):
        cfg = RunConfig(scenario=scfg, intervals=8, workers=m, ratio=r, max_iterations=3, tolerance=1e-300,
                        fine_steps_per_interval=400, coarse_steps_per_interval=0, mode=mode)
        plan = pr.ParallelPlan(horizon=1.0, intervals=8, workers=m, cost_ratio=r, max_iterations=3,
                               tolerance=1e-300, mode=mode)
        return pr.run_gpu(plan, sc, 400, cfg.resolved_coarse_steps(), x0).report.wall_seconds

    wall(pr.PIPELINED, 2, 2.0)  # warm-up: contexts, kernels
    for m in (2, 4):
        wins = sum(wall(pr.PIPELINED, m, 2.0) <= wall(pr.REGULAR, m, 2.0) for _ in range(10))
        assert wins >= 9, (m, wins)
