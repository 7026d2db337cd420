"""GPU Parareal: the native engine with GPU rod propagators and the time-sliced rank driver
(threads transport on one GPU) — parity with the reference's Parareal (golden states from
the reference engine, <= 1e-10 relative position) and bitwise GPU-vs-GPU properties
(exactness, mode / worker / driver independence)."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def small_case():
    from paper_2604_12083_b200.scenario import ScenarioConfig, make_scenario

    return make_scenario(ScenarioConfig(rod_count=1, nodes_per_rod=11, horizon=1.0))


def test_gpu_engine_vs_reference_golden(gpu, golden, oracle):
    from paper_2604_12083_b200 import parareal as pr

    sc = small_case()
    x0 = golden["par_x0"]
    for l in range(1, 5):
        plan = pr.ParallelPlan(horizon=1.0, intervals=4, workers=2, max_iterations=l, tolerance=1e-300,
                               mode=pr.PIPELINED)
        res = pr.run_gpu(plan, sc, 50, 5, x0)
        want = golden[f"par_states_l{l}"]
        for n in range(5):
            assert oracle.position_metric(want[n], res.states[n]) < 1e-10
        assert res.report.iterations_used == l
        np.testing.assert_allclose(res.report.eta_tilde, golden[f"par_eta_tilde_l{l}"], rtol=1e-6, atol=1e-13)


def test_gpu_engine_exactness_and_independence(gpu):
    from paper_2604_12083_b200 import parareal as pr
    from paper_2604_12083_b200.harness import RunConfig, prepare, serial_fine_boundaries
    from paper_2604_12083_b200.scenario import ScenarioConfig

    cfg = RunConfig(scenario=ScenarioConfig(rod_count=1, nodes_per_rod=11, horizon=1.0), intervals=6, workers=2,
                    max_iterations=6, tolerance=1e-300, fine_steps_per_interval=40, coarse_steps_per_interval=4)
    run = prepare(cfg)
    ref = serial_fine_boundaries(run)
    results = []
    for mode in (pr.REGULAR, pr.PIPELINED):
        for workers in (1, 2, 4):
            plan = pr.ParallelPlan(horizon=1.0, intervals=6, workers=workers, max_iterations=3, tolerance=1e-300,
                                   mode=mode)
            results.append(pr.run_gpu(plan, run.scenario, 40, 4, run.x0))
    for r in results:
        assert r.report.eta_tilde == results[0].report.eta_tilde
        for n in range(7):
            assert np.array_equal(r.states[n], results[0].states[n])
        for n in range(4):  # k = 3 iterations pin X[0..3] to the serial fine solution bitwise
            assert np.array_equal(r.states[n], ref[n])


@pytest.mark.parametrize("mode", [0, 1])
def test_sliced_threads_equals_engine(gpu, mode):
    """One slice per rank (4 ranks sharing cuda:0): identical states and reports to the
    task-graph engine, bitwise."""
    from paper_2604_12083_b200 import parareal as pr
    from paper_2604_12083_b200.scenario import ScenarioConfig, build_initial_state, make_scenario

    sc = make_scenario(ScenarioConfig(rod_count=2, nodes_per_rod=32, horizon=4e-3, epsilon=0.08))
    x0 = build_initial_state(sc)
    for l in (1, 2, 4):
        plan = pr.ParallelPlan(horizon=4e-3, intervals=4, workers=4, max_iterations=l, tolerance=1e-300, mode=mode)
        eng = pr.run_gpu(plan, sc, 20, 2, x0)
        sl = pr.run_sliced_threads(plan, sc, 20, 2, x0, [0, 0, 0, 0])
        assert sl.report.eta_tilde == eng.report.eta_tilde
        assert sl.report.iterations_used == l
        for n in range(5):
            assert np.array_equal(sl.states[n], eng.states[n]), (l, n)


def test_sliced_threads_tolerance_stop(gpu):
    from paper_2604_12083_b200 import parareal as pr
    from paper_2604_12083_b200.scenario import ScenarioConfig, build_initial_state, make_scenario

    sc = make_scenario(ScenarioConfig(rod_count=1, nodes_per_rod=21, horizon=0.02))
    x0 = build_initial_state(sc)
    plan = pr.ParallelPlan(horizon=0.02, intervals=4, workers=4, max_iterations=4, tolerance=1e-9, mode=1)
    eng = pr.run_gpu(plan, sc, 100, 10, x0)
    sl = pr.run_sliced_threads(plan, sc, 100, 10, x0, [0, 0, 0, 0])
    assert sl.report.iterations_used == eng.report.iterations_used
    assert sl.report.converged == eng.report.converged
    for n in range(5):
        assert np.array_equal(sl.states[n], eng.states[n])
