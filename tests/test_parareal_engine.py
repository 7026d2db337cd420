"""Native Parareal engine (csrc/parareal.cpp) with host propagators — the reference's
test_parareal.cpp properties: brute-force equality, exactness, mode / worker-count
independence (bitwise), stopping rules, trace sanity, validation.  No GPU needed."""
import numpy as np
import pytest

from toy import brute_force, euler_toy, rk2_toy, serial_fine
from paper_2604_12083_b200 import parareal as pr


def beq(a, b):
    return np.array_equal(np.asarray(a), np.asarray(b))


def test_pointwise_metric():
    m = pr.pointwise_metric(3)
    a = np.array([2, 0, 0, 1, 1, 1.0])
    b = np.array([1, 0, 0, 1, 1, 1.0])
    assert m(a, b) == pytest.approx(0.5)
    assert m(a, a) == 0.0
    assert pr.pointwise_metric(1)([0.0], [3.0]) == pytest.approx(3.0)
    with pytest.raises(ValueError):
        m(a, np.array([1.0]))


def test_serial_blocks_match_brute_force():
    plan = pr.ParallelPlan(horizon=1.5, intervals=5)
    g, f = euler_toy(-1.1, 2), rk2_toy(-1.1, 20)
    x0 = np.array([1.0])
    x = pr.coarse_sweep_initial(plan, g, x0)
    cache = [np.array(v) for v in x]
    for k in range(1, 5):
        xp = pr.fine_parallel(plan, f, x, k)
        x = pr.correct(plan, g, xp, x, cache, k)
        want = brute_force(plan, g, f, x0, k)
        assert all(beq(a, b) for a, b in zip(x, want))


@pytest.mark.parametrize("mode", [pr.REGULAR, pr.PIPELINED])
def test_engine_matches_brute_force(mode):
    g, f = euler_toy(-2.0, 1), rk2_toy(-2.0, 32)
    x0 = np.array([0.7, -0.3, 1.9])
    for l in range(1, 7):
        plan = pr.ParallelPlan(horizon=1.0, intervals=6, workers=3, max_iterations=l, tolerance=1e-300, mode=mode)
        res = pr.run(plan, g, f, x0, pr.pointwise_metric(3))
        want = brute_force(plan, g, f, x0, l)
        assert res.report.iterations_used == l
        assert all(beq(a, b) for a, b in zip(res.states, want))


def test_exactness():
    g, f = euler_toy(-1.3, 2), rk2_toy(-1.3, 40)
    x0 = np.array([1.0, 0.5])
    plan = pr.ParallelPlan(horizon=2.0, intervals=5, workers=2, tolerance=1e-300)
    ref = serial_fine(plan, f, x0)
    for k in range(1, 6):
        for mode in (pr.REGULAR, pr.PIPELINED):
            plan.max_iterations, plan.mode = k, mode
            res = pr.run(plan, g, f, x0, pr.pointwise_metric(2))
            assert all(beq(res.states[i], ref[i]) for i in range(k + 1))


def test_mode_and_worker_independence():
    g, f = euler_toy(0.6, 1), rk2_toy(0.6, 24)
    x0 = np.array([0.2, 0.4, -0.6, 0.8])
    results = []
    for mode in (pr.REGULAR, pr.PIPELINED):
        for workers in (1, 2, 4):
            plan = pr.ParallelPlan(horizon=1.2, intervals=8, max_iterations=4, tolerance=1e-300, mode=mode,
                                   workers=workers)
            results.append(pr.run(plan, g, f, x0, pr.pointwise_metric(4)))
    for r in results[1:]:
        assert r.report.eta_tilde == results[0].report.eta_tilde
        assert all(beq(a, b) for a, b in zip(r.states, results[0].states))


def test_stopping():
    g, f = euler_toy(-0.5, 1), rk2_toy(-0.5, 16)
    x0 = np.array([1.0])
    plan = pr.ParallelPlan(horizon=1.0, intervals=4, workers=2, max_iterations=9, tolerance=float("inf"))
    res = pr.run(plan, g, f, x0, pr.pointwise_metric(1))
    assert res.report.iterations_used == 1 and res.report.converged and len(res.report.eta_tilde) == 1
    plan = pr.ParallelPlan(horizon=1.0, intervals=6, workers=2, max_iterations=2, tolerance=1e-300)
    res = pr.run(plan, g, f, x0, pr.pointwise_metric(1))
    assert res.report.iterations_used == 2 and not res.report.converged
    plan = pr.ParallelPlan(horizon=1.0, intervals=4, workers=2, max_iterations=4, tolerance=1e-14)
    ref = serial_fine(plan, f, x0)
    res = pr.run(plan, g, f, x0, pr.pointwise_metric(1), reference=ref)
    assert res.report.eta and res.report.eta[-1] <= 1e-10


def test_trace_from_live_run():
    g, f = euler_toy(-1.0, 200), rk2_toy(-1.0, 2000)
    plan = pr.ParallelPlan(horizon=1.0, intervals=6, workers=2, max_iterations=3, tolerance=1e-300, mode=pr.PIPELINED)
    res = pr.run(plan, g, f, np.array([1.0]), pr.pointwise_metric(1))
    tr = res.trace
    assert tr.busy_time(pr.COARSE) > 0 and tr.busy_time(pr.FINE) > 0
    fine_events = 0
    cursor = [0.0, 0.0]
    for e in tr.events:
        assert e.t_end >= e.t_start
        assert e.t_start >= cursor[e.worker] - 1e-9
        cursor[e.worker] = max(cursor[e.worker], e.t_end)
        fine_events += e.kind == pr.FINE
    assert fine_events == 15  # 6 + 5 + 4


def test_validation_and_propagator_errors():
    ident = lambda a, b, x: x  # noqa: E731
    with pytest.raises(ValueError):
        pr.run(pr.ParallelPlan(intervals=0), ident, ident, [1.0])
    with pytest.raises(ValueError):
        pr.run(pr.ParallelPlan(intervals=2, tolerance=0.0), ident, ident, [1.0])

    def bad(a, b, x):
        raise RuntimeError("boom")

    with pytest.raises(Exception):
        pr.run(pr.ParallelPlan(intervals=3, workers=2), ident, bad, [1.0])
