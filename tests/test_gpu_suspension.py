"""BASELINE configs[2]/[3] end to end against the reference's OWN runs (SURVEY 8(c),
north_star: "final filament configurations within a stated tolerance of the reference's own
serial and Parareal runs").

Fixture tests/golden/suspension.npz comes from the unmodified reference library
(tests/golden/make_suspension.py: src/propagators.cpp propagate, harness::serial_fine_boundaries,
parareal::run over harness::prepare's propagators) for 64 rods x 256 nodes, epsilon = 0.08,
dt = 1e-6: a 100-step serial RK2 trajectory, n = 4 intervals x (20 RK2 | 2 Euler), Parareal
l = 1..4 pipelined and l = 2 regular at tol = 1e-300.  Per state it keeps every 4th node's
position, the per-rod sums of all 12 packed components, and the SHA-1 of the full state.

Tolerance: 1e-10 relative position (rod_position_metric with the reference state as the
denominator, io.cpp:49-68), the north_star bound; per-rod checksums 1e-10 relative to their
largest entry.  Every GPU driver is checked: the single-device engine, the time-sliced rank
driver (stream-ordered peer copies and the peer-memory hand-off), the hybrid space x time
driver, and the space-parallel propagates (collective and fused peer all-gather)."""
import hashlib
import os
import threading

import numpy as np
import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
TOL = 1e-10


@pytest.fixture(scope="module")
def fx():
    path = os.path.join(ROOT, "tests", "golden", "suspension.npz")
    if not os.path.exists(path):
        pytest.skip("tests/golden/suspension.npz missing")
    return dict(np.load(path))


def scen(fx):
    from paper_2604_12083_b200.scenario import ScenarioConfig, make_scenario

    rods, nodes = int(fx["meta"][0]), int(fx["meta"][1])
    horizon = int(fx["meta"][2]) * int(fx["meta"][3]) * float(fx["params"][1])
    return make_scenario(ScenarioConfig(rod_count=rods, nodes_per_rod=nodes, epsilon=float(fx["params"][0]),
                                        horizon=horizon))


def check(fx, key, state):
    rods, nodes, stride = int(fx["meta"][0]), int(fx["meta"][1]), int(fx["meta"][6])
    x = np.asarray(state).reshape(rods * nodes, 12)
    want = fx[key + "_pos"]
    got = x[::stride, 0:3]
    num = np.sqrt(((got - want) ** 2).sum(axis=1))
    den = np.sqrt((want ** 2).sum(axis=1))
    rel = np.where(den < 1e-14, num, num / np.where(den < 1e-14, 1.0, den)).max()
    assert rel < TOL, (key, rel)
    rs = x.reshape(rods, nodes, 12).sum(axis=1)
    want_rs = fx[key + "_rodsum"]
    assert np.abs(rs - want_rs).max() <= TOL * np.abs(want_rs).max(), key
    return rel


def plan_of(fx, l, mode, workers=None):
    from paper_2604_12083_b200 import parareal as pr

    n = int(fx["meta"][2])
    horizon = n * int(fx["meta"][3]) * float(fx["params"][1])
    return pr.ParallelPlan(horizon=horizon, intervals=n, workers=workers or n, max_iterations=l, tolerance=1e-300,
                           mode=mode)


RUNS = [(1, 1), (1, 2), (1, 3), (1, 4), (0, 2)]


def test_initial_state_bitwise(gpu, fx):
    from paper_2604_12083_b200.scenario import build_initial_state

    x0 = build_initial_state(scen(fx))
    assert hashlib.sha1(np.ascontiguousarray(x0).tobytes()).digest() == bytes(fx["x0_sha1"])


def test_serial_fine_100_steps(gpu, fx):
    import torch

    from paper_2604_12083_b200.propagators import StepperConfig, propagate
    from paper_2604_12083_b200.scenario import build_initial_state

    sc = scen(fx)
    x0 = build_initial_state(sc)
    steps = int(fx["meta"][5])
    out = propagate(torch.as_tensor(x0, device="cuda:0"), 0.0, steps * float(fx["params"][1]),
                    StepperConfig(0.0, 1, steps), sc).cpu().numpy()
    check(fx, "serial100", out)


def test_serial_fine_boundaries(gpu, fx):
    from paper_2604_12083_b200.harness import RunConfig, prepare, serial_fine_boundaries
    from paper_2604_12083_b200.scenario import ScenarioConfig

    n, fine = int(fx["meta"][2]), int(fx["meta"][3])
    cfg = RunConfig(scenario=ScenarioConfig(rod_count=int(fx["meta"][0]), nodes_per_rod=int(fx["meta"][1]),
                                            epsilon=float(fx["params"][0]), horizon=n * fine * float(fx["params"][1])),
                    intervals=n, fine_steps_per_interval=fine, coarse_steps_per_interval=int(fx["meta"][4]))
    b = serial_fine_boundaries(prepare(cfg))
    for i in range(1, n + 1):
        check(fx, f"bounds_n{i}", b[i])


def _eta_close(got, want):
    np.testing.assert_allclose(got, want, rtol=1e-4, atol=1e-14)


@pytest.mark.parametrize("mode,l", RUNS)
def test_engine_vs_reference_parareal(gpu, fx, mode, l):
    from paper_2604_12083_b200 import parareal as pr
    from paper_2604_12083_b200.scenario import build_initial_state

    sc = scen(fx)
    x0 = build_initial_state(sc)
    fine, coarse = int(fx["meta"][3]), int(fx["meta"][4])
    for workers in (2, int(fx["meta"][2]) + 1):
        res = pr.run_gpu(plan_of(fx, l, mode, workers), sc, fine, coarse, x0)
        key = f"par_m{mode}_l{l}"
        for n in range(1, int(fx["meta"][2]) + 1):
            check(fx, f"{key}_n{n}", res.states[n])
        assert res.report.iterations_used == int(fx[key + "_iters"][0])
        _eta_close(res.report.eta_tilde, fx[key + "_eta_tilde"])


@pytest.mark.parametrize("mode,l", RUNS)
@pytest.mark.parametrize("handoff", [False, True])
def test_sliced_driver_vs_reference_parareal(gpu, fx, mode, l, handoff):
    """One slice per rank (4 thread-ranks on cuda:0), fixed-l and eta against the serial fine
    boundaries of the same run, checked against the reference's parareal::run and its eta."""
    from paper_2604_12083_b200 import parareal as pr
    from paper_2604_12083_b200.scenario import build_initial_state

    sc = scen(fx)
    x0 = build_initial_state(sc)
    n, fine, coarse = int(fx["meta"][2]), int(fx["meta"][3]), int(fx["meta"][4])
    bounds = pr.run_sliced_threads(plan_of(fx, n, 1), sc, fine, coarse, x0, [0] * n).states  # X[n] = serial fine
    for i in range(1, n + 1):
        check(fx, f"bounds_n{i}", bounds[i])
    res = pr.run_sliced_threads(plan_of(fx, l, mode), sc, fine, coarse, x0, [0] * n, reference=bounds,
                                handoff=handoff)
    key = f"par_m{mode}_l{l}"
    for i in range(1, n + 1):
        check(fx, f"{key}_n{i}", res.states[i])
    _eta_close(res.report.eta_tilde, fx[key + "_eta_tilde"])
    _eta_close(res.report.eta, fx[key + "_eta"])


def test_tolerance_stop_matches_reference(gpu, fx):
    """tol = 1e-9 stops where the reference's eta_tilde sequence first undercuts it."""
    from paper_2604_12083_b200 import parareal as pr
    from paper_2604_12083_b200.scenario import build_initial_state

    sc = scen(fx)
    x0 = build_initial_state(sc)
    n, fine, coarse = int(fx["meta"][2]), int(fx["meta"][3]), int(fx["meta"][4])
    et = fx["par_m1_l4_eta_tilde"]
    tol = 1e-9
    want = next((k + 1 for k, v in enumerate(et) if v < tol), n)
    plan = plan_of(fx, n, 1)
    plan.tolerance = tol
    for res in (pr.run_gpu(plan, sc, fine, coarse, x0), pr.run_sliced_threads(plan, sc, fine, coarse, x0, [0] * n)):
        assert res.report.iterations_used == want
        assert res.report.converged
        for i in range(1, n + 1):
            check(fx, f"par_m1_l{want}_n{i}", res.states[i])


@pytest.mark.parametrize("mode,l", [(1, 1), (1, 2), (0, 2)])
def test_hybrid_driver_vs_reference_parareal(gpu, fx, mode, l):
    """Hybrid space x time: 4 slices x 2 space members = 8 thread-ranks on cuda:0."""
    from paper_2604_12083_b200 import parareal as pr
    from paper_2604_12083_b200.propagators import ThreadTransports
    from paper_2604_12083_b200.scenario import build_initial_state

    sc = scen(fx)
    x0 = build_initial_state(sc)
    slices, members = int(fx["meta"][2]), 2
    fine, coarse = int(fx["meta"][3]), int(fx["meta"][4])
    plan = plan_of(fx, l, mode)
    time_tr = [ThreadTransports([0] * slices, len_hint=x0.size, slots=l + 2) for _ in range(members)]
    space_c = [ThreadTransports([0] * members) for _ in range(slices)]
    space_f = [ThreadTransports([0] * members) for _ in range(slices)]
    out, errs = {}, []

    def rank(p, q):
        try:
            out[p, q] = pr.run_sliced_rank(plan, sc, fine, coarse, x0, 0, transport=time_tr[q][p],
                                           space=(space_c[p][q], space_f[p][q]))
        except Exception as e:  # pragma: no cover
            errs.append(e)

    th = [threading.Thread(target=rank, args=(p, q)) for p in range(slices) for q in range(members)]
    for t in th:
        t.start()
    for t in th:
        t.join(timeout=600)
    assert not errs, errs
    key = f"par_m{mode}_l{l}"
    for (p, q), res in out.items():
        check(fx, f"{key}_n{p + 1}", res.state)
        _eta_close(res.report.eta_tilde, fx[key + "_eta_tilde"])
    for group in time_tr + space_c + space_f:
        group.close()


@pytest.mark.parametrize("peer", [False, True])
def test_space_parallel_vs_reference_serial(gpu, fx, peer):
    """Space-parallel MRS propagate (targets sharded over 2 thread-ranks; collective or fused
    peer all-gather), 100 RK2 steps, against the reference's serial trajectory."""
    import torch

    from paper_2604_12083_b200.device import Context
    from paper_2604_12083_b200.propagators import (PeerGroup, StepperConfig, ThreadTransports, propagate_sharded,
                                                   propagate_sharded_peer)
    from paper_2604_12083_b200.scenario import build_initial_state

    sc = scen(fx)
    x0 = build_initial_state(sc)
    steps = int(fx["meta"][5])
    cfg = StepperConfig(0.0, 1, steps)
    T = steps * float(fx["params"][1])
    world = 2
    ctxs = [Context(0, sc) for _ in range(world)]
    outs, errs = [None] * world, []
    if peer:
        groups = [PeerGroup(ctxs[r], r, world) for r in range(world)]
        bases = [g.base for g in groups]
        for g in groups:
            g.connect(bases=bases)
        run = lambda r: propagate_sharded_peer(torch.as_tensor(x0, device="cuda:0"), 0.0, T, cfg, sc, groups[r])  # noqa: E731
    else:
        trs = ThreadTransports([0] * world)
        run = lambda r: propagate_sharded(torch.as_tensor(x0, device="cuda:0"), 0.0, T, cfg, sc, trs[r], ctx=ctxs[r])  # noqa: E731

    def rank(r):
        try:
            outs[r] = run(r).cpu().numpy()
        except Exception as e:  # pragma: no cover
            errs.append(e)

    th = [threading.Thread(target=rank, args=(r,)) for r in range(world)]
    for t in th:
        t.start()
    for t in th:
        t.join(timeout=600)
    assert not errs, errs
    for r in range(world):
        check(fx, "serial100", outs[r])
    if peer:
        for g in groups:
            g.close()
    else:
        trs.close()
