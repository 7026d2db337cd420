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


@pytest.mark.parametrize("mode", [0, 1])
def test_sliced_threads_handoff_equals_engine(gpu, mode):
    """Slice states handed off over peer memory (the corrector kernel stores X[k][n] straight
    into rank p+1's slot and releases a system-scope flag): bitwise equal to the engine, and
    to the stream-ordered peer-copy transport."""
    from paper_2604_12083_b200 import parareal as pr
    from paper_2604_12083_b200.scenario import ScenarioConfig, build_initial_state, make_scenario

    sc = make_scenario(ScenarioConfig(rod_count=2, nodes_per_rod=32, horizon=4e-3, epsilon=0.08))
    x0 = build_initial_state(sc)
    for l in (1, 2, 4):
        plan = pr.ParallelPlan(horizon=4e-3, intervals=4, workers=4, max_iterations=l, tolerance=1e-300, mode=mode)
        eng = pr.run_gpu(plan, sc, 20, 2, x0)
        ho = pr.run_sliced_threads(plan, sc, 20, 2, x0, [0, 0, 0, 0], handoff=True)
        assert ho.report.eta_tilde == eng.report.eta_tilde
        assert ho.report.iterations_used == l
        for n in range(5):
            assert np.array_equal(ho.states[n], eng.states[n]), (l, n)


def test_sliced_trace_shows_pipelining(gpu):
    """Rank-driver schedule trace from device timestamps: every rank's tasks with their (k, n);
    in pipelined mode iteration k+1's first corrector starts before iteration k's last one
    ends (the wavefronts overlap), and the fine lanes report idle time W > 0."""
    from paper_2604_12083_b200 import parareal as pr
    from paper_2604_12083_b200.scenario import ScenarioConfig, build_initial_state, make_scenario

    n = 6
    T = n * 40 * 1e-6  # dt = 1e-6 fine, 1e-5 coarse: stable for 64-node rods at eps = 0.08
    sc = make_scenario(ScenarioConfig(rod_count=4, nodes_per_rod=64, horizon=T, epsilon=0.08))
    x0 = build_initial_state(sc)
    plan = pr.ParallelPlan(horizon=T, intervals=n, workers=n, max_iterations=3, tolerance=1e-300,
                           mode=pr.PIPELINED)
    for handoff in (False, True):
        res = pr.run_sliced_threads(plan, sc, 40, 4, x0, [0] * n, handoff=handoff)
        ev = res.trace.events
        corr = [e for e in ev if e.kind == pr.CORRECT]
        fine = [e for e in ev if e.kind == pr.FINE]
        assert len([e for e in ev if e.kind == pr.COARSE]) == n
        assert len(corr) == sum(min(i - 1, 3) for i in range(1, n + 1))
        assert len(fine) == sum(min(i, 3) for i in range(1, n + 1))
        assert all(e.worker == e.interval for e in fine) and all(e.worker == 0 for e in corr)
        assert res.schedule_idle > 0.0
        for k in (1, 2):
            last_k = max(e.t_end for e in corr if e.iteration == k)
            first_k1 = min(e.t_start for e in corr if e.iteration == k + 1)
            assert first_k1 < last_k, (handoff, k, first_k1, last_k)


def _handoff_proc(rank, world, port, q):
    import os

    os.environ.setdefault("CUDA_DEVICE_MAX_CONNECTIONS", "32")
    import torch.distributed as dist

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2604_12083_b200 import parareal as pr
        from paper_2604_12083_b200.scenario import ScenarioConfig, build_initial_state, make_scenario

        sc = make_scenario(ScenarioConfig(rod_count=2, nodes_per_rod=32, horizon=4e-3, epsilon=0.08))
        x0 = build_initial_state(sc)
        out = []
        for mode in (0, 1):
            for l in (1, world):
                plan = pr.ParallelPlan(horizon=4e-3, intervals=world, workers=world, max_iterations=l,
                                       tolerance=1e-300, mode=mode)
                st = pr.StagedTransport(0)  # the metric allreduce / trace gather over gloo
                ho = pr.Handoff(0, x0.size, l + 1)
                dist.barrier()
                res = pr.run_sliced_rank(plan, sc, 20, 2, x0, 0, transport=st.ptr, handoff=ho)
                dist.barrier()  # no rank frees its slots while the previous rank may still write
                ho.close()
                st.close()
                out.append((mode, l, res.state.copy(), res.report.eta_tilde))
        q.put((rank, out))
    except Exception as e:  # pragma: no cover
        q.put((rank, repr(e)))
    finally:
        dist.destroy_process_group()


def test_handoff_ipc_processes(gpu):
    """Two processes on one GPU exchanging CUDA IPC handles of their hand-off slots (the
    one-process-per-GPU layout of an NVSwitch box): every rank's slice state bitwise equal to
    the engine's, regular and pipelined."""
    import socket

    import torch.multiprocessing as mp

    from paper_2604_12083_b200 import parareal as pr
    from paper_2604_12083_b200.scenario import ScenarioConfig, build_initial_state, make_scenario

    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    world = 2
    ps = [ctx.Process(target=_handoff_proc, args=(r, world, port, q)) for r in range(world)]
    for p in ps:
        p.start()
    res = sorted((q.get(timeout=600) for _ in range(world)), key=lambda t: t[0])
    for p in ps:
        p.join(timeout=60)
    sc = make_scenario(ScenarioConfig(rod_count=2, nodes_per_rod=32, horizon=4e-3, epsilon=0.08))
    x0 = build_initial_state(sc)
    for rank, out in res:
        assert isinstance(out, list), out
        for mode, l, state, et in out:
            plan = pr.ParallelPlan(horizon=4e-3, intervals=world, workers=world, max_iterations=l,
                                   tolerance=1e-300, mode=mode)
            eng = pr.run_gpu(plan, sc, 20, 2, x0)
            assert et == eng.report.eta_tilde
            assert np.array_equal(state, eng.states[rank + 1]), (rank, mode, l)
