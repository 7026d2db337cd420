"""Time-sliced rank driver (one slice per rank) over a real multi-process torch.distributed
(gloo) transport on CPU: world sizes 2 and 4, both modes, fixed l and tolerance stop —
every rank's slice state equals the brute-force recurrence bitwise, and the report is the
same on every rank."""
import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp

from toy import brute_force, euler_toy, rk2_toy


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, mode, l, tol, q):
    import torch.distributed as dist

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2604_12083_b200 import parareal as pr

        g, f = euler_toy(-1.7, 2), rk2_toy(-1.7, 24)
        x0 = np.array([1.0, -0.5, 0.25])
        plan = pr.ParallelPlan(horizon=1.0, intervals=world, workers=world, max_iterations=l, tolerance=tol,
                               mode=mode)
        ref = brute_force(plan, g, f, x0, world)  # exact (k = n) boundaries as the true-error reference
        res = pr.run_sliced_rank_host(plan, g, f, x0, pr.pointwise_metric(3), reference_slice=ref[rank + 1])
        lanes = {}
        for e in res.trace.events:
            lanes[(e.worker, e.kind)] = lanes.get((e.worker, e.kind), 0) + 1
        q.put((rank, res.state.tolist(), res.report.eta_tilde, res.report.eta, res.report.iterations_used,
               res.report.converged, lanes, res.schedule_idle))
    finally:
        dist.destroy_process_group()


def _run(world, mode, l, tol):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, mode, l, tol, q)) for r in range(world)]
    for p in procs:
        p.start()
    out = [q.get(timeout=120) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    return sorted(out)


@pytest.mark.parametrize("world,mode,l", [(2, 1, 1), (2, 0, 2), (4, 1, 2), (4, 0, 3), (4, 1, 4)])
def test_rank_driver_matches_brute_force(world, mode, l):
    from paper_2604_12083_b200 import parareal as pr

    out = _run(world, mode, l, 1e-300)
    g, f = euler_toy(-1.7, 2), rk2_toy(-1.7, 24)
    x0 = np.array([1.0, -0.5, 0.25])
    plan = pr.ParallelPlan(horizon=1.0, intervals=world, max_iterations=l, tolerance=1e-300)
    want = brute_force(plan, g, f, x0, l)
    # engine-level reference for the report
    res = pr.run(pr.ParallelPlan(horizon=1.0, intervals=world, workers=2, max_iterations=l, tolerance=1e-300), g, f,
                 x0, pr.pointwise_metric(3))
    for rank, state, et, eta, iters, conv, _, _ in out:
        assert np.array_equal(np.array(state), want[rank + 1]), rank
        assert et == res.report.eta_tilde
        assert iters == l
        assert conv == (l == world)
        assert eta[-1] == 0.0 if l == world else eta[-1] > 0.0


def test_rank_driver_tolerance_stop():
    from paper_2604_12083_b200 import parareal as pr

    out = _run(4, 1, 4, 1e-6)
    g, f = euler_toy(-1.7, 2), rk2_toy(-1.7, 24)
    x0 = np.array([1.0, -0.5, 0.25])
    res = pr.run(pr.ParallelPlan(horizon=1.0, intervals=4, workers=3, max_iterations=4, tolerance=1e-6,
                                 mode=pr.PIPELINED), g, f, x0, pr.pointwise_metric(3))
    iters = {o[4] for o in out}
    assert iters == {res.report.iterations_used}
    for rank, state, et, _, _, conv, _, _ in out:
        assert et == res.report.eta_tilde
        assert conv == res.report.converged
        assert np.array_equal(np.array(state), res.states[rank + 1])


@pytest.mark.parametrize("mode", [0, 1])
def test_rank_driver_schedule_trace(mode):
    """The rank driver's schedule trace (ScheduleTrace semantics, schedule_trace.cpp:17-49):
    gathered from every rank, identical on all ranks; the serial tier (coarse sweep and
    correctors of every rank) on worker 0, rank p's fine solves on worker p+1; idle gaps only
    on fine lanes and W > 0 (no fine lane can start before the coarse sweep reaches it)."""
    world, l = 4, 2
    out = _run(world, mode, l, 1e-300)
    lanes0, idle0 = out[0][6], out[0][7]
    for o in out:
        assert o[6] == lanes0 and o[7] == idle0
    COARSE, FINE, CORRECT, IDLE = 0, 1, 2, 3
    assert lanes0[(0, COARSE)] == world  # one coarse-sweep task per rank
    assert lanes0[(0, CORRECT)] == sum(min(n - 1, l) for n in range(1, world + 1))
    for n in range(1, world + 1):
        assert lanes0[(n, FINE)] == min(n, l)  # F for k = 1..min(n, l)
        assert lanes0.get((n, IDLE), 0) >= 1
    assert (0, IDLE) not in lanes0
    assert idle0 > 0.0


def test_hybrid_rank_layout():
    """Hybrid space x time layout (bench N >= 4): member q of slice p is global rank
    p * members + q; time groups join same-index members, space groups are adjacent ranks."""
    from paper_2604_12083_b200.parareal import hybrid_groups

    tg, sg = hybrid_groups(8, 2)
    assert tg == [[0, 2, 4, 6], [1, 3, 5, 7]]
    assert sg == [[0, 1], [2, 3], [4, 5], [6, 7]]
    tg, sg = hybrid_groups(8, 4)
    assert tg == [[0, 4], [1, 5], [2, 6], [3, 7]] and sg == [[0, 1, 2, 3], [4, 5, 6, 7]]
    for world, members in ((4, 2), (8, 2), (8, 4)):
        tg, sg = hybrid_groups(world, members)
        assert sorted(r for g in tg for r in g) == list(range(world))
        assert sorted(r for g in sg for r in g) == list(range(world))
