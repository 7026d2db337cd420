"""Space-parallel MRS: the propagate with the O(N^2) sum sharded over
in-process ranks sharing cuda:0 (peer-copy all-gather of (u, omega)) is bitwise identical to
the single-GPU propagate, for 2 and 3 ranks and uneven block splits."""
import threading

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("world,kw", [(2, dict(rod_count=4, nodes_per_rod=100)),
                                      (3, dict(rod_count=9, nodes_per_rod=64, epsilon=0.08)),
                                      (4, dict(rod_count=3, nodes_per_rod=200, epsilon=0.08)),
                                      # LJ through the cell list (N >= 2048) inside every rank's rhs
                                      (2, dict(rod_count=40, nodes_per_rod=64, placement=1, lj_well_depth=0.01,
                                               seed=5, epsilon=0.08)),
                                      # 64 x 256: the MRS plan with 37 source chunks
                                      (3, dict(rod_count=64, nodes_per_rod=256, epsilon=0.08))])
def test_sharded_propagate_bitwise(gpu, world, kw):
    import torch
    from paper_2604_12083_b200.device import Context
    from paper_2604_12083_b200.propagators import StepperConfig, ThreadTransports, propagate, propagate_sharded
    from paper_2604_12083_b200.scenario import ScenarioConfig, build_initial_state, make_scenario

    sc = make_scenario(ScenarioConfig(**kw))
    x0 = build_initial_state(sc)
    cfg = StepperConfig(0.0, 1, 6)
    ref_ctx = Context(0, sc)
    ref_ctx.lib.pswim_set_fused(ref_ctx.handle, 0)
    want = propagate(torch.as_tensor(x0, device=gpu), 0.0, 6e-5, cfg, sc, ctx=ref_ctx).cpu().numpy()
    trs = ThreadTransports([0] * world)
    ctxs = [Context(0, sc) for _ in range(world)]
    outs = [None] * world
    errs = []

    def rank(r):
        try:
            outs[r] = propagate_sharded(torch.as_tensor(x0, device=gpu), 0.0, 6e-5, cfg, sc, trs[r],
                                        ctx=ctxs[r]).cpu().numpy()
        except Exception as e:  # pragma: no cover
            errs.append(e)

    th = [threading.Thread(target=rank, args=(r,)) for r in range(world)]
    for t in th:
        t.start()
    for t in th:
        t.join(timeout=300)
    assert not errs, errs
    for r in range(world):
        assert np.array_equal(outs[r], want), r
    trs.close()


@pytest.mark.parametrize("world", [2, 4])
def test_fused_peer_allgather_threads_bitwise(gpu, world):
    """Fused compute + collective: the MRS epilogue stores (u, omega) into every rank's
    exchange block and signals with system-scope atomics (ranks as threads on cuda:0)."""
    import torch
    from paper_2604_12083_b200.device import Context
    from paper_2604_12083_b200.propagators import PeerGroup, StepperConfig, propagate, propagate_sharded_peer
    from paper_2604_12083_b200.scenario import ScenarioConfig, build_initial_state, make_scenario

    sc = make_scenario(ScenarioConfig(rod_count=9, nodes_per_rod=64, epsilon=0.08))
    x0 = build_initial_state(sc)
    cfg = StepperConfig(0.0, 1, 5)
    ref_ctx = Context(0, sc)
    ref_ctx.lib.pswim_set_fused(ref_ctx.handle, 0)
    want = propagate(torch.as_tensor(x0, device=gpu), 0.0, 5e-5, cfg, sc, ctx=ref_ctx).cpu().numpy()
    ctxs = [Context(0, sc) for _ in range(world)]
    groups = [PeerGroup(ctxs[r], r, world) for r in range(world)]
    bases = [g.base for g in groups]
    for g in groups:
        g.connect(bases=bases)
    outs, errs = [None] * world, []

    def rank(r):
        try:
            outs[r] = propagate_sharded_peer(torch.as_tensor(x0, device=gpu), 0.0, 5e-5, cfg, sc, groups[r]).cpu().numpy()
        except Exception as e:  # pragma: no cover
            errs.append(e)

    th = [threading.Thread(target=rank, args=(r,)) for r in range(world)]
    for t in th:
        t.start()
    for t in th:
        t.join(timeout=300)
    assert not errs, errs
    for r in range(world):
        assert np.array_equal(outs[r], want), r
    for g in groups:
        g.close()


def _peer_proc(rank, world, port, q):
    import os

    import torch
    import torch.distributed as dist

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2604_12083_b200.device import Context
        from paper_2604_12083_b200.propagators import PeerGroup, StepperConfig, propagate, propagate_sharded_peer
        from paper_2604_12083_b200.scenario import ScenarioConfig, build_initial_state, make_scenario

        sc = make_scenario(ScenarioConfig(rod_count=4, nodes_per_rod=100, epsilon=0.08))
        x0 = build_initial_state(sc)
        cfg = StepperConfig(0.0, 1, 4)
        ctx = Context(0, sc)
        g = PeerGroup(ctx, rank, world)
        handles = [None] * world
        dist.all_gather_object(handles, g.handle())
        g.connect(handles=handles)
        dist.barrier()
        out = propagate_sharded_peer(torch.as_tensor(x0, device="cuda:0"), 0.0, 4e-5, cfg, sc, g).cpu().numpy()
        dist.barrier()  # no rank frees its block while peers may still write into it
        g.close()
        ref = Context(0, sc)
        ref.lib.pswim_set_fused(ref.handle, 0)
        want = propagate(torch.as_tensor(x0, device="cuda:0"), 0.0, 4e-5, cfg, sc, ctx=ref).cpu().numpy()
        q.put((rank, bool(np.array_equal(out, want))))
    except Exception as e:  # pragma: no cover
        q.put((rank, repr(e)))
    finally:
        dist.destroy_process_group()


def test_fused_peer_allgather_ipc_processes(gpu):
    """Two processes on one GPU exchanging CUDA IPC handles (the one-process-per-GPU layout of
    an NVSwitch box): fused peer all-gather, bitwise identical to one GPU."""
    import socket

    import torch.multiprocessing as mp

    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    ps = [ctx.Process(target=_peer_proc, args=(r, 2, port, q)) for r in range(2)]
    for p in ps:
        p.start()
    res = sorted(q.get(timeout=300) for _ in range(2))
    for p in ps:
        p.join(timeout=60)
    assert res == [(0, True), (1, True)], res
