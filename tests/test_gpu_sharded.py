"""Space-parallel MRS: the propagate with the O(N^2) sum sharded over
in-process ranks sharing cuda:0 (peer-copy all-gather of (u, omega)) is bitwise identical to
the single-GPU propagate, for 2 and 3 ranks and uneven block splits."""
import threading

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("world,kw", [(2, dict(rod_count=4, nodes_per_rod=100)),
                                      (3, dict(rod_count=9, nodes_per_rod=64, epsilon=0.08)),
                                      (4, dict(rod_count=3, nodes_per_rod=200, epsilon=0.08))])
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
