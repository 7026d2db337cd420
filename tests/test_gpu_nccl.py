"""The NCCL transport end to end on one GPU: torch.distributed (nccl, world 1) shares the
unique id, the rank driver runs the single-slice plan, and the result equals the engine."""
import os
import socket

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def test_nccl_rank_driver_world1(gpu):
    import torch.distributed as dist

    from paper_2604_12083_b200 import parareal as pr
    from paper_2604_12083_b200.scenario import ScenarioConfig, build_initial_state, make_scenario

    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK="0", WORLD_SIZE="1")
    dist.init_process_group("nccl", rank=0, world_size=1)
    try:
        sc = make_scenario(ScenarioConfig(rod_count=2, nodes_per_rod=32, epsilon=0.08, horizon=1e-3))
        x0 = build_initial_state(sc)
        plan = pr.ParallelPlan(horizon=1e-3, intervals=1, workers=1, max_iterations=1, tolerance=1e-300, mode=1)
        res = pr.run_sliced_rank(plan, sc, 20, 2, x0, 0)
        eng = pr.run_gpu(plan, sc, 20, 2, x0)
        assert np.array_equal(res.state, eng.states[1])
        assert res.report.iterations_used == 1 and res.report.converged
    finally:
        dist.destroy_process_group()
