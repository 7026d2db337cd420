"""Hybrid space x time: Parareal slices whose coarse and fine propagators
shard the MRS over a space group.  2 slices x 2 members = 4 thread-ranks sharing cuda:0;
every member of every slice must reproduce the task-graph engine's boundary states and
report bitwise (the sharded propagate is bitwise identical to the single-GPU one)."""
import threading

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("mode,l", [(1, 1), (1, 2), (0, 2)])
def test_hybrid_space_time_bitwise_equals_engine(gpu, mode, l):
    from paper_2604_12083_b200 import parareal as pr
    from paper_2604_12083_b200.propagators import ThreadTransports
    from paper_2604_12083_b200.scenario import ScenarioConfig, build_initial_state, make_scenario

    slices, members = 2, 2
    sc = make_scenario(ScenarioConfig(rod_count=9, nodes_per_rod=64, epsilon=0.08, horizon=2e-5))
    x0 = build_initial_state(sc)
    plan = pr.ParallelPlan(horizon=2e-5, intervals=slices, workers=slices, max_iterations=l, tolerance=1e-300,
                           mode=mode)
    eng = pr.run_gpu(plan, sc, 6, 2, x0)

    time_tr = [ThreadTransports([0] * slices, len_hint=x0.size, slots=l + 2) for _ in range(members)]
    space_c = [ThreadTransports([0] * members) for _ in range(slices)]
    space_f = [ThreadTransports([0] * members) for _ in range(slices)]
    out, errs = {}, []

    def rank(p, q):
        try:
            out[p, q] = pr.run_sliced_rank(plan, sc, 6, 2, x0, 0, transport=time_tr[q][p],
                                           space=(space_c[p][q], space_f[p][q]))
        except Exception as e:  # pragma: no cover
            errs.append(e)

    th = [threading.Thread(target=rank, args=(p, q)) for p in range(slices) for q in range(members)]
    for t in th:
        t.start()
    for t in th:
        t.join(timeout=300)
    assert not errs, errs
    for (p, q), res in out.items():
        assert np.array_equal(res.state, eng.states[p + 1]), (p, q)
        assert res.report.eta_tilde == eng.report.eta_tilde
        assert res.report.iterations_used == l
    for group in time_tr + space_c + space_f:
        group.close()
