"""Dev tool: the threads + peer-memory hand-off case of tests/test_gpu_parareal.py in isolation
(run under `timeout`, optionally with cuda-gdb attached to dump host/device state)."""
import faulthandler
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
faulthandler.dump_traceback_later(int(os.environ.get("DUMP_AFTER", "45")), exit=False)

import numpy as np  # noqa: E402

from paper_2604_12083_b200 import parareal as pr  # noqa: E402
from paper_2604_12083_b200.scenario import ScenarioConfig, build_initial_state, make_scenario  # noqa: E402

mode = int(sys.argv[1]) if len(sys.argv) > 1 else 0
handoff = (sys.argv[2] != "0") if len(sys.argv) > 2 else True
sc = make_scenario(ScenarioConfig(rod_count=2, nodes_per_rod=32, horizon=4e-3, epsilon=0.08))
x0 = build_initial_state(sc)
for l in (1, 2, 4):
    plan = pr.ParallelPlan(horizon=4e-3, intervals=4, workers=4, max_iterations=l, tolerance=1e-300, mode=mode)
    t = time.time()
    eng = pr.run_gpu(plan, sc, 20, 2, x0)
    print("engine", l, time.time() - t, flush=True)
    t = time.time()
    ho = pr.run_sliced_threads(plan, sc, 20, 2, x0, [0, 0, 0, 0], handoff=handoff)
    print("sliced", l, time.time() - t, all(np.array_equal(ho.states[n], eng.states[n]) for n in range(5)),
          ho.report.eta_tilde == eng.report.eta_tilde, flush=True)
