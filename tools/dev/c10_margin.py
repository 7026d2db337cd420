"""Dev: the acceptance-C10 margin (pipelined vs regular engine wall time, desk 1 x 31, 8 x 400
RK2, l = 3, r = 2) over 10 repetitions for m = 2, 4."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
from paper_2604_12083_b200 import parareal as pr
from paper_2604_12083_b200.harness import RunConfig
from paper_2604_12083_b200.scenario import ScenarioConfig, build_initial_state, make_scenario

scfg = ScenarioConfig(rod_count=1, nodes_per_rod=31, horizon=1.0, seed=1)
sc = make_scenario(scfg)
x0 = build_initial_state(sc)


def wall(mode, m, r=2.0):
    cfg = RunConfig(scenario=scfg, intervals=8, workers=m, ratio=r, max_iterations=3, tolerance=1e-300,
                    fine_steps_per_interval=400, coarse_steps_per_interval=0, mode=mode)
    plan = pr.ParallelPlan(horizon=1.0, intervals=8, workers=m, cost_ratio=r, max_iterations=3, tolerance=1e-300,
                           mode=mode)
    return pr.run_gpu(plan, sc, 400, cfg.resolved_coarse_steps(), x0).report.wall_seconds


wall(pr.PIPELINED, 2)
for m in (2, 4, 9):
    ps = [wall(pr.PIPELINED, m) for _ in range(10)]
    rs = [wall(pr.REGULAR, m) for _ in range(10)]
    print(f"m={m}: pipelined ms {sorted(round(1e3 * p, 2) for p in ps)}")
    print(f"      regular   ms {sorted(round(1e3 * r, 2) for r in rs)}")
