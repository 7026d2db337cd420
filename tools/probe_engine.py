"""Dev tool: wall time of the single-device Parareal engine (flagellum, n=8 x 1000 RK2 | 100
Euler) per l and lane count, repeated -- the bench's parareal_1gpu leg in isolation."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2604_12083_b200 import parareal as pr  # noqa: E402
from paper_2604_12083_b200.scenario import ScenarioConfig, build_initial_state, make_scenario  # noqa: E402

sc = make_scenario(ScenarioConfig(rod_count=1, nodes_per_rod=100))
x0 = build_initial_state(sc)
n, fine, coarse = 8, 1000, 100
T = n * fine * 1e-6
for workers in (8, 9):
    for l in (1, 2, 3, 1):
        plan = pr.ParallelPlan(horizon=T, intervals=n, workers=workers, max_iterations=l, tolerance=1e-300,
                               mode=pr.PIPELINED)
        walls = []
        for _ in range(3):
            t0 = time.perf_counter()
            res = pr.run_gpu(plan, sc, fine, coarse, x0)
            walls.append((res.report.wall_seconds * 1e3, (time.perf_counter() - t0) * 1e3))
        print(f"workers {workers} l {l}: " + ", ".join(f"{a:.1f}/{b:.1f} ms" for a, b in walls), flush=True)
        ev = res.trace.events
        fines = sorted((e.t_start, e.t_end, e.interval) for e in ev if e.kind == pr.FINE)
        print("   fine spans:", [(round(a * 1e3, 2), round(b * 1e3, 2), k) for a, b, k in fines][:9], flush=True)
