"""Parareal on ONE B200 (dev tool): small systems leave most SMs idle, so n time slices run
concurrently as slice ranks on their own streams (fused cluster kernels side by side).
Reports wall time vs the serial fine integration and the true error eta."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

from paper_2604_12083_b200 import parareal as pr
from paper_2604_12083_b200.device import Context, dptr
from paper_2604_12083_b200.scenario import ScenarioConfig, build_initial_state, make_scenario


def serial_fine(sc, x0, n, fine, T):
    ctx = Context(0, sc)
    dx = torch.as_tensor(x0, device="cuda")
    out = torch.empty_like(dx)
    states = [x0]
    cur = dx.clone()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for i in range(n):
        ctx.check(ctx.lib.pswim_propagate(ctx.handle, dptr(cur), T * i / n, T * (i + 1) / n, 1, fine, 0.0, dptr(out)))
        cur.copy_(out)
        states.append(out.cpu().numpy())
    wall = time.perf_counter() - t0
    ctx.close()
    return states, wall


def main(nodes=100, rods=1, n=8, fine=1000, coarse=100, eps=0.0):
    sc = make_scenario(ScenarioConfig(rod_count=rods, nodes_per_rod=nodes, epsilon=eps))
    x0 = build_initial_state(sc)
    T = n * fine * 1e-6
    ref, wall_serial = serial_fine(sc, x0, n, fine, T)
    # boundary times must match the plan's boundary_time for a bitwise reference
    plan0 = pr.ParallelPlan(horizon=T, intervals=n, workers=n, max_iterations=1, tolerance=1e-300, mode=pr.PIPELINED)
    print(f"{rods}x{nodes}: serial fine {n * fine} RK2 steps: {wall_serial * 1e3:.1f} ms "
          f"({n * fine / wall_serial:,.0f} steps/s)")
    for l in (1, 2, 3):
        plan = pr.ParallelPlan(horizon=T, intervals=n, workers=n, max_iterations=l, tolerance=1e-300,
                               mode=pr.PIPELINED)
        pr.run_sliced_threads(plan, sc, fine, coarse, x0, [0] * n)  # warm-up
        t0 = time.perf_counter()
        res = pr.run_sliced_threads(plan, sc, fine, coarse, x0, [0] * n, reference=ref)
        wall = time.perf_counter() - t0
        w = res.report.wall_seconds
        print(f"  sliced pipelined Parareal l={l}: {w * 1e3:.1f} ms (call {wall * 1e3:.1f})  speedup {wall_serial / w:.2f}x  "
              f"eta={res.report.eta[-1]:.2e}  eta_tilde={res.report.eta_tilde[-1]:.2e}")
        t0 = time.perf_counter()
        eng = pr.run_gpu(plan, sc, fine, coarse, x0, reference=ref)
        wall = time.perf_counter() - t0
        w = eng.report.wall_seconds
        print(f"  engine (m={n} lanes)        l={l}: {w * 1e3:.1f} ms (call {wall * 1e3:.1f})  speedup {wall_serial / w:.2f}x  "
              f"eta={eng.report.eta[-1]:.2e}")


if __name__ == "__main__":
    main()
    main(nodes=51, rods=4, eps=0.0)
