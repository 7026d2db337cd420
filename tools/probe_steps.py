"""Time-step throughput probe (dev tool): RK2 steps/s for the flagellum (1 x 100) with the
fused cluster kernel and with per-step launches, and for the 64 x 256 suspension."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

from paper_2604_12083_b200.device import Context, dptr
from paper_2604_12083_b200.scenario import ScenarioConfig, build_initial_state, make_scenario


def rate(kw, steps, fused, graphs=True):
    sc = make_scenario(ScenarioConfig(**kw))
    ctx = Context(0, sc)
    cs = ctx.lib.pswim_set_fused(ctx.handle, 1 if fused else 0)
    ctx.lib.pswim_set_graphs(ctx.handle, 1 if graphs else 0)
    x = torch.as_tensor(build_initial_state(sc), device="cuda")
    out = torch.empty_like(x)
    L = ctx.lib
    ctx.check(L.pswim_propagate(ctx.handle, dptr(x), 0.0, 10e-6, 1, 10, 0.0, dptr(out)))
    st = ctx.torch_stream()
    a = torch.cuda.Event(enable_timing=True)
    b = torch.cuda.Event(enable_timing=True)
    a.record(st)
    ctx.check(L.pswim_propagate(ctx.handle, dptr(x), 0.0, steps * 1e-6, 1, steps, 0.0, dptr(out)))
    b.record(st)
    b.synchronize()
    sec = a.elapsed_time(b) * 1e-3
    ctx.close()
    return steps / sec, cs


for kw, steps in [(dict(rod_count=1, nodes_per_rod=100), 20000), (dict(rod_count=1, nodes_per_rod=21), 20000),
                  (dict(rod_count=2, nodes_per_rod=128, epsilon=0.08), 5000)]:
    for fused in (True, False):
        r, cs = rate(kw, steps if fused else steps // 10, fused)
        print(f"{kw} fused={fused} cluster={cs}: {r:,.0f} RK2 steps/s")
# the paper's benchmark sizes (4 / 12 / 25 rods x 51 nodes), per-step kernels
for kw in (dict(rod_count=4, nodes_per_rod=51), dict(rod_count=12, nodes_per_rod=51),
           dict(rod_count=25, nodes_per_rod=51), dict(rod_count=3, nodes_per_rod=100)):
    fused = kw["rod_count"] * kw["nodes_per_rod"] <= 256  # fused path where eligible, else per-step kernels
    for graphs in (True, False):
        r, cs = rate(kw, 2048, fused, graphs)
        print(f"{kw} graphs={graphs} fused={fused}: {r:,.0f} RK2 steps/s")
for graphs in (True, False, True, False):
    r, _ = rate(dict(rod_count=64, nodes_per_rod=256, epsilon=0.08), 100, False, graphs)
    print(f"64x256 graphs={graphs}: {r:,.1f} RK2 steps/s")
