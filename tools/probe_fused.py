"""Phase breakdown of the fused small-system propagate (dev tool): in-kernel clock64 phase
timer (pswim_fused_profile) on the flagellum (BASELINE configs[0]) and a 4 x 21 LJ desk."""
import ctypes as C
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

from paper_2604_12083_b200.device import Context, dptr
from paper_2604_12083_b200.scenario import ScenarioConfig, build_initial_state, make_scenario

PHASES = ["front: nodes+stage (+phased)", "front: advance", "front: segments", "mrs_pairs", "reduce+push", "velocity wait", "final advance"]


def profile(kw, steps=2000, cluster=1):
    sc = make_scenario(ScenarioConfig(**kw))
    ctx = Context(0, sc)
    cs = ctx.lib.pswim_set_fused(ctx.handle, cluster)
    x = torch.as_tensor(build_initial_state(sc), device="cuda")
    out = torch.empty_like(x)
    cyc = (C.c_uint64 * 7)()
    ctx.check(ctx.lib.pswim_fused_profile(ctx.handle, dptr(x), 0.0, steps * 1e-6, 1, steps, dptr(out), cyc))
    st = ctx.torch_stream()
    a = torch.cuda.Event(enable_timing=True)
    b = torch.cuda.Event(enable_timing=True)
    a.record(st)
    ctx.check(ctx.lib.pswim_fused_profile(ctx.handle, dptr(x), 0.0, steps * 1e-6, 1, steps, dptr(out), cyc))
    b.record(st)
    b.synchronize()
    us_step = a.elapsed_time(b) * 1e3 / steps
    tot = sum(cyc)
    print(f"{kw}: cluster {cs}, {us_step:.2f} us/RK2 step ({1e6 / us_step:.0f} steps/s incl. timer), "
          f"{tot / steps:.0f} cycles/step")
    for name, c in zip(PHASES, cyc):
        print(f"   {name:28s} {c / steps:8.0f} cycles/step  {100 * c / tot:5.1f} %")
    ctx.close()


def plain(kw, steps=20000, cluster=16):
    """Steps/s of the fused propagate without the phase timer (the bench's configs[0] leg)."""
    sc = make_scenario(ScenarioConfig(**kw))
    ctx = Context(0, sc)
    cs = ctx.lib.pswim_set_fused(ctx.handle, cluster)
    x = torch.as_tensor(build_initial_state(sc), device="cuda")
    out = torch.empty_like(x)
    ctx.check(ctx.lib.pswim_propagate(ctx.handle, dptr(x), 0.0, 1e-5, 1, 10, 0.0, dptr(out)))
    st = ctx.torch_stream()
    a = torch.cuda.Event(enable_timing=True)
    b = torch.cuda.Event(enable_timing=True)
    a.record(st)
    ctx.check(ctx.lib.pswim_propagate(ctx.handle, dptr(x), 0.0, steps * 1e-6, 1, steps, 0.0, dptr(out)))
    b.record(st)
    b.synchronize()
    print(f"{kw}: cluster {cs}: {steps / (a.elapsed_time(b) * 1e-3):.0f} RK2 steps/s (no timer)")
    ctx.close()


if __name__ == "__main__":
    plain(dict(rod_count=1, nodes_per_rod=100))
    profile(dict(rod_count=1, nodes_per_rod=100), cluster=16)
    profile(dict(rod_count=1, nodes_per_rod=100))
    profile(dict(rod_count=4, nodes_per_rod=21, placement=1, lj_well_depth=0.01, seed=2))
