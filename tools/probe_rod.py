"""HBM-roofline microbenchmarks of the rod-side kernels (dev tool, also used by bench.py):
batched sqrt_rotation (144 B/matrix), rod_loads (144 B/node algorithmic), advance_state
(240 B/node) on >= 1e7 elements so the working set is far beyond the 126 MB L2."""
import ctypes as C
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

from paper_2604_12083_b200.device import Context, dptr
from paper_2604_12083_b200.scenario import ScenarioConfig, build_initial_state, make_scenario


def _time(st, fn, reps=5):
    fn()
    torch.cuda.synchronize()
    best = 1e30
    for _ in range(reps):
        a = torch.cuda.Event(enable_timing=True)
        b = torch.cuda.Event(enable_timing=True)
        a.record(st)
        fn()
        b.record(st)
        b.synchronize()
        best = min(best, a.elapsed_time(b))
    return best * 1e-3


def hbm_kernels(device=0, matrices=10_000_000, rods=40_000, m=256):
    out = {}
    ctx = Context(device)
    st = ctx.torch_stream()
    L = ctx.lib
    dev = torch.device("cuda", device)
    # batched sqrt: random rotations via QR of random matrices (det fixed to +1)
    g = torch.Generator(device=dev).manual_seed(0)
    qv = torch.randn(matrices, 4, dtype=torch.float64, device=dev, generator=g)
    qv = qv / qv.norm(dim=1, keepdim=True)
    w_, x_, y_, z_ = qv.unbind(1)
    q = torch.stack([1 - 2 * (y_ * y_ + z_ * z_), 2 * (x_ * y_ - z_ * w_), 2 * (x_ * z_ + y_ * w_),
                     2 * (x_ * y_ + z_ * w_), 1 - 2 * (x_ * x_ + z_ * z_), 2 * (y_ * z_ - x_ * w_),
                     2 * (x_ * z_ - y_ * w_), 2 * (y_ * z_ + x_ * w_), 1 - 2 * (x_ * x_ + y_ * y_)], 1).view(-1, 3, 3)
    del qv, w_, x_, y_, z_
    r9 = q.reshape(-1, 9).contiguous()
    s9 = torch.empty_like(r9)
    t = _time(st, lambda: ctx.check(L.pswim_sqrt_rotation_batched(ctx.handle, dptr(r9), matrices, dptr(s9))))
    out["sqrt_rotation_batched"] = {"elements": matrices, "bytes_per_element": 144, "seconds": t,
                                    "GB_per_s": 144 * matrices / t / 1e9}
    err = (s9.reshape(-1, 3, 3) @ s9.reshape(-1, 3, 3) - q).abs().amax().item()
    out["sqrt_rotation_batched"]["max_abs_residual_S2_minus_R"] = err
    del q, r9, s9
    # rod loads + advance on a rods x m suspension (grid placement), pre-perturbed
    sc = make_scenario(ScenarioConfig(rod_count=rods, nodes_per_rod=m, epsilon=0.08))
    ctx2 = Context(device, sc)
    x0 = torch.as_tensor(build_initial_state(sc), device=dev)
    nodes = rods * m
    f = torch.empty((nodes, 3), dtype=torch.float64, device=dev)
    n = torch.empty_like(f)
    t = _time(ctx2.torch_stream(), lambda: ctx2.check(L.pswim_rod_loads(ctx2.handle, dptr(x0), 0.1, dptr(f), dptr(n), None, None)))
    out["rod_loads"] = {"elements": nodes, "bytes_per_element": 144, "seconds": t, "GB_per_s": 144 * nodes / t / 1e9}
    u = torch.randn((nodes, 3), dtype=torch.float64, device=dev) * 1e-3
    w = torch.randn((nodes, 3), dtype=torch.float64, device=dev)
    xo = torch.empty_like(x0)
    t = _time(ctx2.torch_stream(), lambda: ctx2.check(L.pswim_advance_state(ctx2.handle, dptr(x0), dptr(u), dptr(w), 1e-6, dptr(xo))))
    out["advance_state"] = {"elements": nodes, "bytes_per_element": 240, "seconds": t, "GB_per_s": 240 * nodes / t / 1e9}
    ctx2.sync()
    ctx2.close()
    ctx.close()
    return out


if __name__ == "__main__":
    print(json.dumps(hbm_kernels(), indent=1))
