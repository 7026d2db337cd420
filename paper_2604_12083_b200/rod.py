"""Rod mechanics — mirror of reference include/pintswim/rod.hpp:58-79 on the device.

``rod_loads`` runs internal_loads + nodal_loads (rod.cpp:36-109) for every rod of the
scenario in one kernel; ``lj_repulsion`` is the pair-force kernel (rod.cpp:124-174).
"""
from __future__ import annotations

from .device import dptr, is_device
from .propagators import _device_state, context_for


def rod_loads(state, t: float, sc, ctx=None):
    """Returns (f, n, segment_force, segment_moment) as numpy arrays (device if the input
    state is a CUDA tensor)."""
    import torch

    ctx = ctx or context_for(sc, state.device.index if is_device(state) else 0)
    ds, on_dev = _device_state(state, ctx)
    rods, m = ctx._sc.rod_count, ctx._sc.nodes_per_rod
    f = torch.empty((rods * m, 3), dtype=torch.float64, device=ds.device)
    n = torch.empty_like(f)
    sf = torch.empty((rods * (m - 1), 3), dtype=torch.float64, device=ds.device)
    sn = torch.empty_like(sf)
    ctx.after_torch()
    ctx.check(ctx.lib.pswim_rod_loads(ctx.handle, dptr(ds), float(t), dptr(f), dptr(n), dptr(sf), dptr(sn)))
    ctx.sync()
    out = (f, n, sf, sn)
    return out if on_dev else tuple(a.cpu().numpy() for a in out)


def lj_repulsion(state, sc, ctx=None):
    import torch

    ctx = ctx or context_for(sc, state.device.index if is_device(state) else 0)
    ds, on_dev = _device_state(state, ctx)
    out = torch.empty((ds.numel() // 12, 3), dtype=torch.float64, device=ds.device)
    ctx.after_torch()
    ctx.check(ctx.lib.pswim_lj_forces(ctx.handle, dptr(ds), dptr(out)))
    ctx.sync()
    return out if on_dev else out.cpu().numpy()
