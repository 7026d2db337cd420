"""MRS operator — mirror of the reference's include/pintswim/stokes.hpp.

``evaluate_velocities(targets, sources, loads, kp)`` keeps the reference signature
(stokes.hpp:43-44) and raises ``InvalidArgument`` / ``PswimError`` where the reference
throws (stokes.cpp:11-26).  numpy inputs go through the host-buffer C entry point
(H2D + kernel + D2H); CUDA tensors stay in HBM (stream-ordered device entry point).
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass
from typing import NamedTuple

import numpy as np

from . import _lib
from .device import Context, default_context, dptr, host_f64, hptr, is_device

FREE_SPACE = 0
IMAGE_WALL = 1


@dataclass
class KernelParams:
    """KernelParams, reference stokes.hpp:13-17."""

    epsilon: float = 0.1
    mu: float = 1.0
    wall_mode: int = FREE_SPACE

    def to_c(self) -> _lib.KernelParams:
        return _lib.KernelParams(float(self.epsilon), float(self.mu), int(self.wall_mode), 0)


class LoadSet(NamedTuple):
    """Per-node force / torque densities on the fluid (stokes.hpp:30-33)."""

    f: object
    n: object


class VelocityField(NamedTuple):
    """(stokes.hpp:35-38)"""

    u: object
    omega: object


def evaluate_velocities(targets, sources, loads: LoadSet, kp: KernelParams, ctx: Context | None = None) -> VelocityField:
    if is_device(targets):
        import torch

        ctx = ctx or default_context(targets.device.index or 0)
        nt, ns = targets.shape[0], sources.shape[0]
        if loads.f.shape[0] != ns or loads.n.shape[0] != ns:
            raise _lib.InvalidArgument(1, "stokes: load arrays must match source count")
        u = torch.empty((nt, 3), dtype=torch.float64, device=targets.device)
        w = torch.empty_like(u)
        ctx.after_torch()
        ctx.check(ctx.lib.pswim_mrs_velocities(ctx.handle, dptr(targets), nt, dptr(sources), dptr(loads.f),
                                               dptr(loads.n), ns, C.byref(kp.to_c()), dptr(u), dptr(w)))
        ctx.sync()
        return VelocityField(u, w)
    ctx = ctx or default_context(0)
    t = host_f64(targets, (-1, 3))
    s = host_f64(sources, (-1, 3))
    f = host_f64(loads.f, (-1, 3))
    n = host_f64(loads.n, (-1, 3))
    if len(f) != len(s) or len(n) != len(s):
        raise _lib.InvalidArgument(1, "stokes: load arrays must match source count")
    u = np.zeros_like(t)
    w = np.zeros_like(t)
    ctx.check(ctx.lib.pswim_mrs_velocities_host(ctx.handle, hptr(t), len(t), hptr(s), hptr(f), hptr(n), len(s),
                                                C.byref(kp.to_c()), hptr(u), hptr(w)))
    return VelocityField(u, w)


def h_functions(r, epsilon: float, ctx: Context | None = None) -> np.ndarray:
    """h_functions (stokes.cpp:59-74) evaluated on the device; returns (..., 5)."""
    import torch

    ctx = ctx or default_context(0)
    r = np.atleast_1d(np.asarray(r, dtype=np.float64))
    if epsilon <= 0.0 or np.any(r < 0.0):
        raise _lib.InvalidArgument(1, "h_functions: r >= 0 and epsilon > 0 required")
    dr = torch.as_tensor(r, device=f"cuda:{ctx.device}")
    dh = torch.empty((len(r), 5), dtype=torch.float64, device=dr.device)
    ctx.after_torch()
    ctx.check(ctx.lib.pswim_h_functions(ctx.handle, dptr(dr), len(r), float(epsilon), dptr(dh)))
    ctx.sync()
    return dh.cpu().numpy()
