"""Rotation square root — mirror of reference include/pintswim/rotation.hpp:34
(``sqrt_rotation``), batched on the device (src/rotation.cpp:91-107)."""
from __future__ import annotations

import numpy as np

from .device import Context, default_context, dptr, host_f64, hptr, is_device

K_THETA_LO = 1e-7   # rotation.hpp:42
K_THETA_HI = 1e-2   # rotation.hpp:43


def sqrt_rotation(r, ctx: Context | None = None):
    """S with S @ S = R for every 3x3 rotation in ``r`` (shape (..., 3, 3))."""
    if is_device(r):
        import torch

        ctx = ctx or default_context(r.device.index or 0)
        rr = r.reshape(-1, 9).contiguous()
        out = torch.empty_like(rr)
        ctx.after_torch()
        ctx.check(ctx.lib.pswim_sqrt_rotation_batched(ctx.handle, dptr(rr), rr.shape[0], dptr(out)))
        ctx.sync()
        return out.reshape(r.shape)
    ctx = ctx or default_context(0)
    a = host_f64(r)
    shape = a.shape
    flat = a.reshape(-1, 9).copy()
    out = np.zeros_like(flat)
    ctx.check(ctx.lib.pswim_sqrt_rotation_host(ctx.handle, hptr(flat), len(flat), hptr(out)))
    return out.reshape(shape)
