"""Time integrators — mirror of reference include/pintswim/propagators.hpp:36-65.

States are packed (12 doubles per node, io.cpp:10-25): numpy arrays use the host-buffer
C entry points, float64 CUDA tensors stay in HBM.  Every call runs the sm_100a kernels of
libpswim.so through a per-(device, scenario) :class:`Context`.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass
from typing import Optional

import numpy as np

from . import _lib
from .device import Context, dptr, host_f64, hptr, is_device
from .scenario import Scenario, ScenarioConfig, make_scenario
from .stokes import LoadSet

EULER = 0
RK2 = 1
StiffnessError = _lib.StiffnessError


@dataclass
class StepperConfig:
    """StepperConfig, propagators.hpp:15-20."""

    dt: float = 1e-6
    scheme: int = RK2
    steps_per_interval: int = 0


@dataclass
class SystemVelocities:
    u: object
    omega: object


_ctx_cache: dict = {}


def context_for(sc, device: int = 0) -> Context:
    """Cached context holding the HBM workspaces of scenario `sc` on `device`."""
    if isinstance(sc, ScenarioConfig):
        sc = make_scenario(sc)
    c = sc.to_c()
    key = (device, bytes(c))
    ctx = _ctx_cache.get(key)
    if ctx is None:
        ctx = Context(device, c)
        _ctx_cache[key] = ctx
    return ctx


def _torch():
    import torch

    return torch


def _device_state(state, ctx: Context):
    torch = _torch()
    if is_device(state):
        return state.contiguous(), True
    return torch.as_tensor(host_f64(state).reshape(-1), device=f"cuda:{ctx.device}"), False


def rhs(state, t: float, sc: Scenario, extra: Optional[LoadSet] = None, ctx: Context | None = None) -> SystemVelocities:
    """Elastic + LJ loads through the Stokes mobility (propagators.cpp:38-91)."""
    torch = _torch()
    ctx = ctx or context_for(sc, state.device.index if is_device(state) else 0)
    ds, on_dev = _device_state(state, ctx)
    n = ds.numel() // 12
    u = torch.empty((n, 3), dtype=torch.float64, device=ds.device)
    w = torch.empty_like(u)
    ef = en = None
    if extra is not None:
        ef = torch.as_tensor(host_f64(extra.f, (-1, 3)) if not is_device(extra.f) else extra.f, device=ds.device).contiguous()
        en = torch.as_tensor(host_f64(extra.n, (-1, 3)) if not is_device(extra.n) else extra.n, device=ds.device).contiguous()
        if ef.shape[0] != n or en.shape[0] != n:
            raise _lib.InvalidArgument(1, "rhs: injected LoadSet has wrong node count")
    ctx.after_torch()
    ctx.check(ctx.lib.pswim_rhs(ctx.handle, dptr(ds), float(t), dptr(ef) if ef is not None else None,
                                dptr(en) if en is not None else None, dptr(u), dptr(w)))
    ctx.sync()
    if on_dev:
        return SystemVelocities(u, w)
    return SystemVelocities(u.cpu().numpy(), w.cpu().numpy())


def advance_state(state, vel: SystemVelocities, dt: float, sc: Scenario, ctx: Context | None = None):
    """Forward map over dt (propagators.cpp:93-124): Euler position, Rodrigues triads."""
    torch = _torch()
    ctx = ctx or context_for(sc, state.device.index if is_device(state) else 0)
    ds, on_dev = _device_state(state, ctx)
    n = ds.numel() // 12
    u = torch.as_tensor(vel.u if is_device(vel.u) else host_f64(vel.u, (-1, 3)), device=ds.device).contiguous()
    w = torch.as_tensor(vel.omega if is_device(vel.omega) else host_f64(vel.omega, (-1, 3)), device=ds.device).contiguous()
    if u.shape[0] != n or w.shape[0] != n:
        raise _lib.InvalidArgument(1, "advance_state: velocity sample has wrong node count")
    out = torch.empty_like(ds)
    ctx.after_torch()
    ctx.check(ctx.lib.pswim_advance_state(ctx.handle, dptr(ds), dptr(u), dptr(w), float(dt), dptr(out)))
    ctx.sync()
    return out if on_dev else out.cpu().numpy()


def _step(scheme, state, t, dt, sc, ctx):
    torch = _torch()
    ctx = ctx or context_for(sc, state.device.index if is_device(state) else 0)
    ds, on_dev = _device_state(state, ctx)
    out = torch.empty_like(ds)
    ctx.after_torch()
    ctx.check(ctx.lib.pswim_step(ctx.handle, scheme, dptr(ds), float(t), float(dt), dptr(out)))
    ctx.sync()
    return out if on_dev else out.cpu().numpy()


def step_euler(state, t: float, dt: float, sc: Scenario, ctx: Context | None = None):
    return _step(EULER, state, t, dt, sc, ctx)


def step_rk2(state, t: float, dt: float, sc: Scenario, ctx: Context | None = None):
    return _step(RK2, state, t, dt, sc, ctx)


def propagate(state, t0: float, t1: float, cfg: StepperConfig, sc: Scenario, ctx: Context | None = None):
    """Serial composition of steps over [t0, t1] (propagators.cpp:135-162)."""
    if is_device(state):
        torch = _torch()
        ctx = ctx or context_for(sc, state.device.index or 0)
        ds = state.contiguous()
        out = torch.empty_like(ds)
        ctx.after_torch()
        ctx.check(ctx.lib.pswim_propagate(ctx.handle, dptr(ds), float(t0), float(t1), int(cfg.scheme),
                                          int(cfg.steps_per_interval), float(cfg.dt), dptr(out)))
        return out
    ctx = ctx or context_for(sc, 0)
    x = host_f64(state).reshape(-1).copy()
    out = np.zeros_like(x)
    ctx.check(ctx.lib.pswim_propagate_host(ctx.handle, hptr(x), float(t0), float(t1), int(cfg.scheme),
                                           int(cfg.steps_per_interval), float(cfg.dt), hptr(out)))
    return out


def propagate_sharded(state, t0: float, t1: float, cfg: StepperConfig, sc: Scenario, transport,
                      ctx: Context | None = None):
    """propagate with the O(N^2) MRS sharded across the ranks of `transport` (each rank its
    256-target blocks, one (u, omega) all-gather per rhs).  Every rank passes the same full
    state (CUDA tensor on its device); all ranks must call together.  Bitwise identical to
    :func:`propagate` on one GPU (space-parallel MRS)."""
    torch = _torch()
    ctx = ctx or context_for(sc, state.device.index or 0)
    ds = state.contiguous()
    out = torch.empty_like(ds)
    ctx.after_torch()
    ctx.check(ctx.lib.pswim_propagate_sharded(ctx.handle, transport, dptr(ds), float(t0), float(t1), int(cfg.scheme),
                                              int(cfg.steps_per_interval), float(cfg.dt), dptr(out)))
    return out


class ThreadTransports:
    """`world` in-process ranks (threads) on the given devices (pswim_threads_transports_create)."""

    def __init__(self, devices, len_hint: int = 1, slots: int = 4):
        L = _lib.lib()
        self.world = len(devices)
        devs = (C.c_int * self.world)(*[int(d) for d in devices])
        self.ptr = L.pswim_threads_transports_create(self.world, devs, int(len_hint), int(slots))
        if not self.ptr:
            raise _lib.DeviceError(6, "pswim_threads_transports_create failed")
        self.lib = L

    def __getitem__(self, rank: int):
        return C.pointer(self.ptr[rank])

    def close(self):
        if self.ptr:
            self.lib.pswim_threads_transports_destroy(self.ptr)
            self.ptr = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


class PeerGroup:
    """Exchange block of one rank for the fused sharded-MRS + all-gather over peer memory
    (pswim_peer_group_*).  Share :meth:`handle` (CUDA IPC, other processes) or :attr:`base`
    (ranks of this process), then :meth:`connect`."""

    def __init__(self, ctx: Context, rank: int, world: int):
        self.ctx = ctx
        self.lib = ctx.lib
        self.rank, self.world = int(rank), int(world)
        self.ptr = self.lib.pswim_peer_group_create(ctx.handle, self.rank, self.world)
        if not self.ptr:
            raise _lib.DeviceError(6, "pswim_peer_group_create failed")

    def handle(self) -> bytes:
        buf = (C.c_uint8 * 64)()
        ctx_check = self.lib.pswim_peer_group_handle(self.ptr, buf)
        _lib.raise_for(ctx_check, "cudaIpcGetMemHandle failed")
        return bytes(buf)

    @property
    def base(self) -> int:
        return self.lib.pswim_peer_group_local_base(self.ptr)

    def connect(self, handles=None, bases=None) -> None:
        if handles is not None:
            raw = (C.c_uint8 * (64 * self.world))(*b"".join(handles))
            rc = self.lib.pswim_peer_group_connect(self.ptr, raw, None)
        else:
            arr = (C.c_void_p * self.world)(*bases)
            rc = self.lib.pswim_peer_group_connect(self.ptr, None, arr)
        _lib.raise_for(rc, "pswim_peer_group_connect failed")

    def close(self) -> None:
        if self.ptr:
            self.lib.pswim_peer_group_destroy(self.ptr)
            self.ptr = None


def propagate_sharded_peer(state, t0: float, t1: float, cfg: StepperConfig, sc: Scenario, group: PeerGroup):
    """propagate with the sharded MRS whose all-gather is fused into the kernel epilogue over
    peer memory; bitwise identical to :func:`propagate` on one GPU."""
    torch = _torch()
    ctx = group.ctx
    ds = state.contiguous()
    out = torch.empty_like(ds)
    ctx.after_torch()
    ctx.check(ctx.lib.pswim_propagate_sharded_peer(ctx.handle, group.ptr, dptr(ds), float(t0), float(t1),
                                                   int(cfg.scheme), int(cfg.steps_per_interval), float(cfg.dt),
                                                   dptr(out)))
    return out
