"""Device contexts and tensor plumbing over the C-ABI.

A :class:`Context` owns one ``pswim_ctx`` (device + CUDA stream + HBM workspaces for one
scenario).  PyTorch is used only to hold device memory and to order work against torch's
own streams; all arithmetic runs in libpswim.so's kernels.
"""
from __future__ import annotations

import atexit
import ctypes as C
import weakref
from typing import Optional

import numpy as np

from . import _lib
from ._lib import raise_for


def _torch():
    import torch

    return torch


def as_scenario_struct(sc) -> Optional[_lib.Scenario]:
    if sc is None:
        return None
    if isinstance(sc, _lib.Scenario):
        return sc
    return sc.to_c()


_LIVE: "weakref.WeakSet[Context]" = weakref.WeakSet()


@atexit.register
def _close_live_contexts() -> None:
    # release every context while the CUDA runtime is still up (interpreter teardown would
    # otherwise destroy them in an arbitrary order against torch's own CUDA state)
    for ctx in list(_LIVE):
        try:
            ctx.close()
        except Exception:
            pass


class Context:
    """One device stream with preallocated workspaces (pswim_create, include/pswim_c.h)."""

    def __init__(self, device: int = 0, scenario=None, priority: int = 0):
        L = _lib.lib()
        self.device = int(device)
        self._sc = as_scenario_struct(scenario)
        h = L.pswim_create(self.device, C.byref(self._sc) if self._sc is not None else None, int(priority))
        if not h:
            raise _lib.DeviceError(6, f"pswim_create failed on cuda:{device} (no GPU or bad scenario)")
        self.handle = h
        self.lib = L
        self._torch_stream = None
        _LIVE.add(self)

    def close(self) -> None:
        if getattr(self, "handle", None):
            self.lib.pswim_destroy(self.handle)
            self.handle = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def __enter__(self):
        return self

    def __exit__(self, *exc):
        self.close()

    # -- errors / sync ---------------------------------------------------------------------
    def error(self) -> str:
        return self.lib.pswim_last_error(self.handle).decode()

    def check(self, rc: int) -> None:
        if rc:
            raise_for(rc, self.error())

    def sync(self) -> None:
        self.check(self.lib.pswim_sync(self.handle))

    @property
    def stream_ptr(self) -> int:
        return self.lib.pswim_stream(self.handle)

    def torch_stream(self):
        """The context stream as a torch.cuda.ExternalStream (for event timing / ordering)."""
        if self._torch_stream is None:
            torch = _torch()
            self._torch_stream = torch.cuda.ExternalStream(self.stream_ptr, device=torch.device("cuda", self.device))
        return self._torch_stream

    def after_torch(self) -> None:
        """Order the context stream after torch's current stream (inputs written by torch)."""
        torch = _torch()
        ev = torch.cuda.Event()
        ev.record(torch.cuda.current_stream(self.device))
        self.torch_stream().wait_event(ev)

    def before_torch(self) -> None:
        """Order torch's current stream after the context stream (outputs read by torch)."""
        torch = _torch()
        ev = torch.cuda.Event()
        ev.record(self.torch_stream())
        torch.cuda.current_stream(self.device).wait_event(ev)

    # -- timing ----------------------------------------------------------------------------
    def timing(self, enable: bool = True) -> None:
        self.lib.pswim_timing_enable(self.handle, 1 if enable else 0)

    def timing_reset(self) -> None:
        self.lib.pswim_timing_reset(self.handle)

    def timing_snapshot(self) -> dict:
        t = self.lib.pswim_timing_snapshot(self.handle)
        return {"initialization": t.initialization, "velocity": t.velocity, "triad_update": t.triad_update}

    def dfma_peak(self) -> tuple[float, float]:
        flops = C.c_double()
        ms = C.c_double()
        self.check(self.lib.pswim_dfma_peak(self.handle, C.byref(flops), C.byref(ms)))
        return flops.value, ms.value


def dptr(t) -> int:
    """Device pointer of a contiguous float64 CUDA tensor."""
    torch = _torch()
    if not (isinstance(t, torch.Tensor) and t.is_cuda and t.dtype == torch.float64 and t.is_contiguous()):
        raise _lib.InvalidArgument(1, "expected a contiguous float64 CUDA tensor")
    return t.data_ptr()


def is_device(x) -> bool:
    try:
        torch = _torch()
    except ImportError:  # pragma: no cover
        return False
    return isinstance(x, torch.Tensor) and x.is_cuda


def host_f64(a, shape=None) -> np.ndarray:
    a = np.ascontiguousarray(np.asarray(a, dtype=np.float64))
    if shape is not None:
        a = a.reshape(shape)
    return a


def hptr(a: np.ndarray):
    return a.ctypes.data_as(C.POINTER(C.c_double))


_default_ctx: dict = {}


def default_context(device: int = 0) -> Context:
    """Scenario-less context for the MRS / rotation operators on `device`."""
    ctx = _default_ctx.get(device)
    if ctx is None:
        ctx = Context(device)
        _default_ctx[device] = ctx
    return ctx
