"""Parareal drivers — mirror of reference include/pintswim/parareal.hpp.

* :func:`run` — ``parareal::run(plan, coarse, fine, x0, metric, reference)`` (parareal.hpp:85-86)
  on the native C++ task-graph engine with arbitrary host propagators (Python callables
  ``f(t0, t1, x) -> y`` on numpy vectors).  Used for the physics-agnostic property tests.
* :func:`run_gpu` — the same engine with GPU propagators (coarse Euler / fine RK2 on HBM
  states, one CUDA stream per worker lane) — what ``harness.prepare`` wires up.
* :func:`run_sliced_threads` — one time slice per GPU (or per stream on one GPU), slice
  hand-offs by peer copies, pipelined across iterations.
* :func:`run_sliced_rank` — one process per GPU (torch.distributed launch), NCCL send/recv of
  the slice state + allreduce(max) of the metric; :func:`run_sliced_rank_host` is the same
  rank driver with host propagators and a torch.distributed (gloo) transport for CPU tests.
* :func:`coarse_sweep_initial`, :func:`fine_parallel`, :func:`correct`,
  :func:`pointwise_metric` — the serial building blocks (parareal.cpp:15-89).
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, field
from typing import Callable, List, Optional, Sequence

import numpy as np

from . import _lib

REGULAR = 0
PIPELINED = 1
COARSE, FINE, CORRECT, IDLE = 0, 1, 2, 3
TASK_NAMES = {COARSE: "coarse", FINE: "fine", CORRECT: "correct", IDLE: "idle"}


@dataclass
class ParallelPlan:
    """ParallelPlan, parareal.hpp:30-45."""

    t0: float = 0.0
    horizon: float = 1.0
    intervals: int = 4
    workers: int = 1
    cost_ratio: float = 2.0
    max_iterations: int = 10
    tolerance: float = 1e-10
    mode: int = REGULAR

    def interval_length(self) -> float:
        return self.horizon / self.intervals

    def boundary_time(self, n: int) -> float:
        return self.t0 + (self.horizon / self.intervals) * n

    def to_c(self) -> _lib.Plan:
        return _lib.Plan(float(self.t0), float(self.horizon), int(self.intervals), int(self.workers),
                         float(self.cost_ratio), int(self.max_iterations), int(self.mode), float(self.tolerance))


@dataclass
class ConvergenceReport:
    eta_tilde: List[float] = field(default_factory=list)
    eta: List[float] = field(default_factory=list)
    iterations_used: int = 0
    converged: bool = False
    wall_seconds: float = 0.0


@dataclass
class TraceEvent:
    worker: int
    kind: int
    t_start: float
    t_end: float
    iteration: int = -1  # the task's (k, n) in the Parareal grid; -1 for idle gaps
    interval: int = -1


@dataclass
class ScheduleTrace:
    worker_count: int = 0
    serial_lane: int = 0
    events: List[TraceEvent] = field(default_factory=list)

    def total_idle(self) -> float:
        return sum(e.t_end - e.t_start for e in self.events if e.kind == IDLE)

    def makespan(self) -> float:
        return max((e.t_end for e in self.events), default=0.0)

    def busy_time(self, kind: int) -> float:
        return sum(e.t_end - e.t_start for e in self.events if e.kind == kind)


@dataclass
class RunResult:
    states: List[np.ndarray]
    report: ConvergenceReport
    trace: ScheduleTrace


def _validate(plan: ParallelPlan) -> None:
    # parareal.cpp:38-45
    if plan.intervals < 1 or plan.workers < 1:
        raise _lib.InvalidArgument(1, "parareal: need at least one interval and one worker")
    if plan.max_iterations < 1:
        raise _lib.InvalidArgument(1, "parareal: max_iterations must be >= 1")
    if not plan.tolerance > 0.0:
        raise _lib.InvalidArgument(1, "parareal: tolerance must be positive")
    if plan.horizon <= 0.0:
        raise _lib.InvalidArgument(1, "parareal: horizon must be positive")


# ---- metrics -------------------------------------------------------------------------------
def pointwise_metric(point_dim: int) -> Callable[[np.ndarray, np.ndarray], float]:
    """max_i |x_i - y_i| / |x_i| over consecutive groups of point_dim (parareal.cpp:15-34)."""

    def metric(x, y):
        x = np.asarray(x, dtype=np.float64)
        y = np.asarray(y, dtype=np.float64)
        if point_dim == 0 or x.shape != y.shape or x.size % point_dim:
            raise _lib.InvalidArgument(1, "pointwise_metric: inconsistent state sizes")
        worst = 0.0
        for i in range(0, x.size, point_dim):
            num = 0.0
            den = 0.0
            for c in range(point_dim):
                d = x[i + c] - y[i + c]
                num += d * d
                den += x[i + c] * x[i + c]
            num = np.sqrt(num)
            den = np.sqrt(den)
            worst = max(worst, num if den < 1e-14 else num / den)
        return float(worst)

    metric.dim = point_dim  # type: ignore[attr-defined]
    metric.stride = point_dim  # type: ignore[attr-defined]
    return metric


# ---- serial building blocks (parareal.cpp:58-89) ------------------------------------------
def coarse_sweep_initial(plan: ParallelPlan, coarse, x0) -> List[np.ndarray]:
    _validate(plan)
    x = [np.asarray(x0, dtype=np.float64).copy()]
    for n in range(1, plan.intervals + 1):
        x.append(np.asarray(coarse(plan.boundary_time(n - 1), plan.boundary_time(n), x[n - 1])))
    return x


def fine_parallel(plan: ParallelPlan, fine, x_prev: Sequence[np.ndarray], k: int) -> List[np.ndarray]:
    _validate(plan)
    xp = [np.array(v, copy=True) for v in x_prev]
    for n in range(k, plan.intervals + 1):
        xp[n] = np.asarray(fine(plan.boundary_time(n - 1), plan.boundary_time(n), x_prev[n - 1]))
    return xp


def correct(plan: ParallelPlan, coarse, x_prime, x_prev, g_cache: List[np.ndarray], k: int) -> List[np.ndarray]:
    _validate(plan)
    x = [np.array(v, copy=True) for v in x_prev]
    x[k] = np.array(x_prime[k], copy=True)
    for n in range(k + 1, plan.intervals + 1):
        g_new = np.asarray(coarse(plan.boundary_time(n - 1), plan.boundary_time(n), x[n - 1]))
        x[n] = (x_prime[n] + g_new) - g_cache[n]
        g_cache[n] = g_new
    return x


# ---- native engine ----------------------------------------------------------------------------
def _report_arrays(n: int):
    et = np.zeros(max(n, 1))
    ea = np.zeros(max(n, 1))
    rep = _lib.Report()
    rep.eta_tilde = et.ctypes.data_as(C.POINTER(C.c_double))
    rep.eta = ea.ctypes.data_as(C.POINTER(C.c_double))
    return rep, et, ea


def _finish(rep, et, ea, has_ref) -> ConvergenceReport:
    k = rep.eta_count
    return ConvergenceReport(list(et[:k]), list(ea[:k]) if has_ref else [], int(rep.iterations_used),
                             bool(rep.converged), float(rep.wall_seconds))


def _wrap_propagator(fn):
    def cb(user, t0, t1, xin, xout, length, stream):
        try:
            x = np.ctypeslib.as_array(xin, shape=(length,)).copy()
            y = np.asarray(fn(t0, t1, x), dtype=np.float64)
            if y.shape != (length,):
                return 1  # "parareal: propagator changed the state size"
            np.ctypeslib.as_array(xout, shape=(length,))[:] = y
            return 0
        except _lib.StiffnessError:
            return 4
        except _lib.PswimError as e:
            return e.code
        except Exception:
            return 1

    return _lib.PROPAGATOR_FN(cb)


def run(plan: ParallelPlan, coarse, fine, x0, metric=None, reference: Optional[Sequence[np.ndarray]] = None) -> RunResult:
    """parareal::run on the native engine with host propagators (parareal.hpp:85-86)."""
    _validate(plan)
    L = _lib.lib()
    x0 = np.ascontiguousarray(np.asarray(x0, dtype=np.float64).reshape(-1))
    metric = metric or pointwise_metric(1)
    dim = getattr(metric, "dim", None)
    stride = getattr(metric, "stride", None)
    if dim is None:
        raise _lib.InvalidArgument(1, "run: metric must come from pointwise_metric / rod_position_metric")
    if reference is not None and len(reference) != plan.intervals + 1:
        raise _lib.InvalidArgument(1, "parareal: reference must hold one state per interval boundary")
    n = plan.intervals
    ref = None
    if reference is not None:
        ref = np.ascontiguousarray(np.stack([np.asarray(r, dtype=np.float64).reshape(-1) for r in reference]))
    out = np.zeros((n + 1, x0.size))
    rep, et, ea = _report_arrays(n)
    cap = 64 * (n + 2) * (n + 2) + 64
    trace = (_lib.TraceEvent * cap)()
    tlen = C.c_int64(0)
    cb_c = _wrap_propagator(coarse)
    cb_f = _wrap_propagator(fine)
    rc = L.pswim_parareal_run_host(C.byref(plan.to_c()), cb_c, None, cb_f, None,
                                   x0.ctypes.data_as(C.POINTER(C.c_double)), x0.size, int(dim), int(stride),
                                   ref.ctypes.data_as(C.POINTER(C.c_double)) if ref is not None else None,
                                   out.ctypes.data_as(C.POINTER(C.c_double)), C.byref(rep), trace, cap, C.byref(tlen))
    _lib.raise_for(rc, "parareal::run failed")
    events = _events(trace, tlen)
    return RunResult([out[i].copy() for i in range(n + 1)], _finish(rep, et, ea, ref is not None),
                     ScheduleTrace(plan.workers, 0, events))


def run_gpu(plan: ParallelPlan, scenario, fine_steps: int, coarse_steps: int, x0,
            reference: Optional[Sequence[np.ndarray]] = None, device: int = 0) -> RunResult:
    """parareal::run with GPU rod propagators (coarse Euler, fine RK2; harness.cpp:26-31)."""
    _validate(plan)
    L = _lib.lib()
    sc = scenario.to_c()
    x0 = np.ascontiguousarray(np.asarray(x0, dtype=np.float64).reshape(-1))
    n = plan.intervals
    ref = None
    if reference is not None:
        ref = np.ascontiguousarray(np.stack([np.asarray(r, dtype=np.float64).reshape(-1) for r in reference]))
    out = np.zeros((n + 1, x0.size))
    rep, et, ea = _report_arrays(n)
    cap = 64 * (n + 2) * (n + 2) + 64
    trace = (_lib.TraceEvent * cap)()
    tlen = C.c_int64(0)
    rc = L.pswim_parareal_run_gpu(C.byref(plan.to_c()), C.byref(sc), int(device), int(fine_steps), int(coarse_steps),
                                  x0.ctypes.data_as(C.POINTER(C.c_double)),
                                  ref.ctypes.data_as(C.POINTER(C.c_double)) if ref is not None else None,
                                  out.ctypes.data_as(C.POINTER(C.c_double)), C.byref(rep), trace, cap, C.byref(tlen))
    _lib.raise_for(rc, "parareal::run (gpu) failed")
    events = _events(trace, tlen)
    return RunResult([out[i].copy() for i in range(n + 1)], _finish(rep, et, ea, ref is not None),
                     ScheduleTrace(plan.workers, 0, events))


def _trace_buffers(intervals: int):
    cap = 8 * (intervals + 2) * (intervals + 2) + 64
    return (_lib.TraceEvent * cap)(), cap, C.c_int64(0)


def _events(trace, tlen) -> List[TraceEvent]:
    return [TraceEvent(e.worker, e.kind, e.t_start, e.t_end, e.iteration, e.interval)
            for e in trace[: min(tlen.value, len(trace))]]


def run_sliced_threads(plan: ParallelPlan, scenario, fine_steps: int, coarse_steps: int, x0,
                       devices: Sequence[int], reference: Optional[Sequence[np.ndarray]] = None,
                       handoff: bool = False) -> RunResult:
    """One slice per rank (intervals == len(devices)), ranks as threads of this process.
    ``handoff``: slice states move by the peer-memory hand-off (the producing kernel stores into
    the next rank's slot) instead of stream-ordered peer copies."""
    _validate(plan)
    if len(devices) != plan.intervals:
        raise _lib.InvalidArgument(1, "run_sliced_threads: one device entry per interval")
    L = _lib.lib()
    sc = scenario.to_c()
    x0 = np.ascontiguousarray(np.asarray(x0, dtype=np.float64).reshape(-1))
    n = plan.intervals
    ref = None
    if reference is not None:
        ref = np.ascontiguousarray(np.stack([np.asarray(r, dtype=np.float64).reshape(-1) for r in reference]))
    out = np.zeros((n + 1, x0.size))
    rep, et, ea = _report_arrays(n)
    devs = (C.c_int * n)(*[int(d) for d in devices])
    trace, cap, tlen = _trace_buffers(n)
    rc = L.pswim_parareal_run_threads(C.byref(plan.to_c()), C.byref(sc), devs, int(fine_steps), int(coarse_steps),
                                      x0.ctypes.data_as(C.POINTER(C.c_double)),
                                      ref.ctypes.data_as(C.POINTER(C.c_double)) if ref is not None else None,
                                      out.ctypes.data_as(C.POINTER(C.c_double)), C.byref(rep), int(bool(handoff)),
                                      trace, cap, C.byref(tlen))
    _lib.raise_for(rc, "parareal sliced (threads) failed")
    res = RunResult([out[i].copy() for i in range(n + 1)], _finish(rep, et, ea, ref is not None),
                    ScheduleTrace(n + 1, 0, _events(trace, tlen)))
    res.schedule_idle = float(rep.schedule_idle)
    return res


# ---- one process per rank ----------------------------------------------------------------------
class TorchTransport:
    """pswim_transport over torch.distributed on host buffers (gloo): CPU tests of the rank
    driver logic with world_size > 1."""

    def __init__(self, group=None):
        import torch.distributed as dist

        self.dist = dist
        self.group = group
        rank, world = dist.get_rank(group), dist.get_world_size(group)
        # peers are group ranks; torch.distributed point-to-point calls take global ranks
        self._global = [dist.get_global_rank(group, r) if group is not None else r for r in range(world)]
        self._send = _lib.SEND_FN(self._send_cb)
        self._recv = _lib.RECV_FN(self._recv_cb)
        self._red = _lib.ALLREDUCE_FN(self._red_cb)
        self._gather = _lib.ALLGATHER_FN(self._gather_cb)
        self.c = _lib.Transport(None, rank, world, self._send, self._recv, self._red, self._gather, _lib.HEALTH_FN(),
                                _lib.ABORT_FN())

    def _send_cb(self, user, buf, length, peer, stream):
        import torch

        try:
            t = torch.from_numpy(np.ctypeslib.as_array(buf, shape=(length,)).copy())
            self.dist.send(t, dst=self._global[peer], group=self.group)
            return 0
        except Exception:
            return 7

    def _recv_cb(self, user, buf, length, peer, stream):
        import torch

        try:
            t = torch.empty(length, dtype=torch.float64)
            self.dist.recv(t, src=self._global[peer], group=self.group)
            np.ctypeslib.as_array(buf, shape=(length,))[:] = t.numpy()
            return 0
        except Exception:
            return 7

    def _gather_cb(self, user, send, recv, count, stream):
        import torch

        try:
            t = torch.from_numpy(np.ctypeslib.as_array(send, shape=(count,)).copy())
            out = [torch.empty(count, dtype=torch.float64) for _ in range(self.dist.get_world_size(self.group))]
            self.dist.all_gather(out, t, group=self.group)
            np.ctypeslib.as_array(recv, shape=(count * len(out),))[:] = torch.cat(out).numpy()
            return 0
        except Exception:
            return 7

    def _red_cb(self, user, buf, length, stream):
        import torch

        try:
            arr = np.ctypeslib.as_array(buf, shape=(length,))
            t = torch.from_numpy(arr.copy())
            self.dist.all_reduce(t, op=self.dist.ReduceOp.MAX, group=self.group)
            arr[:] = t.numpy()
            return 0
        except Exception:
            return 7


@dataclass
class RankResult:
    state: np.ndarray  # X[k_final][rank + 1]
    report: ConvergenceReport
    trace: Optional[ScheduleTrace] = None  # every rank's tasks (identical on all ranks)
    schedule_idle: float = 0.0            # W of that trace


def run_sliced_rank_host(plan: ParallelPlan, coarse, fine, x0, metric=None, reference_slice=None,
                         transport: Optional[TorchTransport] = None) -> RankResult:
    """Rank driver with host propagators over a torch.distributed transport."""
    _validate(plan)
    L = _lib.lib()
    tr = transport or TorchTransport()
    metric = metric or pointwise_metric(1)
    x0 = np.ascontiguousarray(np.asarray(x0, dtype=np.float64).reshape(-1))
    out = np.zeros_like(x0)
    rep, et, ea = _report_arrays(plan.intervals)
    ref = None if reference_slice is None else np.ascontiguousarray(np.asarray(reference_slice, dtype=np.float64))
    cb_c = _wrap_propagator(coarse)
    cb_f = _wrap_propagator(fine)
    trace, cap, tlen = _trace_buffers(plan.intervals)
    rc = L.pswim_parareal_rank_host(C.byref(plan.to_c()), cb_c, None, cb_f, None, C.byref(tr.c),
                                    x0.ctypes.data_as(C.POINTER(C.c_double)), x0.size, int(metric.dim),
                                    int(metric.stride),
                                    ref.ctypes.data_as(C.POINTER(C.c_double)) if ref is not None else None,
                                    out.ctypes.data_as(C.POINTER(C.c_double)), C.byref(rep), trace, cap, C.byref(tlen))
    _lib.raise_for(rc, "parareal rank driver failed")
    return RankResult(out, _finish(rep, et, ea, ref is not None), ScheduleTrace(plan.intervals + 1, 0, _events(trace, tlen)),
                      float(rep.schedule_idle))


class StagedTransport:
    """Device-buffer transport over a torch.distributed host wire (gloo), staged through
    pinned memory (pswim_staged_transport_create): the GPU rank drivers with several ranks on
    one GPU, where NCCL refuses duplicate devices.  ``ptr`` is the pswim_transport*."""

    def __init__(self, device: int, group=None):
        L = _lib.lib()
        self.wire = TorchTransport(group)
        self.ptr = L.pswim_staged_transport_create(C.byref(self.wire.c), int(device))
        if not self.ptr:
            raise _lib.PswimError(7, "pswim_staged_transport_create failed")
        self.lib = L

    def close(self):
        if self.ptr:
            self.lib.pswim_staged_transport_destroy(self.ptr)
            self.ptr = None


def _point_at_wheel_nccl() -> None:
    """libpswim dlopens NCCL: prefer the copy torch already loaded, else the nvidia-nccl wheel
    of the running interpreter (PSWIM_NCCL_LIB), else the loader's default search."""
    import os

    if os.environ.get("PSWIM_NCCL_LIB"):
        return
    try:
        import nvidia.nccl as nv  # the CUDA wheel torch depends on

        path = os.path.join(list(nv.__path__)[0], "lib", "libnccl.so.2")
        if os.path.exists(path):
            os.environ["PSWIM_NCCL_LIB"] = path
    except Exception:
        pass


def nccl_transport(device: int):
    """NCCL transport for the current torch.distributed rank (unique id shared via the
    default process group)."""
    import torch.distributed as dist

    _point_at_wheel_nccl()
    L = _lib.lib()
    rank, world = dist.get_rank(), dist.get_world_size()
    uid = (C.c_uint8 * 128)()
    if rank == 0:
        _lib.raise_for(L.pswim_nccl_unique_id(uid), "ncclGetUniqueId failed")
    obj = [bytes(uid) if rank == 0 else None]
    dist.broadcast_object_list(obj, src=0)
    uid = (C.c_uint8 * 128)(*obj[0])
    tr = L.pswim_nccl_transport_create(uid, rank, world, int(device))
    if not tr:
        raise _lib.PswimError(7, "ncclCommInitRank failed")
    return tr


def nccl_group_transports(device: int, groups):
    """One NCCL transport per group this rank belongs to, for a list of disjoint-or-not rank
    groups (each a list of global torch.distributed ranks).  Every rank walks `groups` in the
    same order, so communicator creation never deadlocks; the first rank of a group makes
    its unique id, shared with one all_gather_object.  Returns {group index: transport}."""
    import torch.distributed as dist

    _point_at_wheel_nccl()
    L = _lib.lib()
    rank = dist.get_rank()
    ids = {}
    for gi, g in enumerate(groups):
        if g[0] == rank:
            uid = (C.c_uint8 * 128)()
            _lib.raise_for(L.pswim_nccl_unique_id(uid), "ncclGetUniqueId failed")
            ids[gi] = bytes(uid)
    allids = [None] * dist.get_world_size()
    dist.all_gather_object(allids, ids)
    merged = {}
    for d in allids:
        merged.update(d)
    out = {}
    for gi, g in enumerate(groups):
        if rank in g:
            uid = (C.c_uint8 * 128)(*merged[gi])
            tr = L.pswim_nccl_transport_create(uid, g.index(rank), len(g), int(device))
            if not tr:
                raise _lib.PswimError(7, "ncclCommInitRank failed")
            out[gi] = tr
    return out


def hybrid_groups(world: int, members: int):
    """Rank layout of hybrid space x time: global rank g = p * members + q is member q of
    slice p.  Returns (time groups, space groups): time group q = the q-th members of all
    slices, space group p = the members of slice p (adjacent ranks, NVLink neighbours)."""
    slices = world // members
    time_groups = [[p * members + q for p in range(slices)] for q in range(members)]
    space_groups = [[p * members + q for q in range(members)] for p in range(slices)]
    return time_groups, space_groups


class Handoff:
    """Peer-memory slice hand-off of this rank (pswim_handoff_*): receive slots in this GPU's
    HBM, connected to the next rank's slots through a CUDA IPC handle (NVLink P2P).  Built
    collectively: every rank of the torch.distributed group `group` calls it."""

    def __init__(self, device: int, len_: int, slots: int, group=None):
        import torch.distributed as dist

        L = _lib.lib()
        self.lib = L
        self.h = L.pswim_handoff_create(int(device), int(len_), int(slots))
        if not self.h:
            raise _lib.DeviceError(6, "pswim_handoff_create failed")
        hb = (C.c_uint8 * 64)()
        _lib.raise_for(L.pswim_handoff_handle(self.h, hb), "pswim_handoff_handle failed")
        rank, world = dist.get_rank(group), dist.get_world_size(group)
        handles = [None] * world
        dist.all_gather_object(handles, bytes(hb), group=group)
        nxt = (C.c_uint8 * 64)(*handles[rank + 1]) if rank + 1 < world else None
        _lib.raise_for(L.pswim_handoff_connect(self.h, nxt, None), "pswim_handoff_connect failed")

    def close(self):
        if self.h:
            self.lib.pswim_handoff_destroy(self.h)
            self.h = None


def run_sliced_rank(plan: ParallelPlan, scenario, fine_steps: int, coarse_steps: int, x0, device: int,
                    transport=None, reference_slice=None, space=None, handoff: Optional[Handoff] = None) -> RankResult:
    """This process's slice of a time-sliced pipelined Parareal run on `device` (NCCL).

    ``space=(coarse_transport, fine_transport)``: hybrid space x time -- this rank is one
    member of its slice's space group, and every coarse / fine rhs shards the MRS over that
    group (pswim_parareal_rank_gpu_hybrid); ``transport`` then connects the same-index members
    of all slices.  ``handoff``: slice states move over peer memory (:class:`Handoff`), the
    transport carrying only the metric allreduce."""
    _validate(plan)
    L = _lib.lib()
    own = transport is None
    tr = transport or nccl_transport(device)
    sc = scenario.to_c()
    x0 = np.ascontiguousarray(np.asarray(x0, dtype=np.float64).reshape(-1))
    out = np.zeros_like(x0)
    rep, et, ea = _report_arrays(plan.intervals)
    ref = None if reference_slice is None else np.ascontiguousarray(np.asarray(reference_slice, dtype=np.float64))
    trace, cap, tlen = _trace_buffers(plan.intervals)
    try:
        refp = ref.ctypes.data_as(C.POINTER(C.c_double)) if ref is not None else None
        if space is None:
            rc = L.pswim_parareal_rank_gpu(C.byref(plan.to_c()), C.byref(sc), int(device), tr,
                                           handoff.h if handoff is not None else None, int(fine_steps),
                                           int(coarse_steps), x0.ctypes.data_as(C.POINTER(C.c_double)), refp,
                                           out.ctypes.data_as(C.POINTER(C.c_double)), C.byref(rep), trace, cap,
                                           C.byref(tlen))
        else:
            rc = L.pswim_parareal_rank_gpu_hybrid(C.byref(plan.to_c()), C.byref(sc), int(device), tr, space[0],
                                                  space[1], int(fine_steps), int(coarse_steps),
                                                  x0.ctypes.data_as(C.POINTER(C.c_double)), refp,
                                                  out.ctypes.data_as(C.POINTER(C.c_double)), C.byref(rep), trace, cap,
                                                  C.byref(tlen))
    finally:
        if own:
            L.pswim_nccl_transport_destroy(tr)
    _lib.raise_for(rc, "parareal rank driver (gpu) failed")
    return RankResult(out, _finish(rep, et, ea, ref is not None), ScheduleTrace(plan.intervals + 1, 0, _events(trace, tlen)),
                      float(rep.schedule_idle))
