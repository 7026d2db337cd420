"""ctypes binding of libpswim.so — the C-ABI of include/pswim_c.h.

The library is the product: every numeric entry point runs CUDA kernels for sm_100a.  It
must be built in-tree (``python -m paper_2604_12083_b200.build``); importing the package on
a machine without it raises immediately — there is no CPU fallback.
"""
from __future__ import annotations

import ctypes as C
import os
import threading

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "libpswim.so")

_dp = C.POINTER(C.c_double)
_vp = C.c_void_p
_i64 = C.c_int64
_i32 = C.c_int32


class KernelParams(C.Structure):
    """pswim_kernel_params == KernelParams (reference stokes.hpp:13-17)."""

    _fields_ = [("epsilon", C.c_double), ("mu", C.c_double), ("wall_mode", C.c_int32), ("_pad", C.c_int32)]


class Scenario(C.Structure):
    """pswim_scenario == ScenarioConfig (reference scenario.hpp:16-35)."""

    _fields_ = [
        ("rod_count", C.c_int64), ("nodes_per_rod", C.c_int64), ("rod_length", C.c_double),
        ("a1", C.c_double), ("a2", C.c_double), ("a3", C.c_double),
        ("b1", C.c_double), ("b2", C.c_double), ("b3", C.c_double),
        ("amplitude", C.c_double), ("frequency", C.c_double), ("wavelength", C.c_double),
        ("epsilon", C.c_double), ("mu", C.c_double), ("wall_mode", C.c_int32),
        ("placement", C.c_int32), ("lj_well_depth", C.c_double), ("lj_sigma", C.c_double),
        ("wall_clearance", C.c_double), ("seed", C.c_uint64), ("fine_dt", C.c_double),
        ("horizon", C.c_double),
    ]


class Resolved(C.Structure):
    _fields_ = [("ds", C.c_double), ("epsilon", C.c_double), ("mu", C.c_double),
                ("lj_sigma", C.c_double), ("lj_cutoff", C.c_double),
                ("lj_self_exclusion", C.c_int64), ("total_nodes", C.c_int64)]


class Timing(C.Structure):
    _fields_ = [("initialization", C.c_double), ("velocity", C.c_double), ("triad_update", C.c_double)]


class Plan(C.Structure):
    """pswim_plan == parareal::ParallelPlan (reference parareal.hpp:30-45)."""

    _fields_ = [("t0", C.c_double), ("horizon", C.c_double), ("intervals", C.c_int32),
                ("workers", C.c_int32), ("cost_ratio", C.c_double), ("max_iterations", C.c_int32),
                ("mode", C.c_int32), ("tolerance", C.c_double)]


class Report(C.Structure):
    """pswim_report == parareal::ConvergenceReport (+ wall time, W)."""

    _fields_ = [("eta_tilde", _dp), ("eta", _dp), ("iterations_used", C.c_int32),
                ("converged", C.c_int32), ("eta_count", C.c_int32), ("_pad", C.c_int32),
                ("wall_seconds", C.c_double), ("schedule_idle", C.c_double)]


class TraceEvent(C.Structure):
    _fields_ = [("worker", C.c_int32), ("kind", C.c_int32), ("t_start", C.c_double), ("t_end", C.c_double),
                ("iteration", C.c_int32), ("interval", C.c_int32)]


PROPAGATOR_FN = C.CFUNCTYPE(C.c_int, _vp, C.c_double, C.c_double, _dp, _dp, _i64, _vp)
SEND_FN = C.CFUNCTYPE(C.c_int, _vp, _dp, _i64, _i32, _vp)
RECV_FN = C.CFUNCTYPE(C.c_int, _vp, _dp, _i64, _i32, _vp)
ALLREDUCE_FN = C.CFUNCTYPE(C.c_int, _vp, _dp, _i64, _vp)
ALLGATHER_FN = C.CFUNCTYPE(C.c_int, _vp, _dp, _dp, _i64, _vp)
HEALTH_FN = C.CFUNCTYPE(C.c_int, _vp)
ABORT_FN = C.CFUNCTYPE(None, _vp)


class Transport(C.Structure):
    _fields_ = [("user", _vp), ("rank", C.c_int32), ("world", C.c_int32), ("send", SEND_FN),
                ("recv", RECV_FN), ("allreduce_max", ALLREDUCE_FN), ("allgather", ALLGATHER_FN),
                ("health", HEALTH_FN), ("abort", ABORT_FN)]


# name -> (restype, argtypes); the complete export list of include/pswim_c.h
SIGNATURES = {
    "pswim_scenario_defaults": (None, [C.POINTER(Scenario)]),
    "pswim_scenario_resolve": (C.c_int, [C.POINTER(Scenario), C.POINTER(Resolved)]),
    "pswim_build_initial_state": (C.c_int, [C.POINTER(Scenario), _dp]),
    "pswim_create": (_vp, [C.c_int, C.POINTER(Scenario), C.c_int]),
    "pswim_destroy": (None, [_vp]),
    "pswim_last_error": (C.c_char_p, [_vp]),
    "pswim_stream": (_vp, [_vp]),
    "pswim_sync": (C.c_int, [_vp]),
    "pswim_device": (C.c_int, [_vp]),
    "pswim_mrs_velocities": (C.c_int, [_vp, _vp, _i64, _vp, _vp, _vp, _i64, C.POINTER(KernelParams), _vp, _vp]),
    "pswim_mrs_velocities_host": (C.c_int, [_vp, _dp, _i64, _dp, _dp, _dp, _i64, C.POINTER(KernelParams), _dp, _dp]),
    "pswim_h_functions": (C.c_int, [_vp, _vp, _i64, C.c_double, _vp]),
    "pswim_sqrt_rotation_batched": (C.c_int, [_vp, _vp, _i64, _vp]),
    "pswim_sqrt_rotation_host": (C.c_int, [_vp, _dp, _i64, _dp]),
    "pswim_rod_loads": (C.c_int, [_vp, _vp, C.c_double, _vp, _vp, _vp, _vp]),
    "pswim_lj_forces": (C.c_int, [_vp, _vp, _vp]),
    "pswim_rhs": (C.c_int, [_vp, _vp, C.c_double, _vp, _vp, _vp, _vp]),
    "pswim_advance_state": (C.c_int, [_vp, _vp, _vp, _vp, C.c_double, _vp]),
    "pswim_step": (C.c_int, [_vp, C.c_int, _vp, C.c_double, C.c_double, _vp]),
    "pswim_propagate": (C.c_int, [_vp, _vp, C.c_double, C.c_double, C.c_int, _i64, C.c_double, _vp]),
    "pswim_propagate_host": (C.c_int, [_vp, _dp, C.c_double, C.c_double, C.c_int, _i64, C.c_double, _dp]),
    "pswim_set_fused": (C.c_int, [_vp, C.c_int]),
    "pswim_set_lj_mode": (C.c_int, [_vp, C.c_int]),
    "pswim_set_graphs": (C.c_int, [_vp, C.c_int]),
    "pswim_lj_forces_host": (C.c_int, [_vp, _dp, _dp]),
    "pswim_fused_profile": (C.c_int, [_vp, _vp, C.c_double, C.c_double, C.c_int, C.c_int64, _vp,
                                      C.POINTER(C.c_uint64)]),
    "pswim_timing_enable": (None, [_vp, C.c_int]),
    "pswim_timing_reset": (None, [_vp]),
    "pswim_timing_snapshot": (Timing, [_vp]),
    "pswim_position_metric": (C.c_int, [_vp, _vp, _vp, _i64, _dp]),
    "pswim_parareal_correct": (C.c_int, [_vp, _vp, _vp, _vp, _i64, _vp]),
    "pswim_parareal_run_host": (C.c_int, [C.POINTER(Plan), PROPAGATOR_FN, _vp, PROPAGATOR_FN, _vp, _dp, _i64,
                                          _i32, _i32, _dp, _dp, C.POINTER(Report), C.POINTER(TraceEvent), _i64,
                                          C.POINTER(_i64)]),
    "pswim_parareal_run_gpu": (C.c_int, [C.POINTER(Plan), C.POINTER(Scenario), C.c_int, _i64, _i64, _dp, _dp, _dp,
                                         C.POINTER(Report), C.POINTER(TraceEvent), _i64, C.POINTER(_i64)]),
    "pswim_parareal_rank_gpu": (C.c_int, [C.POINTER(Plan), C.POINTER(Scenario), C.c_int, C.POINTER(Transport), _vp, _i64,
                                          _i64, _dp, _dp, _dp, C.POINTER(Report), C.POINTER(TraceEvent), _i64,
                                          C.POINTER(_i64)]),
    "pswim_parareal_rank_gpu_hybrid": (C.c_int, [C.POINTER(Plan), C.POINTER(Scenario), C.c_int, C.POINTER(Transport),
                                                 C.POINTER(Transport), C.POINTER(Transport), _i64, _i64, _dp, _dp,
                                                 _dp, C.POINTER(Report), C.POINTER(TraceEvent), _i64,
                                                 C.POINTER(_i64)]),
    "pswim_parareal_rank_host": (C.c_int, [C.POINTER(Plan), PROPAGATOR_FN, _vp, PROPAGATOR_FN, _vp,
                                           C.POINTER(Transport), _dp, _i64, _i32, _i32, _dp, _dp, C.POINTER(Report),
                                           C.POINTER(TraceEvent), _i64, C.POINTER(_i64)]),
    "pswim_handoff_create": (_vp, [C.c_int, _i64, _i32]),
    "pswim_handoff_handle": (C.c_int, [_vp, C.POINTER(C.c_uint8)]),
    "pswim_handoff_local_base": (_vp, [_vp]),
    "pswim_handoff_connect": (C.c_int, [_vp, C.POINTER(C.c_uint8), _vp]),
    "pswim_handoff_connect_local": (C.c_int, [_vp, _vp]),
    "pswim_handoff_destroy": (None, [_vp]),
    "pswim_nccl_unique_id": (C.c_int, [C.POINTER(C.c_uint8)]),
    "pswim_nccl_transport_create": (C.POINTER(Transport), [C.POINTER(C.c_uint8), _i32, _i32, C.c_int]),
    "pswim_nccl_transport_destroy": (None, [C.POINTER(Transport)]),
    "pswim_staged_transport_create": (C.POINTER(Transport), [C.POINTER(Transport), C.c_int]),
    "pswim_staged_transport_destroy": (None, [C.POINTER(Transport)]),
    "pswim_threads_transports_create": (C.POINTER(Transport), [C.c_int32, C.POINTER(C.c_int), _i64, C.c_int32]),
    "pswim_threads_transports_destroy": (None, [C.POINTER(Transport)]),
    "pswim_propagate_sharded": (C.c_int, [_vp, C.POINTER(Transport), _vp, C.c_double, C.c_double, C.c_int, _i64,
                                          C.c_double, _vp]),
    "pswim_peer_group_create": (_vp, [_vp, _i32, _i32]),
    "pswim_peer_group_handle": (C.c_int, [_vp, C.POINTER(C.c_uint8)]),
    "pswim_peer_group_local_base": (_vp, [_vp]),
    "pswim_peer_group_connect": (C.c_int, [_vp, C.POINTER(C.c_uint8), C.POINTER(_vp)]),
    "pswim_peer_group_destroy": (None, [_vp]),
    "pswim_propagate_sharded_peer": (C.c_int, [_vp, _vp, _vp, C.c_double, C.c_double, C.c_int, _i64, C.c_double,
                                               _vp]),
    "pswim_parareal_run_threads": (C.c_int, [C.POINTER(Plan), C.POINTER(Scenario), C.POINTER(C.c_int), _i64, _i64,
                                             _dp, _dp, _dp, C.POINTER(Report), _i32, C.POINTER(TraceEvent), _i64,
                                             C.POINTER(_i64)]),
    "pswim_dfma_peak": (C.c_int, [_vp, _dp, _dp]),
    "pswim_dev_fp64_probe": (C.c_int, [_vp, C.c_int, _dp, _dp]),
    "pswim_dev_latency_probe": (C.c_int, [_vp, C.c_int, C.c_int, C.c_int, C.c_int, C.c_int, _dp]),
    "pswim_version": (C.c_char_p, []),
}

_lib = None
_lock = threading.Lock()


def lib() -> C.CDLL:
    """Load libpswim.so (once).  Raises if the CUDA extension was not built."""
    global _lib
    with _lock:
        if _lib is None:
            if not os.path.exists(LIB_PATH):
                raise ImportError(f"{LIB_PATH} is missing: build it with `python -m paper_2604_12083_b200.build` "
                                  "(there is no CPU fallback)")
            handle = C.CDLL(LIB_PATH, mode=C.RTLD_GLOBAL)
            for name, (res, args) in SIGNATURES.items():
                fn = getattr(handle, name)
                fn.restype = res
                fn.argtypes = args
            _lib = handle
    return _lib


ERRORS = {1: "EINVAL", 2: "EUNSUPPORTED_WALL", 3: "ENONFINITE", 4: "ESTIFF", 5: "EDEGENERATE", 6: "ECUDA",
          7: "ECOMM", 8: "ESTATE"}


class PswimError(RuntimeError):
    """Base class; subclasses mirror the reference's exception kinds."""

    def __init__(self, code: int, what: str):
        super().__init__(f"{ERRORS.get(code, code)}: {what}")
        self.code = code
        self.what = what


class InvalidArgument(PswimError, ValueError):
    """std::invalid_argument in the reference."""


class StiffnessError(PswimError):
    """pintswim::StiffnessError (reference propagators.hpp:24-26)."""


class DeviceError(PswimError):
    pass


def raise_for(code: int, what: str) -> None:
    if code == 0:
        return
    if code in (1, 3):
        raise InvalidArgument(code, what)
    if code == 4:
        raise StiffnessError(code, what)
    if code in (2, 5, 8):
        raise PswimError(code, what)
    raise DeviceError(code, what)
