"""paper_2604_12083_b200 — B200-native (sm_100a) MRS / rod / pipelined-Parareal hot path of
arxiv/paper_2604_12083 behind the reference's operator and propagator interfaces.

The compute lives in libpswim.so (CUDA kernels + C++ runtime, C-ABI in include/pswim_c.h);
these modules mirror the reference names (stokes, rotation, rod, propagators, parareal,
harness, io) for callers and tests.
"""
from ._lib import LIB_PATH, InvalidArgument, PswimError, StiffnessError, lib  # noqa: F401

__all__ = ["lib", "LIB_PATH", "PswimError", "InvalidArgument", "StiffnessError"]
