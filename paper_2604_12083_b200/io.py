"""State packing and the convergence metric — mirror of reference include/pintswim/io.hpp:14-21.

Packed layout (io.cpp:10-25): per node 12 doubles [x, d1, d2, d3], rods concatenated.  This
is also the device layout of every state in HBM, so pack/unpack are views, not copies.
"""
from __future__ import annotations

import numpy as np

from . import _lib


def pack_state(rods: np.ndarray) -> np.ndarray:
    """(rods, nodes, 4, 3) or (N, 12) -> flat packed vector."""
    return np.ascontiguousarray(np.asarray(rods, dtype=np.float64)).reshape(-1)


def unpack_state(v, rod_count: int, nodes_per_rod: int) -> np.ndarray:
    """Flat packed vector -> (rods, nodes, 4, 3) view: [..., 0, :] = x, 1..3 = d1, d2, d3."""
    v = np.asarray(v, dtype=np.float64)
    if v.size != 12 * rod_count * nodes_per_rod:
        raise _lib.InvalidArgument(1, "unpack_state: vector size does not match rod layout")
    return v.reshape(rod_count, nodes_per_rod, 4, 3)


def rod_position_metric():
    """max over nodes of |x_i - y_i| / |x_i| on positions only (io.cpp:49-68)."""

    def metric(x, y):
        x = np.asarray(x, dtype=np.float64).reshape(-1)
        y = np.asarray(y, dtype=np.float64).reshape(-1)
        if x.shape != y.shape or x.size % 12:
            raise _lib.InvalidArgument(1, "rod_position_metric: inconsistent packed states")
        px = x.reshape(-1, 12)[:, 0:3]
        py = y.reshape(-1, 12)[:, 0:3]
        d = px - py
        num = np.sqrt((d[:, 0] * d[:, 0] + d[:, 1] * d[:, 1]) + d[:, 2] * d[:, 2])
        den = np.sqrt((px[:, 0] * px[:, 0] + px[:, 1] * px[:, 1]) + px[:, 2] * px[:, 2])
        val = np.where(den < 1e-14, num, num / np.where(den < 1e-14, 1.0, den))
        return float(val.max(initial=0.0))

    metric.dim = 3  # type: ignore[attr-defined]
    metric.stride = 12  # type: ignore[attr-defined]
    return metric
