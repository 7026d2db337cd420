"""State packing and the convergence metric — mirror of reference include/pintswim/io.hpp:14-21.

Packed layout (io.cpp:10-25): per node 12 doubles [x, d1, d2, d3], rods concatenated.  This
is also the device layout of every state in HBM, so pack/unpack are views, not copies.
"""
from __future__ import annotations

import json
import os
from dataclasses import dataclass, field
from typing import List

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


# ---- trajectory files (io.cpp:70-149) ----------------------------------------------------------
class TrajectoryWriter:
    """Binary frames [t, packed state] in native byte order + JSON sidecar <path>.json."""

    def __init__(self, path: str, config):
        self.path = path
        self.config = config
        self.fh = open(path, "wb")
        self.frames = 0
        self.closed = False

    def append(self, t: float, state) -> None:
        np.asarray([t], dtype=np.float64).tofile(self.fh)
        np.ascontiguousarray(np.asarray(state, dtype=np.float64).reshape(-1)).tofile(self.fh)
        self.frames += 1

    def close(self) -> None:
        if self.closed:
            return
        self.closed = True
        self.fh.close()
        c = self.config
        side = {"rod_count": int(c.scenario.rod_count), "nodes_per_rod": int(c.scenario.nodes_per_rod),
                "fine_dt": float(c.scenario.fine_dt), "snapshot_stride": int(c.snapshot_stride),
                "frame_count": self.frames, "seed": int(c.scenario.seed), "config_hash": c.hash(),
                "layout": "frame = [t, per node: x(3), d1(3), d2(3), d3(3)], float64 native order"}
        with open(self.path + ".json", "w") as fh:
            fh.write(json.dumps(side, indent=2, sort_keys=True) + "\n")

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def read_trajectory(path: str):
    """[(t, packed state)], io.cpp:108-132."""
    with open(path + ".json") as fh:
        side = json.load(fh)
    n = 12 * side["rod_count"] * side["nodes_per_rod"]
    raw = np.fromfile(path, dtype=np.float64)
    frames = side["frame_count"]
    if raw.size < frames * (n + 1):
        raise _lib.PswimError(8, f"trajectory: truncated file '{path}'")
    raw = raw[: frames * (n + 1)].reshape(frames, n + 1)
    return [(float(r[0]), r[1:].copy()) for r in raw], side


def export_trajectory_csv(binary_path: str, csv_path: str) -> None:
    """frame,t,rod,node,x,y,z with 17 significant digits (io.cpp:134-149)."""
    frames, side = read_trajectory(binary_path)
    rods, m = side["rod_count"], side["nodes_per_rod"]
    g = lambda v: format(float(v), ".17g")  # noqa: E731
    with open(csv_path, "w") as out:
        out.write("frame,t,rod,node,x,y,z\n")
        for f, (t, st) in enumerate(frames):
            x = st.reshape(rods, m, 12)
            for r in range(rods):
                for k in range(m):
                    out.write(f"{f},{g(t)},{r},{k},{g(x[r, k, 0])},{g(x[r, k, 1])},{g(x[r, k, 2])}\n")


# ---- run records and CSVs (io.cpp:151-184, tools/swim.cpp:133-142) ----------------------------
@dataclass
class RunRecord:
    config: object
    command: str = ""
    eta_tilde: List[float] = field(default_factory=list)
    eta: List[float] = field(default_factory=list)
    iterations_used: int = 0
    converged: bool = True
    wall_seconds: float = 0.0
    schedule_idle: float = 0.0
    timings: dict = field(default_factory=dict)
    artifacts: List[str] = field(default_factory=list)

    def to_dict(self) -> dict:
        t = self.timings or {}
        return {"command": self.command, "config": self.config.flat(), "config_hash": self.config.hash(),
                "seed": int(self.config.scenario.seed),
                "convergence": {"eta_tilde": list(self.eta_tilde), "eta": list(self.eta),
                                "iterations_used": int(self.iterations_used), "converged": bool(self.converged)},
                "schedule": {"wall_seconds": self.wall_seconds, "total_idle": self.schedule_idle},
                "timings": {"initialization": t.get("initialization", 0.0),
                            "velocity_computation": t.get("velocity", 0.0),
                            "triad_update": t.get("triad_update", 0.0)},
                "artifacts": list(self.artifacts)}

    def save(self, path: str) -> None:
        with open(path, "w") as fh:
            fh.write(json.dumps(self.to_dict(), indent=2, sort_keys=True) + "\n")  # nlohmann dumps std::map order


def write_schedule_csv(path: str, trace) -> None:
    """worker,kind,t_start,t_end (io.cpp:176-184)."""
    from .parareal import TASK_NAMES

    g = lambda v: format(float(v), ".17g")  # noqa: E731
    with open(path, "w") as out:
        out.write("worker,kind,t_start,t_end\n")
        for e in trace.events:
            out.write(f"{e.worker},{TASK_NAMES[e.kind]},{g(e.t_start)},{g(e.t_end)}\n")


def write_convergence_csv(path: str, report) -> None:
    """iteration,eta_tilde[,eta] (tools/swim.cpp:133-142)."""
    g = lambda v: format(float(v), ".17g")  # noqa: E731
    with open(path, "w") as out:
        out.write("iteration,eta_tilde" + ("" if not report.eta else ",eta") + "\n")
        for k, et in enumerate(report.eta_tilde):
            out.write(f"{k + 1},{g(et)}" + (f",{g(report.eta[k])}" if report.eta else "") + "\n")
