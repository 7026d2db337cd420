"""Scenario configuration — mirror of reference include/pintswim/scenario.hpp.

``ScenarioConfig`` carries the reference defaults (scenario.hpp:16-35); ``make_scenario``
resolves ds, epsilon = 4 ds, sigma = 3 epsilon and the LJ window (scenario.cpp:10-29) and
``build_initial_state`` returns the packed state (io.cpp:10-25 layout) of
scenario.cpp:71-120, computed by the native host runtime.
"""
from __future__ import annotations

import ctypes as C
import math
from dataclasses import dataclass, field, replace

import numpy as np

from . import _lib

GRID = 0
RANDOM = 1


@dataclass
class MaterialParams:
    a1: float = 0.01
    a2: float = 0.01
    a3: float = 0.01
    b1: float = 2.0
    b2: float = 2.0
    b3: float = 2.0


@dataclass
class WaveformParams:
    amplitude: float = 0.05
    frequency: float = 2.0 * math.pi
    wavelength: float = 1.0


@dataclass
class ScenarioConfig:
    rod_count: int = 1
    nodes_per_rod: int = 51
    rod_length: float = 1.0
    material: MaterialParams = field(default_factory=MaterialParams)
    waveform: WaveformParams = field(default_factory=WaveformParams)
    epsilon: float = 0.0
    mu: float = 1.0
    wall_mode: int = 0
    lj_well_depth: float = 0.0
    lj_sigma: float = 0.0
    wall_clearance: float = 1.0
    seed: int = 1
    fine_dt: float = 1e-6
    horizon: float = 1e-3
    placement: int = GRID

    def to_c(self) -> _lib.Scenario:
        s = _lib.Scenario()
        s.rod_count = int(self.rod_count)
        s.nodes_per_rod = int(self.nodes_per_rod)
        s.rod_length = float(self.rod_length)
        m = self.material
        s.a1, s.a2, s.a3, s.b1, s.b2, s.b3 = (float(v) for v in (m.a1, m.a2, m.a3, m.b1, m.b2, m.b3))
        w = self.waveform
        s.amplitude, s.frequency, s.wavelength = float(w.amplitude), float(w.frequency), float(w.wavelength)
        s.epsilon = float(self.epsilon)
        s.mu = float(self.mu)
        s.wall_mode = int(self.wall_mode)
        s.placement = int(self.placement)
        s.lj_well_depth = float(self.lj_well_depth)
        s.lj_sigma = float(self.lj_sigma)
        s.wall_clearance = float(self.wall_clearance)
        s.seed = int(self.seed)
        s.fine_dt = float(self.fine_dt)
        s.horizon = float(self.horizon)
        return s

    def replace(self, **kw) -> "ScenarioConfig":
        return replace(self, **kw)

    @property
    def total_nodes(self) -> int:
        return int(self.rod_count * self.nodes_per_rod)


@dataclass
class Scenario:
    """Resolved scenario (scenario.hpp:38-44)."""

    cfg: ScenarioConfig
    ds: float
    epsilon: float
    mu: float
    lj_sigma: float
    lj_cutoff: float
    lj_self_exclusion: int

    def to_c(self) -> _lib.Scenario:
        return self.cfg.to_c()

    @property
    def total_nodes(self) -> int:
        return self.cfg.total_nodes


def make_scenario(cfg: ScenarioConfig) -> Scenario:
    L = _lib.lib()
    r = _lib.Resolved()
    c = cfg.to_c()
    rc = L.pswim_scenario_resolve(C.byref(c), C.byref(r))
    if rc:
        _lib.raise_for(rc, "scenario: invalid configuration")
    return Scenario(cfg, r.ds, r.epsilon, r.mu, r.lj_sigma, r.lj_cutoff, int(r.lj_self_exclusion))


def build_initial_state(sc) -> np.ndarray:
    """Packed initial state, shape (rod_count * nodes_per_rod * 12,)."""
    L = _lib.lib()
    cfg = sc.cfg if isinstance(sc, Scenario) else sc
    c = cfg.to_c()
    out = np.zeros(12 * cfg.total_nodes)
    rc = L.pswim_build_initial_state(C.byref(c), out.ctypes.data_as(C.POINTER(C.c_double)))
    if rc:
        _lib.raise_for(rc, "build_initial_state: placement failed after 10000 attempts; enlarge the domain or reduce rod count")
    return out
