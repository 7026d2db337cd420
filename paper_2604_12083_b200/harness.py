"""Run glue — mirror of reference include/pintswim/harness.hpp / src/harness.cpp:5-37.

``prepare(cfg)`` turns a :class:`RunConfig` (config.hpp:20-45 fields) into the resolved
scenario, the Parareal plan, the packed initial state and GPU coarse (Euler) / fine (RK2)
propagators over packed states; ``serial_fine_boundaries`` chains the fine propagator per
interval (bitwise comparable with Parareal iterates).
"""
from __future__ import annotations

from dataclasses import dataclass, field
from typing import Callable, List

import numpy as np

from . import parareal as pr
from .propagators import EULER, RK2, StepperConfig, propagate
from .scenario import Scenario, ScenarioConfig, build_initial_state, make_scenario


@dataclass
class RunConfig:
    scenario: ScenarioConfig = field(default_factory=ScenarioConfig)
    intervals: int = 8
    workers: int = 2
    ratio: float = 2.0
    max_iterations: int = 10
    tolerance: float = 1e-10
    mode: int = pr.PIPELINED
    fine_steps_per_interval: int = 100
    coarse_steps_per_interval: int = 0
    snapshot_stride: int = 1

    def resolved_coarse_steps(self) -> int:
        """config.cpp:247-250: coarse_steps or max(1, llround(2 fine / r))."""
        if self.coarse_steps_per_interval > 0:
            return self.coarse_steps_per_interval
        v = 2.0 * self.fine_steps_per_interval / self.ratio
        return max(1, int(np.floor(v + 0.5)) if v >= 0 else int(np.ceil(v - 0.5)))


@dataclass
class PhysicsRun:
    scenario: Scenario
    plan: pr.ParallelPlan
    x0: np.ndarray
    coarse: Callable
    fine: Callable
    cfg: RunConfig
    device: int = 0

    def run(self, reference: List[np.ndarray] | None = None) -> pr.RunResult:
        """parareal::run with the GPU propagators on the native engine."""
        return pr.run_gpu(self.plan, self.scenario, self.cfg.fine_steps_per_interval,
                          self.cfg.resolved_coarse_steps(), self.x0, reference, self.device)


def prepare(cfg: RunConfig, device: int = 0) -> PhysicsRun:
    sc = make_scenario(cfg.scenario)
    plan = pr.ParallelPlan(t0=0.0, horizon=cfg.scenario.horizon, intervals=cfg.intervals, workers=cfg.workers,
                           cost_ratio=cfg.ratio, max_iterations=cfg.max_iterations, tolerance=cfg.tolerance,
                           mode=cfg.mode)
    x0 = build_initial_state(sc)
    fine_cfg = StepperConfig(0.0, RK2, cfg.fine_steps_per_interval)
    coarse_cfg = StepperConfig(0.0, EULER, cfg.resolved_coarse_steps())

    def fine(t0, t1, x):
        return propagate(x, t0, t1, fine_cfg, sc)

    def coarse(t0, t1, x):
        return propagate(x, t0, t1, coarse_cfg, sc)

    return PhysicsRun(sc, plan, x0, coarse, fine, cfg, device)


def serial_fine_boundaries(run: PhysicsRun) -> List[np.ndarray]:
    """coarse_sweep_initial with the fine propagator (harness.cpp:35-37)."""
    return pr.coarse_sweep_initial(run.plan, run.fine, run.x0)
