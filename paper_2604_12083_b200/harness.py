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

    def flat(self) -> dict:
        """Canonical flat view, config.cpp:191-226 (doubles as %.17g, ints as decimal)."""
        s = self.scenario
        g = lambda v: format(float(v), ".17g")  # noqa: E731  (ostream precision 17)
        m, w = s.material, s.waveform
        return {
            "scenario.rod_count": str(int(s.rod_count)), "scenario.nodes_per_rod": str(int(s.nodes_per_rod)),
            "scenario.rod_length": g(s.rod_length), "scenario.a1": g(m.a1), "scenario.a2": g(m.a2),
            "scenario.a3": g(m.a3), "scenario.b1": g(m.b1), "scenario.b2": g(m.b2), "scenario.b3": g(m.b3),
            "scenario.amplitude": g(w.amplitude), "scenario.wave_frequency": g(w.frequency),
            "scenario.wavelength": g(w.wavelength), "scenario.epsilon": g(s.epsilon), "scenario.mu": g(s.mu),
            "scenario.lj_well_depth": g(s.lj_well_depth), "scenario.lj_sigma": g(s.lj_sigma),
            "scenario.wall_clearance": g(s.wall_clearance), "scenario.seed": str(int(s.seed)),
            "scenario.fine_dt": g(s.fine_dt), "scenario.horizon": g(s.horizon),
            "scenario.placement": "grid" if s.placement == 0 else "random",
            "scenario.wall_mode": "free_space" if s.wall_mode == 0 else "image_wall",
            "parareal.intervals": str(int(self.intervals)), "parareal.workers": str(int(self.workers)),
            "parareal.ratio": g(self.ratio), "parareal.max_iterations": str(int(self.max_iterations)),
            "parareal.tolerance": g(self.tolerance),
            "parareal.mode": "regular" if self.mode == pr.REGULAR else "pipelined",
            "parareal.fine_steps_per_interval": str(int(self.fine_steps_per_interval)),
            "parareal.coarse_steps_per_interval": str(int(self.coarse_steps_per_interval)),
            "output.snapshot_stride": str(int(self.snapshot_stride)),
        }

    def hash(self) -> str:
        """FNV-1a 64 over the canonical view, config.cpp:228-245."""
        h = 1469598103934665603
        for k, v in sorted(self.flat().items()):
            for c in (k + "=" + v + "\n").encode():
                h ^= c
                h = (h * 1099511628211) & 0xFFFFFFFFFFFFFFFF
        return f"{h:016x}"

    def run_tag(self) -> str:
        """io.cpp:172-174."""
        return f"seed{int(self.scenario.seed)}_{self.hash()[:8]}"

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


def simulate(cfg: RunConfig, output_dir: str, fmt: str = "bin", device: int = 0) -> dict:
    """`swim simulate` (tools/swim.cpp:69-115) on the device: serial fine RK2 over the
    horizon at fine_dt, a trajectory frame every snapshot_stride steps, a RunRecord with the
    three stage timers.  Returns the record dict."""
    import os
    import time

    import torch

    from . import io as pio
    from .device import Context, dptr

    sc = make_scenario(cfg.scenario)
    dt = cfg.scenario.fine_dt
    span = cfg.scenario.horizon
    steps = int(np.floor(span / dt + 0.5))
    if steps == 0 or abs(span / dt - steps) > 1e-9 * steps:
        raise ValueError("simulate: horizon must be an integral number of fine_dt steps")
    tag = cfg.run_tag()
    os.makedirs(output_dir, exist_ok=True)
    traj = os.path.join(output_dir, f"traj_{tag}.bin")
    ctx = Context(device, sc)
    ctx.timing(True)
    ctx.timing_reset()
    x = torch.as_tensor(build_initial_state(sc), device=f"cuda:{device}")
    out = torch.empty_like(x)
    writer = pio.TrajectoryWriter(traj, cfg)
    writer.append(0.0, x.cpu().numpy())
    stride = max(1, int(cfg.snapshot_stride))
    t = 0.0
    done = 0
    t_wall = time.perf_counter()
    while done < steps:
        chunk = min(stride - (done % stride), steps - done)
        t1 = t
        for _ in range(chunk):
            t1 += dt  # propagators.cpp:159 accumulation, replicated on the host
        ctx.check(ctx.lib.pswim_propagate(ctx.handle, dptr(x), t, t + chunk * dt, RK2, 0, dt, dptr(out)))
        x, out = out, x
        t = t1
        done += chunk
        if done % stride == 0 or done == steps:
            writer.append(t, x.cpu().numpy())
    wall = time.perf_counter() - t_wall
    writer.close()
    rec = pio.RunRecord(config=cfg, command="simulate", wall_seconds=wall, timings=ctx.timing_snapshot(),
                        artifacts=[traj])
    if fmt == "csv":
        csv_path = os.path.join(output_dir, f"traj_{tag}.csv")
        pio.export_trajectory_csv(traj, csv_path)
        rec.artifacts.append(csv_path)
    rec.save(os.path.join(output_dir, f"record_simulate_{tag}.json"))
    ctx.close()
    return rec.to_dict()
