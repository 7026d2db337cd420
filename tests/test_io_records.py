"""Trace / record / trajectory emission in the reference's schemas:
config hash (config.cpp:191-245), trajectory binary + sidecar (io.cpp:70-132), CSV export,
RunRecord JSON, schedule and convergence CSVs.  No GPU needed."""
import ctypes as C
import json
import os

import numpy as np
import pytest

from oracle.pyoracle import Scenario as OS
from paper_2604_12083_b200 import parareal as pr
from paper_2604_12083_b200.harness import RunConfig
from paper_2604_12083_b200.io import (RunRecord, TrajectoryWriter, export_trajectory_csv, read_trajectory,
                                      write_convergence_csv, write_schedule_csv)
from paper_2604_12083_b200.scenario import RANDOM, ScenarioConfig


CFGS = [RunConfig(),
        RunConfig(scenario=ScenarioConfig(rod_count=64, nodes_per_rod=256, epsilon=0.08, horizon=8e-3),
                  intervals=8, workers=8, ratio=20.0, max_iterations=3, tolerance=1e-300, mode=pr.REGULAR,
                  fine_steps_per_interval=1000, coarse_steps_per_interval=100, snapshot_stride=7),
        RunConfig(scenario=ScenarioConfig(rod_count=3, nodes_per_rod=21, placement=RANDOM, seed=42,
                                          lj_well_depth=0.01))]


def _os_of(cfg):
    s = cfg.scenario
    return OS.make(rod_count=s.rod_count, nodes_per_rod=s.nodes_per_rod, rod_length=s.rod_length,
                   epsilon=s.epsilon, mu=s.mu, placement=s.placement, lj_well_depth=s.lj_well_depth,
                   lj_sigma=s.lj_sigma, seed=s.seed, fine_dt=s.fine_dt, horizon=s.horizon)


@pytest.mark.parametrize("cfg", CFGS)
def test_config_hash_matches_reference(ref, cfg):
    fn = ref.lib.ref_config_hash
    fn.restype = None
    buf = C.create_string_buffer(17)
    fn(C.byref(_os_of(cfg)), cfg.intervals, cfg.workers, C.c_double(cfg.ratio), cfg.max_iterations,
       C.c_double(cfg.tolerance), cfg.mode, cfg.fine_steps_per_interval, cfg.coarse_steps_per_interval,
       cfg.snapshot_stride, buf)
    assert cfg.hash() == buf.value.decode()


def test_trajectory_bytes_match_reference(ref, tmp_path):
    cfg = RunConfig(scenario=ScenarioConfig(rod_count=2, nodes_per_rod=5), snapshot_stride=3)
    rng = np.random.default_rng(0)
    frames = rng.normal(size=(4, 2 * 5 * 12))
    times = np.array([0.0, 0.1, 0.2, 0.3])
    ours = str(tmp_path / "ours.bin")
    theirs = str(tmp_path / "ref.bin")
    w = TrajectoryWriter(ours, cfg)
    for t, f in zip(times, frames):
        w.append(t, f)
    w.close()
    fn = ref.lib.ref_write_trajectory
    fn.restype = C.c_int
    P = C.POINTER(C.c_double)
    assert fn(theirs.encode(), C.byref(_os_of(cfg)), 3, 4, times.ctypes.data_as(P), frames.ctypes.data_as(P)) == 0
    assert open(ours, "rb").read() == open(theirs, "rb").read()
    a, b = json.load(open(ours + ".json")), json.load(open(theirs + ".json"))
    b["config_hash"] = b["config_hash"]  # same schema; hash of the reference's default parareal section differs
    assert set(a) == set(b) and a["frame_count"] == b["frame_count"] == 4 and a["layout"] == b["layout"]
    got, side = read_trajectory(ours)
    assert len(got) == 4 and np.array_equal(got[2][1], frames[2]) and got[3][0] == 0.3
    export_trajectory_csv(ours, str(tmp_path / "t.csv"))
    lines = open(tmp_path / "t.csv").read().splitlines()
    assert lines[0] == "frame,t,rod,node,x,y,z" and len(lines) == 1 + 4 * 10


def test_records_and_csvs(tmp_path):
    g = lambda a, b, x: np.asarray(x) * 0.9  # noqa: E731
    f = lambda a, b, x: np.asarray(x) * 0.91  # noqa: E731
    res = pr.run(pr.ParallelPlan(intervals=4, workers=2, max_iterations=2, tolerance=1e-300), g, f, [1.0, 2.0],
                 pr.pointwise_metric(1))
    write_schedule_csv(str(tmp_path / "s.csv"), res.trace)
    lines = open(tmp_path / "s.csv").read().splitlines()
    assert lines[0] == "worker,kind,t_start,t_end" and len(lines) > 4
    assert {ln.split(",")[1] for ln in lines[1:]} <= {"coarse", "fine", "correct", "idle"}
    write_convergence_csv(str(tmp_path / "c.csv"), res.report)
    assert open(tmp_path / "c.csv").read().splitlines()[0] == "iteration,eta_tilde"
    rec = RunRecord(config=RunConfig(), command="parareal", eta_tilde=res.report.eta_tilde,
                    iterations_used=res.report.iterations_used, converged=res.report.converged,
                    schedule_idle=res.trace.total_idle(), timings={"initialization": 1.0, "velocity": 2.0})
    rec.save(str(tmp_path / "r.json"))
    d = json.load(open(tmp_path / "r.json"))
    assert set(d) == {"command", "config", "config_hash", "seed", "convergence", "schedule", "timings", "artifacts"}
    assert d["timings"]["velocity_computation"] == 2.0 and d["config_hash"] == RunConfig().hash()
