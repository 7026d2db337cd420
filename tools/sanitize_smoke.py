"""Small invocations of every kernel family, for compute-sanitizer (dev tool):

    compute-sanitizer --tool memcheck python tools/sanitize_smoke.py
    compute-sanitizer --tool racecheck python tools/sanitize_smoke.py
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

from paper_2604_12083_b200.propagators import StepperConfig, propagate
from paper_2604_12083_b200 import rotation
from paper_2604_12083_b200.scenario import ScenarioConfig, build_initial_state, make_scenario
from paper_2604_12083_b200.stokes import KernelParams, LoadSet, evaluate_velocities

rng = np.random.default_rng(3)
for n, nt in ((1, None), (300, 77), (1000, None), (3001, 517), (5000, None)):
    s = rng.uniform(-0.5, 0.5, (n, 3))
    t = s if nt is None else rng.uniform(-0.5, 0.5, (nt, 3))
    f, q = rng.uniform(-1, 1, (n, 3)), rng.uniform(-1, 1, (n, 3))
    evaluate_velocities(t, s, LoadSet(f, q), KernelParams(0.1, 1.0))
    d = [torch.as_tensor(a, device="cuda") for a in (t, s, f, q)]
    evaluate_velocities(d[0], d[1], LoadSet(d[2], d[3]), KernelParams(0.1, 1.0))
print("mrs ok")
qm = np.linalg.qr(rng.standard_normal((1000, 3, 3)))[0]
qm = qm * np.sign(np.linalg.det(qm))[:, None, None]
rotation.sqrt_rotation(qm)
print("sqrt ok")
for kw in (dict(rod_count=1, nodes_per_rod=100), dict(rod_count=4, nodes_per_rod=21, placement=1, lj_well_depth=0.01,
                                                          seed=2),
           dict(rod_count=12, nodes_per_rod=51), dict(rod_count=40, nodes_per_rod=64, placement=1, lj_well_depth=0.01,
                                                      seed=5)):
    sc = make_scenario(ScenarioConfig(**kw))
    x = build_initial_state(sc)
    propagate(x, 0.0, 4e-9, StepperConfig(0.0, 1, 4), sc)  # (40 x 64 with LJ: the cell-list path)
    propagate(x, 0.0, 4e-9, StepperConfig(0.0, 0, 4), sc)
    print("propagate ok", kw)
