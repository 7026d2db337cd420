"""Parity at BASELINE.json's full sizes through sampled rows and size-independent properties:
MRS at N = 65,536, 131,072 (configs[4]: 512 x 256) and 1,048,576 (8x beyond it: 3.6 s per
evaluation, 1.8 GB of split-source partials) -- oracle rows, linearity in the loads,
bitwise repeats -- and one RK2 step of the 64 x 256 suspension
(configs[2]) against the reference restatement."""
import os

import numpy as np
import pytest

pytestmark = pytest.mark.gpu
TOL = 1e-10


def _inputs(n, seed):
    rng = np.random.default_rng(seed)
    return (rng.uniform(-0.5, 0.5, (n, 3)) for _ in range(3))


@pytest.mark.parametrize("n", [65536, 131072, 1048576])
def test_mrs_full_size_rows_linearity_repeat(gpu, oracle, n):
    import torch

    from paper_2604_12083_b200.stokes import KernelParams, LoadSet, evaluate_velocities

    x, f, tq = _inputs(n, 11)
    g, h, _ = _inputs(n, 12)
    d = [torch.as_tensor(a, device=gpu) for a in (x, f, tq, g, h)]
    kp = KernelParams(0.08, 1.0)
    a = evaluate_velocities(d[0], d[0], LoadSet(d[1], d[2]), kp)
    b = evaluate_velocities(d[0], d[0], LoadSet(d[1], d[2]), kp)
    assert torch.equal(a.u, b.u) and torch.equal(a.omega, b.omega)  # fixed-order reduction
    # rows of three target blocks (first, middle, last) against the reference restatement
    rows = np.r_[0:32, n // 2 - 16:n // 2 + 16, n - 32:n]
    ou, ow = oracle.evaluate_rows(x[rows], 0, len(rows), x, f, tq, 0.08, 1.0, threads=os.cpu_count() or 1)
    gu, gw = a.u.cpu().numpy()[rows], a.omega.cpu().numpy()[rows]
    scale = max(np.abs(ou).max(), np.abs(ow).max())
    assert max(np.abs(gu - ou).max(), np.abs(gw - ow).max()) / scale < TOL
    # linearity in the loads: u(al F + be G) = al u(F) + be u(G)
    al, be = 0.75, -1.25
    c = evaluate_velocities(d[0], d[0], LoadSet(d[3], d[4]), kp)
    m = evaluate_velocities(d[0], d[0], LoadSet(al * d[1] + be * d[3], al * d[2] + be * d[4]), kp)
    lin_u = (m.u - (al * a.u + be * c.u)).abs().max().item()
    lin_w = (m.omega - (al * a.omega + be * c.omega)).abs().max().item()
    scale = max(m.u.abs().max().item(), m.omega.abs().max().item())
    assert max(lin_u, lin_w) / scale < 1e-12


def test_rk2_step_64x256_vs_oracle(gpu, oracle):
    """BASELINE configs[2] (64 x 256, eps = 0.08, dt = 1e-6): one RK2 step of the GPU
    propagate against the reference restatement (all host threads), <= 1e-10."""
    from oracle.pyoracle import Scenario as OS
    from paper_2604_12083_b200.propagators import StepperConfig, propagate
    from paper_2604_12083_b200.scenario import ScenarioConfig, build_initial_state, make_scenario

    kw = dict(rod_count=64, nodes_per_rod=256, epsilon=0.08)
    sc = make_scenario(ScenarioConfig(**kw))
    x = build_initial_state(sc)
    got = propagate(x, 0.0, 1e-6, StepperConfig(0.0, 1, 1), sc)
    want = oracle.propagate(OS.make(**kw), x, 0.0, 1e-6, 1, steps=1, threads=os.cpu_count() or 1)
    assert oracle.position_metric(want, got) < TOL
    # the triads too (relative to their unit norm)
    assert np.abs(got.reshape(-1, 12)[:, 3:] - want.reshape(-1, 12)[:, 3:]).max() < 1e-10
