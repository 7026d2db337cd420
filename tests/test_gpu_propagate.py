"""GPU parity of rhs / advance_state / step / propagate (reference propagators.cpp:38-162)."""
import os

import numpy as np
import pytest

from helpers import rel_field_err

pytestmark = pytest.mark.gpu


def scen(**kw):
    from paper_2604_12083_b200.scenario import ScenarioConfig, make_scenario

    return make_scenario(ScenarioConfig(**kw))


CASES = [dict(rod_count=1, nodes_per_rod=21), dict(rod_count=1, nodes_per_rod=100),
         dict(rod_count=4, nodes_per_rod=21, placement=1, lj_well_depth=0.01, seed=2),
         dict(rod_count=9, nodes_per_rod=64, epsilon=0.08)]


@pytest.mark.parametrize("kw", CASES)
def test_rhs_matches_oracle(gpu, oracle, kw):
    from paper_2604_12083_b200.propagators import rhs
    from paper_2604_12083_b200.scenario import build_initial_state
    from oracle.pyoracle import Scenario as OS

    sc = scen(**kw)
    x = build_initial_state(sc)
    osc = OS.make(**kw)
    assert np.array_equal(x, oracle.build_initial_state(osc))
    # perturb so every term is active
    rng = np.random.default_rng(1)
    y = x.reshape(-1, 12).copy()
    y[:, 0:3] += rng.normal(scale=1e-3, size=(len(y), 3))
    y = y.reshape(-1)
    got = rhs(y, 0.137, sc)
    want = oracle.rhs(osc, y, 0.137)
    assert rel_field_err((got.u, got.omega), want) < 1e-10


def test_rhs_extra_loads_linear(gpu, oracle):
    from paper_2604_12083_b200.propagators import rhs
    from paper_2604_12083_b200.scenario import build_initial_state
    from paper_2604_12083_b200.stokes import LoadSet
    from oracle.pyoracle import Scenario as OS

    sc = scen(rod_count=1, nodes_per_rod=21)
    x = build_initial_state(sc)
    rng = np.random.default_rng(5)
    ef, en = rng.uniform(-1, 1, (21, 3)), rng.uniform(-1, 1, (21, 3))
    got = rhs(x, 0.1, sc, LoadSet(ef, en))
    want = oracle.rhs(OS.make(rod_count=1, nodes_per_rod=21), x, 0.1, ef.reshape(-1), en.reshape(-1))
    assert rel_field_err((got.u, got.omega), want) < 1e-10


def test_advance_matches_oracle_and_stiffness(gpu, oracle):
    from paper_2604_12083_b200.propagators import StiffnessError, SystemVelocities, advance_state
    from paper_2604_12083_b200.scenario import build_initial_state
    from oracle.pyoracle import Scenario as OS

    sc = scen(rod_count=2, nodes_per_rod=33)
    x = build_initial_state(sc)
    rng = np.random.default_rng(3)
    u = rng.uniform(-0.1, 0.1, (66, 3))
    w = rng.uniform(-2, 2, (66, 3))
    w[5] = 0.0
    got = advance_state(x, SystemVelocities(u, w), 0.01, sc)
    want = oracle.advance_state(OS.make(rod_count=2, nodes_per_rod=33), x, u, w, 0.01)
    assert np.max(np.abs(got - want)) < 1e-14
    with pytest.raises(StiffnessError):
        advance_state(x, SystemVelocities(np.ones((66, 3)), w), 1.0, sc)


@pytest.mark.parametrize("scheme", [0, 1])
def test_propagate_matches_oracle(gpu, oracle, scheme):
    """1 x 100 flagellum (BASELINE config 1), 200 steps at dt=1e-5."""
    from paper_2604_12083_b200.propagators import StepperConfig, propagate
    from paper_2604_12083_b200.scenario import build_initial_state
    from oracle.pyoracle import Scenario as OS

    kw = dict(rod_count=1, nodes_per_rod=100)
    sc = scen(**kw)
    x = build_initial_state(sc)
    got = propagate(x, 0.0, 2e-3, StepperConfig(0.0, scheme, 200), sc)
    want = oracle.propagate(OS.make(**kw), x, 0.0, 2e-3, scheme, steps=200)
    assert oracle.position_metric(want, got) < 1e-10
    moved = oracle.position_metric(x, want)
    assert moved > 1e-6


def test_propagate_64x256_short(gpu, oracle):
    """BASELINE config 3 suspension (64 x 256, eps=0.08): 3 RK2 steps vs the oracle."""
    import torch
    from paper_2604_12083_b200.propagators import StepperConfig, propagate
    from paper_2604_12083_b200.scenario import build_initial_state
    from oracle.pyoracle import Scenario as OS

    kw = dict(rod_count=64, nodes_per_rod=256, epsilon=0.08)
    sc = scen(**kw)
    x = build_initial_state(sc)
    got = propagate(torch.as_tensor(x, device=gpu), 0.0, 3e-6, StepperConfig(1e-6, 1, 0), sc).cpu().numpy()
    want = oracle.propagate(OS.make(**kw), x, 0.0, 3e-6, 1, steps=0, dt=1e-6, threads=8)
    assert oracle.position_metric(want, got) < 1e-10


def test_propagate_bitwise_deterministic_and_composes(gpu):
    from paper_2604_12083_b200.propagators import StepperConfig, propagate
    from paper_2604_12083_b200.scenario import build_initial_state

    sc = scen(rod_count=1, nodes_per_rod=21)
    x = build_initial_state(sc)
    a = propagate(x, 0.0, 0.0625, StepperConfig(0.0, 1, 8), sc)
    b = propagate(x, 0.0, 0.0625, StepperConfig(0.0, 1, 8), sc)
    assert np.array_equal(a, b)
    half = StepperConfig(0.0, 1, 4)
    two = propagate(propagate(x, 0.0, 0.03125, half, sc), 0.03125, 0.0625, half, sc)
    assert np.array_equal(two, a)
    assert np.array_equal(propagate(x, 0.3, 0.3, StepperConfig(0.0, 1, 8), sc), x)
    from paper_2604_12083_b200 import InvalidArgument

    with pytest.raises(InvalidArgument):
        propagate(x, 0.0, 0.1, StepperConfig(0.013, 0, 0), sc)


def test_quiet_rod_zero_rhs(gpu):
    from paper_2604_12083_b200.propagators import rhs
    from paper_2604_12083_b200.scenario import ScenarioConfig, WaveformParams, build_initial_state, make_scenario

    sc = make_scenario(ScenarioConfig(rod_count=1, nodes_per_rod=21, waveform=WaveformParams(0.0, 2 * np.pi, 1.0)))
    v = rhs(build_initial_state(sc), 0.0, sc)
    assert np.abs(v.u).max() < 1e-13 and np.abs(v.omega).max() < 1e-13


@pytest.mark.parametrize("kw,scheme,steps", [(dict(rod_count=1, nodes_per_rod=100), 1, 50),
                                             (dict(rod_count=1, nodes_per_rod=100), 0, 50),
                                             (dict(rod_count=1, nodes_per_rod=21), 1, 40),
                                             (dict(rod_count=4, nodes_per_rod=21, placement=1, lj_well_depth=0.01,
                                                   seed=2), 1, 20),
                                             (dict(rod_count=2, nodes_per_rod=128, epsilon=0.08), 1, 10),
                                             (dict(rod_count=3, nodes_per_rod=60, placement=1, lj_well_depth=0.01,
                                                   seed=3), 0, 7),  # N = 180: 384 threads, LJ, Euler, odd
                                             (dict(rod_count=1, nodes_per_rod=37), 1, 9)])  # 7 chunks, last short
def test_fused_propagate_bitwise_equals_launched_path(gpu, oracle, kw, scheme, steps):
    """The fused cluster kernel (N <= 256) reproduces the per-step launched kernels bitwise
    and the oracle to 1e-10."""
    from paper_2604_12083_b200.device import Context
    from paper_2604_12083_b200.propagators import StepperConfig, propagate
    from paper_2604_12083_b200.scenario import build_initial_state
    from oracle.pyoracle import Scenario as OS

    sc = scen(**kw)
    x = build_initial_state(sc)
    fused = Context(0, sc)
    plain = Context(0, sc)
    cs = fused.lib.pswim_set_fused(fused.handle, 1)
    assert cs >= 1 or kw["nodes_per_rod"] * kw["rod_count"] > 200  # N=256 exceeds the fused smem budget
    plain.lib.pswim_set_fused(plain.handle, 0)
    cfg = StepperConfig(0.0, scheme, steps)
    t1 = steps * 1e-5
    a = propagate(x, 0.0, t1, cfg, sc, ctx=fused)
    b = propagate(x, 0.0, t1, cfg, sc, ctx=plain)
    assert np.array_equal(a, b)
    want = oracle.propagate(OS.make(**kw), x, 0.0, t1, scheme, steps=steps)
    assert oracle.position_metric(want, a) < 1e-10
    fused.close()
    plain.close()


def test_fused_stiffness_and_step_chain(gpu):
    """Stiffness guard raised from inside the fused kernel; fused propagate equals the chain
    of single steps (reference test_propagators.cpp:179-191)."""
    from paper_2604_12083_b200.propagators import StepperConfig, StiffnessError, propagate, step_rk2
    from paper_2604_12083_b200.scenario import build_initial_state

    sc = scen(rod_count=1, nodes_per_rod=21)
    x = build_initial_state(sc)
    horizon = 0.0625
    manual = x
    t = 0.0
    for _ in range(8):
        manual = step_rk2(manual, t, horizon / 8, sc)
        t += horizon / 8
    assert np.array_equal(propagate(x, 0.0, horizon, StepperConfig(0.0, 1, 8), sc), manual)
    with pytest.raises(StiffnessError):
        propagate(x, 0.0, 50.0, StepperConfig(0.0, 1, 5), sc)


def test_simulate_driver(gpu, oracle, tmp_path):
    """`swim simulate` equivalent: frames every snapshot_stride, final frame vs the oracle's
    step chain, RunRecord with the three stage timers (acceptance C7 schema)."""
    import json

    from paper_2604_12083_b200.harness import RunConfig, simulate
    from paper_2604_12083_b200.io import read_trajectory
    from paper_2604_12083_b200.scenario import ScenarioConfig
    from oracle.pyoracle import Scenario as OS

    cfg = RunConfig(scenario=ScenarioConfig(nodes_per_rod=11, fine_dt=0.0005, horizon=0.002), snapshot_stride=3)
    rec = simulate(cfg, str(tmp_path), fmt="csv")
    frames, side = read_trajectory(rec["artifacts"][0])
    assert side["frame_count"] == len(frames) == 3  # t = 0, after 3 steps, after 4 steps
    assert abs(frames[-1][0] - 0.002) < 1e-15
    x = frames[0][1]
    want = x.copy()
    t = 0.0
    for _ in range(4):
        want = oracle.step(OS.make(nodes_per_rod=11), 1, want, t, 0.0005)
        t += 0.0005
    assert oracle.position_metric(want, frames[-1][1]) < 1e-10
    d = json.load(open(os.path.join(str(tmp_path), f"record_simulate_{cfg.run_tag()}.json")))
    for key in ("initialization", "velocity_computation", "triad_update"):
        assert key in d["timings"]
    assert d["timings"]["velocity_computation"] > 0


def test_fused_phase_profile(gpu):
    """pswim_fused_profile: the fused propagate with its in-kernel phase timer on returns the
    same state as the plain fused propagate and non-zero cycles for the phases it runs."""
    import ctypes as C

    import torch

    from paper_2604_12083_b200.device import Context, dptr
    from paper_2604_12083_b200.propagators import StepperConfig, propagate
    from paper_2604_12083_b200.scenario import build_initial_state

    sc = scen(rod_count=1, nodes_per_rod=100)
    x = build_initial_state(sc)
    ctx = Context(0, sc)
    assert ctx.lib.pswim_set_fused(ctx.handle, 1) >= 1
    want = propagate(x, 0.0, 2e-4, StepperConfig(0.0, 1, 20), sc, ctx=ctx)
    dx = torch.as_tensor(x, device=gpu)
    out = torch.empty_like(dx)
    cyc = (C.c_uint64 * 7)()
    ctx.check(ctx.lib.pswim_fused_profile(ctx.handle, dptr(dx), 0.0, 2e-4, 1, 20, dptr(out), cyc))
    assert np.array_equal(out.cpu().numpy(), want)
    assert all(cyc[i] > 0 for i in (0, 1, 2, 3, 4, 5, 6))
    ctx.close()


@pytest.mark.parametrize("kw,scheme,steps", [(dict(rod_count=3, nodes_per_rod=100), 1, 70),
                                             (dict(rod_count=3, nodes_per_rod=100), 0, 64),
                                             (dict(rod_count=4, nodes_per_rod=128, placement=1, lj_well_depth=0.01,
                                                   seed=3, epsilon=0.08), 1, 33)])
def test_graph_replay_bitwise_equals_step_loop(gpu, oracle, kw, scheme, steps):
    """Propagations outside the fused path replay a captured CUDA graph of 32 steps (times
    from device memory): bitwise equal to the launch-per-kernel loop, and to the oracle."""
    from oracle.pyoracle import Scenario as OS
    from paper_2604_12083_b200.device import Context
    from paper_2604_12083_b200.propagators import StepperConfig, propagate
    from paper_2604_12083_b200.scenario import build_initial_state

    sc = scen(**kw)
    x = build_initial_state(sc)
    g, p = Context(0, sc), Context(0, sc)
    assert g.lib.pswim_set_fused(g.handle, 0) == 0  # N > 256: not fused-eligible anyway
    p.lib.pswim_set_fused(p.handle, 0)
    assert p.lib.pswim_set_graphs(p.handle, 0) == 1
    cfg = StepperConfig(0.0, scheme, steps)
    t1 = steps * 1e-6
    a = propagate(x, 0.0, t1, cfg, sc, ctx=g)
    b = propagate(x, 0.0, t1, cfg, sc, ctx=p)
    assert np.array_equal(a, b)
    # a second interval reuses the captured graph at new times
    a2 = propagate(a, t1, 2 * t1, cfg, sc, ctx=g)
    b2 = propagate(b, t1, 2 * t1, cfg, sc, ctx=p)
    assert np.array_equal(a2, b2)
    want = oracle.propagate(OS.make(**kw), x, 0.0, t1, scheme, steps=steps)
    assert oracle.position_metric(want, a) < 1e-10
    g.close()
    p.close()


@pytest.mark.parametrize("kw", [dict(rod_count=1, nodes_per_rod=3), dict(rod_count=2, nodes_per_rod=3),
                                dict(rod_count=5, nodes_per_rod=3), dict(rod_count=130, nodes_per_rod=3),
                                dict(rod_count=1, nodes_per_rod=257), dict(rod_count=3, nodes_per_rod=86)])
def test_edge_sizes_vs_oracle(gpu, oracle, kw):
    """Ragged and extreme layouts: the shortest rods the reference accepts (3 nodes), one rod
    just over the fused limit,
    node counts that are not multiples of the warp tile (30 / 31 nodes) or of the MRS target
    block (256): rhs and a short RK2 propagate against the oracle; fused and launched paths
    (and the graph replay) agree bitwise where both apply."""
    from oracle.pyoracle import Scenario as OS
    from paper_2604_12083_b200.device import Context
    from paper_2604_12083_b200.propagators import StepperConfig, propagate, rhs
    from paper_2604_12083_b200.scenario import build_initial_state

    kw = dict(kw, epsilon=0.08)
    sc = scen(**kw)
    x = build_initial_state(sc)
    osc = OS.make(**kw)
    v = rhs(x, 0.0, sc)
    ou, ow = oracle.rhs(osc, x, 0.0)
    scale = max(np.abs(ou).max(), np.abs(ow).max(), 1e-300)
    assert max(np.abs(v.u - ou).max(), np.abs(v.omega - ow).max()) <= 1e-10 * scale
    steps = 40
    cfg = StepperConfig(0.0, 1, steps)
    a_ctx, b_ctx = Context(0, sc), Context(0, sc)
    b_ctx.lib.pswim_set_fused(b_ctx.handle, 0)
    b_ctx.lib.pswim_set_graphs(b_ctx.handle, 0)
    a = propagate(x, 0.0, steps * 1e-6, cfg, sc, ctx=a_ctx)
    b = propagate(x, 0.0, steps * 1e-6, cfg, sc, ctx=b_ctx)
    assert np.array_equal(a, b)
    want = oracle.propagate(osc, x, 0.0, steps * 1e-6, 1, steps=steps)
    assert oracle.position_metric(want, a) < 1e-10
    a_ctx.close()
    b_ctx.close()


def test_fused_cluster_cap_bitwise(gpu):
    """pswim_set_fused(ctx, 16): the flagellum on 16-CTA clusters, bitwise equal to the
    default 8-CTA cluster and to the launched path (the cluster size only splits targets)."""
    from paper_2604_12083_b200.device import Context
    from paper_2604_12083_b200.propagators import StepperConfig, propagate
    from paper_2604_12083_b200.scenario import build_initial_state

    sc = scen(rod_count=1, nodes_per_rod=100)
    x = build_initial_state(sc)
    c16, c8, cl = Context(0, sc), Context(0, sc), Context(0, sc)
    assert c16.lib.pswim_set_fused(c16.handle, 16) == 16
    assert c8.lib.pswim_set_fused(c8.handle, 1) == 8
    cl.lib.pswim_set_fused(cl.handle, 0)
    cfg = StepperConfig(0.0, 1, 30)
    outs = [propagate(x, 0.0, 3e-5, cfg, sc, ctx=c) for c in (c16, c8, cl)]
    assert np.array_equal(outs[0], outs[1]) and np.array_equal(outs[0], outs[2])
    for c in (c16, c8, cl):
        c.close()


@pytest.mark.parametrize("kw,steps", [(dict(rod_count=1, nodes_per_rod=21), 4),      # fused cluster path
                                      (dict(rod_count=9, nodes_per_rod=64, epsilon=0.08), 40)])  # graph path
def test_propagate_rejects_image_wall(gpu, kw, steps):
    """image_wall throws in the reference (stokes.cpp:15-17) on every path, including the fused
    and graph-replay propagates that never reach rhs()."""
    from paper_2604_12083_b200 import PswimError
    from paper_2604_12083_b200.propagators import StepperConfig, propagate
    from paper_2604_12083_b200.scenario import build_initial_state

    sc = scen(wall_mode=1, **kw)
    x = build_initial_state(scen(**kw))
    with pytest.raises(PswimError) as ei:
        propagate(x, 0.0, steps * 1e-6, StepperConfig(0.0, 1, steps), sc)
    assert ei.value.code == 2
