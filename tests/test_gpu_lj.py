"""Cell-list LJ: the hashed cell-list pair search (lj_cells.cu) against the
all-pairs kernel and the reference restatement of lj_repulsion (src/rod.cpp:124-174), on
suspensions large enough for the cell list (N >= 2048) with many pairs inside the cutoff."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _suspension(noise, shift=0.0, rods=40, m=64, seed=5):
    from paper_2604_12083_b200.scenario import RANDOM, ScenarioConfig, build_initial_state, make_scenario

    sc = make_scenario(ScenarioConfig(rod_count=rods, nodes_per_rod=m, placement=RANDOM, lj_well_depth=0.01,
                                      seed=seed))
    x = build_initial_state(sc).reshape(-1, 12)
    rng = np.random.default_rng(seed)
    x[:, 0:3] += rng.normal(scale=noise, size=(len(x), 3)) + shift
    return sc, x.reshape(-1)


def _forces(ctx, x, mode):
    import torch

    from paper_2604_12083_b200.device import dptr

    ctx.lib.pswim_set_lj_mode(ctx.handle, mode)
    dx = torch.as_tensor(x, device="cuda:0")
    out = torch.empty((dx.numel() // 12, 3), dtype=torch.float64, device="cuda:0")
    ctx.after_torch()
    ctx.check(ctx.lib.pswim_lj_forces(ctx.handle, dptr(dx), dptr(out)))
    ctx.sync()
    return out.cpu().numpy()


@pytest.mark.parametrize("noise,shift", [(0.08, 0.0), (0.15, 0.0), (0.08, 12345.5), (0.08, -3.0e4)])
def test_cell_list_matches_all_pairs_and_oracle(gpu, oracle, noise, shift):
    from paper_2604_12083_b200.device import Context

    sc, x = _suspension(noise, shift)
    ctx = Context(0, sc)
    cells = _forces(ctx, x, 2)
    pairs = _forces(ctx, x, 1)
    want = oracle.lj_repulsion(x, 40, 64, 0.01, sc.lj_sigma, sc.lj_self_exclusion)
    scale = np.abs(want).max()
    assert scale > 0 and np.count_nonzero(np.abs(want).sum(1)) > 100  # many interacting nodes
    assert np.max(np.abs(cells - pairs)) <= 1e-13 * scale
    assert np.max(np.abs(cells - want)) <= 1e-12 * scale
    # auto mode picks the cell list at this size; repeat runs are bitwise identical
    again = _forces(ctx, x, 0)
    assert np.array_equal(again, cells)
    ctx.close()


def test_cell_list_near_collisions_and_coincident_nodes(gpu, oracle):
    """Pairs closer than the clamp radius and exactly coincident nodes of different rods
    (rod.cpp:155-160: dir = (1,0,0) for r = 0, the sign fixed by pair order)."""
    from paper_2604_12083_b200.device import Context

    sc, x = _suspension(0.08)
    xs = x.reshape(-1, 12)
    xs[64 * 7 + 10, 0:3] = xs[64 * 3 + 20, 0:3]  # coincident (rods 3 and 7)
    xs[64 * 9 + 5, 0:3] = xs[64 * 11 + 40, 0:3] + 1e-6 * sc.lj_sigma  # inside r_min
    x = xs.reshape(-1)
    ctx = Context(0, sc)
    cells = _forces(ctx, x, 2)
    pairs = _forces(ctx, x, 1)
    want = oracle.lj_repulsion(x, 40, 64, 0.01, sc.lj_sigma, sc.lj_self_exclusion)
    scale = np.abs(want).max()
    assert np.max(np.abs(cells - want)) <= 1e-12 * scale
    assert np.max(np.abs(cells - pairs)) <= 1e-13 * scale
    ctx.close()


def test_rhs_with_cell_list_lj_matches_oracle(gpu, oracle):
    """rhs (propagators.cpp:38-91) with LJ active at N = 2560: the GPU rhs through the cell
    list against the reference restatement's rhs."""
    import torch

    from oracle.pyoracle import Scenario as OS
    from paper_2604_12083_b200.device import Context
    from paper_2604_12083_b200.propagators import rhs

    sc, x = _suspension(0.08)
    ctx = Context(0, sc)
    ctx.lib.pswim_set_lj_mode(ctx.handle, 2)
    vel = rhs(torch.as_tensor(x, device="cuda:0"), 0.01, sc, ctx=ctx)
    u, w = vel.u.cpu().numpy(), vel.omega.cpu().numpy()
    osc = OS.make(rod_count=40, nodes_per_rod=64, placement=1, lj_well_depth=0.01, seed=5)
    ou, ow = oracle.rhs(osc, x, 0.01, threads=8)
    scale = max(np.abs(ou).max(), np.abs(ow).max())
    assert max(np.abs(u - ou).max(), np.abs(w - ow).max()) <= 1e-10 * scale
    ctx.close()


@pytest.mark.parametrize("squeeze", [0.02, 0.002])
def test_cell_list_crowded_buckets(gpu, oracle, squeeze):
    """Crowded cells: the suspension squeezed towards its centre so that buckets hold tens to
    hundreds of nodes -- the per-bucket sort's warp network (<= 128 members) and its in-place
    fallback (> 128) -- against the all-pairs kernel, the oracle, and a bitwise repeat."""
    from paper_2604_12083_b200.device import Context

    sc, x = _suspension(0.02)
    xs = x.reshape(-1, 12)
    c = xs[:, 0:3].mean(axis=0)
    xs[:, 0:3] = c + squeeze * (xs[:, 0:3] - c)
    x = xs.reshape(-1)
    rc = 2.0 ** (1.0 / 6.0) * sc.lj_sigma
    cell = np.floor(xs[:, 0:3] / rc).astype(np.int64)
    _, counts = np.unique(cell, axis=0, return_counts=True)
    assert counts.max() > (16 if squeeze > 0.01 else 128)
    ctx = Context(0, sc)
    cells = _forces(ctx, x, 2)
    pairs = _forces(ctx, x, 1)
    want = oracle.lj_repulsion(x, 40, 64, 0.01, sc.lj_sigma, sc.lj_self_exclusion)
    scale = np.abs(want).max()
    assert scale > 0
    assert np.max(np.abs(cells - pairs)) <= 1e-12 * scale
    assert np.max(np.abs(cells - want)) <= 1e-12 * scale
    assert np.array_equal(_forces(ctx, x, 2), cells)
    ctx.close()
