"""GPU parity of the MRS kernel against the oracle (reference stokes.cpp semantics).

Tolerance: 1e-10 relative to the max |u|,|omega| over targets (BASELINE.json north_star);
observed ~1e-14.  Determinism: bitwise-identical repeated runs (fixed-order reduction).
"""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu
TOL = 1e-10


def rel_err(got, want):
    scale = max(np.abs(want[0]).max(), np.abs(want[1]).max(), 1e-300)
    return max(np.abs(got[0] - want[0]).max(), np.abs(got[1] - want[1]).max()) / scale


def rand_inputs(n, seed, scale=0.5, nt=None):
    rng = np.random.default_rng(seed)
    s = rng.uniform(-scale, scale, (n, 3))
    f = rng.uniform(-0.5, 0.5, (n, 3))
    tq = rng.uniform(-0.5, 0.5, (n, 3))
    t = s if nt is None else rng.uniform(-scale, scale, (nt, 3))
    return t, s, f, tq


@pytest.mark.parametrize("n", [1, 7, 100, 255, 256, 257, 1000, 2053])
def test_mrs_matches_oracle(gpu, oracle, n):
    from paper_2604_12083_b200.stokes import KernelParams, LoadSet, evaluate_velocities

    t, s, f, tq = rand_inputs(n, 100 + n)
    got = evaluate_velocities(t, s, LoadSet(f, tq), KernelParams(0.1, 1.3))
    want = oracle.evaluate_velocities(t, s, f, tq, 0.1, 1.3)
    assert rel_err(got, want) < TOL


def test_mrs_rectangular_and_device_path(gpu, oracle):
    import torch
    from paper_2604_12083_b200.stokes import KernelParams, LoadSet, evaluate_velocities

    t, s, f, tq = rand_inputs(3001, 5, nt=517)
    want = oracle.evaluate_velocities(t, s, f, tq, 0.07, 0.9)
    d = [torch.as_tensor(a, device=gpu) for a in (t, s, f, tq)]
    got = evaluate_velocities(d[0], d[1], LoadSet(d[2], d[3]), KernelParams(0.07, 0.9))
    assert rel_err((got.u.cpu().numpy(), got.omega.cpu().numpy()), want) < TOL


def test_mrs_16k_rows_vs_oracle_and_bitwise_repeat(gpu, oracle):
    """BASELINE config 2 inputs (N=16384, eps=0.1, mu=1), rows checked against the oracle."""
    import torch
    from paper_2604_12083_b200.stokes import KernelParams, LoadSet, evaluate_velocities

    t, s, f, tq = rand_inputs(16384, 7)
    d = [torch.as_tensor(a, device=gpu) for a in (t, s, f, tq)]
    a = evaluate_velocities(d[0], d[1], LoadSet(d[2], d[3]), KernelParams(0.1, 1.0))
    b = evaluate_velocities(d[0], d[1], LoadSet(d[2], d[3]), KernelParams(0.1, 1.0))
    assert torch.equal(a.u, b.u) and torch.equal(a.omega, b.omega)
    rows = np.r_[0:64, 8000:8064, 16320:16384]
    ou, ow = oracle.evaluate_velocities(t[rows], s, f, tq, 0.1, 1.0)
    gu, gw = a.u.cpu().numpy()[rows], a.omega.cpu().numpy()[rows]
    assert rel_err((gu, gw), (ou, ow)) < TOL


def test_mrs_known_answers(gpu, oracle):
    from paper_2604_12083_b200.stokes import KernelParams, LoadSet, evaluate_velocities, h_functions

    # zero loads -> zero field (test_stokes.cpp:82-88)
    t, s, f, tq = rand_inputs(8, 3)
    z = evaluate_velocities(t, s, LoadSet(np.zeros((8, 3)), np.zeros((8, 3))), KernelParams(0.25, 1.7))
    assert np.all(z.u == 0.0) and np.all(z.omega == 0.0)
    # origin isotropy: u = f H1(0)/mu, omega = 0 (test_stokes.cpp:62-77)
    node = np.array([[0.5, -0.2, 1.0]])
    fl = np.array([[1.0, 2.0, -0.5]])
    fld = evaluate_velocities(node, node, LoadSet(fl, np.zeros((1, 3))), KernelParams(0.8, 3.0))
    h0 = oracle.h_functions(0.0, 0.8)
    assert np.linalg.norm(fld.u[0] - fl[0] * (h0[0] / 3.0)) < 1e-15
    assert np.linalg.norm(fld.omega[0]) < 1e-15
    # mirror symmetry (test_stokes.cpp:90-99)
    m = evaluate_velocities(np.zeros((1, 3)), np.array([[0, 0, 1.0], [0, 0, -1.0]]),
                            LoadSet(np.array([[1.0, 0.5, 0.3], [1.0, 0.5, -0.3]]), np.zeros((2, 3))),
                            KernelParams(0.25, 1.7))
    assert abs(m.u[0, 2]) < 1e-16
    # h_functions device twin equals the oracle
    r = np.array([0.0, 1e-3, 0.37, 1.0, 5.0, 1e3])
    hd = h_functions(r, 0.37)
    ho = np.array([oracle.h_functions(x, 0.37) for x in r])
    assert np.max(np.abs(hd - ho) / np.abs(ho)) < 1e-14


def test_mrs_dense_oracle_n12(gpu, oracle):
    """Independent dense-oracle equivalence at N=12 (test_stokes.cpp:118-135), <1e-12."""
    from paper_2604_12083_b200.stokes import KernelParams, LoadSet, evaluate_velocities

    rng = np.random.default_rng(42)
    nodes = rng.uniform(-0.8, 0.8, (12, 3))
    f = rng.uniform(-1, 1, (12, 3))
    tq = rng.uniform(-1, 1, (12, 3))
    got = evaluate_velocities(nodes, nodes, LoadSet(f, tq), KernelParams(0.15, 2.3))
    want = oracle.dense_mobility_apply(nodes, f, tq, 0.15, 2.3)
    assert rel_err(got, want) < 1e-12


def test_mrs_errors(gpu):
    from paper_2604_12083_b200 import InvalidArgument, PswimError
    from paper_2604_12083_b200.stokes import KernelParams, LoadSet, evaluate_velocities

    t, s, f, tq = rand_inputs(8, 3)
    bad = f.copy()
    bad[3, 1] = np.inf
    with pytest.raises(InvalidArgument):
        evaluate_velocities(t, s, LoadSet(bad, tq), KernelParams(0.25, 1.7))
    with pytest.raises(PswimError):
        evaluate_velocities(t, s, LoadSet(f, tq), KernelParams(0.25, 1.7, wall_mode=1))
    with pytest.raises(InvalidArgument):
        evaluate_velocities(t, s, LoadSet(f, tq), KernelParams(0.0, 1.7))
    with pytest.raises(InvalidArgument):
        evaluate_velocities(t, s, LoadSet(f[:5], tq), KernelParams(0.1, 1.0))
    # the error is cleared: a valid call afterwards succeeds
    evaluate_velocities(t, s, LoadSet(f, tq), KernelParams(0.25, 1.7))


def test_mrs_empty(gpu):
    from paper_2604_12083_b200.stokes import KernelParams, LoadSet, evaluate_velocities

    e = evaluate_velocities(np.zeros((0, 3)), np.ones((4, 3)), LoadSet(np.ones((4, 3)), np.ones((4, 3))), KernelParams())
    assert e.u.shape == (0, 3)
    z = evaluate_velocities(np.ones((4, 3)), np.zeros((0, 3)), LoadSet(np.zeros((0, 3)), np.zeros((0, 3))), KernelParams())
    assert np.all(z.u == 0.0)
