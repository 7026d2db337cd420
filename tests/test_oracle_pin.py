"""Pins the oracle (plain-C restatement) against the reference: bitwise against the
reference library itself when it is built here, and against the committed golden vectors
(generated from the reference by tests/golden/make_golden.py) everywhere."""
import numpy as np
import pytest

from oracle.pyoracle import Scenario


def test_oracle_vs_golden_mrs(oracle, golden):
    u, w = oracle.evaluate_velocities(golden["mrs12_nodes"], golden["mrs12_nodes"], golden["mrs12_f"],
                                      golden["mrs12_n"], 0.15, 2.3)
    assert np.array_equal(u, golden["mrs12_u"]) and np.array_equal(w, golden["mrs12_w"])
    x = golden["mrs1k_x"]
    u, w = oracle.evaluate_velocities(x, x, golden["mrs1k_f"], golden["mrs1k_n"], 0.1, 1.0)
    assert np.array_equal(u, golden["mrs1k_u"]) and np.array_equal(w, golden["mrs1k_w"])
    du, dw = oracle.dense_mobility_apply(golden["mrs12_nodes"], golden["mrs12_f"], golden["mrs12_n"], 0.15, 2.3)
    assert np.array_equal(du, golden["mrs12_dense_u"]) and np.array_equal(dw, golden["mrs12_dense_w"])
    # reference test bound: evaluator vs independent dense oracle < 1e-12 (test_stokes.cpp:118-135)
    scale = max(np.abs(du).max(), np.abs(dw).max())
    assert max(np.abs(golden["mrs12_u"] - du).max(), np.abs(golden["mrs12_w"] - dw).max()) / scale < 1e-12


def test_oracle_vs_golden_h_and_sqrt(oracle, golden):
    h = np.array([oracle.h_functions(r, 0.37) for r in golden["h_r"]])
    assert np.array_equal(h, golden["h_vals"])
    # H vs radial quadrature of the blob (test_stokes.cpp:34-47): rel < 1e-6
    assert np.max(np.abs(golden["h_vals"][1:6] - golden["h_quad"]) / np.abs(golden["h_quad"])) < 1e-6
    s = np.array([oracle.sqrt_rotation(m) for m in golden["sqrt_in"]])
    assert np.array_equal(s, golden["sqrt_out"])


def test_oracle_vs_golden_rod(oracle, golden):
    rod = golden["rod9_state"]
    fo, mo = oracle.internal_loads(rod, 1.0, golden["rod9_mat"], golden["rod9_wave"], 0.25)
    assert np.array_equal(fo, golden["rod9_seg_f"]) and np.array_equal(mo, golden["rod9_seg_n"])
    nf, nn = oracle.nodal_loads(rod, 1.0, fo, mo)
    assert np.array_equal(nf, golden["rod9_f"]) and np.array_equal(nn, golden["rod9_n"])
    e = oracle.elastic_energy(rod, 1.0, golden["rod9_mat"], golden["rod9_wave"], 0.25)
    assert e == golden["rod9_energy"][0]


def test_oracle_vs_golden_propagators(oracle, golden):
    desk = Scenario.make(rod_count=1, nodes_per_rod=21)
    x0 = oracle.build_initial_state(desk)
    assert np.array_equal(x0, golden["desk_x0"])
    u, w = oracle.rhs(desk, x0, 0.1)
    assert np.array_equal(u, golden["desk_rhs_u"]) and np.array_equal(w, golden["desk_rhs_w"])
    assert np.array_equal(oracle.propagate(desk, x0, 0.0, 0.0625, 1, steps=8), golden["desk_rk2_8"])
    assert np.array_equal(oracle.propagate(desk, x0, 0.0, 0.0625, 0, steps=8), golden["desk_euler_8"])
    lj = Scenario.make(rod_count=4, nodes_per_rod=21, placement=1, lj_well_depth=0.01, seed=2)
    xl = oracle.build_initial_state(lj)
    assert np.array_equal(xl, golden["lj_x0"])
    u, w = oracle.rhs(lj, xl, 0.05)
    assert np.array_equal(u, golden["lj_rhs_u"]) and np.array_equal(w, golden["lj_rhs_w"])
    r = oracle.resolve(lj)
    assert np.array_equal(oracle.lj_repulsion(xl, 4, 21, 0.01, r.lj_sigma, r.lj_self_exclusion), golden["lj_forces"])
    flag = Scenario.make(rod_count=1, nodes_per_rod=100)
    xf = oracle.build_initial_state(flag)
    assert np.array_equal(oracle.propagate(flag, xf, 0.0, 1e-3, 1, steps=100), golden["flag_rk2_100"])


def test_oracle_parareal_vs_golden(oracle, golden):
    """Brute-force Parareal recurrence == the reference's threaded engine, bitwise, l=1..4."""
    import ctypes as C

    sm = Scenario.make(rod_count=1, nodes_per_rod=11, horizon=1.0)
    xs = golden["par_x0"]
    for l in range(1, 5):
        states = np.zeros((5, xs.size))
        et = np.zeros(l)
        rc = oracle.parareal_rod_(C.byref(sm), 0.0, 1.0, 4, l, 50, 5, xs.ctypes.data_as(C.POINTER(C.c_double)),
                                  states.ctypes.data_as(C.POINTER(C.c_double)), et.ctypes.data_as(C.POINTER(C.c_double)), 1)
        assert rc == 0
        assert np.array_equal(states, golden[f"par_states_l{l}"])
        assert np.array_equal(et, golden[f"par_eta_tilde_l{l}"])
        # exactness: k iterations pin X[0..k] to the serial fine solution (test_parareal.cpp:192-212)
        for n in range(l + 1):
            assert np.array_equal(states[n], golden["par_serial_fine"][n])


def test_oracle_bitwise_vs_reference_library(oracle, ref):
    """The restatement reproduces the compiled reference bitwise on fresh random inputs."""
    rng = np.random.default_rng(0)
    t = rng.uniform(-1, 1, (300, 3))
    f, n = rng.uniform(-1, 1, (300, 3)), rng.uniform(-1, 1, (300, 3))
    a = oracle.evaluate_velocities(t, t, f, n, 0.05, 0.7)
    b = ref.evaluate_velocities(t, t, f, n, 0.05, 0.7)
    assert np.array_equal(a[0], b[0]) and np.array_equal(a[1], b[1])
    for _ in range(500):
        ax = rng.normal(size=3)
        ax /= np.linalg.norm(ax)
        th = rng.choice([rng.uniform(0, np.pi), rng.uniform(0, 1e-7), np.pi - rng.uniform(0, 1e-2)])
        R = ref.from_axis_angle(ax, th)
        assert np.array_equal(oracle.sqrt_rotation(R), ref.sqrt_rotation(R))
    for kw in (dict(rod_count=3, nodes_per_rod=17, placement=1, lj_well_depth=0.02, seed=9),
               dict(rod_count=4, nodes_per_rod=40, epsilon=0.08)):
        sc = Scenario.make(**kw)
        x = oracle.build_initial_state(sc)
        assert np.array_equal(x, ref.build_initial_state(sc))
        for scheme in (0, 1):
            assert np.array_equal(oracle.propagate(sc, x, 0.0, 5e-4, scheme, steps=5),
                                  ref.propagate(sc, x, 0.0, 5e-4, scheme, steps=5))


def test_oracle_errors(oracle):
    from oracle.pyoracle import OracleError

    t = np.zeros((2, 3))
    f = np.ones((2, 3))
    f[1, 0] = np.nan
    with pytest.raises(OracleError):
        oracle.evaluate_velocities(t, t, f, np.ones((2, 3)), 0.1, 1.0)
    with pytest.raises(OracleError):
        oracle.evaluate_velocities(t, t, np.ones((2, 3)), np.ones((2, 3)), 0.1, 1.0, wall=1)
    rod = np.zeros((4, 12))
    rod[:, 0] = [0, 1, 1, 2]
    rod[:, 3:6] = [0, 1, 0]
    rod[:, 6:9] = [0, 0, 1]
    rod[:, 9:12] = [1, 0, 0]
    with pytest.raises(OracleError):
        oracle.internal_loads(rod, 1.0, [1] * 6, [0, 0, 1], 0.0)
