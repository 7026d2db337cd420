"""Generates tests/golden/golden.npz from the UNMODIFIED reference library.

Run here (where /root/reference exists):   make -C oracle ref && python tests/golden/make_golden.py

Every array comes from oracle/_ref/libpintswim_ref.so (reference proj/src + tests/oracles.cpp
compiled in place by oracle/Makefile), with inputs drawn exactly as the reference's own tests
draw them where a test is named (std::mt19937_64 seeds of test_stokes / test_rotation /
test_rod / acceptance).  The committed fixture pins the oracle restatement and the GPU path
on machines without the reference.
"""
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)

from oracle.pyoracle import Oracle, Scenario  # noqa: E402


def uniforms(ref, seed, count):
    return ref.random_draws(seed, 0, count, 0.0, 1.0)


def main():
    ref = Oracle("ref")
    g = {}
    # --- MRS: test_stokes.cpp:118-135 inputs (seed 42: 12 nodes at scale 0.8, then f,n per node)
    u = uniforms(ref, 42, 12 * 3 + 24 * 3)
    nodes = (-0.8 + 1.6 * u[:36]).reshape(12, 3)
    fl = np.zeros((12, 3))
    nl = np.zeros((12, 3))
    rest = u[36:]
    for i in range(12):
        fl[i] = -1.0 + 2.0 * rest[6 * i:6 * i + 3]
        nl[i] = -1.0 + 2.0 * rest[6 * i + 3:6 * i + 6]
    g["mrs12_nodes"], g["mrs12_f"], g["mrs12_n"] = nodes, fl, nl
    g["mrs12_u"], g["mrs12_w"] = ref.evaluate_velocities(nodes, nodes, fl, nl, 0.15, 2.3)
    g["mrs12_dense_u"], g["mrs12_dense_w"] = ref.dense_mobility_apply(nodes, fl, nl, 0.15, 2.3)
    # --- MRS: BASELINE config-2 style inputs (bench_kernels.cpp:46-63: mt19937_64(7), u - 0.5), N=1024
    n = 1024
    u = uniforms(ref, 7, 9 * n).reshape(n, 3, 3) - 0.5
    x, f, tq = u[:, 0], u[:, 1], u[:, 2]
    g["mrs1k_x"], g["mrs1k_f"], g["mrs1k_n"] = x, f, tq
    g["mrs1k_u"], g["mrs1k_w"] = ref.evaluate_velocities(x, x, f, tq, 0.1, 1.0, parallel=True)
    # --- h functions + quadrature oracle (test_stokes.cpp:34-47)
    rs = np.array([0.0, 0.0037, 0.185, 0.37, 0.74, 1.85, 37.0, 370.0])
    g["h_r"] = rs
    g["h_eps"] = np.array([0.37])
    g["h_vals"] = np.array([ref.h_functions(r, 0.37) for r in rs])
    g["h_quad"] = np.array([ref.h_quadrature(r, 0.37) for r in rs[1:6]])
    # --- sqrt_rotation over all branches (test_rotation.cpp:88-168 sampling)
    mats = []
    axes = ref.random_draws(2024, 1, 64)
    angles = ref.random_draws(5, 0, 64, 0.0, np.pi)
    for i in range(64):
        mats.append(ref.from_axis_angle(axes[i], angles[i]))
        mats.append(ref.from_axis_angle(axes[i], np.pi - 1e-3 * angles[i] / np.pi))
        mats.append(ref.from_axis_angle(axes[i], 1e-8 * angles[i]))
    for ax in np.eye(3):
        mats.append(ref.from_axis_angle(ax, np.pi))
    mats = np.array(mats)
    g["sqrt_in"] = mats
    g["sqrt_out"] = np.array([ref.sqrt_rotation(m) for m in mats])
    # --- rod loads on perturbed_rod (test_rod.cpp:126-155: seed 2023, M=9, jitters 0.08/0.25)
    rod = ref.perturbed_rod(9, 1.0, 2023, 0.08, 0.25)
    mat6 = np.array([0.8, 0.8, 1.2, 3.0, 3.0, 5.0])
    wave3 = np.array([0.2, 1.5, 1.0])
    fo, mo = ref.internal_loads(rod, 1.0, mat6, wave3, 0.25)
    nf, nn = ref.nodal_loads(rod, 1.0, fo, mo)
    g["rod9_state"], g["rod9_mat"], g["rod9_wave"] = rod, mat6, wave3
    g["rod9_seg_f"], g["rod9_seg_n"], g["rod9_f"], g["rod9_n"] = fo, mo, nf, nn
    g["rod9_energy"] = np.array([ref.elastic_energy(rod, 1.0, mat6, wave3, 0.25)])
    # --- scenario + rhs + propagate
    desk = Scenario.make(rod_count=1, nodes_per_rod=21)
    x0 = ref.build_initial_state(desk)
    g["desk_x0"] = x0
    g["desk_rhs_u"], g["desk_rhs_w"] = ref.rhs(desk, x0, 0.1)
    g["desk_rk2_8"] = ref.propagate(desk, x0, 0.0, 0.0625, 1, steps=8)
    g["desk_euler_8"] = ref.propagate(desk, x0, 0.0, 0.0625, 0, steps=8)
    lj = Scenario.make(rod_count=4, nodes_per_rod=21, placement=1, lj_well_depth=0.01, seed=2)
    xl = ref.build_initial_state(lj)
    g["lj_x0"] = xl
    g["lj_rhs_u"], g["lj_rhs_w"] = ref.rhs(lj, xl, 0.05)
    g["lj_forces"] = ref.lj_repulsion(xl, 4, 21, 0.01, ref.resolve(lj).lj_sigma, ref.resolve(lj).lj_self_exclusion)
    flag = Scenario.make(rod_count=1, nodes_per_rod=100)
    xf = ref.build_initial_state(flag)
    g["flag_x0"] = xf
    g["flag_rk2_100"] = ref.propagate(flag, xf, 0.0, 1e-3, 1, steps=100)
    # --- Parareal on a reduced desk run (acceptance_main.cpp:127-143 shape), fixed l
    sm = Scenario.make(rod_count=1, nodes_per_rod=11, horizon=1.0)
    xs = ref.build_initial_state(sm)
    nI, fine, coarse = 4, 50, 5
    states = np.zeros((nI + 1, xs.size))
    for l in range(1, nI + 1):
        et = np.zeros(nI)
        iters = np.zeros(1, dtype=np.int32)
        conv = np.zeros(1, dtype=np.int32)
        import ctypes as C

        rc = ref.parareal_rod_(C.byref(sm), 0.0, 1.0, nI, 2, l, 1e-300, 1, fine, coarse,
                               xs.ctypes.data_as(C.POINTER(C.c_double)), None,
                               states.ctypes.data_as(C.POINTER(C.c_double)),
                               et.ctypes.data_as(C.POINTER(C.c_double)), None,
                               iters.ctypes.data_as(C.POINTER(C.c_int)), conv.ctypes.data_as(C.POINTER(C.c_int)), None)
        assert rc == 0
        g[f"par_states_l{l}"] = states.copy()
        g[f"par_eta_tilde_l{l}"] = et[:l].copy()
    serial = np.zeros((nI + 1, xs.size))
    rc = ref.serial_fine_boundaries_(C.byref(sm), 0.0, 1.0, nI, fine, xs.ctypes.data_as(C.POINTER(C.c_double)),
                                     serial.ctypes.data_as(C.POINTER(C.c_double)))
    assert rc == 0
    g["par_x0"] = xs
    g["par_serial_fine"] = serial
    out = os.path.join(HERE, "golden.npz")
    np.savez_compressed(out, **g)
    print(f"wrote {out}: {len(g)} arrays, {os.path.getsize(out)} bytes")


if __name__ == "__main__":
    main()
