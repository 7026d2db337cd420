"""Generates tests/golden/suspension.npz: BASELINE configs[2]/[3] end-to-end fixtures from the
UNMODIFIED reference library (oracle/_ref, reference proj/src compiled in place).

Run here (where /root/reference exists):   make -C oracle ref && python tests/golden/make_suspension.py

Scenario: 64 rods x 256 nodes, grid placement, epsilon = 0.08 (SURVEY 8(d) configs[2]-[4]; the
default 4 ds is not stable at dt = 1e-6), desk moduli, LJ off, dt = 1e-6.
  * serial fine: the reference's `propagate` (src/propagators.cpp:135-162), 100 RK2 steps;
  * serial fine boundaries: harness::serial_fine_boundaries (src/harness.cpp:35-37),
    n = 4 intervals x 20 RK2 steps;
  * Parareal: the reference's own parareal::run (src/parareal.cpp:430-438) over the
    harness::prepare propagators (fine RK2 x 20, coarse Euler x 2 per interval), n = 4,
    pipelined l = 1..4 and regular l = 2, tolerance 1e-300 (fixed l), eta against the serial
    fine boundaries.
A full state is 1.57 MB, so the fixture keeps, per state: positions of every 4th node
(4096 x 3), the per-rod sums of all 12 packed components (64 x 12; a checksum that still
compares at a relative tolerance), and the SHA-1 of the full packed state (bitwise pin of
the oracle restatement, which must reproduce the reference exactly).
"""
import ctypes as C
import hashlib
import os
import sys
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)

from oracle.pyoracle import Oracle, Scenario  # noqa: E402

RODS, NODES, EPS = 64, 256, 0.08
DT = 1e-6
N_INT, FINE, COARSE = 4, 20, 2
SERIAL_STEPS = 100
STRIDE = 4  # sampled nodes


def digest(state):
    s = np.ascontiguousarray(state, dtype=np.float64)
    return np.frombuffer(hashlib.sha1(s.tobytes()).digest(), dtype=np.uint8).copy()


def reduce(state):
    x = np.asarray(state).reshape(RODS * NODES, 12)
    return x[::STRIDE, 0:3].copy(), x.reshape(RODS, NODES, 12).sum(axis=1)


def put(g, key, state):
    g[key + "_pos"], g[key + "_rodsum"] = reduce(state)
    g[key + "_sha1"] = digest(state)


def main():
    ref = Oracle("ref")
    ref.set_threads_(os.cpu_count() or 1)
    sc = Scenario.make(rod_count=RODS, nodes_per_rod=NODES, epsilon=EPS)
    x0 = ref.build_initial_state(sc)
    g = {"x0_sha1": digest(x0), "meta": np.array([RODS, NODES, N_INT, FINE, COARSE, SERIAL_STEPS, STRIDE]),
         "params": np.array([EPS, DT])}
    t = time.time()
    serial = ref.propagate(sc, x0, 0.0, SERIAL_STEPS * DT, 1, steps=SERIAL_STEPS)
    put(g, "serial100", serial)
    print(f"serial {SERIAL_STEPS} RK2 steps: {time.time() - t:.1f} s", flush=True)

    horizon = N_INT * FINE * DT
    len_ = x0.size
    bounds = np.zeros((N_INT + 1, len_))
    t = time.time()
    rc = ref.serial_fine_boundaries_(C.byref(sc), 0.0, horizon, N_INT, FINE, x0.ctypes.data_as(C.POINTER(C.c_double)),
                                     bounds.ctypes.data_as(C.POINTER(C.c_double)))
    assert rc == 0
    for n in range(1, N_INT + 1):
        put(g, f"bounds_n{n}", bounds[n])
    print(f"serial fine boundaries: {time.time() - t:.1f} s", flush=True)

    runs = [(1, l) for l in (1, 2, 3, 4)] + [(0, 2)]
    for mode, l in runs:
        states = np.zeros((N_INT + 1, len_))
        et = np.zeros(N_INT)
        ea = np.zeros(N_INT)
        iters = np.zeros(1, dtype=np.int32)
        conv = np.zeros(1, dtype=np.int32)
        t = time.time()
        P = C.POINTER(C.c_double)
        rc = ref.parareal_rod_(C.byref(sc), 0.0, horizon, N_INT, 1, l, 1e-300, mode, FINE, COARSE,
                               x0.ctypes.data_as(P), bounds.ctypes.data_as(P), states.ctypes.data_as(P),
                               et.ctypes.data_as(P), ea.ctypes.data_as(P), iters.ctypes.data_as(C.POINTER(C.c_int)),
                               conv.ctypes.data_as(C.POINTER(C.c_int)), None)
        assert rc == 0, rc
        key = f"par_m{mode}_l{l}"
        for n in range(1, N_INT + 1):
            put(g, f"{key}_n{n}", states[n])
        g[key + "_eta_tilde"] = et[:iters[0]].copy()
        g[key + "_eta"] = ea[:iters[0]].copy()
        g[key + "_iters"] = np.array([iters[0], conv[0]])
        print(f"parareal mode {mode} l {l}: {time.time() - t:.1f} s, eta_tilde {et[:iters[0]]}, eta {ea[:iters[0]]}",
              flush=True)
    out = os.path.join(HERE, "suspension.npz")
    np.savez_compressed(out, **g)
    print(f"wrote {out}: {len(g)} arrays, {os.path.getsize(out)} bytes")


if __name__ == "__main__":
    main()
