"""ctypes bindings of the oracle libraries — TEST INFRASTRUCTURE ONLY.

* ``Oracle("or")``  -> oracle/liboracle.so, the plain-C restatement (pswim_oracle.c)
* ``Oracle("ref")`` -> oracle/_ref/libpintswim_ref.so, the unmodified reference library
  (arxiv/paper_2604_12083 proj/src, built by oracle/Makefile) behind ref_shim.cpp

Both expose the same calls (prefix ``or_`` / ``ref_``), numpy in / numpy out.  Only
tests/, __graft_entry__.smoke() and bench.py's CPU-baseline legs import this module.
"""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATHS = {
    "or": os.path.join(HERE, "liboracle.so"),
    "ref": os.path.join(HERE, "_ref", "libpintswim_ref.so"),
}

_dp = C.POINTER(C.c_double)
_i64 = C.c_int64


class Scenario(C.Structure):
    """pswim_scenario (include/pswim_c.h) == ScenarioConfig (scenario.hpp:16-35)."""

    _fields_ = [
        ("rod_count", C.c_int64), ("nodes_per_rod", C.c_int64), ("rod_length", C.c_double),
        ("a1", C.c_double), ("a2", C.c_double), ("a3", C.c_double),
        ("b1", C.c_double), ("b2", C.c_double), ("b3", C.c_double),
        ("amplitude", C.c_double), ("frequency", C.c_double), ("wavelength", C.c_double),
        ("epsilon", C.c_double), ("mu", C.c_double), ("wall_mode", C.c_int32),
        ("placement", C.c_int32), ("lj_well_depth", C.c_double), ("lj_sigma", C.c_double),
        ("wall_clearance", C.c_double), ("seed", C.c_uint64), ("fine_dt", C.c_double),
        ("horizon", C.c_double),
    ]

    @classmethod
    def make(cls, **kw) -> "Scenario":
        s = cls()
        # ScenarioConfig defaults, scenario.hpp:16-35
        d = dict(rod_count=1, nodes_per_rod=51, rod_length=1.0, a1=0.01, a2=0.01, a3=0.01,
                 b1=2.0, b2=2.0, b3=2.0, amplitude=0.05, frequency=2.0 * np.pi, wavelength=1.0,
                 epsilon=0.0, mu=1.0, wall_mode=0, placement=0, lj_well_depth=0.0, lj_sigma=0.0,
                 wall_clearance=1.0, seed=1, fine_dt=1e-6, horizon=1e-3)
        d.update(kw)
        for k, v in d.items():
            setattr(s, k, v)
        return s

    def total_nodes(self) -> int:
        return int(self.rod_count * self.nodes_per_rod)


class Resolved(C.Structure):
    _fields_ = [("ds", C.c_double), ("epsilon", C.c_double), ("mu", C.c_double),
                ("lj_sigma", C.c_double), ("lj_cutoff", C.c_double),
                ("lj_self_exclusion", C.c_int64), ("total_nodes", C.c_int64)]


class OracleError(RuntimeError):
    def __init__(self, code: int, what: str):
        super().__init__(f"{what}: code {code}")
        self.code = code


def _p(a: np.ndarray):
    return a.ctypes.data_as(_dp)


def _f64(a, shape=None) -> np.ndarray:
    a = np.ascontiguousarray(np.asarray(a, dtype=np.float64))
    if shape is not None:
        a = a.reshape(shape)
    return a


class Oracle:
    def __init__(self, kind: str = "or"):
        path = LIB_PATHS[kind]
        if not os.path.exists(path):
            raise FileNotFoundError(f"{path} missing: run `make -C oracle {'ref' if kind == 'ref' else 'liboracle'}`")
        self.kind = kind
        self.pre = "or_" if kind == "or" else "ref_"
        self.lib = C.CDLL(path)
        self._sig()

    def _fn(self, name, restype, argtypes):
        f = getattr(self.lib, self.pre + name)
        f.restype = restype
        f.argtypes = argtypes
        return f

    def _sig(self):
        S = C.POINTER(Scenario)
        self.h_functions_ = self._fn("h_functions", None, [C.c_double, C.c_double, _dp])
        ev_args = [_dp, _i64, _dp, _dp, _dp, _i64, C.c_double, C.c_double, C.c_int, _dp, _dp]
        if self.kind == "ref":
            ev_args = ev_args + [C.c_int]
        self.evaluate_velocities_ = self._fn("evaluate_velocities", C.c_int, ev_args)
        self.grand_mobility_ = self._fn("grand_mobility", C.c_int, [_dp, _i64, C.c_double, C.c_double, _dp])
        self.from_axis_angle_ = self._fn("from_axis_angle", C.c_int, [_dp, C.c_double, _dp])
        self.to_axis_angle_ = self._fn("to_axis_angle", None, [_dp, _dp, _dp])
        self.sqrt_rotation_ = self._fn("sqrt_rotation", None, [_dp, _dp])
        self.rotation_residual_ = self._fn("rotation_residual", C.c_double, [_dp])
        self.internal_loads_ = self._fn("internal_loads", C.c_int, [_dp, _i64, C.c_double, _dp, _dp, C.c_double, _dp, _dp])
        self.nodal_loads_ = self._fn("nodal_loads", C.c_int, [_dp, _i64, C.c_double, _dp, _dp, _dp, _dp])
        self.lj_repulsion_ = self._fn("lj_repulsion", None, [_dp, _i64, _i64, C.c_double, C.c_double, _i64, _dp])
        self.reorthonormalize_ = self._fn("reorthonormalize", _i64, [_dp, _i64, C.c_double])
        self.resolve_ = self._fn("resolve", C.c_int, [S, C.POINTER(Resolved)])
        self.build_initial_state_ = self._fn("build_initial_state", C.c_int, [S, _dp])
        rhs_args = [S, _dp, C.c_double, _dp, _dp, _dp, _dp]
        step_args = [S, C.c_int, _dp, C.c_double, C.c_double, _dp]
        prop_args = [S, _dp, C.c_double, C.c_double, C.c_int, _i64, C.c_double, _dp]
        if self.kind == "or":
            rhs_args = rhs_args + [C.c_int]
            step_args = step_args + [C.c_int]
            prop_args = prop_args + [C.c_int]
        self.rhs_ = self._fn("rhs", C.c_int, rhs_args)
        self.advance_state_ = self._fn("advance_state", C.c_int, [S, _dp, _dp, _dp, C.c_double, _dp])
        self.step_ = self._fn("step", C.c_int, step_args)
        self.propagate_ = self._fn("propagate", C.c_int, prop_args)
        self.position_metric_ = self._fn("position_metric", C.c_double, [_dp, _dp, _i64])
        self.pointwise_metric_ = self._fn("pointwise_metric", C.c_double, [_dp, _dp, _i64, _i64])
        self.dense_mobility_apply_ = self._fn("dense_mobility_apply", None,
                                              [_dp, _i64, _dp, _dp, C.c_double, C.c_double, _dp, _dp])
        self.elastic_energy_ = self._fn("elastic_energy", C.c_double, [_dp, _i64, C.c_double, _dp, _dp, C.c_double])
        if self.kind == "or":
            self.evaluate_rows_ = self._fn("evaluate_velocities_rows", C.c_int,
                                           [_dp, _i64, _i64, _dp, _dp, _dp, _i64, C.c_double, C.c_double, _dp, _dp, C.c_int])
            self.parareal_rod_ = self._fn("parareal_rod", C.c_int,
                                          [S, C.c_double, C.c_double, C.c_int, C.c_int, _i64, _i64, _dp, _dp, _dp, C.c_int])
        else:
            self.set_threads_ = self._fn("set_threads", None, [C.c_int])
            self.max_threads_ = self._fn("max_threads", C.c_int, [])
            self.random_draws_ = self._fn("random_draws", None, [C.c_uint64, C.c_int, C.c_double, C.c_double, _i64, _dp])
            self.perturbed_rod_ = self._fn("perturbed_rod", None, [_i64, C.c_double, C.c_uint64, C.c_double, C.c_double, _dp])
            self.h_quadrature_ = self._fn("h_quadrature", None, [C.c_double, C.c_double, _dp])
            self.parareal_rod_ = self._fn("parareal_rod", C.c_int,
                                          [S, C.c_double, C.c_double, C.c_int, C.c_int, C.c_int, C.c_double, C.c_int,
                                           _i64, _i64, _dp, _dp, _dp, _dp, _dp, C.POINTER(C.c_int),
                                           C.POINTER(C.c_int), _dp])
            self.serial_fine_boundaries_ = self._fn("serial_fine_boundaries", C.c_int,
                                                    [S, C.c_double, C.c_double, C.c_int, _i64, _dp, _dp])

    @staticmethod
    def _check(rc, what):
        if rc:
            raise OracleError(rc, what)

    # ---- stokes ----
    def h_functions(self, r, eps):
        h = np.zeros(5)
        self.h_functions_(float(r), float(eps), _p(h))
        return h

    def evaluate_velocities(self, tgt, src, f, n, eps, mu, wall=0, parallel=False):
        tgt, src, f, n = (_f64(a, (-1, 3)) for a in (tgt, src, f, n))
        u = np.zeros_like(tgt)
        w = np.zeros_like(tgt)
        args = [_p(tgt), len(tgt), _p(src), _p(f), _p(n), len(src), float(eps), float(mu), int(wall), _p(u), _p(w)]
        if self.kind == "ref":
            args.append(1 if parallel else 0)
        self._check(self.evaluate_velocities_(*args), "evaluate_velocities")
        return u, w

    def evaluate_rows(self, tgt, t0, t1, src, f, n, eps, mu, threads=1):
        tgt, src, f, n = (_f64(a, (-1, 3)) for a in (tgt, src, f, n))
        u = np.zeros_like(tgt)
        w = np.zeros_like(tgt)
        self.evaluate_rows_(_p(tgt), t0, t1, _p(src), _p(f), _p(n), len(src), eps, mu, _p(u), _p(w), threads)
        return u[t0:t1], w[t0:t1]

    def grand_mobility(self, nodes, eps, mu):
        nodes = _f64(nodes, (-1, 3))
        m = np.zeros((6 * len(nodes), 6 * len(nodes)))
        self._check(self.grand_mobility_(_p(nodes), len(nodes), eps, mu, _p(m)), "grand_mobility")
        return m

    # ---- rotation ----
    def from_axis_angle(self, axis, angle):
        axis = _f64(axis, (3,))
        r = np.zeros(9)
        self._check(self.from_axis_angle_(_p(axis), float(angle), _p(r)), "from_axis_angle")
        return r.reshape(3, 3)

    def to_axis_angle(self, r):
        r = _f64(r, (9,))
        axis = np.zeros(3)
        ang = np.zeros(1)
        self.to_axis_angle_(_p(r), _p(axis), _p(ang))
        return axis, float(ang[0])

    def sqrt_rotation(self, r):
        r = _f64(r, (9,))
        s = np.zeros(9)
        self.sqrt_rotation_(_p(r), _p(s))
        return s.reshape(3, 3)

    def rotation_residual(self, r):
        return float(self.rotation_residual_(_p(_f64(r, (9,)))))

    # ---- rod ----
    def internal_loads(self, rod12, length, mat6, wave3, t):
        rod12 = _f64(rod12, (-1, 12))
        m = len(rod12)
        fo = np.zeros((m - 1, 3))
        mo = np.zeros((m - 1, 3))
        self._check(self.internal_loads_(_p(rod12), m, length, _p(_f64(mat6)), _p(_f64(wave3)), t, _p(fo), _p(mo)),
                    "internal_loads")
        return fo, mo

    def nodal_loads(self, rod12, length, force, moment):
        rod12 = _f64(rod12, (-1, 12))
        m = len(rod12)
        f = np.zeros((m, 3))
        n = np.zeros((m, 3))
        self._check(self.nodal_loads_(_p(rod12), m, length, _p(_f64(force, (-1, 3))), _p(_f64(moment, (-1, 3))),
                                      _p(f), _p(n)), "nodal_loads")
        return f, n

    def lj_repulsion(self, state12, rods, m, well, sigma, excl):
        state12 = _f64(state12)
        out = np.zeros((rods * m, 3))
        self.lj_repulsion_(_p(state12), rods, m, well, sigma, excl, _p(out))
        return out

    def reorthonormalize(self, rod12, tol=1e-9):
        rod12 = _f64(rod12, (-1, 12)).copy()
        touched = self.reorthonormalize_(_p(rod12), len(rod12), tol)
        return rod12, int(touched)

    # ---- scenario / propagators ----
    def resolve(self, sc):
        r = Resolved()
        self._check(self.resolve_(C.byref(sc), C.byref(r)), "resolve")
        return r

    def build_initial_state(self, sc):
        out = np.zeros(12 * sc.total_nodes())
        self._check(self.build_initial_state_(C.byref(sc), _p(out)), "build_initial_state")
        return out

    def rhs(self, sc, state, t, extra_f=None, extra_n=None, threads=1):
        state = _f64(state)
        n = sc.total_nodes()
        u = np.zeros((n, 3))
        w = np.zeros((n, 3))
        ef = _p(_f64(extra_f)) if extra_f is not None else None
        en = _p(_f64(extra_n)) if extra_n is not None else None
        args = [C.byref(sc), _p(state), t, ef, en, _p(u), _p(w)]
        if self.kind == "or":
            args.append(threads)
        self._check(self.rhs_(*args), "rhs")
        return u, w

    def advance_state(self, sc, state, u, w, dt):
        state = _f64(state)
        out = np.zeros_like(state)
        self._check(self.advance_state_(C.byref(sc), _p(state), _p(_f64(u)), _p(_f64(w)), dt, _p(out)),
                    "advance_state")
        return out

    def step(self, sc, scheme, state, t, dt, threads=1):
        state = _f64(state)
        out = np.zeros_like(state)
        args = [C.byref(sc), scheme, _p(state), t, dt, _p(out)]
        if self.kind == "or":
            args.append(threads)
        self._check(self.step_(*args), "step")
        return out

    def propagate(self, sc, state, t0, t1, scheme, steps=0, dt=0.0, threads=1):
        state = _f64(state)
        out = np.zeros_like(state)
        args = [C.byref(sc), _p(state), t0, t1, scheme, steps, dt, _p(out)]
        if self.kind == "or":
            args.append(threads)
        self._check(self.propagate_(*args), "propagate")
        return out

    def position_metric(self, x, y):
        x = _f64(x)
        y = _f64(y)
        return float(self.position_metric_(_p(x), _p(y), len(x)))

    def pointwise_metric(self, x, y, dim):
        x = _f64(x)
        y = _f64(y)
        return float(self.pointwise_metric_(_p(x), _p(y), len(x), dim))

    def dense_mobility_apply(self, nodes, f, n, eps, mu):
        nodes, f, n = (_f64(a, (-1, 3)) for a in (nodes, f, n))
        u = np.zeros_like(nodes)
        w = np.zeros_like(nodes)
        self.dense_mobility_apply_(_p(nodes), len(nodes), _p(f), _p(n), eps, mu, _p(u), _p(w))
        return u, w

    def elastic_energy(self, rod12, length, mat6, wave3, t):
        rod12 = _f64(rod12, (-1, 12))
        return float(self.elastic_energy_(_p(rod12), len(rod12), length, _p(_f64(mat6)), _p(_f64(wave3)), t))

    # ---- ref-only helpers ----
    def random_draws(self, seed, kind, count, lo=0.0, hi=1.0):
        out = np.zeros(count * (1 if kind == 0 else 3))
        self.random_draws_(seed, kind, lo, hi, count, _p(out))
        return out if kind == 0 else out.reshape(count, 3)

    def perturbed_rod(self, m, length, seed, pj, aj):
        out = np.zeros((m, 12))
        self.perturbed_rod_(m, length, seed, pj, aj, _p(out))
        return out

    def h_quadrature(self, r, eps):
        h = np.zeros(5)
        self.h_quadrature_(float(r), float(eps), _p(h))
        return h
