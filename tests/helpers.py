"""Shared test helpers (numpy only)."""
import numpy as np


def perturbed_rod(oracle, m, length, rng, pj, aj):
    """Straight rod along +x with jittered positions and exactly-orthonormal rotated triads
    (the construction of the reference's tests/oracles.cpp:204-222, numpy RNG)."""
    ds = length / (m - 1)
    rod = np.zeros((m, 12))
    for k in range(m):
        rod[k, 0:3] = np.array([k * ds, 0.0, 0.0]) + rng.uniform(-pj * ds, pj * ds, 3)
        ax = rng.normal(size=3)
        ax /= np.linalg.norm(ax)
        q = oracle.from_axis_angle(ax, rng.uniform(0.0, aj))
        rod[k, 3:6] = q @ np.array([0.0, 1.0, 0.0])
        rod[k, 6:9] = q @ np.array([0.0, 0.0, 1.0])
        rod[k, 9:12] = q @ np.array([1.0, 0.0, 0.0])
    return rod


def raw_rodrigues(n, theta):
    c, s = np.cos(theta), np.sin(theta)
    k = np.array([[0, -n[2], n[1]], [n[2], 0, -n[0]], [-n[1], n[0], 0]])
    return c * np.eye(3) + (1 - c) * np.outer(n, n) + s * k


def rel_field_err(got, want):
    scale = max(np.abs(np.asarray(want[0])).max(), np.abs(np.asarray(want[1])).max(), 1e-300)
    return max(np.abs(np.asarray(got[0]) - want[0]).max(), np.abs(np.asarray(got[1]) - want[1]).max()) / scale
