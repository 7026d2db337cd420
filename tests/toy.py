"""Toy scalar ODE x' = lambda x propagators and the brute-force Parareal recurrence
(the reference's tests/test_parareal.cpp:15-65 fake physics), numpy."""
import numpy as np


def euler_toy(lam, steps):
    def f(t0, t1, x):
        dt = (t1 - t0) / steps
        y = np.array(x, dtype=np.float64, copy=True)
        for _ in range(steps):
            y = y + dt * lam * y
        return y

    return f


def rk2_toy(lam, steps):
    def f(t0, t1, x):
        dt = (t1 - t0) / steps
        y = np.array(x, dtype=np.float64, copy=True)
        for _ in range(steps):
            mid = y + 0.5 * dt * lam * y
            y = y + dt * lam * mid
        return y

    return f


def brute_force(plan, coarse, fine, x0, iterations):
    n = plan.intervals
    bt = plan.boundary_time
    x = [None] * (n + 1)
    g_old = [None] * (n + 1)
    x[0] = np.asarray(x0, dtype=np.float64)
    for i in range(1, n + 1):
        g_old[i] = coarse(bt(i - 1), bt(i), x[i - 1])
        x[i] = g_old[i]
    for k in range(1, iterations + 1):
        xp = [None] * (n + 1)
        for i in range(k, n + 1):
            xp[i] = fine(bt(i - 1), bt(i), x[i - 1])
        xn = list(x)
        if k <= n:
            xn[k] = xp[k]
        for i in range(k + 1, n + 1):
            g_new = coarse(bt(i - 1), bt(i), xn[i - 1])
            xn[i] = (xp[i] + g_new) - g_old[i]
            g_old[i] = g_new
        x = xn
    return x


def serial_fine(plan, fine, x0):
    ref = [np.asarray(x0, dtype=np.float64)]
    for i in range(1, plan.intervals + 1):
        ref.append(fine(plan.boundary_time(i - 1), plan.boundary_time(i), ref[i - 1]))
    return ref
