"""CPU check of the algebra the MRS kernel uses (mrs.cu): H kernels on powers of Q^-1/2,
1/(8 pi mu) folded into the loads, and the rotlet identity
sum h3 n x (t - s) = (sum h3 n) x t - sum h3 (n x s) in block-origin coordinates.
A numpy emulation of the kernel's per-pair formulas must match the oracle to 1e-12."""
import numpy as np


def emulate(t, s, f, n, eps, mu):
    e2 = eps * eps
    scale = (1.0 / (8.0 * np.pi)) / mu
    o = t[0]
    tp, sp = t - o, s - o
    fp, nq = f * scale, n * scale
    mf, mn = np.cross(fp, sp), np.cross(nq, sp)
    r = tp[:, None, :] - sp[None, :, :]
    q = (r * r).sum(-1) + e2
    y = 1.0 / np.sqrt(q)
    y2 = y * y
    y3 = y * y2
    y5 = y3 * y2
    y7 = y5 * y2
    h1 = e2 * y3 + y
    h3 = 1.5 * e2 * y5 + y3
    g4 = -7.5 * e2 * e2 * y7 + h3          # H4 = -g4 / 2
    g5 = 2.5 * e2 * y7 + y5                # H5 = 3 g5 / 2
    fr = (fp[None] * r).sum(-1)
    n3r = ((-3.0 * nq)[None] * r).sum(-1)  # staged n3 = -3 n'
    u = (h1[..., None] * fp[None]).sum(1) + ((y3 * fr)[..., None] * r).sum(1)
    w = -0.5 * ((g4[..., None] * nq[None]).sum(1) + ((g5 * n3r)[..., None] * r).sum(1))
    an, bn = h3 @ nq, h3 @ mn
    af, bf = h3 @ fp, h3 @ mf
    u += np.cross(an, tp) - bn
    w += np.cross(af, tp) - bf
    return u, w


def test_kernel_algebra_matches_oracle(oracle):
    rng = np.random.default_rng(3)
    for n_, eps, mu, spread in [(64, 0.1, 1.0, 0.5), (200, 0.04, 2.3, 3.0), (50, 0.3, 0.7, 20.0)]:
        s = rng.uniform(-spread, spread, (n_, 3))
        f = rng.uniform(-1, 1, (n_, 3))
        tq = rng.uniform(-1, 1, (n_, 3))
        got = emulate(s, s, f, tq, eps, mu)
        want = oracle.evaluate_velocities(s, s, f, tq, eps, mu)
        scale = max(np.abs(want[0]).max(), np.abs(want[1]).max())
        err = max(np.abs(got[0] - want[0]).max(), np.abs(got[1] - want[1]).max()) / scale
        assert err < 1e-12, err
