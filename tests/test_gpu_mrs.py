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
    # far field approaches the singular kernels (test_stokes.cpp:49-60), < 1e-3
    eps = 0.2
    r = np.array([1e2, 1e3]) * eps
    hf = h_functions(r, eps)
    sing = np.stack([1 / (8 * np.pi * r), 1 / (8 * np.pi * r**3), 1 / (8 * np.pi * r**3), -1 / (16 * np.pi * r**3),
                     3 / (16 * np.pi * r**5)], axis=1)
    assert np.max(np.abs(hf - sing) / np.abs(sing)) < 1e-3


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


def test_mrs_linearity_permutation_curl(gpu):
    """test_stokes.cpp:154-206 and :279-302 on the GPU operator: linearity in the loads,
    source-permutation invariance (< 1e-12), and omega = curl(u)/2 by central differences
    (< 1e-4)."""
    from paper_2604_12083_b200.stokes import KernelParams, LoadSet, evaluate_velocities

    rng = np.random.default_rng(21)
    nodes = rng.uniform(-1, 1, (10, 3))
    kp = KernelParams(0.2, 1.0)
    la = (rng.uniform(-1, 1, (10, 3)), rng.uniform(-1, 1, (10, 3)))
    lb = (rng.uniform(-1, 1, (10, 3)), rng.uniform(-1, 1, (10, 3)))
    al, be = 0.7, -1.3
    combo = LoadSet(al * la[0] + be * lb[0], al * la[1] + be * lb[1])
    fa = evaluate_velocities(nodes, nodes, LoadSet(*la), kp)
    fb = evaluate_velocities(nodes, nodes, LoadSet(*lb), kp)
    fc = evaluate_velocities(nodes, nodes, combo, kp)
    scale = np.abs(fc.u).max()
    assert np.abs(fc.u - (al * fa.u + be * fb.u)).max() / scale < 1e-12
    assert np.abs(fc.omega - (al * fa.omega + be * fb.omega)).max() / scale < 1e-12

    src = rng.uniform(-1, 1, (15, 3))
    f, n = rng.uniform(-1, 1, (15, 3)), rng.uniform(-1, 1, (15, 3))
    tg = rng.uniform(-1, 1, (6, 3))
    kp = KernelParams(0.3, 1.0)
    base = evaluate_velocities(tg, src, LoadSet(f, n), kp)
    perm = rng.permutation(15)
    sh = evaluate_velocities(tg, src[perm], LoadSet(f[perm], n[perm]), kp)
    scale = np.abs(base.u).max()
    assert np.abs(base.u - sh.u).max() / scale < 1e-12 and np.abs(base.omega - sh.omega).max() / scale < 1e-12

    src = rng.uniform(-0.5, 0.5, (6, 3))
    f, n = rng.uniform(-1, 1, (6, 3)), rng.uniform(-1, 1, (6, 3))
    kp = KernelParams(0.2, 1.4)
    h = 1e-4 * kp.epsilon
    for _ in range(10):
        p = rng.uniform(-0.8, 0.8, 3)
        pts = np.array([p + h * e for e in np.eye(3)] + [p - h * e for e in np.eye(3)] + [p])
        v = evaluate_velocities(pts, src, LoadSet(f, n), kp)
        du = [(v.u[k] - v.u[3 + k]) / (2 * h) for k in range(3)]
        half_curl = 0.5 * np.array([du[1][2] - du[2][1], du[2][0] - du[0][2], du[0][1] - du[1][0]])
        w = v.omega[6]
        assert np.linalg.norm(w - half_curl) / np.linalg.norm(w) < 1e-4


def test_mrs_equals_grand_mobility_matvec(gpu, oracle):
    """test_stokes.cpp:237-276: the dense 6N x 6N mobility (reference assemble_grand_mobility,
    oracle restatement) applied to the loads equals the GPU operator (< 1e-12)."""
    from paper_2604_12083_b200.stokes import KernelParams, LoadSet, evaluate_velocities

    rng = np.random.default_rng(55)
    nodes = rng.uniform(-0.6, 0.6, (12, 3))
    f, n = rng.uniform(-1, 1, (12, 3)), rng.uniform(-1, 1, (12, 3))
    m = oracle.grand_mobility(nodes, 0.4, 1.9)
    x = np.concatenate([f, n], axis=1).reshape(-1)
    y = (m @ x).reshape(12, 6)
    got = evaluate_velocities(nodes, nodes, LoadSet(f, n), KernelParams(0.4, 1.9))
    scale = np.abs(got.u).max()
    assert np.abs(y[:, :3] - got.u).max() / scale < 1e-12
    assert np.abs(y[:, 3:] - got.omega).max() / scale < 1e-12


def test_mrs_golden_vectors(gpu, golden):
    """Reference golden outputs (tests/golden/golden.npz, generated from the reference)."""
    from paper_2604_12083_b200.stokes import KernelParams, LoadSet, evaluate_velocities

    x = golden["mrs1k_x"]
    got = evaluate_velocities(x, x, LoadSet(golden["mrs1k_f"], golden["mrs1k_n"]), KernelParams(0.1, 1.0))
    assert rel_err(got, (golden["mrs1k_u"], golden["mrs1k_w"])) < TOL
    nd = golden["mrs12_nodes"]
    got = evaluate_velocities(nd, nd, LoadSet(golden["mrs12_f"], golden["mrs12_n"]), KernelParams(0.15, 2.3))
    assert rel_err(got, (golden["mrs12_dense_u"], golden["mrs12_dense_w"])) < 1e-12


@pytest.mark.parametrize("n,nt", [(16384, None), (5000, 3001), (700, None), (300, 77)])
def test_mrs_host_entry_pinned_and_pageable(gpu, oracle, n, nt):
    """pswim_mrs_velocities_host (the e2e entry): outputs in page-locked memory are written by
    the kernel itself (mapped host memory), pageable ones are copied back; page-locked inputs
    go through the SM upload kernel (16-B and, for an 8-B-aligned view, scalar loads).
    Bitwise equal to the device-pointer entry on the same inputs, for pinned (aligned and
    not) and pageable host buffers, over repeated calls."""
    import ctypes as C

    import torch

    from paper_2604_12083_b200 import _lib
    from paper_2604_12083_b200.device import Context, dptr

    t, s, f, tq = rand_inputs(n, 900 + n, nt=nt)
    ctx = Context(0)
    L, kp, P = ctx.lib, _lib.KernelParams(0.1, 1.0, 0, 0), C.POINTER(C.c_double)
    m = len(t)
    d = [torch.as_tensor(a, device=gpu) for a in (t, s, f, tq)]
    du, dw = torch.empty_like(d[0]), torch.empty_like(d[0])
    ctx.after_torch()
    ctx.check(L.pswim_mrs_velocities(ctx.handle, dptr(d[0]), m, dptr(d[1]), dptr(d[2]), dptr(d[3]), n, C.byref(kp),
                                     dptr(du), dptr(dw)))
    ctx.sync()
    ref_u, ref_w = du.cpu().numpy(), dw.cpu().numpy()
    want = oracle.evaluate_velocities(t[:64], s, f, tq, 0.1, 1.0)
    assert rel_err((ref_u[:64], ref_w[:64]), want) < TOL

    def hp(a):
        return C.cast(a.data_ptr(), P) if isinstance(a, torch.Tensor) else a.ctypes.data_as(P)

    same = nt is None

    def pinned_view(a, off):
        # page-locked copy of `a` starting `off` doubles into its allocation (off = 1: 8-B
        # aligned only, the upload kernel's scalar path)
        buf = torch.empty(a.size + off, dtype=torch.float64).pin_memory()
        v = buf[off:].view(a.shape)
        v.copy_(torch.as_tensor(a))
        return v

    for pinned in (True, "unaligned", False):
        if pinned:
            off = 1 if pinned == "unaligned" else 0
            hs, hf, hn = (pinned_view(a, off) for a in (s, f, tq))
            ht = hs if same else pinned_view(t, off)
            hu, hw = torch.zeros((m, 3), dtype=torch.float64).pin_memory(), torch.zeros((m, 3), dtype=torch.float64).pin_memory()
        else:
            hs, hf, hn = (np.ascontiguousarray(a) for a in (s, f, tq))
            ht = hs if same else np.ascontiguousarray(t)
            hu, hw = np.zeros((m, 3)), np.zeros((m, 3))
        for _ in range(3):
            ctx.check(L.pswim_mrs_velocities_host(ctx.handle, hp(ht), m, hp(hs), hp(hf), hp(hn), n, C.byref(kp), hp(hu),
                                                  hp(hw)))
            gu = hu.numpy() if pinned else hu
            gw = hw.numpy() if pinned else hw
            assert np.array_equal(gu, ref_u) and np.array_equal(gw, ref_w)
            (hu.zero_() if pinned else hu.fill(0.0))
            (hw.zero_() if pinned else hw.fill(0.0))
        del hs, hf, hn, ht, hu, hw
    torch.cuda.synchronize()
    ctx.close()


def test_mrs_kernel_variants_bitwise(gpu):
    """The four all-pairs kernel variants (PSWIM_MRS_TPT = 1..4: one, two (2 and 3 CTAs/SM)
    and four targets per thread) run the same per-target operation sequence on the same
    chunk plan, so their outputs are bitwise identical (the variant is read once per
    process, hence one subprocess each)."""
    import subprocess
    import sys

    code = ("import hashlib, numpy as np, torch\n"
            "from paper_2604_12083_b200.stokes import KernelParams, LoadSet, evaluate_velocities\n"
            "rng = np.random.default_rng(5)\n"
            "for n in (300, 2053, 16384):\n"
            "    d = [torch.as_tensor(rng.uniform(-0.5, 0.5, (n, 3)), device='cuda') for _ in range(3)]\n"
            "    r = evaluate_velocities(d[0], d[0], LoadSet(d[1], d[2]), KernelParams(0.1, 1.0))\n"
            "    print(hashlib.sha1(r.u.cpu().numpy().tobytes() + r.omega.cpu().numpy().tobytes()).hexdigest())\n")
    import os

    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    outs = []
    for v in ("1", "2", "3", "4"):
        env = dict(os.environ, PSWIM_MRS_TPT=v)
        r = subprocess.run([sys.executable, "-c", code], capture_output=True, text=True, env=env, cwd=root,
                           timeout=600)
        assert r.returncode == 0, r.stderr[-2000:]
        outs.append(r.stdout.split())
    assert all(o == outs[0] for o in outs) and len(outs[0]) == 3, outs
