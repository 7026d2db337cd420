"""Where the e2e (host-buffer C-ABI) MRS time goes at N = 16384 (dev tool).

Times, on one B200: the whole pswim_mrs_velocities_host call (wall, as bench.py), the same
with no L2 flush, the pieces on the device (H2D copies, kernel, D2H copies) with CUDA events,
and the host overhead of a tiny call."""
import ctypes as C
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

from paper_2604_12083_b200 import _lib
from paper_2604_12083_b200.device import Context, dptr

ctx = Context(0)
L = ctx.lib
kp = _lib.KernelParams(0.1, 1.0, 0, 0)
st = ctx.torch_stream()
P = C.POINTER(C.c_double)
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")


def hp(t):
    return C.cast(t.data_ptr(), P)


def wall(fn, reps=50, do_flush=True):
    for _ in range(3):
        fn()
    ts = []
    for _ in range(reps):
        if do_flush:
            with torch.cuda.stream(st):
                flush.zero_()
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        fn()
        ts.append(time.perf_counter() - t0)
    return 1e6 * float(np.mean(ts)), 1e6 * float(np.median(ts))


def events(fn, reps=50):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    ts = []
    for _ in range(reps):
        a = torch.cuda.Event(enable_timing=True)
        b = torch.cuda.Event(enable_timing=True)
        a.record(st)
        fn()
        b.record(st)
        b.synchronize()
        ts.append(a.elapsed_time(b) * 1e3)
    return float(np.mean(ts))


def probe(n):
    rng = np.random.default_rng(7)
    hx, hf, hn = (torch.as_tensor(rng.uniform(-0.5, 0.5, (n, 3))).pin_memory() for _ in range(3))
    hu = torch.empty((n, 3), dtype=torch.float64).pin_memory()
    hw = torch.empty((n, 3), dtype=torch.float64).pin_memory()  # (empty_like does not pin)
    dx, df, dn = (t.cuda() for t in (hx, hf, hn))
    du, dw = torch.empty_like(dx), torch.empty_like(dx)

    def e2e():
        ctx.check(L.pswim_mrs_velocities_host(ctx.handle, hp(hx), n, hp(hx), hp(hf), hp(hn), n, C.byref(kp), hp(hu),
                                              hp(hw)))

    def kern():
        ctx.check(L.pswim_mrs_velocities(ctx.handle, dptr(dx), n, dptr(dx), dptr(df), dptr(dn), n, C.byref(kp),
                                         dptr(du), dptr(dw)))

    def h2d():
        with torch.cuda.stream(st):
            for d, h in ((dx, hx), (df, hf), (dn, hn)):
                d.copy_(h, non_blocking=True)

    def d2h():
        with torch.cuda.stream(st):
            hu.copy_(du, non_blocking=True)
            hw.copy_(dw, non_blocking=True)

    print(f"N={n}")
    print("  e2e wall (flush)     mean/median us: %.1f / %.1f" % wall(e2e))
    print("  e2e wall (no flush)  mean/median us: %.1f / %.1f" % wall(e2e, do_flush=False))
    print("  kernel events        us: %.1f" % events(kern))
    print("  kernel wall+sync     mean/median us: %.1f / %.1f" % wall(lambda: (kern(), ctx.sync())))
    print("  H2D 3 arrays events  us: %.1f" % events(h2d))
    print("  D2H 2 arrays events  us: %.1f" % events(d2h))
    print("  e2e events           us: %.1f" % events(e2e))
    # pinned / pageable inputs x outputs (pipelined upload needs pinned inputs; direct output
    # writes need pinned outputs)
    px, pf, pn = (np.ascontiguousarray(t.numpy()) for t in (hx, hf, hn))
    pu, pw = np.zeros((n, 3)), np.zeros((n, 3))

    def npp(a):
        return a.ctypes.data_as(P)

    for name, ins, outs in (("in pinned,   out pageable", (hp(hx), hp(hf), hp(hn)), (npp(pu), npp(pw))),
                            ("in pageable, out pinned  ", (npp(px), npp(pf), npp(pn)), (hp(hu), hp(hw))),
                            ("in pageable, out pageable", (npp(px), npp(pf), npp(pn)), (npp(pu), npp(pw)))):
        def call(ins=ins, outs=outs):
            ctx.check(L.pswim_mrs_velocities_host(ctx.handle, ins[0], n, ins[0], ins[1], ins[2], n, C.byref(kp),
                                                  outs[0], outs[1]))
        print("  e2e %s  mean/median us: %.1f / %.1f" % ((name,) + wall(call)))
    torch.cuda.synchronize()


# pinned tensors used on the context's stream are released (inside probe) before it closes
for n in [int(a) for a in (sys.argv[1:] or ["16384", "256"])]:
    probe(n)
ctx.close()
