"""Per-CTA timeline of one MRS launch (dev tool).

    python tools/probe_mrs_trace.py build      # here: libpswim_trace.so (-DPSWIM_MRS_TRACE)
    python tools/probe_mrs_trace.py [N]        # on the GPU: SM occupancy over time

Each CTA records its globaltimer start / end, SM and whether it ran its target block's
reduction; the summary shows the ramp-up, the drain, and the busy-slot fraction."""
import ctypes as C
import os
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
sys.path.insert(0, ROOT)
TRACE_LIB = os.path.join(HERE, "libpswim_trace.so")


def build():
    from paper_2604_12083_b200 import build as b

    b.COMMON = b.COMMON + ["-DPSWIM_MRS_TRACE"]
    b.BUILD = os.path.join(ROOT, "build", "pswim_trace")
    b.LIB = TRACE_LIB
    b.build(verbose=True)


def run(n):
    import numpy as np
    import torch

    from paper_2604_12083_b200 import _lib

    _lib.LIB_PATH = TRACE_LIB
    from paper_2604_12083_b200.device import Context, dptr

    ctx = Context(0)
    L = ctx.lib
    kp = _lib.KernelParams(0.1, 1.0, 0, 0)
    rng = np.random.default_rng(7)
    x, f, t = (torch.as_tensor(rng.uniform(-0.5, 0.5, (n, 3)), device="cuda") for _ in range(3))
    u, w = torch.empty_like(x), torch.empty_like(x)
    tr = torch.zeros(3 * 64 * 1024, dtype=torch.int64, device="cuda")
    L.pswim_mrs_trace_set.argtypes = [C.c_void_p]
    for rep in range(3):
        ctx.check(L.pswim_mrs_trace_set(C.c_void_p(tr.data_ptr())))
        tr.zero_()
        torch.cuda.synchronize()
        ctx.check(L.pswim_mrs_velocities(ctx.handle, dptr(x), n, dptr(x), dptr(f), dptr(t), n, C.byref(kp), dptr(u),
                                         dptr(w)))
        ctx.sync()
    r = tr.cpu().numpy().reshape(-1, 3)
    r = r[r[:, 1] > 0]
    t0 = r[:, 0].min()
    s, e = (r[:, 0] - t0) / 1e3, (r[:, 1] - t0) / 1e3  # us
    sm, last = r[:, 2] & 0xFFFF, r[:, 2] >> 16
    T = e.max()
    dur = e - s
    print(f"N={n}: {len(r)} CTAs, span {T:.1f} us, CTA duration median {np.median(dur):.1f} us "
          f"(min {dur.min():.1f}, max {dur.max():.1f}); reduction CTAs {int(last.sum())}, their median "
          f"{np.median(dur[last == 1]):.1f} us")
    # busy CTA-slots over time (3 slots per SM)
    grid = np.linspace(0, T, 400)
    busy = np.array([((s <= g) & (e > g)).sum() for g in grid])
    slots = 148 * 3
    print(f"busy fraction of {slots} slots: mean {busy.mean() / slots:.3f}")
    for frac in (0.0, 0.01, 0.02, 0.05, 0.9, 0.95, 0.98, 0.99, 1.0):
        i = min(len(grid) - 1, int(frac * (len(grid) - 1)))
        print(f"  t = {grid[i]:7.1f} us  busy {busy[i]:4d}")
    first_end = np.sort(e)[:5]
    print("first CTA ends (us):", np.round(first_end, 1), " last CTA starts:", np.round(np.sort(s)[-5:], 1))
    ctx.close()


if __name__ == "__main__":
    if len(sys.argv) > 1 and sys.argv[1] == "build":
        build()
    else:
        for a in (sys.argv[1:] or ["16384", "65536"]):
            run(int(a))
