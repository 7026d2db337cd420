"""Dev: how much of the host-buffer MRS call is the input upload?  Times (N = 16384, no L2
flush, 50 reps, host wall clock): the full pswim_mrs_velocities_host call; the device-input
call writing its outputs straight into mapped page-locked host memory (no upload); the
device-input, device-output call (DESIGN §10 item 3)."""
import ctypes as C
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import numpy as np
import torch

from paper_2604_12083_b200 import _lib
from paper_2604_12083_b200.device import Context, dptr

ctx = Context(0)
L = ctx.lib
kp = _lib.KernelParams(0.1, 1.0, 0, 0)
n = 16384
rng = np.random.default_rng(7)
hx, hf, hn = (torch.as_tensor(rng.uniform(-0.5, 0.5, (n, 3))).pin_memory() for _ in range(3))
hu = torch.empty((n, 3), dtype=torch.float64).pin_memory()
hw = torch.empty((n, 3), dtype=torch.float64).pin_memory()
dx, df, dn = (t.cuda() for t in (hx, hf, hn))
du, dw = torch.empty_like(dx), torch.empty_like(dx)
P = C.POINTER(C.c_double)


def hp(t):
    return C.cast(t.data_ptr(), P)


def mapped(t):
    # device view of a page-locked tensor (cudaHostGetDevicePointer through torch's allocator:
    # pinned memory is mapped with unified addressing, so the host pointer is valid on device)
    return C.c_void_p(t.data_ptr())


def wall(fn, reps=50):
    for _ in range(5):
        fn()
    torch.cuda.synchronize()
    ts = []
    for _ in range(reps):
        t0 = time.perf_counter()
        fn()
        ts.append(time.perf_counter() - t0)
    return 1e6 * float(np.median(ts))


def host():
    ctx.check(L.pswim_mrs_velocities_host(ctx.handle, hp(hx), n, hp(hx), hp(hf), hp(hn), n, C.byref(kp), hp(hu), hp(hw)))


def dev_in_host_out():
    ctx.check(L.pswim_mrs_velocities(ctx.handle, dptr(dx), n, dptr(dx), dptr(df), dptr(dn), n, C.byref(kp), mapped(hu),
                                     mapped(hw)))
    ctx.sync()


def dev_only():
    ctx.check(L.pswim_mrs_velocities(ctx.handle, dptr(dx), n, dptr(dx), dptr(df), dptr(dn), n, C.byref(kp), dptr(du),
                                     dptr(dw)))
    ctx.sync()


print(f"host call (upload + kernel + direct output): {wall(host):.1f} us")
print(f"device inputs, outputs to mapped host memory: {wall(dev_in_host_out):.1f} us")
print(f"device inputs and outputs:                    {wall(dev_only):.1f} us")
ctx.close()
