"""MRS throughput for rectangular problems (dev tool): nt targets x ns sources, device path."""
import ctypes as C
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

from paper_2604_12083_b200 import _lib
from paper_2604_12083_b200.device import Context, dptr

ctx = Context(0)
peak, _ = ctx.dfma_peak()
kp = _lib.KernelParams(0.1, 1.0, 0, 0)
for spec in (sys.argv[1:] or ["16384x16384", "16384x65536", "65536x16384", "4096x65536"]):
    nt, ns = (int(v) for v in spec.split("x"))
    rng = np.random.default_rng(7)
    t = torch.as_tensor(rng.uniform(-0.5, 0.5, (nt, 3)), device="cuda")
    s, f, n = (torch.as_tensor(rng.uniform(-0.5, 0.5, (ns, 3)), device="cuda") for _ in range(3))
    u, w = torch.empty_like(t), torch.empty_like(t)
    st = ctx.torch_stream()

    def call():
        ctx.check(ctx.lib.pswim_mrs_velocities(ctx.handle, dptr(t), nt, dptr(s), dptr(f), dptr(n), ns, C.byref(kp),
                                               dptr(u), dptr(w)))

    for _ in range(3):
        call()
    ctx.sync()
    ts = []
    for _ in range(5):
        a = torch.cuda.Event(enable_timing=True)
        b = torch.cuda.Event(enable_timing=True)
        a.record(st)
        call()
        b.record(st)
        b.synchronize()
        ts.append(a.elapsed_time(b))
    ms = min(ts)
    gp = nt * ns / (ms * 1e-3) / 1e9
    print(f"{nt} x {ns}: {ms:.3f} ms  {gp:.1f} Gpair/s  frac={gp * 103e9 / peak:.3f}")
ctx.close()
