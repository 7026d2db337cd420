"""Quick MRS throughput probe (dev tool): Gpair/s at several N + DFMA peak."""
import sys, os, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import ctypes as C
from paper_2604_12083_b200.device import Context, dptr
from paper_2604_12083_b200 import _lib

ctx = Context(0)
peak, ms = ctx.dfma_peak()
print(f"dfma peak {peak/1e12:.2f} TFLOP/s ({ms:.2f} ms)")
kp = _lib.KernelParams(0.1, 1.0, 0, 0)
for n in [int(a) for a in (sys.argv[1:] or ["16384", "65536", "131072"])]:
    rng = np.random.default_rng(7)
    d = [torch.as_tensor(rng.uniform(-0.5, 0.5, (n, 3)), device="cuda") for _ in range(3)]
    u = torch.empty_like(d[0]); w = torch.empty_like(d[0])
    st = ctx.torch_stream()
    torch.cuda.synchronize()
    for _ in range(3):
        ctx.check(ctx.lib.pswim_mrs_velocities(ctx.handle, dptr(d[0]), n, dptr(d[0]), dptr(d[1]), dptr(d[2]), n, C.byref(kp), dptr(u), dptr(w)))
    ctx.sync()
    reps = 5 if n <= 65536 else 2
    ts = []
    for _ in range(reps):
        a = torch.cuda.Event(enable_timing=True); b = torch.cuda.Event(enable_timing=True)
        a.record(st)
        ctx.check(ctx.lib.pswim_mrs_velocities(ctx.handle, dptr(d[0]), n, dptr(d[0]), dptr(d[1]), dptr(d[2]), n, C.byref(kp), dptr(u), dptr(w)))
        b.record(st)
        b.synchronize()
        ts.append(a.elapsed_time(b))
    t = min(ts)
    gp = n * n / (t * 1e-3) / 1e9
    print(f"N={n}: {t:.3f} ms  {gp:.1f} Gpair/s  {gp*103/1e3:.2f} TFLOP/s(103/pair)  frac={gp*103e9/peak:.3f}")
    import hashlib
    print(f"  sha1(u,w) = {hashlib.sha1(u.cpu().numpy().tobytes() + w.cpu().numpy().tobytes()).hexdigest()[:16]}")
