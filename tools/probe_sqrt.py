"""Dev: batched sqrt_rotation HBM throughput only (1e7 matrices), for kernel variant sweeps."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

from paper_2604_12083_b200.device import Context, dptr
from tools.probe_rod import _time

ctx = Context(0)
st = ctx.torch_stream()
n = 10_000_000
g = torch.Generator(device="cuda").manual_seed(0)
qv = torch.randn(n, 4, dtype=torch.float64, device="cuda", generator=g)
qv = qv / qv.norm(dim=1, keepdim=True)
w_, x_, y_, z_ = qv.unbind(1)
q = torch.stack([1 - 2 * (y_ * y_ + z_ * z_), 2 * (x_ * y_ - z_ * w_), 2 * (x_ * z_ + y_ * w_),
                 2 * (x_ * y_ + z_ * w_), 1 - 2 * (x_ * x_ + z_ * z_), 2 * (y_ * z_ - x_ * w_),
                 2 * (x_ * z_ - y_ * w_), 2 * (y_ * z_ + x_ * w_), 1 - 2 * (x_ * x_ + y_ * y_)], 1)
r9 = q.contiguous()
s9 = torch.empty_like(r9)
t = _time(st, lambda: ctx.check(ctx.lib.pswim_sqrt_rotation_batched(ctx.handle, dptr(r9), n, dptr(s9))), reps=10)
print(f"PSWIM_SQRT_CTA={os.environ.get('PSWIM_SQRT_CTA', '0')}: {144 * n / t / 1e9:.0f} GB/s")
