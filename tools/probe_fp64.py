"""FP64 pipe microbenchmarks (dev tool): DFMA/DMUL rates by operand pattern."""
import ctypes as C
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2604_12083_b200.device import Context

ctx = Context(0)
names = {0: "DFMA constant operands", 1: "DFMA shared reg operands (reuse)", 2: "DFMA 3 distinct reg pairs",
         3: "DMUL 2 distinct reg pairs", 4: "DFMA 3 distinct + MUFU.RSQ64H every 48",
         5: "DMMA m8n8k4 only (FMA equivalents)", 6: "half warps DFMA + half warps DMMA (FMA equiv)"}
for k in range(7):
    r = C.c_double()
    ms = C.c_double()
    ctx.check(ctx.lib.pswim_dev_fp64_probe(ctx.handle, k, C.byref(r), C.byref(ms)))
    print(f"kind {k}: {r.value / 1e12:7.3f} T ops/s  ({names[k]})  {ms.value:.2f} ms")
