"""Dev sweep: fused-kernel per-rhs phase floors (pswim_dev_latency_probe) for alternative MRS
item decompositions of the 100-node flagellum on a 16-CTA cluster (7 targets per CTA)."""
import ctypes as C
import math
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2604_12083_b200.device import Context
from paper_2604_12083_b200.scenario import ScenarioConfig, make_scenario

sc = make_scenario(ScenarioConfig(rod_count=1, nodes_per_rod=100))
ctx = Context(0, sc)
n, tpc = 100, 7
for ns in (1, 2, 3, 4, 5, 6, 8):
    chunks = math.ceil(n / ns)
    warps = math.ceil(tpc * chunks / 32)
    for w in sorted({min(warps, 12), 12, 8, 6, 4}):
        if w < min(warps, 12):
            continue
        out = (C.c_double * 4)()
        rc = ctx.lib.pswim_dev_latency_probe(ctx.handle, ns, w, min(chunks, 64), 6 * tpc, 6 * n, out)
        print(f"ns {ns} chunks {chunks} item-warps needed {warps} run on {w}: front {out[0]:.0f} items {out[1]:.0f} "
              f"reduce {out[2]:.0f} exchange {out[3]:.0f} rc {rc}")
