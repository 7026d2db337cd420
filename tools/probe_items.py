"""Dev sweep: fused-kernel per-rhs phase floors (pswim_dev_latency_probe) for alternative MRS
item decompositions of an N-node system with tpc targets per CTA (N = 100: tpc 7 on a
16-CTA cluster, 13 on 8 CTAs)."""
import ctypes as C
import math
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2604_12083_b200.device import Context
from paper_2604_12083_b200.scenario import ScenarioConfig, make_scenario

sc = make_scenario(ScenarioConfig(rod_count=1, nodes_per_rod=100))
ctx = Context(0, sc)
n = int(sys.argv[1]) if len(sys.argv) > 1 else 100
for tpc in [int(v) for v in (sys.argv[2] if len(sys.argv) > 2 else "7,13").split(",")]:
    for ns in (2, 3, 4, 5, 6, 7, 8):
        chunks = math.ceil(n / ns)
        warps = math.ceil(tpc * chunks / 32)
        if warps > 12:
            continue
        out = (C.c_double * 4)()
        rc = ctx.lib.pswim_dev_latency_probe(ctx.handle, ns, warps, min(chunks, 64), 6 * tpc, 6 * n, out)
        print(f"n {n} tpc {tpc} ns {ns} chunks {chunks} warps {warps}: items {out[1]:.0f} reduce {out[2]:.0f} "
              f"sum {out[1] + out[2]:.0f} rc {rc}")
