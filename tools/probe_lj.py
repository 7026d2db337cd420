"""LJ pair-search probe (dev tool, also used by bench.py): all-pairs tiles vs the hashed cell
list on the BASELINE suspensions with LJ enabled (lj_well_depth = 0.01), ms per evaluation."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

from paper_2604_12083_b200.device import Context, dptr
from paper_2604_12083_b200.scenario import ScenarioConfig, build_initial_state, make_scenario


def lj_times(device=0, sizes=((64, 256), (512, 256)), reps=5):
    out = {}
    for rods, m in sizes:
        sc = make_scenario(ScenarioConfig(rod_count=rods, nodes_per_rod=m, epsilon=0.08, lj_well_depth=0.01))
        x = build_initial_state(sc).reshape(-1, 12)
        rng = np.random.default_rng(1)
        x[:, 0:3] += rng.normal(scale=0.5 * sc.lj_sigma, size=(len(x), 3))  # bring rods into contact
        ctx = Context(device, sc)
        dx = torch.as_tensor(x.reshape(-1), device=f"cuda:{device}")
        f = torch.empty((rods * m, 3), dtype=torch.float64, device=dx.device)
        st = ctx.torch_stream()
        res = {}
        for mode, name in ((1, "all_pairs"), (2, "cell_list")):
            ctx.lib.pswim_set_lj_mode(ctx.handle, mode)
            ctx.check(ctx.lib.pswim_lj_forces(ctx.handle, dptr(dx), dptr(f)))
            ctx.sync()
            best = 1e30
            for _ in range(reps if mode == 2 or rods * m <= 20000 else 1):
                a = torch.cuda.Event(enable_timing=True)
                b = torch.cuda.Event(enable_timing=True)
                a.record(st)
                ctx.check(ctx.lib.pswim_lj_forces(ctx.handle, dptr(dx), dptr(f)))
                b.record(st)
                b.synchronize()
                best = min(best, a.elapsed_time(b))
            res[name + "_ms"] = best
            res[name + "_sum"] = float(f.abs().sum())
        res["nodes"] = rods * m
        out[f"{rods}x{m}"] = res
        ctx.close()
    return out


if __name__ == "__main__":
    print(json.dumps(lj_times(), indent=1))
