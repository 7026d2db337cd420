"""Coarse/fine contention on one B200 (dev tool): the time-sliced Parareal rank runs its
coarse (Euler) chain on a high-priority stream while its fine (RK2) solve occupies the GPU
on a low-priority stream.  Measures T_F, T_G alone, and T_G while F runs, for the 64 x 256
suspension with the bench's per-interval plan (50 RK2 / 5 Euler steps), and prints the
pipelined-Parareal speedup those numbers predict at n = 2, 4, 8 slices (l = 1)."""
import os
import sys
import threading
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import ctypes as C

import torch

from paper_2604_12083_b200 import _lib
from paper_2604_12083_b200.device import dptr
from paper_2604_12083_b200.scenario import ScenarioConfig, build_initial_state, make_scenario


def main(fine=50, coarse=5):
    L = _lib.lib()
    sc = make_scenario(ScenarioConfig(rod_count=64, nodes_per_rod=256, epsilon=0.08))
    cs = sc.to_c()
    cf = L.pswim_create(0, C.byref(cs), 0)
    cg = L.pswim_create(0, C.byref(cs), -5)
    x = torch.as_tensor(build_initial_state(sc), device="cuda")
    of, og = torch.empty_like(x), torch.empty_like(x)

    def run_f():
        L.pswim_propagate(cf, dptr(x), 0.0, fine * 1e-6, 1, fine, 0.0, dptr(of))

    def run_g():
        L.pswim_propagate(cg, dptr(x), 0.0, fine * 1e-6, 0, coarse, 0.0, dptr(og))

    for fn in (run_f, run_g):
        fn()
    t0 = time.perf_counter(); run_f(); tf = time.perf_counter() - t0
    t0 = time.perf_counter(); run_g(); tg = time.perf_counter() - t0
    res = {}
    th = threading.Thread(target=run_f)
    th.start()
    time.sleep(0.2 * tf)
    t0 = time.perf_counter(); run_g(); res["g_under_f"] = time.perf_counter() - t0
    th.join()
    tgc = res["g_under_f"]
    print(f"T_F = {tf * 1e3:.1f} ms, T_G alone = {tg * 1e3:.2f} ms, T_G while F runs = {tgc * 1e3:.2f} ms")
    for n in (2, 4, 8):
        # pipelined, l = 1, one slice per GPU.  If a rank starts its fine solve as soon as its
        # input arrives, each coarse link of the iteration-0 wavefront shares the GPU with that
        # rank's own fine solve: wall ~ (n - 1) T_G,contended + T_F + T_G.  The rank driver
        # instead starts F after its own coarse of the same input (parareal.cpp launch_fine):
        # the wavefront runs uncontended and F starts T_G later: wall ~ n T_G + T_F.
        wall_c = (n - 1) * tgc + tf + tg
        wall = n * tg + tf
        print(f"n = {n}: predicted speedup vs serial fine {n * tf / wall:.2f} "
              f"(fine started with the coarse: {n * tf / wall_c:.2f})")
    L.pswim_destroy(cf)
    L.pswim_destroy(cg)


if __name__ == "__main__":
    main()
