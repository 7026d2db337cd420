#!/usr/bin/env python
"""bench.py — MRS Gpair-interactions/s (+ simulated RK2 time-steps/s) on B200.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]

One JSON line on rank 0:

* value        MRS all-pairs evaluation, BASELINE.json configs[1] (N = 16384 regularized
               points, targets = sources, eps = 0.1, mu = 1, inputs ~ U[-0.5,0.5)^3), inputs
               resident in HBM, L2 flushed (256 MiB write) before every timed step, each step
               timed with CUDA events on the launching stream; whole-job Gpair/s = N_gpus *
               N^2 / max-over-ranks step time (weak scaling: every rank evaluates its own
               suspension, no data-path collective).
* e2e          the same evaluation through the C-ABI host entry point
               (pswim_mrs_velocities_host): pinned host buffers, H2D + kernel + D2H + sync
               inside the timed region.
* roofline     dominant kernel (mrs_kernel): 103 FLOP/pair (stokes.cpp:29-55 as
               written) x N^2 / average launch time, against the FP64 DFMA peak measured
               live in this run (MEASURED_PEAKS.json has no FP64 entry).
* time_steps   secondary metric: simulated RK2 time-steps/s.  N=1: serial fine RK2 on
               configs[2] (64 x 256 suspension, eps = 0.08, dt = 1e-6).  N>1: pipelined
               Parareal, one time slice per GPU over NCCL (configs[3]).
* cpu_baseline the reference's own evaluate_velocities (oracle/_ref, OpenMP, all host
               threads) on a bounded target sample of the same workload (rank 0, N=1).

``--impl reference`` times that reference CPU path alone (rank 0; other ranks exit 0).
"""
from __future__ import annotations

import argparse
import ctypes as C
import json
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)
# more hardware work queues than the default 8, so that the streams of one process (coarse,
# fine, comm, engine lanes) do not serialise behind each other's device-side waits
os.environ.setdefault("CUDA_DEVICE_MAX_CONNECTIONS", "32")
# every device / transport wait of the rank drivers completes in well under a minute in these
# legs; a peer that died aborts the leg after 5 min instead of the library's 15 min default
os.environ.setdefault("PSWIM_COMM_TIMEOUT_S", "300")

N_POINTS = 16384
EPS, MU = 0.1, 1.0
FLOP_PER_PAIR = 103
WORKLOAD = "MRS all-pairs velocity evaluation, N=16384 regularized points (BASELINE configs[1])"


def _jsonable(o):
    """numpy scalars / arrays in the JSON line as plain numbers / lists."""
    if isinstance(o, np.generic):
        return o.item()
    if isinstance(o, np.ndarray):
        return o.tolist()
    raise TypeError(f"not JSON serializable: {type(o).__name__}")


class Mt19937_64:
    """std::mt19937_64 (the C++ standard's 64-bit Mersenne Twister), so the bench draws exactly
    the inputs of the reference's own timer (tools/bench_kernels.cpp:46-50)."""

    N, M = 312, 156
    MASK = (1 << 64) - 1

    def __init__(self, seed: int = 5489):
        mt = [seed & self.MASK]
        for i in range(1, self.N):
            mt.append((6364136223846793005 * (mt[-1] ^ (mt[-1] >> 62)) + i) & self.MASK)
        self.mt, self.i = mt, self.N

    def _twist(self):
        mt, n, m = self.mt, self.N, self.M
        for i in range(n):
            x = (mt[i] & 0xFFFFFFFF80000000) | (mt[(i + 1) % n] & 0x7FFFFFFF)
            xa = x >> 1
            if x & 1:
                xa ^= 0xB5026F5AA96619E9
            mt[i] = mt[(i + m) % n] ^ xa
        self.i = 0

    def __call__(self) -> int:
        if self.i >= self.N:
            self._twist()
        y = self.mt[self.i]
        self.i += 1
        y ^= (y >> 29) & 0x5555555555555555
        y ^= (y << 17) & 0x71D67FFFEDA60000
        y ^= (y << 37) & 0xFFF7EEE000000000
        y ^= y >> 43
        return y & self.MASK


def synthetic_inputs(n: int, seed: int):
    """x, f, n per point in that order, each component (rng() >> 11) * 2^-53 - 0.5 from
    std::mt19937_64(seed) -- bench_kernels.cpp:46-50 / :59-63 (seed 7 there)."""
    rng = Mt19937_64(seed)
    u = np.array([rng() >> 11 for _ in range(9 * n)], dtype=np.float64) * 2.0 ** -53 - 0.5
    u = u.reshape(n, 3, 3)
    return [np.ascontiguousarray(u[:, i, :]) for i in range(3)]


# ------------------------------------------------------------------------------------------
class ClockSampler:
    """SM clocks + throttle reasons sampled during the timed region (NVML; nvidia-smi fallback)."""

    FIELDS = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.samples = []
        self._stop = threading.Event()
        self._t = threading.Thread(target=self._run, daemon=True)

    def _nvml(self):
        # NVML directly (~1 ms per sample) so a ~0.1 s timed region still gets tens of samples
        try:
            import pynvml as nv

            nv.nvmlInit()
            h = nv.nvmlDeviceGetHandleByIndex(self.index)
            smax = nv.nvmlDeviceGetMaxClockInfo(h, nv.NVML_CLOCK_SM)
            get_reasons = getattr(nv, "nvmlDeviceGetCurrentClocksEventReasons", None) or \
                nv.nvmlDeviceGetCurrentClocksThrottleReasons
        except Exception:
            return False
        bits = (0x8, 0x40, 0x20, 0x4)  # hw_slowdown, hw_thermal, sw_thermal, sw_power_cap
        while not self._stop.is_set():
            try:
                sm = nv.nvmlDeviceGetClockInfo(h, nv.NVML_CLOCK_SM)
                r = get_reasons(h)
                self.samples.append([str(sm), str(smax), ""] + ["Active" if r & b else "Not Active" for b in bits])
            except Exception:
                pass
            self._stop.wait(0.005)
        return True

    def _run(self):
        if self._nvml():
            return
        while not self._stop.is_set():
            try:
                out = subprocess.run(["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.FIELDS}",
                                      "--format=csv,noheader,nounits"], capture_output=True, text=True, timeout=5)
                parts = [p.strip() for p in out.stdout.strip().split(",")]
                if len(parts) == 7:
                    self.samples.append(parts)
            except Exception:
                pass
            self._stop.wait(0.05)

    def __enter__(self):
        self._t.start()
        return self

    def __exit__(self, *exc):
        self._stop.set()
        self._t.join(timeout=10)

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        sm = [float(s[0]) for s in self.samples if s[0].replace(".", "").isdigit()]
        smax = [float(s[1]) for s in self.samples if s[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for s in self.samples for i in range(4) if s[3 + i].lower() == "active"})
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(smax) if smax else None,
                "reasons": reasons, "samples": len(self.samples)}


# ------------------------------------------------------------------------------------------
def dist_env():
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return world, rank, local


WIRE = "nccl"  # "gloo": test mode -- ranks may share a GPU, transports staged over gloo


def reduce_max(value: float, device=None) -> float:
    import torch
    import torch.distributed as dist

    if not (dist.is_available() and dist.is_initialized()):
        return value
    t = torch.tensor([value], dtype=torch.float64, device=device if WIRE == "nccl" else "cpu")
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def barrier():
    import torch.distributed as dist

    if dist.is_available() and dist.is_initialized():
        dist.barrier()


# ------------------------------------------------------------------------------------------
_INPUTS = {}


def inputs_cached(n: int, seed: int):
    if (n, seed) not in _INPUTS:
        _INPUTS[n, seed] = synthetic_inputs(n, seed)
    return _INPUTS[n, seed]


def cpu_reference_mrs(n_targets: int, reps: int, threads: int | None = None):
    """The reference's evaluate_velocities (OpenMP) on n_targets x N_POINTS pairs."""
    from oracle.pyoracle import Oracle

    ref = Oracle("ref")
    full = ref.max_threads_()
    ref.set_threads_(threads or full)
    cores = ref.max_threads_()
    x, f, tq = inputs_cached(N_POINTS, 7)
    tgt = np.ascontiguousarray(x[:n_targets])
    ref.evaluate_velocities(tgt[:64], x, f, tq, EPS, MU, parallel=True)  # OpenMP team warm-up
    times = []
    for _ in range(reps):
        t0 = time.perf_counter()
        ref.evaluate_velocities(tgt, x, f, tq, EPS, MU, parallel=True)
        times.append(time.perf_counter() - t0)
    ref.set_threads_(full)
    return times, cores


def run_reference_arm(args) -> None:
    """The reference's own evaluate_velocities (oracle/_ref, OpenMP, every host thread) on the
    SAME workload as our arm: the full N x N evaluation of the same mt19937_64(7) inputs, each
    step one evaluation.  Also one evaluation with a single thread (the reference's serial
    path cost), with the host's core count."""
    world, rank, _ = dist_env()
    if rank != 0:
        return
    n_targets = args.ref_targets
    times, cores = cpu_reference_mrs(n_targets, args.steps + args.warmup)
    t = times[args.warmup:] or times
    per = sum(t) / len(t)
    value = n_targets * N_POINTS / per / 1e9
    one, _ = cpu_reference_mrs(n_targets, 1, threads=1)
    sample = (f"{n_targets} targets x {N_POINTS} sources per step" +
              (" (the full all-pairs evaluation of our arm's workload)" if n_targets == N_POINTS else
               " (bounded sample of the N=16384 all-pairs workload)"))
    line = {
        "impl": "reference", "metric": "MRS Gpair-interactions/s", "value": value, "unit": "Gpair/s",
        "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * per,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": WORKLOAD, "points": N_POINTS, "epsilon": EPS, "mu": MU, "targets_equal_sources": True,
                   "inputs": "std::mt19937_64(7), (rng() >> 11) * 2^-53 - 0.5 per component (bench_kernels.cpp:46-50)",
                   "l2": "n/a (CPU)"},
        "cpu_baseline": {"value": value, "unit": "Gpair/s", "cores": cores, "kind": "reference", "sample": sample,
                         "nproc": os.cpu_count(),
                         "single_thread": {"value": n_targets * N_POINTS / one[0] / 1e9, "unit": "Gpair/s",
                                           "cores": 1, "sample": "one evaluation of the same workload, "
                                                                 "OMP team of 1 thread"}},
        "e2e": {"value": value, "unit": "Gpair/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line, default=_jsonable), flush=True)


# ------------------------------------------------------------------------------------------
def run_ours(args) -> None:
    import torch
    import torch.distributed as dist

    world, rank, local = dist_env()
    if WIRE != "nccl":
        local = local % torch.cuda.device_count()  # test mode: ranks may share a GPU
    if world > 1 and not dist.is_initialized():
        if WIRE == "nccl":
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        else:
            dist.init_process_group("gloo")
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)

    from paper_2604_12083_b200 import _lib
    from paper_2604_12083_b200.device import Context, dptr

    L = _lib.lib()
    ctx = Context(local)
    st = ctx.torch_stream()
    kp = _lib.KernelParams(EPS, MU, 0, 0)
    n = N_POINTS

    # --- measured FP64 peak (roofline denominator) ---
    dfma_peak, _ = ctx.dfma_peak()

    # --- device-resident inputs (every rank its own suspension of the same size) ---
    x, f, tq = inputs_cached(n, 7 + rank)
    dx, df, dn = (torch.as_tensor(a, device=dev) for a in (x, f, tq))
    du = torch.empty_like(dx)
    dw = torch.empty_like(dx)
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)  # > 126 MB L2

    def launch():
        ctx.check(L.pswim_mrs_velocities(ctx.handle, dptr(dx), n, dptr(dx), dptr(df), dptr(dn), n, C.byref(kp),
                                         dptr(du), dptr(dw)))

    torch.cuda.synchronize()
    for _ in range(args.warmup):
        launch()
    ctx.sync()
    barrier()
    torch.cuda.synchronize()
    times = []
    with ClockSampler(local) as clk:
        for _ in range(args.steps):
            with torch.cuda.stream(st):
                flush.zero_()
            a = torch.cuda.Event(enable_timing=True)
            b = torch.cuda.Event(enable_timing=True)
            a.record(st)
            launch()
            b.record(st)
            b.synchronize()
            times.append(a.elapsed_time(b))
    ctx.sync()
    torch.cuda.synchronize()
    barrier()
    ms = sum(times) / len(times)
    ms_max = reduce_max(ms, dev)
    value = world * n * n / (ms_max * 1e-3) / 1e9

    # --- e2e through the C-ABI host entry point, pinned host buffers ---
    hx, hf, hn = (torch.as_tensor(a).pin_memory() for a in (x, f, tq))
    hu = torch.empty((n, 3), dtype=torch.float64).pin_memory()
    hw = torch.empty((n, 3), dtype=torch.float64).pin_memory()  # (empty_like does not pin)
    P = C.POINTER(C.c_double)

    def hp(t):
        return C.cast(t.data_ptr(), P)

    def e2e_call():
        ctx.check(L.pswim_mrs_velocities_host(ctx.handle, hp(hx), n, hp(hx), hp(hf), hp(hn), n, C.byref(kp),
                                              hp(hu), hp(hw)))

    for _ in range(max(1, args.warmup)):
        e2e_call()
    barrier()
    e2e_t = []
    for _ in range(args.steps):
        with torch.cuda.stream(st):
            flush.zero_()
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        e2e_call()
        e2e_t.append(time.perf_counter() - t0)
    e2e_s = reduce_max(sum(e2e_t) / len(e2e_t), dev)
    e2e_value = world * n * n / e2e_s / 1e9
    h2d = 3 * n * 3 * 8  # positions (targets = sources: copied once), f, n
    d2h = 2 * n * 3 * 8

    # parity spot check of the device run's output (after the e2e timing: no host threads
    # of the oracle around while it runs) against the reference restatement (rows)
    parity = None
    if rank == 0 and not args.no_cpu:
        from oracle.pyoracle import Oracle

        rows = np.r_[0:32, n // 2:n // 2 + 32, n - 32:n]
        ou, ow = Oracle("or").evaluate_velocities(x[rows], x, f, tq, EPS, MU)
        gu, gw = du.cpu().numpy()[rows], dw.cpu().numpy()[rows]
        scale = max(np.abs(ou).max(), np.abs(ow).max())
        parity = float(max(np.abs(gu - ou).max(), np.abs(gw - ow).max()) / scale)

    # --- roofline of the dominant kernel ---
    achieved = FLOP_PER_PAIR * n * n / (ms * 1e-3) / 1e12
    traffic = None
    tpath = os.path.join(ROOT, "profiles", "mrs_kernel_traffic.json")
    if os.path.exists(tpath):
        try:
            traffic = json.load(open(tpath)).get("dram_bytes_per_launch")
        except Exception:
            traffic = None
    roofline = {"bound": "compute", "pipe": "FP64 FMA (CUDA cores; FP64 is not a dense contraction)",
                "achieved": achieved, "peak": dfma_peak / 1e12, "unit": "TFLOP/s", "frac": achieved / (dfma_peak / 1e12),
                "traffic": traffic, "kernel": "mrs_kernel<split, variant %s>" % os.environ.get("PSWIM_MRS_TPT", "3"),
                "flop_per_pair": FLOP_PER_PAIR, "peak_source": "DFMA microbenchmark measured in this run "
                "(MEASURED_PEAKS.json has no FP64 entry)", "dp_instructions_per_pair_loop": 51}

    # --- the north_star's MRS target sizes (N >= 64k), rank 0 at N = 1 ---
    sweep = None
    if rank == 0 and world == 1 and not args.no_sweep:
        try:
            sweep = mrs_sweep_leg(ctx, L, kp, dev, local, dfma_peak, flush)
        except Exception as e:
            sweep = {"error": f"{type(e).__name__}: {e}"}

    # --- secondary: simulated RK2 time-steps/s ---
    time_steps = None
    if not args.no_steps:
        try:
            time_steps = time_steps_leg(args, world, rank, local, dev)
        except Exception as e:  # the MRS line must still be reported
            time_steps = {"error": f"{type(e).__name__}: {e}"}

    # --- HBM-bound rod-side kernels on >= 1e7 elements (rank 0, N=1) ---
    hbm = None
    if rank == 0 and world == 1 and not args.no_steps:
        sys.path.insert(0, os.path.join(ROOT, "tools"))
        from probe_rod import hbm_kernels

        with ClockSampler(local) as hclk:
            hbm = hbm_kernels(local)
        for v in hbm.values():
            v["frac_of_measured_hbm"] = v["GB_per_s"] / _hbm_peak()
        hbm["clocks"] = hclk.summary()
        try:
            from probe_lj import lj_times

            hbm["lj_repulsion"] = {"workload": "LJ pair forces (lj_well_depth = 0.01, grid suspensions perturbed "
                                               "by 0.5 sigma into contact), ms per evaluation",
                                   **lj_times(local)}
        except Exception as e:
            hbm["lj_repulsion"] = {"error": f"{type(e).__name__}: {e}"}

    # --- CPU baseline (reference, host cores) ---
    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu:
        from oracle.pyoracle import LIB_PATHS

        if os.path.exists(LIB_PATHS["ref"]):
            nt = args.ref_targets
            ct, cores = cpu_reference_mrs(nt, 3)
            best = min(ct)
            cpu = {"value": nt * n / best / 1e9, "unit": "Gpair/s", "cores": cores, "kind": "reference",
                   "nproc": os.cpu_count(),
                   "sample": f"best of 3: {nt} targets x {n} sources of the N=16384 workload, the same "
                             "mt19937_64(7) inputs (oracle/_ref = reference evaluate_velocities, OpenMP)"}
        else:
            cpu = {"value": None, "unit": "Gpair/s", "cores": 0, "kind": "reference",
                   "sample": "oracle/_ref not built on this box"}

    if rank == 0:
        line = {
            "metric": "MRS Gpair-interactions/s", "value": value, "unit": "Gpair/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms_max, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"workload": WORKLOAD, "points": n, "epsilon": EPS, "mu": MU, "targets_equal_sources": True,
                       "l2": "flushed (256 MiB write) before every timed step", "parallelism": f"replicas{world}"},
            "clocks": clk.summary(),
            "e2e": {"value": e2e_value, "unit": "Gpair/s", "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h,
                    "ms_per_step": 1e3 * e2e_s, "ms_per_step_median_rank0": 1e3 * float(np.median(e2e_t)),
                    "api": "pswim_mrs_velocities_host (C-ABI)"},
            "gpu_launches": args.steps,
            "roofline": roofline,
            "cpu_baseline": cpu,
            "parity_rel_err_vs_oracle": parity,
            "mrs_sweep": sweep,
            "time_steps": time_steps,
            "hbm_kernels": hbm,
        }
        print(json.dumps(line, default=_jsonable), flush=True)
    ctx.close()
    if world > 1:
        barrier()
        dist.destroy_process_group()


def mrs_sweep_leg(ctx, L, kp, dev, local, dfma_peak, flush, sizes=(65536, 131072), reps=5):
    """MRS at the north_star's sizes (>= 60 % of FP64 peak at N >= 64k): same inputs recipe
    (mt19937_64(7)), targets = sources, L2 flushed before every timed launch, CUDA events on
    the launching stream, clocks sampled during the timed launches."""
    import torch

    from paper_2604_12083_b200.device import dptr

    st = ctx.torch_stream()
    out = {"workload": "MRS all-pairs evaluation, targets = sources, eps=0.1, mu=1, mt19937_64(7) inputs "
                       "(BASELINE configs[1] recipe at the north_star's N >= 64k)", "points": {}}
    for n in sizes:
        x, f, tq = inputs_cached(n, 7)
        dx, df, dn = (torch.as_tensor(a, device=dev) for a in (x, f, tq))
        du, dw = torch.empty_like(dx), torch.empty_like(dx)

        def launch():
            ctx.check(L.pswim_mrs_velocities(ctx.handle, dptr(dx), n, dptr(dx), dptr(df), dptr(dn), n, C.byref(kp),
                                             dptr(du), dptr(dw)))

        for _ in range(3):
            launch()
        ctx.sync()
        times = []
        with ClockSampler(local) as clk:
            for _ in range(reps):
                with torch.cuda.stream(st):
                    flush.zero_()
                a = torch.cuda.Event(enable_timing=True)
                b = torch.cuda.Event(enable_timing=True)
                a.record(st)
                launch()
                b.record(st)
                b.synchronize()
                times.append(a.elapsed_time(b))
        ctx.sync()
        ms = sum(times) / len(times)
        achieved = FLOP_PER_PAIR * n * n / (ms * 1e-3) / 1e12
        out["points"][str(n)] = {"value": n * n / (ms * 1e-3) / 1e9, "unit": "Gpair/s", "ms": ms,
                                 "roofline_frac": achieved / (dfma_peak / 1e12), "achieved_tflops": achieved,
                                 "clocks": clk.summary(), "launches": reps}
        del dx, df, dn, du, dw
    out["peak_tflops"] = dfma_peak / 1e12
    return out


def time_steps_leg(args, world, rank, local, dev):
    """Simulated RK2 time-steps/s: serial fine (N=1) or sliced pipelined Parareal (N>1)."""
    import torch

    from paper_2604_12083_b200 import parareal as pr
    from paper_2604_12083_b200.device import Context, dptr
    from paper_2604_12083_b200.scenario import ScenarioConfig, build_initial_state, make_scenario

    sc = make_scenario(ScenarioConfig(rod_count=64, nodes_per_rod=256, epsilon=0.08, fine_dt=1e-6))
    x0 = build_initial_state(sc)
    if world == 1:
        ctx = Context(local, sc)
        L = ctx.lib
        dx = torch.as_tensor(x0, device=dev)
        out = torch.empty_like(dx)
        steps = args.serial_steps
        ctx.check(L.pswim_propagate(ctx.handle, dptr(dx), 0.0, 3e-6, 1, 3, 0.0, dptr(out)))  # warm-up
        st = ctx.torch_stream()
        a = torch.cuda.Event(enable_timing=True)
        b = torch.cuda.Event(enable_timing=True)
        a.record(st)
        ctx.check(L.pswim_propagate(ctx.handle, dptr(dx), 0.0, steps * 1e-6, 1, steps, 0.0, dptr(out)))
        b.record(st)
        b.synchronize()
        sec = a.elapsed_time(b) * 1e-3
        ctx.close()
        leg = {"metric": "simulated RK2 time-steps/s", "value": steps / sec, "unit": "steps/s",
               "config": {"workload": "serial fine RK2, 64 x 256 suspension, eps=0.08, dt=1e-6 (BASELINE configs[2])",
                          "steps": steps}, "gpu_launches_per_step": 6}
        if not args.no_cpu:
            from oracle.pyoracle import LIB_PATHS, Oracle, Scenario as OS

            if os.path.exists(LIB_PATHS["ref"]):
                ref = Oracle("ref")
                osc = OS.make(rod_count=64, nodes_per_rod=256, epsilon=0.08)
                t0 = time.perf_counter()
                ref.propagate(osc, x0, 0.0, 2e-6, 1, steps=2)
                cpu = 2 / (time.perf_counter() - t0)
                leg["cpu_baseline"] = {"value": cpu, "unit": "steps/s", "cores": ref.max_threads_(),
                                       "kind": "reference",
                                       "sample": "2 RK2 steps of the same suspension (reference propagate, OpenMP)"}
        leg["flagellum"] = flagellum_leg(args, local, dev)
        try:
            leg["gpu_vs_reference_parareal"] = reduced_parity(local)
        except Exception as e:
            leg["gpu_vs_reference_parareal"] = {"error": f"{type(e).__name__}: {e}"}
        return leg
    # N > 1: one Parareal slice per GPU (BASELINE configs[3])
    tr = _transport(local)
    try:
        leg = parareal_sweep_leg(args, sc, x0, world, rank, local, dev, tr)
        try:
            sp = space_parallel_leg(sc, x0, local, dev, tr, world)
            # strong scaling of the exact serial fine integration (no Parareal error) against the
            # 1-GPU serial fine rate measured in the sweep leg
            base = leg.get("serial_fine_steps_per_s")
            if base:
                sp["speedup_vs_1gpu_serial_fine"] = sp["value"] / base
                if "value" in sp.get("fused_peer_allgather", {}):
                    sp["fused_peer_allgather"]["speedup_vs_1gpu_serial_fine"] = sp["fused_peer_allgather"]["value"] / base
            leg["space_parallel"] = sp
        except Exception as e:
            leg["space_parallel"] = {"error": f"{type(e).__name__}: {e}"}
        if world >= 4 and world % 2 == 0:
            try:
                leg["hybrid_space_time"] = hybrid_leg(args, sc, x0, local, dev, world, members=2)
            except Exception as e:
                leg["hybrid_space_time"] = {"error": f"{type(e).__name__}: {e}"}
        if not args.no_large:
            try:
                leg["large_suspension"] = large_leg(args, local, dev, tr, world, rank)
            except Exception as e:
                leg["large_suspension"] = {"error": f"{type(e).__name__}: {e}"}
    finally:
        _lib_destroy(tr)
    return leg


def serial_fine_boundaries_gpu(sc, x0, plan, fine, local, dev):
    """harness::serial_fine_boundaries (harness.cpp:35-37) on one GPU: the fine propagator
    chained over the plan's intervals at boundary_time(n).  Returns (states, seconds)."""
    import torch

    from paper_2604_12083_b200.device import Context, dptr

    ctx = Context(local, sc)
    cur = torch.as_tensor(x0, device=dev)
    nxt = torch.empty_like(cur)
    ctx.check(ctx.lib.pswim_propagate(ctx.handle, dptr(cur), 0.0, 2e-6, 1, 2, 0.0, dptr(nxt)))  # warm-up
    states = [cur.clone()]
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for i in range(plan.intervals):
        ctx.check(ctx.lib.pswim_propagate(ctx.handle, dptr(cur), plan.boundary_time(i), plan.boundary_time(i + 1), 1,
                                          fine, 0.0, dptr(nxt)))
        cur, nxt = nxt, cur
        states.append(cur.clone())
    torch.cuda.synchronize()
    sec = time.perf_counter() - t0
    ctx.close()
    return states, sec


def parareal_sweep_leg(args, sc, x0, world, rank, local, dev, tr):
    """BASELINE configs[3] as BASELINE.md states it: n = m = world intervals of `fine` RK2 steps
    (dt = 1e-6) with `coarse` Euler steps (r = 2 fine / coarse rhs), pipelined Parareal with one
    slice per GPU, l = 1..min(4, world) at tol = 1e-300 (fixed l) and one tol = 1e-10 run.  Per
    run: simulated steps/s, speedup over the 1-GPU serial fine integration of the same horizon,
    eta = true error vs that serial fine solution (max over ranks, rod_position_metric), and the
    schedule idle W of the rank-driver trace."""
    import torch
    import torch.distributed as dist

    from paper_2604_12083_b200 import parareal as pr

    fine, coarse = args.fine_steps, max(1, min(args.coarse_steps, args.fine_steps // 10))
    T = world * fine * 1e-6

    def plan(l, tol=1e-300):
        return pr.ParallelPlan(t0=0.0, horizon=T, intervals=world, workers=world, max_iterations=l, tolerance=tol,
                               mode=pr.PIPELINED)

    # serial fine on rank 0: the speedup denominator and every rank's true-error reference
    barrier()
    buf = torch.empty((world + 1, x0.size), dtype=torch.float64, device=dev if WIRE == "nccl" else "cpu")
    serial = torch.zeros(1, dtype=torch.float64, device=buf.device)
    if rank == 0:
        states, sec = serial_fine_boundaries_gpu(sc, x0, plan(1), fine, local, dev)
        buf.copy_(torch.stack(states))
        serial.fill_(sec)
    dist.broadcast(buf, 0)
    dist.broadcast(serial, 0)
    serial_s = float(serial.item())
    ref_slice = buf[rank + 1].cpu().numpy()
    warm = pr.ParallelPlan(t0=0.0, horizon=world * 1e-6, intervals=world, workers=world, max_iterations=1,
                           tolerance=1e-300, mode=pr.PIPELINED)
    pr.run_sliced_rank(warm, sc, 1, 1, x0, local, transport=tr)  # contexts, kernels, plans

    def timed(p, handoff=None):
        barrier()
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        res = pr.run_sliced_rank(p, sc, fine, coarse, x0, local, transport=tr, reference_slice=ref_slice,
                                 handoff=handoff)
        call = reduce_max(time.perf_counter() - t0, dev)
        wall = reduce_max(res.report.wall_seconds, dev)  # start barrier -> result downloaded, max over ranks
        eta = float(res.report.eta[-1]) if res.report.eta else None
        return res, {"iterations": res.report.iterations_used, "converged": res.report.converged,
                     "value": world * fine / wall, "unit": "steps/s", "wall_s": wall,
                     "speedup_vs_serial_fine": serial_s / wall, "eta_vs_serial_fine": eta,
                     "within_tolerance_1e-10": bool(eta is not None and eta <= 1e-10),
                     "eta_tilde": res.report.eta_tilde, "schedule_idle_s": res.schedule_idle,
                     "call_s_incl_setup": call}

    sweep = [timed(plan(l))[1] for l in range(1, min(4, world) + 1)]
    _, tol_run = timed(plan(world, 1e-10))
    leg = {"metric": "simulated RK2 time-steps/s", "value": tol_run["value"], "unit": "steps/s",
           "speedup_vs_serial_fine": tol_run["speedup_vs_serial_fine"],
           "eta_vs_serial_fine": tol_run["eta_vs_serial_fine"],
           "config": {"workload": "pipelined Parareal, one slice per GPU, 64 x 256 suspension, eps=0.08, dt=1e-6 "
                                  "(BASELINE configs[3]); headline = the tol=1e-10 run", "intervals": world,
                      "fine_rk2_steps_per_interval": fine, "coarse_euler_steps_per_interval": coarse,
                      "cost_ratio_r": 2.0 * fine / coarse, "tolerance": 1e-10,
                      "iterations": tol_run["iterations"], "eta_tilde": tol_run["eta_tilde"]},
           "serial_fine_s": serial_s, "serial_fine_steps_per_s": world * fine / serial_s,
           "speedup_denominator": "1-GPU serial fine integration of the same world x fine RK2 steps, measured",
           "tolerance_run": tol_run, "iteration_sweep": sweep}
    # the same l = 2 run with the peer-memory hand-off (corrector stores into the next rank's
    # HBM slot over NVLink, CUDA IPC) instead of NCCL send/recv
    try:
        ho = pr.Handoff(local, x0.size, min(2, world) + 1)
        barrier()
        _, hrun = timed(plan(min(2, world)), handoff=ho)
        barrier()
        ho.close()
        leg["peer_handoff"] = hrun
    except Exception as e:
        leg["peer_handoff"] = {"error": f"{type(e).__name__}: {e}"}
    if rank == 0:
        leg["gpu_vs_reference_parareal"] = reduced_parity(local)
    return leg


def reduced_parity(local):
    """GPU Parareal(l) against the reference's own parareal::run at reduced size (fixture
    tests/golden/suspension.npz: 64 x 256, n = 4, 20 RK2 | 2 Euler per interval): max relative
    position difference over every 4th node of every boundary state (rod_position_metric)."""
    from paper_2604_12083_b200 import parareal as pr
    from paper_2604_12083_b200.scenario import ScenarioConfig, build_initial_state, make_scenario

    path = os.path.join(ROOT, "tests", "golden", "suspension.npz")
    if not os.path.exists(path):
        return {"error": "tests/golden/suspension.npz missing"}
    fx = np.load(path)
    rods, nodes, n, fine, coarse, _, stride = (int(v) for v in fx["meta"])
    sc = make_scenario(ScenarioConfig(rod_count=rods, nodes_per_rod=nodes, epsilon=float(fx["params"][0])))
    x0 = build_initial_state(sc)
    T = n * fine * float(fx["params"][1])
    out = {"workload": f"{rods} x {nodes}, n={n}, {fine} RK2 | {coarse} Euler per interval, pipelined, tol=1e-300 "
                       "(the reference ran parareal::run on the CPU; tests/golden/make_suspension.py)"}
    for l in range(1, n + 1):
        res = pr.run_gpu(pr.ParallelPlan(horizon=T, intervals=n, workers=n + 1, max_iterations=l, tolerance=1e-300,
                                         mode=pr.PIPELINED), sc, fine, coarse, x0, device=local)
        worst = 0.0
        for i in range(1, n + 1):
            got = res.states[i].reshape(-1, 12)[::stride, 0:3]
            want = fx[f"par_m1_l{l}_n{i}_pos"]
            worst = max(worst, float((np.sqrt(((got - want) ** 2).sum(1)) / np.sqrt((want ** 2).sum(1))).max()))
        out[f"l{l}"] = worst
    return out


def large_leg(args, local, dev, tr, world, rank):
    """BASELINE configs[4]: the 512 x 256 suspension (N = 131,072), pipelined Parareal with one
    slice per GPU, swept over the iteration count l.  Simulated RK2 steps/s, the speedup over
    the same fine propagation serially on one GPU, and the Parareal defect eta_tilde per l."""
    import torch

    from paper_2604_12083_b200 import parareal as pr
    from paper_2604_12083_b200.device import Context, dptr
    from paper_2604_12083_b200.scenario import ScenarioConfig, build_initial_state, make_scenario

    rods = int(os.environ.get("PSWIM_BENCH_LARGE_RODS", "512"))  # (tests shrink it)
    sc = make_scenario(ScenarioConfig(rod_count=rods, nodes_per_rod=256, epsilon=0.08, fine_dt=1e-6))
    x0 = build_initial_state(sc)
    fine, coarse = args.large_fine_steps, 1
    # serial fine reference time: one interval on rank 0 (x world intervals)
    serial = None
    barrier()
    if rank == 0:
        sctx = Context(local, sc)
        dx = torch.as_tensor(x0, device=dev)
        dout = torch.empty_like(dx)
        sctx.check(sctx.lib.pswim_propagate(sctx.handle, dptr(dx), 0.0, 1e-6, 1, 1, 0.0, dptr(dout)))  # warm-up
        torch.cuda.synchronize()
        t1 = time.perf_counter()
        sctx.check(sctx.lib.pswim_propagate(sctx.handle, dptr(dx), 0.0, fine * 1e-6, 1, fine, 0.0, dptr(dout)))
        torch.cuda.synchronize()
        serial = world * (time.perf_counter() - t1)
        sctx.close()
    barrier()
    warm = pr.ParallelPlan(t0=0.0, horizon=world * 1e-6, intervals=world, workers=world, max_iterations=1,
                           tolerance=1e-300, mode=pr.PIPELINED)
    pr.run_sliced_rank(warm, sc, 1, coarse, x0, local, transport=tr)  # contexts, kernels, plans
    sweep = []
    for l in range(1, min(world, args.large_max_iters) + 1):
        plan = pr.ParallelPlan(t0=0.0, horizon=world * fine * 1e-6, intervals=world, workers=world,
                               max_iterations=l, tolerance=1e-300, mode=pr.PIPELINED)
        barrier()
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        res = pr.run_sliced_rank(plan, sc, fine, coarse, x0, local, transport=tr)
        wall = reduce_max(res.report.wall_seconds, dev)
        sweep.append({"iterations": res.report.iterations_used, "value": world * fine / wall, "unit": "steps/s",
                      "wall_s": wall, "speedup_vs_serial_fine": (serial / wall) if serial else None,
                      "eta_tilde": res.report.eta_tilde})
    return {"metric": "simulated RK2 time-steps/s", "unit": "steps/s",
            "config": {"workload": f"pipelined Parareal, one slice per GPU, {rods} x 256 suspension (BASELINE configs[4])",
                       "points": rods * 256, "intervals": world, "fine_rk2_steps_per_interval": fine,
                       "coarse_euler_steps_per_interval": coarse},
            "serial_fine_s": serial, "iteration_sweep": sweep}


def hybrid_leg(args, sc, x0, local, dev, world, members):
    """Hybrid space x time: world / members Parareal slices, each propagated by a space group
    of `members` GPUs that shards every rhs's MRS (NCCL all-gather); slice hand-offs between
    same-index members."""
    import torch.distributed as dist

    from paper_2604_12083_b200 import parareal as pr

    rank = dist.get_rank()
    slices = world // members
    tg, sg = pr.hybrid_groups(world, members)
    groups = tg + sg + sg  # time, space (coarse), space (fine): every rank creates them in this order
    trs = _group_transports(local, groups)
    q, p = rank % members, rank // members
    t_tr, c_tr, f_tr = trs[q], trs[len(tg) + p], trs[len(tg) + len(sg) + p]
    fine_steps, coarse_steps = args.fine_steps, max(1, min(args.coarse_steps, args.fine_steps // 10))
    plan = pr.ParallelPlan(t0=0.0, horizon=slices * fine_steps * 1e-6, intervals=slices, workers=slices,
                           max_iterations=args.parareal_iters, tolerance=1e-300, mode=pr.PIPELINED)
    try:
        pr.run_sliced_rank(plan, sc, fine_steps, coarse_steps, x0, local, transport=t_tr, space=(c_tr, f_tr))
        barrier()
        t0 = time.perf_counter()
        res = pr.run_sliced_rank(plan, sc, fine_steps, coarse_steps, x0, local, transport=t_tr, space=(c_tr, f_tr))
        wall = reduce_max(res.report.wall_seconds, dev)
    finally:
        for tr in trs.values():
            _lib_destroy(tr)
    return {"metric": "simulated RK2 time-steps/s", "value": slices * fine_steps / wall, "unit": "steps/s",
            "config": {"workload": f"pipelined Parareal, {slices} slices x {members} GPUs per slice (MRS sharded "
                                   "inside each slice), 64 x 256 suspension", "fine_rk2_steps_per_interval": fine_steps,
                       "coarse_euler_steps_per_interval": coarse_steps, "iterations": res.report.iterations_used}}


def space_parallel_leg(sc, x0, local, dev, tr, world, steps=20):
    """Serial fine RK2 of the 64 x 256 suspension with the MRS sharded over the ranks (each
    rank its 256-target blocks, NCCL all-gather of (u, omega) per rhs; bitwise identical to
    one GPU): strong scaling of the time-step rate."""
    import torch

    from paper_2604_12083_b200.device import Context, dptr

    ctx = Context(local, sc)
    dx = torch.as_tensor(x0, device=dev)
    out = torch.empty_like(dx)
    L = ctx.lib
    ctx.check(L.pswim_propagate_sharded(ctx.handle, tr, dptr(dx), 0.0, 2e-6, 1, 2, 0.0, dptr(out)))  # warm-up
    barrier()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    ctx.check(L.pswim_propagate_sharded(ctx.handle, tr, dptr(dx), 0.0, steps * 1e-6, 1, steps, 0.0, dptr(out)))
    wall = reduce_max(time.perf_counter() - t0, dev)
    leg = {"metric": "simulated RK2 time-steps/s", "value": steps / wall, "unit": "steps/s", "scaling": "strong",
           "config": {"workload": "serial fine RK2, 64 x 256 suspension, MRS targets sharded over the GPUs "
                                  "(NCCL all-gather of u, omega per rhs)", "gpus": world, "steps": steps}}
    # the same with the all-gather fused into the MRS kernel epilogue over peer memory (IPC)
    try:
        import torch.distributed as dist

        from paper_2604_12083_b200.propagators import PeerGroup

        rank = dist.get_rank()
        g = PeerGroup(ctx, rank, world)
        handles = [None] * world
        dist.all_gather_object(handles, g.handle())
        g.connect(handles=handles)
        barrier()
        ctx.check(L.pswim_propagate_sharded_peer(ctx.handle, g.ptr, dptr(dx), 0.0, 2e-6, 1, 2, 0.0, dptr(out)))
        barrier()
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        ctx.check(L.pswim_propagate_sharded_peer(ctx.handle, g.ptr, dptr(dx), 0.0, steps * 1e-6, 1, steps, 0.0,
                                                 dptr(out)))
        wall = reduce_max(time.perf_counter() - t0, dev)
        barrier()
        g.close()
        leg["fused_peer_allgather"] = {"value": steps / wall, "unit": "steps/s",
                                       "kernel": "mrs_kernel<.., kPeer> epilogue stores (u, omega) into every "
                                                 "rank's HBM over NVLink (CUDA IPC) + system-scope arrivals"}
    except Exception as e:
        leg["fused_peer_allgather"] = {"error": f"{type(e).__name__}: {e}"}
    ctx.close()
    return leg


def flagellum_leg(args, local, dev):
    """BASELINE configs[0]: one 100-node flagellum, serial fine RK2 (dt = 1e-6): fused
    single-cluster propagate kernel vs the reference's own propagate on the host cores."""
    import torch

    from paper_2604_12083_b200.device import Context, dptr
    from paper_2604_12083_b200.scenario import ScenarioConfig, build_initial_state, make_scenario

    kw = dict(rod_count=1, nodes_per_rod=100)
    sc = make_scenario(ScenarioConfig(**kw))
    x0 = build_initial_state(sc)
    ctx = Context(local, sc)
    cs = ctx.lib.pswim_set_fused(ctx.handle, 16)  # a lone system: 16-CTA clusters
    dx = torch.as_tensor(x0, device=dev)
    out = torch.empty_like(dx)
    L = ctx.lib
    ctx.check(L.pswim_propagate(ctx.handle, dptr(dx), 0.0, 1e-5, 1, 10, 0.0, dptr(out)))
    steps = 20000
    st = ctx.torch_stream()
    a = torch.cuda.Event(enable_timing=True)
    b = torch.cuda.Event(enable_timing=True)
    with ClockSampler(local) as fclk:
        a.record(st)
        ctx.check(L.pswim_propagate(ctx.handle, dptr(dx), 0.0, steps * 1e-6, 1, steps, 0.0, dptr(out)))
        b.record(st)
        b.synchronize()
    gpu = steps / (a.elapsed_time(b) * 1e-3)
    leg = {"metric": "simulated RK2 time-steps/s", "value": gpu, "unit": "steps/s",
           "config": {"workload": "single flagellum, 1 x 100 nodes, serial fine RK2, dt=1e-6 (BASELINE configs[0])",
                      "steps": steps, "kernel": f"fused propagate, cluster of {cs} CTAs, 1 launch per interval"},
           "clocks": fclk.summary()}
    leg["latency_roofline"] = latency_roofline(ctx, sc, cs, gpu, fclk.summary())
    ctx.close()
    leg["parareal_1gpu"] = parareal_1gpu_leg(sc, x0, local)
    if not args.no_cpu:
        from oracle.pyoracle import LIB_PATHS, Oracle, Scenario as OS

        if os.path.exists(LIB_PATHS["ref"]):
            ref = Oracle("ref")
            osc = OS.make(**kw)
            csteps = 2000
            full = ref.max_threads_()
            rates = {}
            for threads in (full, 1):  # BASELINE §3: the OpenMP team and one thread (the faster one counts)
                ref.set_threads_(threads)
                t0 = time.perf_counter()
                ref.propagate(osc, x0, 0.0, csteps * 1e-6, 1, steps=csteps)
                rates[threads] = csteps / (time.perf_counter() - t0)
            ref.set_threads_(full)
            best = max(rates, key=rates.get)
            leg["cpu_baseline"] = {"value": rates[best], "unit": "steps/s", "cores": best, "kind": "reference",
                                   "sample": f"{csteps} RK2 steps of the same flagellum (reference propagate; best of "
                                             f"the {full}-thread OpenMP team and 1 thread)",
                                   "by_threads": {str(k): v for k, v in rates.items()}, "nproc": os.cpu_count()}
    return leg


def latency_roofline(ctx, sc, cs, steps_per_s, clocks):
    """Latency roofline of the fused small-system kernel: the per-rhs phases'
    floors measured live on this GPU by pswim_dev_latency_probe, each phase alone on an idle
    SM with the kernel's own decomposition -- the front-pass chain on one warp per SMSP, the
    MRS items (warps x sources per item), the in-order chunk reduction, the 16-CTA velocity
    exchange -- summed over the two rhs of an RK2 step, against the measured cycles per step."""
    import ctypes as C

    import math

    n = sc.total_nodes
    chunks = max(1, (n + 5) // 6)  # mrs_plan's single-block small-system plan (6 sources per chunk)
    tpc = (n + cs - 1) // cs
    warps = math.ceil(tpc * chunks / 32)
    ns = math.ceil(n / chunks)
    out = (C.c_double * 4)()
    rc = ctx.lib.pswim_dev_latency_probe(ctx.handle, ns, min(warps, 12), chunks, 6 * tpc, 6 * n, out)
    if rc != 0:
        return {"error": f"pswim_dev_latency_probe rc={rc}"}
    floor_rhs = sum(out)
    mhz = clocks.get("sm_mhz") or 1965.0
    measured = mhz * 1e6 / steps_per_s
    return {"bound": "latency", "unit": "cycles/RK2 step", "floor": 2 * floor_rhs, "measured": measured,
            "frac": 2 * floor_rhs / measured,
            "floor_per_rhs": {"front_chain": out[0], f"mrs_items_{warps}w_x_{ns}src": out[1],
                              f"chunk_reduction_{chunks}": out[2], f"exchange_cluster{cs}": out[3]},
            "note": "each phase timed alone on an idle SM (clock64, pswim_dev_latency_probe); measured = "
                    "SM clock / steps per s"}


def parareal_1gpu_leg(sc, x0, local, n=8, fine=1000, coarse=100):
    """Time-parallel on ONE B200: a small system leaves most SMs idle, so the n fine solves
    of a Parareal iteration run concurrently (fused cluster kernels on n+1 engine lanes).
    Simulated steps/s = n * fine / wall; eta = error vs the serial fine solution."""
    from paper_2604_12083_b200 import parareal as pr

    T = n * fine * 1e-6
    plan = pr.ParallelPlan(horizon=T, intervals=n, workers=n + 1, max_iterations=1, tolerance=1e-300,
                           mode=pr.PIPELINED)
    serial = pr.run_gpu(pr.ParallelPlan(horizon=T, intervals=n, workers=1, max_iterations=n, tolerance=1e-300),
                        sc, fine, coarse, x0, device=local)  # k = n: exact serial fine boundaries
    # serial fine wall time: the same n fine propagations back to back, in the fastest serial
    # configuration (16-CTA cluster, the flagellum leg's) -- the speedup denominator
    import torch

    from paper_2604_12083_b200.device import Context, dptr

    ctx = Context(local, sc)
    ctx.lib.pswim_set_fused(ctx.handle, 16)
    cur = torch.as_tensor(x0, device=f"cuda:{local}")
    out = torch.empty_like(cur)
    ctx.check(ctx.lib.pswim_propagate(ctx.handle, dptr(cur), 0.0, 10e-6, 1, 10, 0.0, dptr(out)))  # warm-up
    ctx.sync()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for i in range(n):
        ctx.check(ctx.lib.pswim_propagate(ctx.handle, dptr(cur), plan.boundary_time(i), plan.boundary_time(i + 1), 1,
                                          fine, 0.0, dptr(out)))
        cur, out = out, cur
    serial_wall = time.perf_counter() - t0
    ctx.close()
    out = {}
    for l in (1, 2):
        plan.max_iterations = l
        pr.run_gpu(plan, sc, fine, coarse, x0, device=local)  # warm-up
        with ClockSampler(local) as pclk:
            res = pr.run_gpu(plan, sc, fine, coarse, x0, reference=serial.states, device=local)
        out[f"clocks_l{l}"] = pclk.summary()
        out[f"l{l}"] = {"value": n * fine / res.report.wall_seconds, "unit": "steps/s",
                        "speedup_vs_serial_fine": serial_wall / res.report.wall_seconds, "eta": res.report.eta[-1]}
    return {"workload": f"pipelined Parareal on one B200, flagellum 1x100, n={n} intervals x {fine} RK2 "
                        f"(coarse {coarse} Euler), {n + 1} engine lanes", "serial_fine_steps_per_s": n * fine / serial_wall,
            "serial_fine_config": "the same n fine propagations back to back on a 16-CTA cluster (fastest serial)",
            **out}


def _hbm_peak() -> float:
    try:
        return float(json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))["hbm_gbs"])
    except Exception:
        return 6650.0  # B200_PROFILING.md fallback


_STAGED = {}  # transport pointer address -> StagedTransport (test-mode wire)


def _transport(local):
    """The rank's device transport over the whole world: NCCL, or (test mode) staged gloo."""
    from paper_2604_12083_b200 import parareal as pr

    if WIRE == "nccl":
        return pr.nccl_transport(local)
    st = pr.StagedTransport(local)
    _STAGED[C.addressof(st.ptr.contents)] = st
    return st.ptr


def _group_transports(local, groups):
    import torch.distributed as dist

    from paper_2604_12083_b200 import parareal as pr

    if WIRE == "nccl":
        return pr.nccl_group_transports(local, groups)
    out = {}
    rank = dist.get_rank()
    for gi, g in enumerate(groups):
        pg = dist.new_group(g)  # collective over the world, every rank in the same order
        if rank in g:
            st = pr.StagedTransport(local, pg)
            _STAGED[C.addressof(st.ptr.contents)] = st
            out[gi] = st.ptr
    return out


def _lib_destroy(tr):
    from paper_2604_12083_b200 import _lib

    st = _STAGED.pop(C.addressof(tr.contents), None)
    if st is not None:
        st.close()
    else:
        _lib.lib().pswim_nccl_transport_destroy(tr)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=100)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--ref-targets", type=int, default=N_POINTS,
                    help="targets of the CPU legs (default: all, the full N x N evaluation)")
    ap.add_argument("--fine-steps", type=int, default=1000, help="RK2 steps per interval, N>1 Parareal legs")
    ap.add_argument("--coarse-steps", type=int, default=100, help="Euler steps per interval, N>1 Parareal legs")
    ap.add_argument("--serial-steps", type=int, default=200, help="RK2 steps of the N=1 serial fine leg")
    ap.add_argument("--parareal-iters", type=int, default=1, help="iterations of the hybrid space x time leg")
    ap.add_argument("--no-cpu", action="store_true", help="skip the CPU baseline (profiling runs)")
    ap.add_argument("--no-steps", action="store_true", help="skip the time-step leg")
    ap.add_argument("--no-sweep", action="store_true", help="skip the N = 64k / 131k MRS points")
    ap.add_argument("--no-large", action="store_true", help="skip the N > 1 large-suspension sweep (configs[4])")
    ap.add_argument("--large-fine-steps", type=int, default=8, help="RK2 steps per interval, large sweep")
    ap.add_argument("--large-max-iters", type=int, default=4, help="largest Parareal iteration count swept")
    ap.add_argument("--wire", default="nccl", choices=["nccl", "gloo"],
                    help="N>1 transport; gloo = test mode (ranks may share one GPU, staged host transports)")
    args = ap.parse_args()
    global WIRE
    WIRE = args.wire
    if args.warmup < 3:
        args.warmup = 3
    if args.impl == "reference":
        run_reference_arm(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
