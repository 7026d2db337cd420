"""The bench's N > 1 code path end to end on one B200: torchrun with 2 and 4 ranks sharing
cuda:0, `--wire gloo` (NCCL refuses two ranks on one device, so the slice hand-offs,
all-gathers and metric allreduce go through pswim_staged_transport over gloo).  Exercises
the time-sliced Parareal leg, the space-parallel legs (collective and fused peer all-gather
over CUDA IPC) and, at 4 ranks, the hybrid space x time leg, and checks the JSON line."""
import json
import os
import socket
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


@pytest.mark.parametrize("world", [2, 4])
def test_bench_multirank_gloo_wire(gpu, world):
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={world}",
           "--master-addr", "127.0.0.1", f"--master-port={_port()}", os.path.join(ROOT, "bench.py"),
           "--gpus", str(world), "--steps", "3", "--warmup", "3", "--wire", "gloo", "--fine-steps", "4",
           "--no-cpu"]
    env = dict(os.environ, PSWIM_BENCH_LARGE_RODS="4")  # the configs[4] sweep code path, shrunk
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=900, cwd=ROOT, env=env)
    lines = [l for l in r.stdout.splitlines() if l.startswith("{")]
    assert r.returncode == 0 and lines, r.stdout[-3000:] + r.stderr[-3000:]
    d = json.loads(lines[-1])
    assert d["n_gpus"] == world and d["value"] > 0
    ts = d["time_steps"]
    assert "error" not in ts and ts["value"] > 0 and ts["config"]["intervals"] == world, ts
    assert ts["speedup_vs_serial_fine"] > 0
    sw = ts["iteration_sweep"]
    assert [x["iterations"] for x in sw] == list(range(1, min(world, 4) + 1)), sw
    assert all(x["eta_vs_serial_fine"] is not None for x in sw)
    assert sw[-1]["eta_vs_serial_fine"] <= sw[0]["eta_vs_serial_fine"]
    assert "error" not in ts["peer_handoff"], ts["peer_handoff"]
    assert ts["tolerance_run"]["converged"]
    gp = ts["gpu_vs_reference_parareal"]
    assert "error" not in gp and all(gp[f"l{l}"] < 1e-10 for l in range(1, 5)), gp
    sp = ts["space_parallel"]
    assert "error" not in sp and sp["value"] > 0, sp
    assert "error" not in sp["fused_peer_allgather"], sp
    lg = ts["large_suspension"]
    assert "error" not in lg and len(lg["iteration_sweep"]) == min(world, 4), lg
    assert all(x["value"] > 0 and x["iterations"] == i + 1 for i, x in enumerate(lg["iteration_sweep"]))
    if world >= 4:
        hy = ts["hybrid_space_time"]
        assert "error" not in hy and hy["value"] > 0 and hy["config"]["iterations"] == 1, hy
