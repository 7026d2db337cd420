"""Drop-in A/B: the reference's OWN parareal::run (compiled unmodified into
oracle/_ref/ab_parareal) driving the B200 propagators through include/pswim/pintswim_gpu.hpp,
against the same engine with the reference CPU propagators (acceptance criterion 1 shape)."""
import json
import os
import subprocess

import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
AB = os.path.join(ROOT, "oracle", "_ref", "ab_parareal")


def test_reference_engine_drives_gpu_propagators(gpu):
    if not os.path.exists(AB):
        pytest.skip("oracle/_ref/ab_parareal not built (needs /root/reference at build time)")
    r = subprocess.run([AB], capture_output=True, text=True, timeout=600)
    print(r.stdout, r.stderr[-2000:])
    line = json.loads(r.stdout.strip().splitlines()[-1])
    assert r.returncode == 0, line
    assert line["ok"] and line["max_position_metric_gpu_vs_cpu"] <= 1e-10
    assert line["iterations_cpu"] == line["iterations_gpu"] and line["gpu_bitwise_modes_workers"]
