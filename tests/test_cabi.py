"""The C-ABI library loads and exports every symbol include/pswim_c.h declares (no GPU)."""
import os
import re

from paper_2604_12083_b200 import _lib

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def header_functions():
    text = open(os.path.join(ROOT, "include", "pswim_c.h")).read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    names = set(re.findall(r"\b(pswim_[a-z0-9_]+)\s*\(", text))
    types = set(re.findall(r"typedef\s+int\s+\(\*\s*(pswim_[a-z0-9_]+)\)", text))
    return sorted(names - types)


def test_library_exports_every_header_symbol():
    L = _lib.lib()
    names = header_functions()
    assert len(names) > 30
    missing = [n for n in names if not hasattr(L, n)]
    assert not missing, missing
    assert set(names) == set(_lib.SIGNATURES), set(names) ^ set(_lib.SIGNATURES)


def test_library_is_sm100a_cuda():
    import subprocess

    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "--list-elf", _lib.LIB_PATH], capture_output=True, text=True)
    assert "sm_100a" in out.stdout


def test_version_and_host_entry_points():
    import ctypes as C

    import numpy as np

    L = _lib.lib()
    assert b"sm_100a" in L.pswim_version()
    sc = _lib.Scenario()
    L.pswim_scenario_defaults(C.byref(sc))
    assert sc.nodes_per_rod == 51 and sc.b1 == 2.0
    r = _lib.Resolved()
    assert L.pswim_scenario_resolve(C.byref(sc), C.byref(r)) == 0
    assert abs(r.epsilon - 4 * r.ds) < 1e-15
    out = np.zeros(12 * 51)
    assert L.pswim_build_initial_state(C.byref(sc), out.ctypes.data_as(C.POINTER(C.c_double))) == 0
    sc.nodes_per_rod = 2
    assert L.pswim_scenario_resolve(C.byref(sc), C.byref(r)) == 1
