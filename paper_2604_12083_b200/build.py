"""In-tree build of libpswim.so (CUDA sm_100a + C++ host runtime) with nvcc.

    python -m paper_2604_12083_b200.build        # or __graft_entry__.build()

Each translation unit is compiled in parallel with
``-gencode arch=compute_100a,code=sm_100a -lineinfo -O3`` and linked into
paper_2604_12083_b200/libpswim.so, next to this file, so it travels with the repo snapshot.
ptxas resource usage (registers / spills / smem per kernel) is written to build/ptxas.log.
"""
from __future__ import annotations

import concurrent.futures as cf
import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
CSRC = os.path.join(HERE, "csrc")
BUILD = os.path.join(ROOT, "build", "pswim")
LIB = os.path.join(HERE, "libpswim.so")
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
HOST_CXX = "/usr/bin/g++"
# -fmad=false: no automatic FMA contraction.  Contraction decisions depend on the inlining
# context (e.g. whether a product has other uses), so the same device routine inlined into
# two kernels could round differently; the fused small-system kernel and the launched
# kernels must agree bitwise.  Every FMA on the path is an explicit fma() call instead.
COMMON = ["-O3", "-std=c++17", "-lineinfo", "-fmad=false", "-Xcompiler", "-fPIC", "-ccbin", HOST_CXX,
          "-I" + os.path.join(ROOT, "include")]


def _sources():
    return sorted(f for f in os.listdir(CSRC) if f.endswith((".cu", ".cpp")))


def _compile(src: str) -> tuple[str, str]:
    obj = os.path.join(BUILD, src + ".o")
    path = os.path.join(CSRC, src)
    deps = [path] + [os.path.join(CSRC, h) for h in os.listdir(CSRC) if h.endswith((".h", ".cuh"))]
    deps.append(os.path.join(ROOT, "include", "pswim_c.h"))
    deps.append(os.path.join(ROOT, "include", "pswim", "device_math.cuh"))
    if os.path.exists(obj) and os.path.getmtime(obj) >= max(os.path.getmtime(d) for d in deps):
        return obj, ""
    cmd = [NVCC, *ARCH, *COMMON, "-Xptxas", "-v", "-c", path, "-o", obj]
    if src.endswith(".cpp"):
        cmd = [NVCC, *ARCH, *COMMON, "-x", "cu", "-c", path, "-o", obj]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError(f"nvcc failed for {src}:\n{r.stdout}\n{r.stderr}")
    return obj, r.stderr


def build(verbose: bool = False) -> str:
    os.makedirs(BUILD, exist_ok=True)
    # objects are rebuilt when the compile flags change, not only when sources do
    stamp = os.path.join(BUILD, "flags.txt")
    flags = " ".join([NVCC, *ARCH, *COMMON])
    if not os.path.exists(stamp) or open(stamp).read() != flags:
        for f in os.listdir(BUILD):
            if f.endswith(".o"):
                os.remove(os.path.join(BUILD, f))
        with open(stamp, "w") as fh:
            fh.write(flags)
    srcs = _sources()
    with cf.ThreadPoolExecutor(max_workers=min(8, len(srcs))) as ex:
        results = list(ex.map(_compile, srcs))
    objs = [o for o, _ in results]
    log = "".join(f"== {s}\n{l}" for s, (_, l) in zip(srcs, results) if l)
    if log:
        with open(os.path.join(ROOT, "build", "ptxas.log"), "w") as fh:
            fh.write(log)
    newest = max(os.path.getmtime(o) for o in objs)
    if not os.path.exists(LIB) or os.path.getmtime(LIB) < newest:
        cmd = [NVCC, *ARCH, "-shared", "-ccbin", HOST_CXX, "-o", LIB, *objs,
               "-lpthread", "-ldl"]
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            raise RuntimeError(f"link failed:\n{r.stdout}\n{r.stderr}")
    if verbose:
        print(f"built {LIB}")
    return LIB


if __name__ == "__main__":
    build(verbose=True)
    sys.exit(0)
