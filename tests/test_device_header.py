"""The public device header include/pswim/device_math.cuh (reference rotation.hpp:34's
sqrt_rotation as a __device__ function) is self-contained: a foreign translation unit that
includes only it compiles for sm_100a and emits the routine (no GPU needed)."""
import os
import subprocess
import tempfile

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")

SRC = r'''
#include <pswim/device_math.cuh>
__global__ void user_kernel(const double* r9, double* s9, int n) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n) pswim_sqrt_rotation_dev(r9 + 9 * i, s9 + 9 * i);
}
__global__ void user_kernel_m33(const double* r9, double* out, int n) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    pswim::m33 r;
    for (int k = 0; k < 9; ++k) r.m[k] = r9[9 * i + k];
    const pswim::m33 s = pswim::sqrt_rotation(r);
    const pswim::m33 s2 = pswim::mm(s, s);  // S^2 = R
    for (int k = 0; k < 9; ++k) out[9 * i + k] = s2.m[k];
}
'''


def test_public_device_header_compiles_standalone():
    with tempfile.TemporaryDirectory() as d:
        src = os.path.join(d, "user.cu")
        open(src, "w").write(SRC)
        obj = os.path.join(d, "user.o")
        r = subprocess.run([NVCC, "-gencode", "arch=compute_100a,code=sm_100a", "-fmad=false", "-O3",
                            "-I" + os.path.join(ROOT, "include"), "-c", src, "-o", obj],
                           capture_output=True, text=True)
        assert r.returncode == 0, r.stderr
        sass = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "-sass", obj], capture_output=True, text=True).stdout
        assert "user_kernel" in sass and "MUFU.RSQ64H" in sass  # the rsqrt-based half-angle sqrt
