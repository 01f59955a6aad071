"""Build recipe of the CUDA product (libh2d.so) for sm_100a.

Bit-exactness against the reference needs IEEE fp64 without contraction:
-fmad=false (no DFMA fusion of a*b+c), no fast-math; division and sqrt in
double precision are IEEE round-to-nearest in CUDA by default.
"""
import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(HERE, "csrc")
OUT = os.path.join(HERE, "libh2d.so")
SOURCES = ["h2d_kernels.cu", "h2d_scalar.cu", "h2d_capi.cu", "hydro_api.cpp", "hydro_harness.cpp", "h2d_io.cpp"]
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
FLAGS = ["-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-lineinfo", "-fmad=false", "-std=c++17",
         "-Xcompiler", "-fPIC", "-Xcompiler", "-ffp-contract=off", "-Xptxas", "-v"]


def build(verbose: bool = False) -> str:
    srcs = [os.path.join(CSRC, s) for s in SOURCES]
    deps = srcs + [os.path.join(CSRC, h) for h in os.listdir(CSRC) if h.endswith((".cuh", ".h"))]
    deps.append(os.path.join(HERE, "..", "include", "h2d.h"))
    deps.append(os.path.join(HERE, "..", "include", "hydro", "b200.hpp"))
    if os.path.exists(OUT) and all(os.path.getmtime(OUT) >= os.path.getmtime(d) for d in deps):
        return OUT
    cmd = [NVCC, *FLAGS, "-I" + os.path.join(HERE, "..", "include"), "-shared", "-o", OUT + ".tmp", *srcs,
           "-lcudart"]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        sys.stderr.write(r.stdout + r.stderr)
        raise RuntimeError("nvcc failed building libh2d.so")
    if verbose:
        sys.stderr.write(r.stderr)
    os.replace(OUT + ".tmp", OUT)
    return OUT


if __name__ == "__main__":
    print(build(verbose="-v" in sys.argv))
