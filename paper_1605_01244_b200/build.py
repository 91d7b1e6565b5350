"""Build libvfnfft.so in-tree with nvcc for sm_100a (no torch JIT cache)."""

from __future__ import annotations

import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(HERE, "csrc")
LIB = os.path.join(HERE, "libvfnfft.so")
SOURCES = ["vfn_host.cpp", "vfn_kernels.cu", "vfn_gather.cu", "vfn_gather_m6.cu", "vfn_rect.cu", "vfn_direct.cu", "vfn_util.cu", "vfn_tube.cu", "vfn_api.cu"]
CUDA_HOME = os.environ.get("CUDA_HOME", "/usr/local/cuda")
NVCC = os.path.join(CUDA_HOME, "bin", "nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]


def build(verbose: bool = False, force: bool = False) -> str:
    srcs = [os.path.join(CSRC, s) for s in SOURCES]
    deps = srcs + [os.path.join(CSRC, h) for h in os.listdir(CSRC) if h.endswith((".cuh", ".h"))]
    deps.append(os.path.join(os.path.dirname(HERE), "include", "vfnfft.h"))
    if not force and os.path.exists(LIB):
        t = os.path.getmtime(LIB)
        if all(os.path.getmtime(d) <= t for d in deps):
            return LIB
    cmd = [
        NVCC, *ARCH, "-O3", "-lineinfo", "-std=c++17", "-shared", "-Xcompiler", "-fPIC",
        "-Xptxas", "-v" if verbose else "-O3",
        "--cudart", "static",
        "-o", LIB, *srcs,
        "-L" + os.path.join(CUDA_HOME, "lib64"), "-lcufft", "-lcublas",
        "-Xlinker", "-rpath=" + os.path.join(CUDA_HOME, "lib64"),
    ]
    if verbose:
        print(" ".join(cmd))
    res = subprocess.run(cmd, capture_output=True, text=True)
    if verbose or res.returncode != 0:
        sys.stderr.write(res.stdout + res.stderr)
    if res.returncode != 0:
        raise RuntimeError("nvcc build of libvfnfft.so failed")
    return LIB


if __name__ == "__main__":
    build(verbose="-v" in sys.argv, force=True)
    print(LIB)
