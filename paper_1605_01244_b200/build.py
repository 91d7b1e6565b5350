"""Build libvfnfft.so in-tree with nvcc for sm_100a (no torch JIT cache).

Every translation unit is compiled to an object in parallel, then linked
(static cudart; cuFFT from the CUDA toolkit via rpath)."""

from __future__ import annotations

import concurrent.futures as cf
import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(HERE, "csrc")
OBJ = os.path.join(HERE, "build")
LIB = os.path.join(HERE, "libvfnfft.so")
LIB_CHECKS = os.path.join(HERE, "libvfnfft_checks.so")
SOURCES = ["vfn_host.cpp", "vfn_stage.cpp", "vfn_kernels.cu", "vfn_gather.cu", "vfn_gather_tc.cu", "vfn_rect.cu",
           "vfn_direct.cu", "vfn_util.cu", "vfn_tube.cu", "vfn_io.cpp", "vfn_io_kernels.cu", "vfn_shard.cu", "vfn_zgemm.cu", "vfn_rect_nufft.cu", "vfn_sort.cu", "vfn_api.cu"]
CUDA_HOME = os.environ.get("CUDA_HOME", "/usr/local/cuda")
NVCC = os.path.join(CUDA_HOME, "bin", "nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
FLAGS = [*ARCH, "-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC"]


def _deps():
    hdrs = [os.path.join(CSRC, h) for h in os.listdir(CSRC) if h.endswith((".cuh", ".h"))]
    hdrs.append(os.path.join(os.path.dirname(HERE), "include", "vfnfft.h"))
    return hdrs


def _compile(src: str, verbose: bool, checks: bool = False) -> tuple[str, subprocess.CompletedProcess]:
    obj = os.path.join(OBJ + ("_checks" if checks else ""), os.path.splitext(src)[0] + ".o")
    cmd = [NVCC, *FLAGS, *(["-DVFN_CHECKS"] if checks else []), "-c", os.path.join(CSRC, src), "-o", obj]
    if verbose:
        cmd[1:1] = ["-Xptxas", "-v"]
    return obj, subprocess.run(cmd, capture_output=True, text=True)


def build(verbose: bool = False, force: bool = False, checks: bool = False) -> str:
    """checks=True: the debug variant libvfnfft_checks.so with device-side
    bounds checks (VFN_DCHECK); select it at run time with VFN_LIB=checks."""
    lib = LIB_CHECKS if checks else LIB
    srcs = [os.path.join(CSRC, s) for s in SOURCES]
    if not force and os.path.exists(lib):
        t = os.path.getmtime(lib)
        if all(os.path.getmtime(d) <= t for d in srcs + _deps()):
            return lib
    os.makedirs(OBJ + ("_checks" if checks else ""), exist_ok=True)
    workers = max(1, min(len(SOURCES), os.cpu_count() or 1))
    with cf.ThreadPoolExecutor(workers) as ex:
        results = list(ex.map(lambda s: _compile(s, verbose, checks), SOURCES))
    failed = False
    for (obj, res), src in zip(results, SOURCES):
        if verbose or res.returncode != 0:
            sys.stderr.write(res.stdout + res.stderr)
        failed |= res.returncode != 0
    if failed:
        raise RuntimeError("nvcc build of libvfnfft.so failed")
    link = [NVCC, *ARCH, "-shared", "--cudart", "static", "-o", lib, *[o for o, _ in results],
            "-L" + os.path.join(CUDA_HOME, "lib64"), "-lcufft",
            "-Xlinker", "-rpath=" + os.path.join(CUDA_HOME, "lib64")]
    res = subprocess.run(link, capture_output=True, text=True)
    if verbose or res.returncode != 0:
        sys.stderr.write(res.stdout + res.stderr)
    if res.returncode != 0:
        raise RuntimeError("linking libvfnfft.so failed")
    return lib


if __name__ == "__main__":
    print(build(verbose="-v" in sys.argv, force=True, checks="--checks" in sys.argv))
