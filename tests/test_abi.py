"""The C ABI library builds for sm_100a, loads without a GPU and exports every
entry point include/vfnfft.h declares (no compute calls here)."""

import ctypes
import os
import re
import subprocess

import pytest

from conftest import REPO

HEADER = os.path.join(REPO, "include", "vfnfft.h")


def declared_functions():
    text = open(HEADER).read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"^\s*(?:const\s+)?\w+\*?\s+\**(vfn_\w+)\s*\(", text, flags=re.M)))


def test_header_declares_the_boundary():
    names = declared_functions()
    for required in ("vfn_plan_create", "vfn_plan_eval", "vfn_plan_destroy", "vfn_rect_eval",
                     "vfn_map_to_torus", "vfn_plan_bin", "vfn_direct_eval", "vfn_last_error"):
        assert required in names


def test_library_exports_every_declared_symbol():
    from paper_1605_01244_b200 import _lib

    lib = _lib.load()
    for name in declared_functions():
        assert hasattr(lib, name), name
        assert name in _lib.SIGNATURES, f"{name} has no ctypes signature"
    assert lib.vfn_version().decode().startswith("vfnfft")


def test_exported_symbols_match_header_exactly():
    from paper_1605_01244_b200 import _lib

    out = subprocess.run(["nm", "-D", "--defined-only", _lib.LIB_PATH], capture_output=True, text=True).stdout
    exported = sorted({l.split()[-1] for l in out.splitlines() if l.split()[-1].startswith("vfn_")})
    assert exported == declared_functions()


def test_sass_is_sm100a():
    from paper_1605_01244_b200 import _lib

    res = subprocess.run(["cuobjdump", "--list-elf", _lib.LIB_PATH], capture_output=True, text=True)
    if res.returncode != 0:
        pytest.skip("cuobjdump unavailable")
    assert "sm_100a" in res.stdout


def test_invalid_arguments_fail_without_a_gpu():
    from paper_1605_01244_b200 import _lib

    lib = _lib.load()
    h = ctypes.c_void_p()
    st = lib.vfn_plan_create(ctypes.byref(h), 0, _lib.i64x3((8, 8, 8)), _lib.f64x3((0, 0, 0)),
                             _lib.f64x3((1, 1, 1)), 2.0, 0, ctypes.c_void_p(1), 0, None)
    assert st == _lib.VFN_ERR_INVALID
    assert "cutoff" in lib.vfn_last_error().decode()
    st = lib.vfn_plan_create(ctypes.byref(h), 0, _lib.i64x3((10, 10, 10)), _lib.f64x3((0, 0, 0)),
                             _lib.f64x3((1, 1, 1)), 1.5, 6, ctypes.c_void_p(1), 0, None)
    assert st == _lib.VFN_ERR_INVALID
    assert "even" in lib.vfn_last_error().decode()


def test_warp_threshold_matches_header():
    """The Python launch accounting uses the header's VFN_WARP_MAX_M."""
    import re

    from paper_1605_01244_b200 import nufft

    hdr = open(os.path.join(REPO, "include", "vfnfft.h")).read()
    assert int(re.search(r"#define VFN_WARP_MAX_M (\d+)", hdr).group(1)) == nufft.WARP_MAX_M
