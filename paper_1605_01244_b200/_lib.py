"""ctypes binding of libvfnfft.so (the C ABI declared in include/vfnfft.h).

The library is built in-tree by `paper_1605_01244_b200/build.py` (called from
`__graft_entry__.build()`).  There is no fallback: if the shared library is
missing or cannot be loaded, importing the evaluators raises.
"""

from __future__ import annotations

import ctypes
import os

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
# VFN_LIB=checks loads the debug build with device-side bounds checks
# (python paper_1605_01244_b200/build.py --checks)
LIB_PATH = os.path.join(HERE, "libvfnfft_checks.so" if os.environ.get("VFN_LIB") == "checks" else "libvfnfft.so")

VFN_OK = 0
VFN_ERR_INVALID = -1
VFN_ERR_OUTSIDE = -2
VFN_ERR_IO = -7

_c_i64_3 = ctypes.c_int64 * 3
_c_f64_3 = ctypes.c_double * 3
_vp = ctypes.c_void_p
_cp = ctypes.c_char_p


class SnapshotInfo(ctypes.Structure):
    """vfn_snapshot_info (include/vfnfft.h): the SFS1 header fields."""

    _fields_ = [("a", ctypes.c_double * 3), ("b", ctypes.c_double * 3),
                ("shape", ctypes.c_int64 * 3), ("mirror", ctypes.c_int * 3),
                ("time", ctypes.c_double)]

# name -> (restype, argtypes); mirrors include/vfnfft.h
SIGNATURES = {
    "vfn_version": (ctypes.c_char_p, []),
    "vfn_last_error": (ctypes.c_char_p, []),
    "vfn_plan_create": (
        ctypes.c_int,
        [ctypes.POINTER(_vp), ctypes.c_int, _c_i64_3, _c_f64_3, _c_f64_3, ctypes.c_double,
         ctypes.c_int, _vp, ctypes.c_int, _vp],
    ),
    "vfn_plan_eval": (
        ctypes.c_int,
        [_vp, _vp, ctypes.c_int64, _vp, ctypes.c_int, ctypes.POINTER(ctypes.c_int64), _vp],
    ),
    "vfn_plan_destroy": (ctypes.c_int, [_vp]),
    "vfn_plan_info": (ctypes.c_int, [_vp, _c_i64_3, ctypes.POINTER(ctypes.c_double)]),
    "vfn_plan_grid": (ctypes.c_int, [_vp, _vp]),
    "vfn_plan_bin": (
        ctypes.c_int,
        [_vp, _vp, ctypes.c_int64, _vp, _vp, ctypes.c_int, ctypes.POINTER(ctypes.c_int64), _vp],
    ),
    "vfn_map_to_torus": (
        ctypes.c_int,
        [ctypes.c_int, _c_f64_3, _c_f64_3, _vp, ctypes.c_int64, _vp, ctypes.c_int, _vp],
    ),
    "vfn_rect_eval": (
        ctypes.c_int,
        [ctypes.c_int, _c_i64_3, _c_f64_3, _c_f64_3, _vp, _vp, ctypes.c_int64, _vp,
         ctypes.c_int64, _vp, ctypes.c_int64, _vp, ctypes.c_int, _vp],
    ),
    "vfn_rect_eval_nufft": (
        ctypes.c_int,
        [ctypes.c_int, _c_i64_3, _c_f64_3, _c_f64_3, _vp, _vp, ctypes.c_int64, _vp,
         ctypes.c_int64, _vp, ctypes.c_int64, ctypes.c_double, ctypes.c_int, _vp, ctypes.c_int, _vp],
    ),
    "vfn_direct_eval": (
        ctypes.c_int,
        [ctypes.c_int, _c_i64_3, _c_f64_3, _c_f64_3, _vp, _vp, ctypes.c_int64, _vp,
         ctypes.c_int, ctypes.POINTER(ctypes.c_int64), _vp],
    ),
    "vfn_plan_set_gather": (ctypes.c_int, [_vp, ctypes.c_int]),
    "vfn_plan_set_box": (ctypes.c_int, [_vp, ctypes.c_int]),
    "vfn_plan_key_shift": (ctypes.c_int, [_vp, ctypes.c_int64, ctypes.POINTER(ctypes.c_int)]),
    "vfn_plan_set_graphs": (ctypes.c_int, [_vp, ctypes.c_int]),
    "vfn_plan_geometry": (
        ctypes.c_int, [_vp, ctypes.c_int64, ctypes.c_int * 3, ctypes.c_int * 3]
    ),
    "vfn_bench_fp64_peak": (
        ctypes.c_int,
        [ctypes.c_int, ctypes.c_double, ctypes.POINTER(ctypes.c_double), ctypes.POINTER(ctypes.c_double)],
    ),
    "vfn_decompose": (
        ctypes.c_int,
        [ctypes.c_int, _vp, _c_i64_3, _c_f64_3, _c_f64_3, ctypes.c_int * 3, _vp, ctypes.c_int, _vp],
    ),
    "vfn_synthesize": (
        ctypes.c_int,
        [ctypes.c_int, _vp, _c_i64_3, _c_f64_3, _c_f64_3, _vp, ctypes.c_int, _vp],
    ),
    "vfn_tube_eval": (
        ctypes.c_int,
        [ctypes.POINTER(_vp), ctypes.c_int, _vp, _c_i64_3, _c_f64_3, _c_f64_3, ctypes.c_int * 3,
         _vp, ctypes.c_int, ctypes.c_int, ctypes.c_double, ctypes.c_double, ctypes.c_int,
         ctypes.POINTER(ctypes.c_int64), ctypes.POINTER(ctypes.c_int), _vp],
    ),
    "vfn_tube_copy": (ctypes.c_int, [_vp, _vp, _vp, _vp]),
    "vfn_tube_destroy": (ctypes.c_int, [_vp]),
    "vfn_snapshot_info_read": (ctypes.c_int, [_cp, ctypes.POINTER(SnapshotInfo)]),
    "vfn_snapshot_read": (
        ctypes.c_int,
        [_cp, ctypes.POINTER(SnapshotInfo), _vp, ctypes.c_int64, ctypes.c_int, ctypes.c_int, _vp],
    ),
    "vfn_snapshot_write": (
        ctypes.c_int, [_cp, ctypes.POINTER(SnapshotInfo), _vp, ctypes.c_int, ctypes.c_int, _vp]
    ),
    "vfn_csv_read": (
        ctypes.c_int,
        [_cp, ctypes.POINTER(_vp), ctypes.POINTER(ctypes.c_int64), ctypes.POINTER(ctypes.c_int)],
    ),
    "vfn_table_name": (ctypes.c_int, [_vp, ctypes.c_int, ctypes.POINTER(_cp)]),
    "vfn_table_column": (ctypes.c_int, [_vp, ctypes.c_int, _vp]),
    "vfn_table_points": (
        ctypes.c_int, [_vp, ctypes.c_int * 3, _vp, ctypes.c_int, ctypes.c_int, _vp]
    ),
    "vfn_table_destroy": (ctypes.c_int, [_vp]),
    "vfn_csv_write": (
        ctypes.c_int,
        [_cp, _vp, ctypes.c_int64, ctypes.c_int, ctypes.POINTER(_cp), ctypes.POINTER(_vp),
         ctypes.POINTER(ctypes.c_int64), ctypes.POINTER(ctypes.c_int)],
    ),
    "vfn_density": (
        ctypes.c_int, [ctypes.c_int, _vp, ctypes.c_int64, _vp, ctypes.c_int, _vp]
    ),
    "vfn_field_write": (
        ctypes.c_int,
        [_cp, _cp, _cp, _cp, _cp, _c_i64_3, _vp * 3, _vp, _vp, ctypes.c_int, ctypes.c_double,
         ctypes.c_int, ctypes.c_int, _vp],
    ),
    "vfn_vtk_write": (
        ctypes.c_int,
        [_cp, _cp, _c_i64_3, _vp * 3, ctypes.c_int, ctypes.POINTER(_cp), ctypes.POINTER(_vp),
         ctypes.c_int, ctypes.c_int, _vp],
    ),
    "vfn_plan_part_keys": (
        ctypes.c_int, [_vp, _vp, ctypes.c_int64, ctypes.c_int64, ctypes.c_int64, _vp, _vp]
    ),
    "vfn_plan_partition": (
        ctypes.c_int,
        [_vp, _vp, ctypes.c_int64, ctypes.c_int64, _vp, ctypes.c_int, _vp, _vp, _vp,
         ctypes.POINTER(ctypes.c_int64), _vp],
    ),
    "vfn_plan_partition_count": (
        ctypes.c_int,
        [_vp, _vp, ctypes.c_int64, ctypes.c_int64, _vp, ctypes.c_int, ctypes.POINTER(ctypes.c_int64),
         ctypes.POINTER(ctypes.c_int64), _vp],
    ),
    "vfn_plan_partition_scatter_peers": (
        ctypes.c_int,
        [_vp, _vp, ctypes.c_int64, ctypes.c_int, ctypes.POINTER(ctypes.c_int64), ctypes.POINTER(_vp),
         ctypes.POINTER(_vp), _vp],
    ),
    "vfn_gather_values": (ctypes.c_int, [ctypes.c_int, _vp, _vp, ctypes.c_int64, _vp, _vp]),
    "vfn_plan_decide": (
        ctypes.c_int,
        [_vp, ctypes.c_int64, _vp, ctypes.c_int, ctypes.POINTER(ctypes.c_int), ctypes.POINTER(ctypes.c_int), _vp],
    ),
    "vfn_plan_eval_to_peers": (
        ctypes.c_int,
        [_vp, _vp, ctypes.c_int64, _vp, ctypes.c_int, ctypes.POINTER(ctypes.c_int64), ctypes.POINTER(_vp),
         ctypes.POINTER(ctypes.c_int64), _vp],
    ),
    "vfn_ipc_alloc": (ctypes.c_int, [ctypes.c_int, ctypes.c_int64, ctypes.POINTER(_vp), ctypes.c_ubyte * 64]),
    "vfn_ipc_open": (ctypes.c_int, [ctypes.c_int, ctypes.c_ubyte * 64, ctypes.POINTER(_vp)]),
    "vfn_ipc_close": (ctypes.c_int, [ctypes.c_int, _vp]),
    "vfn_ipc_free": (ctypes.c_int, [ctypes.c_int, _vp]),
    "vfn_copy_device": (ctypes.c_int, [ctypes.c_int, _vp, _vp, ctypes.c_int64, _vp]),
    "vfn_plan_build_timing": (ctypes.c_int, [_vp, ctypes.c_float * 5]),
    "vfn_pool_release": (ctypes.c_int, [ctypes.c_int]),
    "vfn_plan_last_timing": (
        ctypes.c_int, [_vp, ctypes.POINTER(ctypes.c_float), ctypes.POINTER(ctypes.c_float)]
    ),
}

_lib = None


def load() -> ctypes.CDLL:
    """Load libvfnfft.so (once).  Raises if it is absent — no CPU fallback."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise ImportError(
            f"{LIB_PATH} is missing; build it with `python -c 'import __graft_entry__ as g; g.build()'`"
        )
    lib = ctypes.CDLL(LIB_PATH)
    for name, (res, args) in SIGNATURES.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    _lib = lib
    return lib


class VfnError(RuntimeError):
    pass


def check(status: int) -> None:
    if status == VFN_OK:
        return
    msg = load().vfn_last_error().decode(errors="replace")
    if status in (VFN_ERR_INVALID, VFN_ERR_OUTSIDE):
        raise ValueError(msg)
    if status == VFN_ERR_IO:
        raise OSError(msg)
    raise VfnError(f"vfnfft error {status}: {msg}")


def i64x3(v) -> ctypes.Array:
    return _c_i64_3(*[int(x) for x in v])


def f64x3(v) -> ctypes.Array:
    return _c_f64_3(*[float(x) for x in v])


def ptr(a) -> int:
    """Data pointer of a C-contiguous numpy array or torch tensor."""
    if isinstance(a, np.ndarray):
        return a.ctypes.data
    return a.data_ptr()
