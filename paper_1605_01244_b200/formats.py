"""File formats on either side of the evaluation path: the
reference's ``snapshots`` and ``fields`` modules with the same names,
arguments, outputs (byte for byte) and ValueError texts, implemented by the
native readers / writers of libvfnfft.so (csrc/vfn_io.cpp):

* ``read_snapshot`` / ``write_snapshot`` — SFS1 files (snapshots.py:29-72);
  ``read_snapshot(path, device=d)`` streams the payload into HBM through
  pinned chunks, so ``snapshot_spectral`` / ``tube_eval`` start on the device;
* ``read_points_csv`` / ``write_points_csv`` — points CSV (fields.py:146-174),
  parsed and formatted on all host threads (numbers as Python ``float()`` /
  ``repr()``); ``read_points`` gives the (M, 3) points directly (host or HBM);
* ``write_field`` / ``read_field`` — rectilinear field files (fields.py:67-117);
* ``write_vtk_rectilinear`` — legacy VTK (fields.py:119-143), scalars packed
  on the device when they live there;
* ``equispaced_axes`` / ``clustered_axes`` — evaluation axes (fields.py:30-64).
"""

from __future__ import annotations

import ctypes
import os
from pathlib import Path

import numpy as np

from . import _lib
from .fourier import DomainBox
from .nufft import _device_of, _is_cuda_tensor, _stream_of, _torch
from .tube import Snapshot

__all__ = [
    "clustered_axes",
    "density",
    "equispaced_axes",
    "read_field",
    "read_points",
    "read_points_csv",
    "read_snapshot",
    "write_field",
    "write_points_csv",
    "write_snapshot",
    "write_vtk_rectilinear",
]

_FORMAT = "rectilinear-field-v1"


def _path(p) -> bytes:
    return os.fsencode(os.fspath(p))


_check = _lib.check  # INVALID -> ValueError, IO -> OSError


# ------------------------------------------------------------------ snapshots


def read_snapshot(path, device=None) -> Snapshot:
    """SFS1 file -> Snapshot (snapshots.py:50-72).  With ``device`` (an int
    or torch device) the values land in HBM as a complex128 CUDA tensor."""
    lib = _lib.load()
    info = _lib.SnapshotInfo()
    _check(lib.vfn_snapshot_info_read(_path(path), ctypes.byref(info)))
    shape = tuple(int(v) for v in info.shape)
    count = shape[0] * shape[1] * shape[2]
    if device is not None:
        t = _torch() or __import__("torch")
        values = t.empty(shape, dtype=t.complex128, device=t.device("cuda", _dev_index(device)))
        dev = values.device.index
        _check(lib.vfn_snapshot_read(_path(path), ctypes.byref(info), values.data_ptr(), count, 1, dev,
                                     _stream_of(dev)))
    else:
        values = np.empty(shape, dtype=np.complex128)
        _check(lib.vfn_snapshot_read(_path(path), ctypes.byref(info), values.ctypes.data, count, 0, 0,
                                     None))
    dom = DomainBox(tuple(info.a), tuple(info.b))
    return Snapshot(dom, values, tuple(bool(m) for m in info.mirror), float(info.time))


def write_snapshot(path, snap) -> None:
    """Snapshot -> SFS1 file (snapshots.py:34-47); device values stream out
    through pinned chunks."""
    info = _lib.SnapshotInfo()
    info.a[:] = [float(v) for v in snap.domain.a]
    info.b[:] = [float(v) for v in snap.domain.b]
    values = snap.values
    if _is_cuda_tensor(values):
        values = values.to(_torch().complex128).contiguous()
        on_dev, dev = 1, _device_of(values)
    else:
        values = np.ascontiguousarray(values, dtype=np.complex128)
        on_dev, dev = 0, 0
    info.shape[:] = [int(s) for s in values.shape]
    info.mirror[:] = [1 if m else 0 for m in snap.mirror]
    info.time = float(snap.time)
    _check(_lib.load().vfn_snapshot_write(_path(path), ctypes.byref(info), _lib.ptr(values), on_dev, dev,
                                          _stream_of(dev) if on_dev else None))


def _dev_index(device) -> int:
    if isinstance(device, int):
        return device
    t = _torch() or __import__("torch")
    d = t.device(device)
    return d.index if d.index is not None else t.cuda.current_device()


# ------------------------------------------------------------------ points CSV


class _Table:
    def __init__(self, path):
        self.lib = _lib.load()
        self.h = ctypes.c_void_p()
        rows, cols = ctypes.c_int64(0), ctypes.c_int(0)
        _check(self.lib.vfn_csv_read(_path(path), ctypes.byref(self.h), ctypes.byref(rows),
                                     ctypes.byref(cols)))
        self.rows, self.cols = rows.value, cols.value
        self.names = []
        for c in range(self.cols):
            name = ctypes.c_char_p()
            _check(self.lib.vfn_table_name(self.h, c, ctypes.byref(name)))
            self.names.append(name.value.decode())

    def column(self, c) -> np.ndarray:
        out = np.empty(self.rows)
        _check(self.lib.vfn_table_column(self.h, c, out.ctypes.data))
        return out

    def close(self):
        if self.h:
            self.lib.vfn_table_destroy(self.h)
            self.h = ctypes.c_void_p()

    def __enter__(self):
        return self

    def __exit__(self, *exc):
        self.close()


def read_points_csv(path) -> dict[str, np.ndarray]:
    """Columns of a points CSV as float arrays keyed by header name
    (fields.py:160-174); a repeated name keeps its last column, as a dict
    comprehension does."""
    with _Table(path) as t:
        return {name: t.column(c) for c, name in enumerate(t.names)}


def read_points(path, device=None):
    """The x1, x2, x3 columns of a points CSV as (M, 3) float64 points — a
    numpy array, or with ``device`` a CUDA tensor filled through pinned
    chunks.  Missing columns raise as cli.py:110-112 does."""
    with _Table(path) as t:
        idx = {name: c for c, name in enumerate(t.names)}
        for need in ("x1", "x2", "x3"):
            if need not in idx:
                raise ValueError(f"points file lacks column {need!r}")
        cols = (ctypes.c_int * 3)(idx["x1"], idx["x2"], idx["x3"])
        if device is not None:
            tt = _torch() or __import__("torch")
            pts = tt.empty((t.rows, 3), dtype=tt.float64, device=tt.device("cuda", _dev_index(device)))
            dev = pts.device.index
            _check(t.lib.vfn_table_points(t.h, cols, pts.data_ptr(), 1, dev, _stream_of(dev)))
        else:
            pts = np.empty((t.rows, 3))
            _check(t.lib.vfn_table_points(t.h, cols, pts.ctypes.data, 0, 0, None))
        return pts


def _host_column(col, n):
    """(array, kind, stride) of one extra CSV column: float64 (repr of a
    float), int64 (repr of an int) or bool (True/False), as .item() gives."""
    if _is_cuda_tensor(col):
        col = col.detach().cpu().numpy()
    a = np.asarray(col)
    if a.dtype.kind == "c":
        raise TypeError("complex CSV columns are not supported; write re and im separately")
    if a.dtype.kind == "f":
        a = np.asarray(a, dtype=np.float64)
        kind = 0
    elif a.dtype.kind in "iu":
        a = np.asarray(a, dtype=np.int64)
        kind = 1
    elif a.dtype.kind == "b":
        a = np.asarray(a, dtype=np.uint8)
        kind = 2
    else:
        raise TypeError(f"unsupported CSV column dtype {a.dtype}")
    a = a.reshape(-1)
    if a.size < n:
        raise IndexError(f"index {a.size} is out of bounds for axis 0 with size {a.size}")
    # strided views (e.g. .real / .imag of complex values) are passed as is
    stride = a.strides[0] // a.itemsize if a.strides[0] % a.itemsize == 0 else None
    if stride is None or stride <= 0:
        a = np.ascontiguousarray(a)
        stride = 1
    return a, kind, stride


def write_points_csv(path, points, columns: dict) -> None:
    """CSV with x1,x2,x3 plus named extra columns, one row per point, numbers
    as Python repr() (fields.py:146-157)."""
    if _is_cuda_tensor(points):
        points = points.detach().cpu().numpy()
    pts = np.ascontiguousarray(np.asarray(points, dtype=float).reshape(-1, 3))
    M = pts.shape[0]
    names, arrays, kinds, strides = [], [], [], []
    for name, col in columns.items():
        a, k, s = _host_column(col, M)
        names.append(str(name).encode())
        arrays.append(a)
        kinds.append(k)
        strides.append(s)
    nc = len(names)
    c_names = (ctypes.c_char_p * max(nc, 1))(*names)
    c_cols = (ctypes.c_void_p * max(nc, 1))(*[a.ctypes.data for a in arrays])
    c_str = (ctypes.c_int64 * max(nc, 1))(*strides)
    c_kind = (ctypes.c_int * max(nc, 1))(*kinds)
    _check(_lib.load().vfn_csv_write(_path(path), pts.ctypes.data, M, nc, c_names, c_cols, c_str, c_kind))


# ------------------------------------------------------------------ fields


def equispaced_axes(sizes, bounds) -> list[np.ndarray]:
    """Three linspace vectors over [a_d, b_d], endpoints included (fields.py:30-39)."""
    out = []
    for d in range(3):
        m = int(sizes[d])
        a, b = bounds[2 * d], bounds[2 * d + 1]
        if m < 1 or b <= a:
            raise ValueError(f"bad grid request in direction {d}: {m} points on [{a}, {b}]")
        out.append(np.linspace(a, b, m))
    return out


def clustered_axes(sizes, bounds, strength: float = 1.0) -> list[np.ndarray]:
    """Sinh-stretched axes denser around the midpoints, endpoints pinned
    (fields.py:42-64): y = c + s sinh(u asinh(h / s)), u in [-1, 1]."""
    if strength <= 0:
        raise ValueError("clustering strength must be positive")
    out = []
    for d in range(3):
        m = int(sizes[d])
        a, b = bounds[2 * d], bounds[2 * d + 1]
        if m < 1 or b <= a:
            raise ValueError(f"bad grid request in direction {d}: {m} points on [{a}, {b}]")
        c, h = 0.5 * (a + b), 0.5 * (b - a)
        y = c + strength * np.sinh(np.linspace(-1.0, 1.0, m) * np.arcsinh(h / strength))
        y[0], y[-1] = a, b
        out.append(y)
    return out


def density(values):
    """|psi|^2 as numpy's values.real**2 + values.imag**2 (cli.py:94):
    computed on the device for CUDA tensors, else with numpy."""
    if _is_cuda_tensor(values):
        t = _torch()
        v = values.to(t.complex128).contiguous()
        rho = t.empty(v.shape, dtype=t.float64, device=v.device)
        dev = _device_of(v)
        _check(_lib.load().vfn_density(dev, v.data_ptr(), v.numel(), rho.data_ptr(), 1, _stream_of(dev)))
        return rho
    v = np.asarray(values)
    return v.real**2 + v.imag**2


def _coords_arg(coords):
    cs = []
    for c in coords:
        if _is_cuda_tensor(c):
            c = c.detach().cpu().numpy()
        cs.append(np.ascontiguousarray(np.asarray(c, dtype=np.float64).reshape(-1)))
    return cs, (ctypes.c_void_p * 3)(*[c.ctypes.data for c in cs])


def _payload(x, dtype, torch_dtype):
    if _is_cuda_tensor(x):
        return x.to(torch_dtype).contiguous(), 1
    return np.ascontiguousarray(x, dtype=dtype), 0


def write_field(base, coords, values, density, time=None) -> list[Path]:
    """Header + payloads for a field on the tensor grid of coords
    (fields.py:67-95): base.hdr, base.psi.f64, base.rho.f64.  Values and
    density may be CUDA tensors (streamed out through pinned chunks)."""
    base = Path(base)
    shape = tuple(len(c) for c in coords)
    vshape = tuple(values.shape)
    dshape = tuple(density.shape)
    if vshape != shape or dshape != shape:
        raise ValueError(f"payload shape {vshape} does not match grid {shape}")
    psi_path = base.with_suffix(".psi.f64")
    rho_path = base.with_suffix(".rho.f64")
    hdr_path = base.with_suffix(".hdr")
    cs, c_coords = _coords_arg(coords)
    t = _torch()
    v, v_dev = _payload(values, np.complex128, t.complex128 if t else None)
    r, r_dev = _payload(density, np.float64, t.float64 if t else None)
    on_dev = v_dev and r_dev
    if v_dev != r_dev:  # one on the device, one on the host: bring both home
        v = v.cpu().numpy() if v_dev else v
        r = r.cpu().numpy() if r_dev else r
    dev = _device_of(v) if on_dev else 0
    _check(_lib.load().vfn_field_write(
        _path(hdr_path), _path(psi_path), _path(rho_path), psi_path.name.encode(), rho_path.name.encode(),
        _lib.i64x3(shape), c_coords, _lib.ptr(v), _lib.ptr(r), int(time is not None),
        float(time) if time is not None else 0.0, int(on_dev), dev, _stream_of(dev) if on_dev else None))
    return [hdr_path, psi_path, rho_path]


def read_field(base):
    """Inverse of write_field: (coords, values, density, meta) (fields.py:98-116)."""
    base = Path(base)
    meta = {}
    for line in base.with_suffix(".hdr").read_text().splitlines():
        line = line.split("#", 1)[0].strip()
        if not line:
            continue
        key, _, val = line.partition("=")
        meta[key.strip()] = val.strip()
    if meta.get("format") != _FORMAT:
        raise ValueError(f"{base}: unknown field format {meta.get('format')!r}")
    shape = tuple(int(v) for v in meta["size"].split())
    coords = [np.array([float(v) for v in meta[f"coords_{d + 1}"].split()]) for d in range(3)]
    values = np.fromfile(base.with_suffix(".psi.f64"), dtype="<c16")
    dens = np.fromfile(base.with_suffix(".rho.f64"), dtype="<f8")
    return coords, values.reshape(shape), dens.reshape(shape), meta


def write_vtk_rectilinear(path, coords, scalars: dict, title="field") -> None:
    """Legacy binary VTK rectilinear grid (fields.py:119-143); scalars on the
    device are transposed / converted / byte-swapped there."""
    shape = tuple(len(c) for c in coords)
    t = _torch()
    names, arrays = [], []
    on_dev = None
    for name, data in scalars.items():
        dshape = tuple(data.shape)
        if dshape != shape:
            raise ValueError(f"scalar {name} shape {dshape} does not match grid {shape}")
        a, dflag = _payload(data, np.float64, t.float64 if t else None)
        on_dev = dflag if on_dev is None else on_dev
        if dflag != on_dev:
            raise ValueError("all VTK scalars must live on the same side (host or device)")
        names.append(str(name).encode())
        arrays.append(a)
    on_dev = on_dev or 0
    dev = _device_of(arrays[0]) if on_dev else 0
    cs, c_coords = _coords_arg(coords)
    n = len(names)
    c_names = (ctypes.c_char_p * max(n, 1))(*names)
    c_data = (ctypes.c_void_p * max(n, 1))(*[_lib.ptr(a) for a in arrays])
    _check(_lib.load().vfn_vtk_write(_path(path), str(title).encode(), _lib.i64x3(shape), c_coords, n,
                                     c_names, c_data, on_dev, dev, _stream_of(dev) if on_dev else None))
