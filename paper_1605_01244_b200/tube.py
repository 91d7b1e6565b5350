"""The next rows after the hot path on the device:

* ``snapshot_spectral`` — snapshot samples -> centred coefficients on the
  computational box (mirror extension + forward FFT + shift + scale;
  gpe.py:90-113, fourier.py:183-188) -> vfn_decompose;
* ``tube_eval`` — adaptive low-density point extraction that reuses one
  evaluation plan over its refinement passes (tube.py:58-127) ->
  vfn_tube_eval.  Same arguments, warnings, errors and output type as the
  reference.

Snapshots are duck-typed on ``.domain``, ``.values``, ``.mirror`` (the
reference's ``gpe.Snapshot`` works unchanged).
"""

from __future__ import annotations

import ctypes
import math
import warnings
from dataclasses import dataclass

import numpy as np

from . import _lib
from .fourier import DomainBox, SpectralField
from .nufft import MAX_CUTOFF, NufftParams, _device_of, _is_cuda_tensor, _stream_of, _torch, _warn_accuracy

__all__ = ["Snapshot", "TubePointCloud", "computational_domain", "snapshot_spectral", "tube_eval"]


@dataclass(frozen=True)
class Snapshot:
    """Samples on the physical grid plus mirror flags (gpe.py:62-78).
    ``values`` is a complex128 numpy array or a CUDA tensor (a snapshot file
    read straight into HBM, formats.read_snapshot(..., device=...))."""

    domain: DomainBox
    values: np.ndarray
    mirror: tuple
    time: float = 0.0

    def __post_init__(self):
        object.__setattr__(self, "mirror", tuple(bool(m) for m in self.mirror))
        if _is_cuda_tensor(self.values):
            object.__setattr__(self, "values", self.values.to(_torch().complex128).contiguous())
        else:
            object.__setattr__(self, "values", np.ascontiguousarray(self.values, dtype=np.complex128))
        if self.values.ndim != 3:
            raise ValueError("snapshot values must be a 3D array")


@dataclass(frozen=True)
class TubePointCloud:
    """Points with their densities and first-appearance pass (tube.py:33-47)."""

    points: np.ndarray
    density: np.ndarray
    level: np.ndarray

    def __post_init__(self):
        if self.points.shape != (self.density.size, 3) or self.density.size != self.level.size:
            raise ValueError("inconsistent point cloud arrays")

    def __len__(self) -> int:
        return self.density.size


def computational_domain(domain, mirror) -> DomainBox:
    """Physical box extended to [a, a + 2 (b - a)) where mirrored (gpe.py:81-87)."""
    b = list(domain.b)
    for d in range(3):
        if mirror[d]:
            b[d] = domain.a[d] + 2.0 * (domain.b[d] - domain.a[d])
    return DomainBox(domain.a, tuple(b))


def _snap_args(snap):
    """(values, on_device, mirror flags): CUDA tensors stay on the device."""
    if _is_cuda_tensor(snap.values):
        values = snap.values.to(_torch().complex128).contiguous()
        on_dev = 1
    else:
        values = np.ascontiguousarray(np.asarray(snap.values), dtype=np.complex128)
        on_dev = 0
    if values.ndim != 3:
        raise ValueError("snapshot values must be a 3D array")
    mirror = (ctypes.c_int * 3)(*[1 if m else 0 for m in snap.mirror])
    return values, on_dev, mirror


def snapshot_spectral(snap) -> SpectralField:
    """Coefficients of the snapshot's mirror-extended field on the
    computational box (gpe.py:110-113), computed on the device.  Device
    samples give device coefficients (no host round trip); host samples give
    host coefficients."""
    values, on_dev, mirror = _snap_args(snap)
    dom = computational_domain(snap.domain, snap.mirror)
    shape = tuple(int(s) * (2 if m else 1) for s, m in zip(values.shape, snap.mirror))
    dev = _device_of(values)
    if on_dev:
        t = _torch()
        out = t.empty(shape, dtype=t.complex128, device=values.device)
    else:
        out = np.empty(shape, dtype=np.complex128)
    _lib.check(
        _lib.load().vfn_decompose(dev, _lib.ptr(values), _lib.i64x3(values.shape),
                                  _lib.f64x3(snap.domain.a), _lib.f64x3(snap.domain.b), mirror,
                                  _lib.ptr(out), on_dev, _stream_of(dev))
    )
    return SpectralField(dom, out)


def _empty_cloud() -> TubePointCloud:
    return TubePointCloud(np.empty((0, 3)), np.empty(0), np.empty(0, dtype=np.int64))


def tube_eval(snap, thresholds, final_filter: float | None = None,
              params: NufftParams | None = None) -> TubePointCloud:
    """Extract and refine the low-density point set of a snapshot
    (tube.py:58-127): the first threshold selects seeds among the stored
    samples, each later one the parents of the next 3x refinement."""
    thresholds = [float(t) for t in np.atleast_1d(thresholds)]
    if not thresholds or any(t <= 0 for t in thresholds):
        raise ValueError("thresholds must be a nonempty sequence of positive values")
    params = params or NufftParams()
    values, _, mirror = _snap_args(snap)
    if params.cutoff > MAX_CUTOFF:
        raise ValueError(f"cutoff must be <= {MAX_CUTOFF}")
    thr = np.asarray(thresholds, dtype=np.float64)
    dev = _device_of(values)
    lib = _lib.load()
    handle = ctypes.c_void_p()
    count = ctypes.c_int64(0)
    no_seeds = ctypes.c_int(0)
    ff = float(final_filter) if final_filter is not None else math.nan
    _lib.check(
        lib.vfn_tube_eval(ctypes.byref(handle), dev, _lib.ptr(values), _lib.i64x3(values.shape),
                          _lib.f64x3(snap.domain.a), _lib.f64x3(snap.domain.b), mirror,
                          thr.ctypes.data, len(thresholds), int(final_filter is not None), ff,
                          float(params.oversampling), int(params.cutoff), ctypes.byref(count),
                          ctypes.byref(no_seeds), _stream_of(dev))
    )
    try:
        if no_seeds.value:
            warnings.warn(
                f"no grid point has density <= {thresholds[0]}; returning an empty cloud",
                RuntimeWarning,
                stacklevel=2,
            )
            return _empty_cloud()
        # the reference builds its plan once seeds exist (tube.py:100), which
        # is where its accuracy warnings come from (nufft.py:199-212)
        _warn_accuracy(params, stacklevel=3)
        n = count.value
        if n == 0:
            return _empty_cloud()
        pts = np.empty((n, 3))
        dens = np.empty(n)
        lev = np.empty(n, dtype=np.int64)
        _lib.check(lib.vfn_tube_copy(handle, pts.ctypes.data, dens.ctypes.data, lev.ctypes.data))
        return TubePointCloud(pts, dens, lev)
    finally:
        lib.vfn_tube_destroy(handle)
