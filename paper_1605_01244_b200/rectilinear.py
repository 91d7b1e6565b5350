"""Rectilinear tensor-grid evaluation (vortexfourier/rectilinear.py) on the
B200 C ABI: ``eval_rectilinear`` -> vfn_rect_eval (three exact separable 1D
non-uniform passes, K5).  ``basis_matrix`` keeps the reference's
host helper and its argument checks (rectilinear.py:22-44), which
``eval_rectilinear`` also applies before calling the device."""

from __future__ import annotations

import numpy as np

from . import _lib
from .nufft import _device_of, _is_cuda_tensor, _stream_of, _torch

__all__ = ["basis_matrix", "eval_rectilinear"]


def _check_axis(domain, n: int, axis: int, coords) -> np.ndarray:
    # rectilinear.py:28-41
    if axis not in (0, 1, 2):
        raise ValueError(f"axis must be 0, 1 or 2, got {axis}")
    if n <= 0 or n % 2 != 0:
        raise ValueError(f"mode count must be positive and even, got {n}")
    y = np.asarray(coords, dtype=float)
    if y.ndim != 1:
        raise ValueError("coordinate vector must be one-dimensional")
    a, b = domain.a[axis], domain.b[axis]
    if y.size and (y.min() < a or y.max() >= b or np.isnan(y).any()):
        bad = y[(y < a) | (y >= b) | np.isnan(y)][0]
        raise ValueError(
            f"coordinate {bad} outside [{a}, {b}) in direction {axis}; "
            "the right endpoint aliases the left under periodicity and is rejected"
        )
    return np.ascontiguousarray(y)


def basis_matrix(domain, n: int, axis: int, coords) -> np.ndarray:
    """E[m, k] = exp(2 pi i (y_m - a)(k - n/2)/(b - a)) / sqrt(b - a) (host helper)."""
    y = _check_axis(domain, n, axis, coords)
    a, b = domain.a[axis], domain.b[axis]
    k = np.arange(n) - n // 2
    return np.exp(2j * np.pi * np.outer(y - a, k) / (b - a)) / np.sqrt(b - a)


def eval_rectilinear(spec, coords, out=None, *, mode: str = "exact", params=None):
    """Series values on the tensor grid coords[0] x coords[1] x coords[2];
    complex (M1, M2, M3) (rectilinear.py:47-64).  ``out`` (extension, like
    ``NufftPlan.evaluate``'s): a C-contiguous complex128 (M1, M2, M3) array on
    the coefficients' side (numpy for host coefficients, a CUDA tensor for
    device ones) that receives the values; pinned host memory makes the
    result download overlap the last pass.

    ``mode`` (extension): "exact" (default; the reference's dense separable
    contractions, to rounding) or "nufft" (three 1D type-2 NUFFT passes with
    ``params`` — NufftParams, default sigma 2, m 6 — accurate to the plan's
    ~10^-(2m+1); needs sigma * N a power of two <= 4096 per axis)."""
    if mode not in ("exact", "nufft"):
        raise ValueError("mode must be 'exact' or 'nufft'")
    if len(coords) != 3:
        raise ValueError("need exactly three coordinate vectors")
    coeffs = spec.coeffs
    shape = tuple(int(s) for s in coeffs.shape)
    on_dev = 1 if _is_cuda_tensor(coeffs) else 0
    ys = []
    for d in range(3):
        c = coords[d]
        if _is_cuda_tensor(c):
            c = c.detach().cpu().numpy()
        ys.append(_check_axis(spec.domain, shape[d], d, c))
    M = tuple(int(y.size) for y in ys)
    if on_dev:
        t = _torch()
        dev = _device_of(coeffs)
        coeffs = coeffs.to(t.complex128).contiguous()
        ys = [t.as_tensor(y, device=coeffs.device) for y in ys]
        if out is None:
            out = t.empty(M, dtype=t.complex128, device=coeffs.device)
        elif not (_is_cuda_tensor(out) and out.device == coeffs.device and tuple(out.shape) == M
                  and out.dtype == t.complex128 and out.is_contiguous()):
            raise ValueError(f"out must be a contiguous complex128 CUDA tensor of shape {M} on {coeffs.device}")
    else:
        dev = _device_of(None)
        coeffs = np.ascontiguousarray(np.asarray(coeffs), dtype=np.complex128)
        if out is None:
            out = np.empty(M, dtype=np.complex128)
        elif not (isinstance(out, np.ndarray) and out.shape == M and out.dtype == np.complex128
                  and out.flags.c_contiguous):
            raise ValueError(f"out must be a C-contiguous complex128 numpy array of shape {M}")
    if 0 in M:
        return out
    lib = _lib.load()
    if mode == "nufft":
        from .nufft import NufftParams

        params = params or NufftParams()
        _lib.check(
            lib.vfn_rect_eval_nufft(dev, _lib.i64x3(shape), _lib.f64x3(spec.domain.a),
                                    _lib.f64x3(spec.domain.b), _lib.ptr(coeffs), _lib.ptr(ys[0]), M[0],
                                    _lib.ptr(ys[1]), M[1], _lib.ptr(ys[2]), M[2], float(params.oversampling),
                                    int(params.cutoff), _lib.ptr(out), on_dev, _stream_of(dev))
        )
        return out
    _lib.check(
        lib.vfn_rect_eval(dev, _lib.i64x3(shape), _lib.f64x3(spec.domain.a),
                          _lib.f64x3(spec.domain.b), _lib.ptr(coeffs), _lib.ptr(ys[0]), M[0],
                          _lib.ptr(ys[1]), M[1], _lib.ptr(ys[2]), M[2], _lib.ptr(out), on_dev,
                          _stream_of(dev))
    )
    return out
