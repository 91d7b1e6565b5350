"""Boundary types of the hot path, with the reference's names and checks.

`DomainBox` and `SpectralField` mirror the reference's types
(fourier.py:56-91, :147-164, value checks :118-125) so that callers of the
reference evaluators can pass the same objects.  Any object with `.a`/`.b`
(domain) or `.domain`/`.coeffs` (field) attributes is accepted by duck typing,
so reference instances work unchanged.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

__all__ = ["DomainBox", "PhysicalField", "SpectralField", "decompose", "fft_workers", "regular_grid",
           "set_fft_workers", "synthesize_regular"]

_fft_workers = -1


def set_fft_workers(n: int | None) -> None:
    """The reference's CPU FFT thread knob (fourier.py:47-54), kept for
    compatibility: every transform here runs on the GPU (cuFFT), so the
    value is only stored and reported back."""
    global _fft_workers
    _fft_workers = -1 if n is None else int(n)


def fft_workers() -> int:
    return _fft_workers


@dataclass(frozen=True)
class DomainBox:
    """Axis-aligned half-open box prod_d [a_d, b_d) (fourier.py:56-91)."""

    a: tuple
    b: tuple

    def __post_init__(self):
        a = tuple(float(v) for v in self.a)
        b = tuple(float(v) for v in self.b)
        if len(a) != 3 or len(b) != 3:
            raise ValueError("DomainBox needs exactly three bounds per side")
        for d in range(3):
            if not (np.isfinite(a[d]) and np.isfinite(b[d])):
                raise ValueError("domain bounds must be finite")
            if not a[d] < b[d]:
                raise ValueError(
                    f"domain bounds must satisfy a < b, got [{a[d]}, {b[d]}) in direction {d}"
                )
        object.__setattr__(self, "a", a)
        object.__setattr__(self, "b", b)

    @property
    def widths(self) -> np.ndarray:
        return np.array(self.b) - np.array(self.a)

    @property
    def volume(self) -> float:
        return float(np.prod(self.widths))

    def contains(self, points: np.ndarray) -> np.ndarray:
        pts = np.atleast_2d(np.asarray(points, dtype=float))
        return np.all((pts >= np.asarray(self.a)) & (pts < np.asarray(self.b)), axis=1)


def _check_values(values):
    # fourier.py:118-125; CUDA torch tensors are kept on the device
    mod = type(values).__module__
    if mod.startswith("torch") and getattr(values, "is_cuda", False):
        import torch

        if values.dim() != 3:
            raise ValueError(f"expected a 3D array, got shape {tuple(values.shape)}")
        if any(v % 2 for v in values.shape):
            raise ValueError(f"array dimensions must be even, got shape {tuple(values.shape)}")
        return values.to(torch.complex128).contiguous()
    values = np.asarray(values)
    if values.ndim != 3:
        raise ValueError(f"expected a 3D array, got shape {values.shape}")
    for v in values.shape:
        if v % 2 != 0:
            raise ValueError(f"array dimensions must be even, got shape {values.shape}")
    return np.ascontiguousarray(values, dtype=np.complex128)


@dataclass(frozen=True)
class PhysicalField:
    """Complex samples on the regular grid of a DomainBox (fourier.py:128-145)."""

    domain: DomainBox
    values: np.ndarray

    def __post_init__(self):
        object.__setattr__(self, "values", _check_values(self.values))

    @property
    def step(self) -> np.ndarray:
        return np.asarray(self.domain.widths) / np.array(tuple(self.values.shape))


@dataclass(frozen=True)
class SpectralField:
    """Centred-order Fourier coefficients on a DomainBox (fourier.py:147-164)."""

    domain: DomainBox
    coeffs: np.ndarray

    def __post_init__(self):
        object.__setattr__(self, "coeffs", _check_values(self.coeffs))

    def wavenumbers(self, axis: int) -> np.ndarray:
        n = self.coeffs.shape[axis]
        return np.arange(n) - n // 2


def regular_grid(domain, size) -> list:
    """x_d = a_d + j h_d, j = 0..N_d-1 (fourier.py:167-180)."""
    size = tuple(int(v) for v in size)
    return [np.linspace(domain.a[d], domain.b[d], size[d] + 1)[: size[d]] for d in range(3)]


def _transform(fn_name, domain, arr, extra=()):
    # shared plumbing of decompose / synthesize_regular: numpy in -> numpy out,
    # CUDA torch tensors in -> CUDA tensors out (no host round trip)
    from . import _lib
    from .nufft import _device_of, _is_cuda_tensor, _stream_of, _torch

    on_dev = 1 if _is_cuda_tensor(arr) else 0
    shape = tuple(int(s) for s in arr.shape)
    if on_dev:
        t = _torch()
        out = t.empty(shape, dtype=t.complex128, device=arr.device)
    else:
        out = np.empty(shape, dtype=np.complex128)
    dev = _device_of(arr)
    fn = getattr(_lib.load(), fn_name)
    _lib.check(fn(dev, _lib.ptr(arr), _lib.i64x3(shape), _lib.f64x3(domain.a), _lib.f64x3(domain.b), *extra,
                  _lib.ptr(out), on_dev, _stream_of(dev)))
    return out


def decompose(field) -> SpectralField:
    """Grid samples to centred Fourier coefficients on the device
    (fourier.py:183-188): fftshift(fftn(values)) * prod_d sqrt(w_d) / N_d."""
    import ctypes

    values = _check_values(field.values)
    mirror = (ctypes.c_int * 3)(0, 0, 0)
    return SpectralField(field.domain, _transform("vfn_decompose", field.domain, values, (mirror,)))


def synthesize_regular(spec) -> PhysicalField:
    """Inverse of decompose: the samples on the regular grid of spec.domain
    (fourier.py:191-196), on the device."""
    coeffs = _check_values(spec.coeffs)
    return PhysicalField(spec.domain, _transform("vfn_synthesize", spec.domain, coeffs))
