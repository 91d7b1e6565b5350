"""Seeded synthetic inputs for the five BASELINE.json configurations.

No public dataset is involved: the reference's benchmarks are synthetic
spectra and point clouds, restated here from SURVEY.md 8(d).  Seeds:
coefficients ``default_rng(1000 + c)``, points ``default_rng(2000 + c)``.

* c1  N=32^3,  decay 64,   M=1e4 uniform in [-1/2,1/2)^3
* c2  N=64^3,  decay 256,  M=1e6 uniform
* c3  N=128^3 from two perpendicular straight vortex lines on [-8,8)^3,
      M=1e7 Gaussian cloud (std 0.05) at the origin
* c4  N=128^3, decay 1024, rectilinear 256^3 tanh-clustered tensor grid
* c5  N=256^3, decay 4096, M=2^28 uniform (generated on the device)

The spectrum follows the reference fixture pattern (conftest.py:24-27:
real then imaginary standard normals) times exp(-|k|^2/decay).
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

UNIT_BOX = ((-0.5, -0.5, -0.5), (0.5, 0.5, 0.5))
VORTEX_BOX = ((-8.0, -8.0, -8.0), (8.0, 8.0, 8.0))


@dataclass(frozen=True)
class Workload:
    name: str
    modes: tuple
    box: tuple
    npoints: int
    decay: float | None
    kind: str  # "uniform" | "cluster" | "rectilinear"


WORKLOADS = {
    "c1": Workload("c1", (32, 32, 32), UNIT_BOX, 10_000, 64.0, "uniform"),
    "c2": Workload("c2", (64, 64, 64), UNIT_BOX, 1_000_000, 256.0, "uniform"),
    "c3": Workload("c3", (128, 128, 128), VORTEX_BOX, 10_000_000, None, "cluster"),
    "c4": Workload("c4", (128, 128, 128), UNIT_BOX, 256 ** 3, 1024.0, "rectilinear"),
    "c5": Workload("c5", (256, 256, 256), UNIT_BOX, 1 << 28, 4096.0, "uniform"),
}


def decaying_spectrum(shape, decay: float, seed: int) -> np.ndarray:
    """N(0,1) + i N(0,1) coefficients times exp(-|k|^2 / decay), centred order."""
    rng = np.random.default_rng(seed)
    c = rng.standard_normal(shape) + 1j * rng.standard_normal(shape)
    k2 = np.zeros(shape)
    for d, n in enumerate(shape):
        k = (np.arange(n) - n // 2).astype(float)
        view = [1, 1, 1]
        view[d] = -1
        k2 = k2 + (k * k).reshape(view)
    return np.ascontiguousarray(c * np.exp(-k2 / decay))


def _transverse_frame(direction):
    # same convention as the reference's straight-vortex frame
    # (vortex.py:246-255): lowest-index smallest component picks the helper axis
    d = np.asarray(direction, dtype=float)
    d = d / np.linalg.norm(d)
    e = np.zeros(3)
    e[int(np.argmin(np.abs(d)))] = 1.0
    u1 = np.cross(d, e)
    u1 /= np.linalg.norm(u1)
    u2 = np.cross(d, u1)
    return u1, u2


def vortex_pair_field(shape=(128, 128, 128), box=VORTEX_BOX) -> np.ndarray:
    """psi = prod_i tanh(r_i/sqrt2) e^{i theta_i} sampled on the box's grid for a
    line through (0,0,+1/2) along x and one through (0,0,-1/2) along y
    (reference frame vortex.py:246-284)."""
    a, b = np.asarray(box[0]), np.asarray(box[1])
    axes = [a[d] + (b[d] - a[d]) * np.arange(shape[d]) / shape[d] for d in range(3)]
    psi = np.ones(shape, dtype=np.complex128)
    for pos, direction in (((0.0, 0.0, 0.5), (1.0, 0.0, 0.0)), ((0.0, 0.0, -0.5), (0.0, 1.0, 0.0))):
        u1, u2 = _transverse_frame(direction)
        w = [axes[d] - pos[d] for d in range(3)]
        s1 = w[0][:, None, None] * u1[0] + w[1][None, :, None] * u1[1] + w[2][None, None, :] * u1[2]
        s2 = w[0][:, None, None] * u2[0] + w[1][None, :, None] * u2[1] + w[2][None, None, :] * u2[2]
        psi *= np.tanh(np.hypot(s1, s2) / np.sqrt(2.0)) * np.exp(1j * np.arctan2(s2, s1))
    return psi


def vortex_pair_spectrum(shape=(128, 128, 128), box=VORTEX_BOX) -> np.ndarray:
    """Centred coefficients of vortex_pair_field, transformed like the
    reference's decompose (fourier.py:183-188)."""
    a, b = np.asarray(box[0]), np.asarray(box[1])
    psi = vortex_pair_field(shape, box)
    import scipy.fft

    scale = float(np.prod(np.sqrt(b - a) / np.asarray(shape)))
    return np.ascontiguousarray(np.fft.fftshift(scipy.fft.fftn(psi, workers=-1)) * scale)


def coefficients(name: str) -> np.ndarray:
    w = WORKLOADS[name]
    c = int(name[1:])
    if w.kind == "cluster":
        return vortex_pair_spectrum(w.modes, w.box)
    return decaying_spectrum(w.modes, w.decay, 1000 + c)


def points(name: str, count: int | None = None) -> np.ndarray:
    """Host-side points for c1..c3 (c5 is generated on the device by bench.py)."""
    w = WORKLOADS[name]
    c = int(name[1:])
    m = w.npoints if count is None else count
    rng = np.random.default_rng(2000 + c)
    if w.kind == "cluster":
        return rng.normal(0.0, 0.05, (m, 3))
    return rng.uniform(-0.5, 0.5, (m, 3))


def rect_axes(count: int = 256):
    """c4 coordinates x_j = 0.5 tanh(3 u_j)/tanh(3), u_j = -1 + 2j/count."""
    u = -1.0 + 2.0 * np.arange(count) / count
    x = 0.5 * np.tanh(3.0 * u) / np.tanh(3.0)
    return [x.copy(), x.copy(), x.copy()]


DEVICE_CHUNK = 1 << 22  # generation unit of the device-side c5 set


def device_points(name: str, lo: int, hi: int, device):
    """Rows [lo, hi) of the workload's point set as a CUDA tensor.  c5's 2^28
    uniform points are generated on the device in 2^22-point chunks, chunk k
    from its own seed, so any rank's block of the ONE global set is the same
    whatever the rank count (strong scaling shards one set)."""
    import torch

    w = WORKLOADS[name]
    if name != "c5":
        return torch.as_tensor(points(name)[lo:hi]).to(device)
    out = torch.empty((hi - lo, 3), dtype=torch.float64, device=device)
    gen = torch.Generator(device=device)
    k0, k1 = lo // DEVICE_CHUNK, -(-hi // DEVICE_CHUNK)
    for k in range(k0, k1):
        c0, c1 = k * DEVICE_CHUNK, min((k + 1) * DEVICE_CHUNK, w.npoints)
        gen.manual_seed(2005 + 7919 * k)
        chunk = torch.rand((c1 - c0, 3), dtype=torch.float64, device=device, generator=gen) - 0.5
        a, b = max(lo, c0), min(hi, c1)
        out[a - lo:b - lo] = chunk[a - c0:b - c0]
    return out
