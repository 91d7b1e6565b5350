"""Scattered-point evaluation of a spectral field: the reference operator API
(vortexfourier/nufft.py) on top of the B200 C ABI (include/vfnfft.h).

Same names, argument meaning, warnings and error texts as the reference:

* ``NufftParams``        nufft.py:46-78   (host dataclass, identical rules)
* ``AccuracyWarning``    nufft.py:42-43
* ``NufftPlan``          nufft.py:190-272 -> vfn_plan_create / vfn_plan_eval
* ``eval_nufft``         nufft.py:275-279
* ``eval_direct``        nufft.py:129-149 -> vfn_direct_eval (device NDFT)
* ``map_to_torus``       nufft.py:81-92   -> vfn_map_to_torus (bit-exact)
* ``rescale_coeffs``     nufft.py:95-112  (host helper; the plan fuses it into K2)
* ``_kb_beta`` / ``_kb_values`` / ``_kb_transform`` / ``_oversampled_size``
  (nufft.py:152-187) are host helpers kept for callers that import them.

Points and coefficients may be numpy arrays (host; results come back as
numpy) or CUDA torch tensors (device-resident; results stay on the device).
There is no CPU evaluation path: without libvfnfft.so this module raises.
"""

from __future__ import annotations

import ctypes
import sys
import warnings
from dataclasses import dataclass
from math import ceil, log10

import numpy as np

from . import _lib

__all__ = [
    "AccuracyWarning",
    "NufftParams",
    "NufftPlan",
    "map_to_torus",
    "rescale_coeffs",
    "eval_direct",
    "eval_nufft",
]


class AccuracyWarning(UserWarning):
    """Requested evaluation accuracy is unlikely to be met (nufft.py:42-43)."""


@dataclass(frozen=True)
class NufftParams:
    """Oversampling sigma, window half-width m ('cutoff') and target eps
    (nufft.py:46-78)."""

    oversampling: float = 2.0
    cutoff: int = 6
    eps: float = 1e-12

    def __post_init__(self):
        if self.oversampling < 1.0:
            raise ValueError("oversampling must be >= 1")
        if self.cutoff < 1:
            raise ValueError("cutoff must be >= 1")
        if not 0 < self.eps < 1:
            raise ValueError("eps must be in (0, 1)")

    @classmethod
    def for_accuracy(cls, eps: float) -> "NufftParams":
        if not 0 < eps < 1:
            raise ValueError("eps must be in (0, 1)")
        return cls(cutoff=max(1, min(13, ceil(-log10(eps) / 2))), eps=eps)

    def reached_eps(self) -> float:
        return 10.0 ** (-(2 * self.cutoff + 1))


# ------------------------------------------------------------------ host helpers


def _kb_beta(cutoff: int, oversampling: float) -> float:
    w = 2 * cutoff + 1
    return float(np.pi * np.sqrt((w / oversampling) ** 2 * (oversampling - 0.5) ** 2 - 0.8))


def _kb_values(v: np.ndarray, cutoff: int, beta: float) -> np.ndarray:
    half = cutoff + 0.5
    return np.i0(beta * np.sqrt(np.clip(1.0 - (v / half) ** 2, 0.0, None))) / np.i0(beta)


def _kb_transform(k: np.ndarray, n: int, cutoff: int, beta: float) -> np.ndarray:
    w = (cutoff + 0.5) / n
    t = 2.0 * np.pi * w * np.asarray(k, dtype=float)
    s2 = beta * beta - t * t
    sq = np.sqrt(np.abs(s2))
    out = np.where(s2 > 0, np.sinh(sq) / np.where(sq == 0, 1.0, sq), np.sinc(sq / np.pi))
    out[sq == 0] = 1.0
    return 2.0 * w * out / np.i0(beta)


def _oversampled_size(n: int, oversampling: float) -> int:
    target = oversampling * n
    rounded = int(round(target))
    if abs(target - rounded) > 1e-9 or rounded % 2 != 0 or rounded < n:
        raise ValueError(
            f"oversampling {oversampling} of {n} modes gives grid size {target}; "
            "need an even integer no smaller than the mode count"
        )
    return rounded


def rescale_coeffs(spec) -> np.ndarray:
    """Torus-restatement coefficients (nufft.py:95-112); host helper."""
    out = np.asarray(spec.coeffs)
    for axis in range(3):
        n = out.shape[axis]
        k = np.arange(n) - n // 2
        view = [1, 1, 1]
        view[axis] = -1
        out = out * (1.0 - 2.0 * (np.abs(k) % 2)).reshape(view)
    return out * (1.0 / np.sqrt(np.prod(np.asarray(spec.domain.b) - np.asarray(spec.domain.a))))


# ------------------------------------------------------------------ array plumbing


def _torch():
    return sys.modules.get("torch")


def _is_cuda_tensor(x) -> bool:
    t = _torch()
    return t is not None and isinstance(x, t.Tensor) and x.is_cuda


def _stream_of(device: int):
    t = _torch()
    if t is None:
        return None
    # the raw-handle getter costs ~0.1 us against ~2.5 us for
    # is_available() + current_stream(); same stream
    raw = getattr(t._C, "_cuda_getCurrentRawStream", None)
    if raw is not None and t.cuda.is_initialized():
        return ctypes.c_void_p(raw(device))
    if not t.cuda.is_available():
        return None
    return ctypes.c_void_p(t.cuda.current_stream(device).cuda_stream)


def _points_arg(points):
    """(array, on_device, M) for a points argument; shape errors as nufft.py:116-118."""
    if _is_cuda_tensor(points):
        t = _torch()
        if points.dim() != 2 or points.shape[1] != 3:
            raise ValueError(f"points must be an (M, 3) array, got shape {tuple(points.shape)}")
        pts = points.to(t.float64).contiguous()
        return pts, 1, int(pts.shape[0])
    t = _torch()
    if t is not None and isinstance(points, t.Tensor):
        points = points.detach().cpu().numpy()
    pts = np.ascontiguousarray(np.asarray(points, dtype=float))
    if pts.ndim != 2 or pts.shape[1] != 3:
        raise ValueError(f"points must be an (M, 3) array, got shape {pts.shape}")
    return pts, 0, int(pts.shape[0])


def _outside_message(pts, row: int, domain) -> str:
    # the reference's text (nufft.py:122-125)
    if _is_cuda_tensor(pts):
        bad = pts[row].detach().cpu().numpy()
    else:
        bad = np.asarray(pts[row])
    return (
        f"point {bad.tolist()} (row {row}) lies outside the domain "
        f"{list(domain.a)} .. {list(domain.b)}"
    )


def _empty_like_points(pts, on_device, M):
    if on_device:
        t = _torch()
        return t.empty(M, dtype=t.complex128, device=pts.device)
    return np.empty(M, dtype=np.complex128)


def _device_of(x, default=None) -> int:
    if _is_cuda_tensor(x):
        return x.device.index if x.device.index is not None else 0
    if default is not None:
        return default
    t = _torch()
    if t is not None and t.cuda.is_available() and t.cuda.is_initialized():
        return t.cuda.current_device()
    return 0


# ------------------------------------------------------------------ operators


def map_to_torus(points, domain) -> np.ndarray:
    """zeta = mod((x - a)/(a - b), 1) - 1/2, computed on the GPU bit-exactly
    (nufft.py:81-92)."""
    pts, on_dev, M = _points_arg(points)
    dev = _device_of(pts)
    out = np.empty((M, 3)) if not on_dev else _torch().empty_like(pts)
    lib = _lib.load()
    _lib.check(
        lib.vfn_map_to_torus(dev, _lib.f64x3(domain.a), _lib.f64x3(domain.b), _lib.ptr(pts), M,
                             _lib.ptr(out), on_dev, _stream_of(dev))
    )
    return out


def eval_direct(spec, points):
    """Exact series sum at each point, on the device (nufft.py:129-149)."""
    pts, on_dev, M = _points_arg(points)
    out = _empty_like_points(pts, on_dev, M)
    if M == 0:
        return out
    dev = _device_of(pts)
    coeffs = spec.coeffs
    if on_dev and not _is_cuda_tensor(coeffs):
        t = _torch()
        coeffs = t.as_tensor(np.ascontiguousarray(coeffs, dtype=np.complex128), device=pts.device)
    elif not on_dev:
        coeffs = np.ascontiguousarray(np.asarray(coeffs), dtype=np.complex128)
    lib = _lib.load()
    bad = ctypes.c_int64(-1)
    st = lib.vfn_direct_eval(dev, _lib.i64x3(coeffs.shape), _lib.f64x3(spec.domain.a),
                             _lib.f64x3(spec.domain.b), _lib.ptr(coeffs), _lib.ptr(pts), M,
                             _lib.ptr(out), on_dev, ctypes.byref(bad), _stream_of(dev))
    if st == _lib.VFN_ERR_OUTSIDE:
        raise ValueError(_outside_message(pts, bad.value, spec.domain))
    _lib.check(st)
    return out


# Largest window half-width the kernels are instantiated for: the reference's
# NufftParams.for_accuracy clamps to 13 (nufft.py:67-73); an explicit larger
# cutoff is rejected with ValueError instead of being evaluated.
MAX_CUTOFF = 13


def _warn_accuracy(params: "NufftParams", stacklevel: int = 2) -> None:
    """The plan's accuracy warnings (nufft.py:199-212), shared with tube_eval
    whose reference builds a NufftPlan (tube.py:100)."""
    if params.cutoff < 2:
        warnings.warn(
            f"cutoff {params.cutoff} gives a degraded window; expect at "
            "best ~1e-3 relative accuracy",
            AccuracyWarning,
            stacklevel=stacklevel,
        )
    elif params.reached_eps() > params.eps:
        warnings.warn(
            f"cutoff {params.cutoff} reaches ~{params.reached_eps():.0e}, "
            f"short of the requested eps {params.eps:.0e}",
            AccuracyWarning,
            stacklevel=stacklevel,
        )


# Evaluates of at most this many points run the unbinned warp-per-point
# gather (one launch instead of ~25; include/vfnfft.h VFN_WARP_MAX_M).  Its
# values agree with the binned gather's to rounding, not bitwise.
WARP_MAX_M = 32768


class NufftPlan:
    """Reusable evaluator for one SpectralField (nufft.py:190-272).

    Building the plan deconvolves, pads and FFTs on the device; the grid
    stays resident in HBM so repeated ``evaluate`` calls cost only the
    map/bin/gather kernels.
    """

    def __init__(self, spec, params: NufftParams | None = None, *, device: int | None = None):
        params = params or NufftParams()
        _warn_accuracy(params, stacklevel=3)
        if params.cutoff > MAX_CUTOFF:
            # the reference accepts any cutoff >= 1; for_accuracy never asks
            # for more than 13 (nufft.py:67-73), the kernels stop there
            raise ValueError(f"cutoff must be <= {MAX_CUTOFF}")
        self.domain = spec.domain
        self.params = params
        coeffs = spec.coeffs
        shape = tuple(int(s) for s in coeffs.shape)
        self._n = tuple(_oversampled_size(v, params.oversampling) for v in shape)
        self._beta = _kb_beta(params.cutoff, params.oversampling)
        self._modes = shape
        self._handle = None
        self._gather = 0
        self._box = 0
        on_dev = 1 if _is_cuda_tensor(coeffs) else 0
        if not on_dev:
            coeffs = np.ascontiguousarray(np.asarray(coeffs), dtype=np.complex128)
        else:
            coeffs = coeffs.to(_torch().complex128).contiguous()
        self.device = _device_of(coeffs, device)
        lib = _lib.load()
        handle = ctypes.c_void_p()
        _lib.check(
            lib.vfn_plan_create(ctypes.byref(handle), self.device, _lib.i64x3(shape),
                                _lib.f64x3(self.domain.a), _lib.f64x3(self.domain.b),
                                float(params.oversampling), int(params.cutoff), _lib.ptr(coeffs),
                                on_dev, _stream_of(self.device))
        )
        self._handle = handle

    def __del__(self):
        po = getattr(self, "_peer_buffers", None)
        if po is not None:
            try:
                po.close()
            except Exception:
                pass
        h = getattr(self, "_handle", None)
        if h is not None and _lib is not None and _lib._lib is not None:
            try:
                _lib._lib.vfn_plan_destroy(h)
            except Exception:
                pass
            self._handle = None

    @property
    def _grid(self) -> np.ndarray:
        """The oversampled grid (nufft.py:242), copied to the host."""
        out = np.empty(self._n, dtype=np.complex128)
        _lib.check(_lib.load().vfn_plan_grid(self._handle, out.ctypes.data))
        return out

    def set_gather(self, variant: int) -> None:
        """0 = automatic (the warp-per-point gather up to WARP_MAX_M points, the
        binned tensor-core gather above), 1 = thread-per-point gather, 2 = DMMA
        box gather, 3 = unbinned warp-per-point gather, 4 = binned with the
        automatic kernel at any M."""
        _lib.check(_lib.load().vfn_plan_set_gather(self._handle, int(variant)))
        self._gather = int(variant)

    def set_graphs(self, enable: bool) -> None:
        """Replay binned evaluates below 2^20 points as one CUDA graph when the call
        repeats (same buffers, M, geometry); on by default, values identical."""
        _lib.check(_lib.load().vfn_plan_set_graphs(self._handle, int(bool(enable))))

    def set_box(self, bxy: int) -> None:
        """Gather box width: 0 = automatic (by the points' local density), 1 or 2.
        Fix it when results must be bitwise identical across batches/GPU counts."""
        _lib.check(_lib.load().vfn_plan_set_box(self._handle, int(bxy)))
        self._box = int(bxy)

    # ---- multi-GPU steps (parallel.evaluate_sharded; include/vfnfft.h)

    DENSITY_SAMPLE = 16384  # rows j * (M // 16384) decide the box width from 2^20 points

    def decide(self, M: int, sample=None) -> tuple[int, int]:
        """(gather variant, box width) an evaluate of M points takes: variant 3
        (warp per point) or 4 (binned), box 1 or 2.  ``sample``: CUDA tensor of
        the DENSITY_SAMPLE rows j * (M // DENSITY_SAMPLE) of the whole set
        (needed from 2^20 points)."""
        v, b = ctypes.c_int(), ctypes.c_int()
        ptr = 0
        ns = 0
        if sample is not None:
            sample = sample.to(_torch().float64).contiguous()
            ptr, ns = _lib.ptr(sample), int(sample.shape[0])
        _lib.check(_lib.load().vfn_plan_decide(self._handle, int(M), ptr, ns, ctypes.byref(v), ctypes.byref(b),
                                               _stream_of(self.device)))
        return v.value, b.value

    def pin(self, variant: int, box: int) -> None:
        """Fix the gather variant and box width (what ``decide`` returned)."""
        self.set_gather(variant)
        self.set_box(box)

    def part_keys(self, points, stride: int = 1, row0: int = 0):
        """Partition keys (tile << 32 | row0 + row) of rows 0, stride, ... of a
        CUDA (M, 3) tensor, as a uint64 tensor (int64 storage)."""
        t = _torch()
        M = int(points.shape[0])
        n = -(-M // stride) if M else 0
        keys = t.empty(n, dtype=t.int64, device=points.device)
        if n:
            _lib.check(_lib.load().vfn_plan_part_keys(self._handle, _lib.ptr(points), M, int(stride), int(row0),
                                                      _lib.ptr(keys), _stream_of(self.device)))
        return keys

    def partition(self, points, splitters, row0: int = 0, raise_outside: bool = True):
        """Stable split of a CUDA (M, 3) tensor by key range: (send points,
        per-destination counts (list), pos (int32 send position per row)), plus
        the first out-of-domain local row (-1 if none) when not
        ``raise_outside``.  ``splitters``: ascending int64 CUDA tensor of
        nparts - 1 keys."""
        t = _torch()
        M = int(points.shape[0])
        nparts = int(splitters.shape[0]) + 1
        send = t.empty_like(points)
        pos = t.empty(M, dtype=t.int32, device=points.device)
        counts = (ctypes.c_int64 * nparts)()
        bad = ctypes.c_int64(-1)
        st = _lib.load().vfn_plan_partition(self._handle, _lib.ptr(points), M, int(row0),
                                            _lib.ptr(splitters) if nparts > 1 else None, nparts,
                                            _lib.ptr(send), _lib.ptr(pos), counts, ctypes.byref(bad),
                                            _stream_of(self.device))
        if st == _lib.VFN_ERR_OUTSIDE:
            if raise_outside:
                raise ValueError(_outside_message(points, bad.value, self.domain))
            return send, [0] * nparts, pos, bad.value
        _lib.check(st)
        if raise_outside:
            return send, list(counts), pos
        return send, list(counts), pos, -1

    def evaluate_to_peers(self, points, rows, seg_off, outs, M: int | None = None) -> None:
        """Evaluate received points (CUDA (M, 3), or a device address with
        ``M``) and store each value at outs[o][rows[i]] for its owner o
        (seg_off[o] <= i < seg_off[o + 1]); ``outs``: device addresses (ints)
        of the owners' IPC-mapped buffers; ``rows``: CUDA int32 tensor or
        device address (include/vfnfft.h vfn_plan_eval_to_peers)."""
        if M is None:
            M = int(points.shape[0])
        pp = points if isinstance(points, int) else _lib.ptr(points)
        rp = rows if isinstance(rows, int) else _lib.ptr(rows)
        n = len(outs)
        off = (ctypes.c_int64 * (n + 1))(*[int(x) for x in seg_off])
        ptrs = (ctypes.c_void_p * n)(*[int(x) for x in outs])
        bad = ctypes.c_int64(-1)
        st = _lib.load().vfn_plan_eval_to_peers(self._handle, pp if M else None, M, rp if M else None, n, off,
                                                ptrs, ctypes.byref(bad), _stream_of(self.device))
        if st == _lib.VFN_ERR_OUTSIDE:
            raise ValueError(_outside_message(points, bad.value, self.domain))
        _lib.check(st)

    def partition_count(self, points, splitters, row0: int = 0):
        """Count phase of a partition scattered straight to the receiving ranks:
        (per-destination counts, first out-of-domain local row or -1)."""
        M = int(points.shape[0])
        nparts = int(splitters.shape[0]) + 1
        counts = (ctypes.c_int64 * nparts)()
        bad = ctypes.c_int64(-1)
        st = _lib.load().vfn_plan_partition_count(self._handle, _lib.ptr(points) if M else None, M, int(row0),
                                                  _lib.ptr(splitters) if nparts > 1 else None, nparts, counts,
                                                  ctypes.byref(bad), _stream_of(self.device))
        if st == _lib.VFN_ERR_OUTSIDE:
            return [0] * nparts, bad.value
        _lib.check(st)
        return list(counts), -1

    def partition_scatter_peers(self, points, dst_off, recv_pts, recv_rows) -> None:
        """Scatter phase: this rank's points into the destinations' receive
        buffers (device addresses), at dst_off[d] + position (vfn_plan_partition_scatter_peers)."""
        M = int(points.shape[0])
        n = len(dst_off)
        off = (ctypes.c_int64 * n)(*[int(x) for x in dst_off])
        rp = (ctypes.c_void_p * n)(*[int(x) for x in recv_pts])
        rr = (ctypes.c_void_p * n)(*[int(x) for x in recv_rows])
        _lib.check(_lib.load().vfn_plan_partition_scatter_peers(self._handle, _lib.ptr(points) if M else None, M, n,
                                                                off, rp, rr, _stream_of(self.device)))

    def build_timing(self) -> dict:
        """Where the plan build went (ms): host wall time of the whole
        construction, the three grid kernels (CUDA events) and the host
        setup before them (allocations, window fit, tables)."""
        v = (ctypes.c_float * 5)()
        _lib.check(_lib.load().vfn_plan_build_timing(self._handle, v))
        return {"total": v[0], "deconv_pad": v[1], "fft": v[2], "halo": v[3], "host_setup": v[4]}

    def last_timing(self) -> tuple[float, float]:
        """(gather_ms, device_total_ms) of the last evaluate, CUDA-event timed."""
        g, t = ctypes.c_float(), ctypes.c_float()
        _lib.check(_lib.load().vfn_plan_last_timing(self._handle, ctypes.byref(g), ctypes.byref(t)))
        return g.value, t.value

    def evaluate(self, points, chunk: int = 4096, *, out=None):
        """Series values at M points, in input order (nufft.py:244-272).

        ``chunk`` is accepted for signature compatibility; the device path
        has no chunk loop and results do not depend on it.  ``out`` (optional)
        is a caller-owned complex128 buffer of length M on the same side as
        ``points`` (e.g. pinned host memory), written in place and returned."""
        pts, on_dev, M = _points_arg(points)
        if M and chunk == 0:  # the reference's chunk loop is range(0, M, chunk)
            raise ValueError("range() arg 3 must not be zero")
        if out is None:
            out = _empty_like_points(pts, on_dev, M)
        else:
            ok = out.shape == (M,) and (
                (on_dev and _is_cuda_tensor(out) and out.dtype == _torch().complex128 and out.is_contiguous())
                or (not on_dev and isinstance(out, np.ndarray) and out.dtype == np.complex128
                    and out.flags.c_contiguous)
            )
            if not ok:
                raise ValueError("out must be a contiguous complex128 buffer of shape (M,) next to points")
        if on_dev and (pts.device.index or 0) != self.device:
            raise ValueError(f"points are on cuda:{pts.device.index}, plan on cuda:{self.device}")
        if on_dev and (out.device.index or 0) != self.device:
            raise ValueError(f"out is on cuda:{out.device.index}, plan on cuda:{self.device}")
        if M == 0:
            return out
        lib = _lib.load()
        bad = ctypes.c_int64(-1)
        st = lib.vfn_plan_eval(self._handle, _lib.ptr(pts), M, _lib.ptr(out), on_dev,
                               ctypes.byref(bad), _stream_of(self.device))
        if st == _lib.VFN_ERR_OUTSIDE:
            raise ValueError(_outside_message(pts, bad.value, self.domain))
        _lib.check(st)
        return out

    def geometry(self, M: int) -> tuple[tuple, tuple]:
        """(box, tile) cell sizes of the bin key of the last evaluate/bin call
        (else the point-independent choice for M points)."""
        box = (ctypes.c_int * 3)()
        tile = (ctypes.c_int * 3)()
        _lib.check(_lib.load().vfn_plan_geometry(self._handle, int(M), box, tile))
        return tuple(box), tuple(tile)

    def key_shift(self, M: int = 0) -> int:
        """Depth resolution of the bin key of the last evaluate/bin call (else
        the point-independent choice for M points): 1 = depth pairs, 0 = depths."""
        v = ctypes.c_int()
        _lib.check(_lib.load().vfn_plan_key_shift(self._handle, int(M), ctypes.byref(v)))
        return v.value

    def launch_count(self, M: int) -> int:
        """Kernels of this library one evaluate of M points launches (for M above
        CUB's single-tile sort threshold): map+key, the onesweep radix sort
        (histogram, exclusive sum, 2 kernels per 8 key bits), box counts and
        their scan, the unit/work-item builders and the gather
        (profiles/r01/launches_c5_v8.md lists them)."""
        if M == 0:
            return 0
        if (self._gather == 0 and M <= WARP_MAX_M) or self._gather == 3:
            return 2  # unbinned warp-per-point gather + the bad-row store
        box, tile = self.geometry(M)
        ntiles = 1
        for d in range(3):
            ntiles *= -(-self._n[d] // tile[d])
        nkeys = ntiles * (tile[0] // box[0]) * (tile[1] // box[1]) * (tile[2] // box[2])
        sh = self.key_shift(M)
        nkeys *= (box[2] + (1 << sh) - 1) >> sh  # key slots per box (include/vfnfft.h vfn_plan_bin)
        bits = max(1, int(nkeys - 1).bit_length())
        sort = 2 + 2 * -(-bits // 8)
        if 2 <= self.params.cutoff <= 7 and tile[2] == 20 - 2 * self.params.cutoff:
            prep = 1 + 2 + (1 + 2 + 1) + (1 + 2 + 1)  # box counts+scan, units+scan+write, items
        else:
            prep = 1 + 2 + 1 + 2 + 1                  # box counts+scan, tile units+scan, items
        return 1 + sort + prep + 1

    def bin(self, points):
        """(keys, perm) of the device bin sort as numpy arrays."""
        pts, on_dev, M = _points_arg(points)
        if on_dev:
            pts = pts.cpu().numpy()
        keys = np.empty(M, dtype=np.uint32)
        perm = np.empty(M, dtype=np.int32)
        if M == 0:
            return keys, perm
        bad = ctypes.c_int64(-1)
        st = _lib.load().vfn_plan_bin(self._handle, _lib.ptr(pts), M, _lib.ptr(keys), _lib.ptr(perm),
                                      0, ctypes.byref(bad), None)
        if st == _lib.VFN_ERR_OUTSIDE:
            raise ValueError(_outside_message(pts, bad.value, self.domain))
        _lib.check(st)
        return keys, perm


def gather_values(values, pos, out=None):
    """out[i] = values[pos[i]] on the device (values back in input order
    after a key-range exchange; include/vfnfft.h vfn_gather_values)."""
    t = _torch()
    M = int(pos.shape[0])
    if out is None:
        out = t.empty(M, dtype=t.complex128, device=pos.device)
    dev = _device_of(pos)
    _lib.check(_lib.load().vfn_gather_values(dev, _lib.ptr(values), _lib.ptr(pos), M, _lib.ptr(out),
                                             _stream_of(dev)))
    return out


def eval_nufft(spec, points, params: NufftParams | None = None):
    """One-shot scattered evaluation (nufft.py:275-279)."""
    return NufftPlan(spec, params).evaluate(points)
