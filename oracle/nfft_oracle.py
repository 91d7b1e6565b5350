"""CPU oracle for the 3D NFFT trafo hot path — TEST INFRASTRUCTURE ONLY.

This module restates, in plain numpy/scipy, the algorithm of the reference
package `vortexfourier` (mounted read-only at /root/reference during
development; it does not travel to the GPU box).  It exists so that the
parity tests (`tests/`), `__graft_entry__.smoke()` and the `cpu_baseline` /
`--impl reference` legs of `bench.py` have a checker.  The product path
(`paper_1605_01244_b200`) never imports it.

Pinning: `tests/golden/make_golden.py` imports the real reference and writes
golden vectors under `tests/golden/`; `tests/test_oracle_golden.py` checks this
restatement against every one of them (bit-exact where the arithmetic is the
same numpy sequence, <=1e-14 relative elsewhere).

Every function cites the reference file:line it follows.  Paths are relative
to /root/reference/pkg/src/vortexfourier/.
"""

from __future__ import annotations

import cmath
import math

import numpy as np
import scipy.fft

__all__ = [
    "centered_wavenumbers",
    "kb_beta",
    "kb_window",
    "kb_hat",
    "grid_size",
    "torus_map",
    "torus_coeffs",
    "oversampled_grid",
    "nearest_cells",
    "gather_eval",
    "nufft_eval",
    "ndft",
    "basis_matrix",
    "rectilinear",
    "bin_keys",
    "bin_permutation",
    "domain_violation",
    "partition_keys",
    "partition",
]


def centered_wavenumbers(n: int) -> np.ndarray:
    """k = j - n/2 for j = 0..n-1 (fourier.py:161-164)."""
    return np.arange(n) - n // 2


def kb_beta(m: int, sigma: float) -> float:
    """Kaiser-Bessel shape parameter for a window of 2m+1 cells (nufft.py:152-156)."""
    width = 2 * m + 1
    inner = (width / sigma) ** 2 * (sigma - 0.5) ** 2 - 0.8
    return float(np.pi * np.sqrt(inner))


def kb_window(v: np.ndarray, m: int, beta: float) -> np.ndarray:
    """Window value at signed cell distance v (nufft.py:159-164)."""
    half = m + 0.5
    radial = np.clip(1.0 - (v / half) ** 2, 0.0, None)
    return np.i0(beta * np.sqrt(radial)) / np.i0(beta)


def kb_hat(k: np.ndarray, n: int, m: int, beta: float) -> np.ndarray:
    """Continuous Fourier transform of the window at integer k (nufft.py:167-176)."""
    half_width = (m + 0.5) / n
    t = 2.0 * np.pi * half_width * np.asarray(k, dtype=float)
    d = beta * beta - t * t
    r = np.sqrt(np.abs(d))
    safe = np.where(r == 0, 1.0, r)
    val = np.where(d > 0, np.sinh(r) / safe, np.sinc(r / np.pi))
    val[r == 0] = 1.0
    return 2.0 * half_width * val / np.i0(beta)


def grid_size(modes: int, sigma: float) -> int:
    """Oversampled grid size: an even integer >= modes (nufft.py:179-187)."""
    target = sigma * modes
    n = int(round(target))
    if abs(target - n) > 1e-9 or n % 2 != 0 or n < modes:
        raise ValueError(
            f"oversampling {sigma} of {modes} modes gives grid size {target}; "
            "need an even integer no smaller than the mode count"
        )
    return n


def domain_violation(points: np.ndarray, a, b) -> int:
    """Index of the first row outside prod [a, b) (NaN counts as outside), or -1
    (nufft.py:115-126 with fourier.py:86-91)."""
    pts = np.asarray(points, dtype=float)
    a = np.asarray(a, dtype=float)
    b = np.asarray(b, dtype=float)
    ok = np.all((pts >= a) & (pts < b), axis=1)
    bad = np.flatnonzero(~ok)
    return int(bad[0]) if bad.size else -1


def torus_map(points: np.ndarray, a, b) -> np.ndarray:
    """zeta = mod((x - a) / (a - b), 1) - 1/2 (nufft.py:81-92)."""
    pts = np.asarray(points, dtype=float)
    a = np.asarray(a, dtype=float)
    b = np.asarray(b, dtype=float)
    return np.mod((pts - a) / (a - b), 1.0) - 0.5


def torus_coeffs(coeffs: np.ndarray, a, b) -> np.ndarray:
    """(-1)^(|k1|+|k2|+|k3|) / sqrt(vol) rescale of centred coefficients
    (nufft.py:95-112)."""
    widths = np.asarray(b, dtype=float) - np.asarray(a, dtype=float)
    out = np.asarray(coeffs)
    for d in range(3):
        k = centered_wavenumbers(coeffs.shape[d])
        sign = 1.0 - 2.0 * (np.abs(k) % 2)
        shape = [1, 1, 1]
        shape[d] = -1
        out = out * sign.reshape(shape)
    return out * (1.0 / np.sqrt(np.prod(widths)))


def oversampled_grid(coeffs: np.ndarray, a, b, sigma: float = 2.0, m: int = 6):
    """Deconvolve, zero-pad into the 8 corner octants and forward-FFT
    (nufft.py:213-242).  Returns (grid, n, beta)."""
    shape = coeffs.shape
    n = tuple(grid_size(s, sigma) for s in shape)
    beta = kb_beta(m, sigma)
    fh = torus_coeffs(coeffs, a, b)
    for d in range(3):
        phat = kb_hat(centered_wavenumbers(shape[d]), n[d], m, beta)
        view = [1, 1, 1]
        view[d] = -1
        fh = fh / phat.reshape(view)
    fh /= float(np.prod(n))
    grid = np.zeros(n, dtype=np.complex128)
    # centred index j (wavenumber j - N/2) lands at (j - N/2) mod n
    idx = [np.mod(centered_wavenumbers(shape[d]), n[d]) for d in range(3)]
    grid[np.ix_(idx[0], idx[1], idx[2])] = fh
    grid = scipy.fft.fftn(grid, overwrite_x=True, workers=-1)
    return grid, n, beta


def nearest_cells(points: np.ndarray, a, b, n):
    """u = z * n and l0 = floor(u + 1/2) exactly as the reference gather
    computes them (nufft.py:248-257).  l0 may equal n (survey fact 5)."""
    zeta = torus_map(points, a, b)
    z = np.where(zeta < 0, zeta + 1.0, zeta)
    u = z * np.asarray(n)
    l0 = np.floor(u + 0.5).astype(np.int64)
    return u, l0


def gather_eval(grid: np.ndarray, n, m: int, beta: float, points, a, b, chunk: int = 4096):
    """Window-weighted (2m+1)^3 gather from the oversampled grid
    (nufft.py:244-272)."""
    pts = np.asarray(points, dtype=float)
    out = np.empty(pts.shape[0], dtype=np.complex128)
    if pts.shape[0] == 0:
        return out
    u_all, l0_all = nearest_cells(pts, a, b, n)
    offs = np.arange(-m, m + 1)
    for s in range(0, pts.shape[0], chunk):
        u = u_all[s : s + chunk]
        l0 = l0_all[s : s + chunk]
        w = []
        ix = []
        for d in range(3):
            v = u[:, d : d + 1] - l0[:, d : d + 1] - offs
            w.append(kb_window(v, m, beta))
            ix.append((l0[:, d : d + 1] + offs) % n[d])
        block = grid[ix[0][:, :, None, None], ix[1][:, None, :, None], ix[2][:, None, None, :]]
        t = np.einsum("pabc,pc->pab", block, w[2])
        t = np.einsum("pab,pb->pa", t, w[1])
        out[s : s + chunk] = np.einsum("pa,pa->p", t, w[0])
    return out


def nufft_eval(coeffs, a, b, points, sigma: float = 2.0, m: int = 6):
    """One-shot plan + gather (nufft.py:275-279)."""
    grid, n, beta = oversampled_grid(coeffs, a, b, sigma, m)
    return gather_eval(grid, n, m, beta, points, a, b)


def ndft(coeffs: np.ndarray, a, b, points) -> np.ndarray:
    """Exact series sum per point, O(N1 N2 N3) each (nufft.py:129-149)."""
    pts = np.asarray(points, dtype=float)
    a = np.asarray(a, dtype=float)
    widths = np.asarray(b, dtype=float) - a
    ks = [centered_wavenumbers(s) for s in coeffs.shape]
    scale = 1.0 / np.sqrt(np.prod(widths))
    out = np.empty(pts.shape[0], dtype=np.complex128)
    for i in range(pts.shape[0]):
        t = (pts[i] - a) / widths
        e = [np.exp(2j * np.pi * ks[d] * t[d]) for d in range(3)]
        out[i] = np.einsum("abc,a,b,c->", coeffs, e[0], e[1], e[2]) * scale
    return out


def series_scalar(coeffs: np.ndarray, a, b, point) -> complex:
    """The series at one point summed term by term in plain Python complex
    arithmetic, first axis innermost — an order independent of both the
    tensor contraction of eval_direct (nufft.py:129-149) and the device
    NDFT; the reference pins eval_direct against such a sum
    (tests/oracles.py:19-33, test_nufft.py:60-67).  Small cases only."""
    n = coeffs.shape
    w = [float(b[d]) - float(a[d]) for d in range(3)]
    ph = [[cmath.exp(2j * cmath.pi * (j - n[d] // 2) * (float(point[d]) - float(a[d])) / w[d])
           for j in range(n[d])] for d in range(3)]
    acc = 0j
    for j3 in range(n[2]):
        for j2 in range(n[1]):
            e23 = ph[2][j3] * ph[1][j2]
            for j1 in range(n[0]):
                acc += complex(coeffs[j1, j2, j3]) * (e23 * ph[0][j1])
    return acc / math.sqrt(w[0] * w[1] * w[2])


def basis_matrix(a_d: float, b_d: float, nmodes: int, coords) -> np.ndarray:
    """E[m, k] = exp(2 pi i (y_m - a)(k - N/2)/(b - a)) / sqrt(b - a)
    (rectilinear.py:22-44)."""
    y = np.asarray(coords, dtype=float)
    k = centered_wavenumbers(nmodes)
    return np.exp(2j * np.pi * np.outer(y - a_d, k) / (b_d - a_d)) / np.sqrt(b_d - a_d)


def rectilinear(coeffs: np.ndarray, a, b, coords) -> np.ndarray:
    """Tensor-grid evaluation by three mode contractions (rectilinear.py:47-64)."""
    e = [basis_matrix(a[d], b[d], coeffs.shape[d], coords[d]) for d in range(3)]
    t = np.matmul(coeffs.transpose(2, 0, 1), e[1].T)
    t = np.matmul(e[0], t)
    return np.tensordot(t, e[2], axes=([0], [1]))


# ---------------------------------------------------------------------------
# N1 (new, no reference counterpart): the bin-sort key.
# A point's nearest oversampled cell c_d = l0_d mod n_d (nufft.py:248-257) is
# grouped into gather boxes of (bi, bj, bk) cells; boxes are numbered
# row-major inside tiles of (ti, tj, tk) cells, tiles row-major over the grid
# (the row-major convention of tube.py:50-51).  Inside a box the key keeps
# the cell's depth (c_z mod bk) >> s only, s = 1 (depth pairs) except for
# odd m on the tensor-core gather (s = 0): key = (tile * boxes_per_tile +
# box) * ceil(bk / 2^s) + (depth >> s).  The permutation is a stable sort on that
# key (precedent: the stable argsort of tube.py:125).
# ---------------------------------------------------------------------------


def bin_keys(points, a, b, n, box=(1, 1, 4), tile=(4, 4, 4), key_shift: int = 1) -> np.ndarray:
    """Sort key of every point; see the block comment above.  Inside a box the
    key is the depth >> key_shift (1: depth pairs), so a box's points sort by it."""
    _, l0 = nearest_cells(points, a, b, n)
    cell = l0 % np.asarray(n)
    box = np.asarray(box)
    tile = np.asarray(tile)
    ntile = -(-np.asarray(n) // tile)
    t = cell // tile
    rem = cell % tile
    inner = rem // box
    c = rem % box
    nbox = tile // box
    tile_id = (t[:, 0] * ntile[1] + t[:, 1]) * ntile[2] + t[:, 2]
    box_id = (inner[:, 0] * nbox[1] + inner[:, 1]) * nbox[2] + inner[:, 2]
    slots = (int(box[2]) + (1 << key_shift) - 1) >> key_shift
    key = (tile_id * int(np.prod(nbox)) + box_id) * slots + (c[:, 2] >> key_shift)
    return key.astype(np.int64)


def bin_permutation(points, a, b, n, box=(1, 1, 4), tile=(4, 4, 4), key_shift: int = 1) -> np.ndarray:
    """Stable argsort of bin_keys: sorted position -> input row."""
    return np.argsort(bin_keys(points, a, b, n, box, tile, key_shift), kind="stable")


def partition_keys(points, a, b, n, tile, row0: int = 0) -> np.ndarray:
    """Key of the multi-GPU key-range partition (new): the
    row-major index of the tile holding the nearest cell (same cell as the
    reference gather, nufft.py:248-257) shifted left by 32, or'ed with the
    global input row.  uint64 values < 2^63, returned as int64."""
    _, l0 = nearest_cells(points, a, b, n)
    cell = l0 % np.asarray(n)
    tile = np.asarray(tile)
    ntile = -(-np.asarray(n) // tile)
    t = cell // tile
    tile_id = (t[:, 0] * ntile[1] + t[:, 1]) * ntile[2] + t[:, 2]
    return (tile_id.astype(np.int64) << 32) | (np.arange(len(points), dtype=np.int64) + row0)


def partition(points, a, b, n, tile, splitters, row0: int = 0):
    """Stable split by destination d = #{splitters <= key}: (send rows in
    destination-major, input order within a destination; counts per
    destination; pos = send position of every input row)."""
    keys = partition_keys(points, a, b, n, tile, row0)
    dest = np.searchsorted(np.asarray(splitters, dtype=np.int64), keys, side="right")
    order = np.argsort(dest, kind="stable")
    pos = np.empty(len(points), dtype=np.int64)
    pos[order] = np.arange(len(points))
    counts = np.bincount(dest, minlength=len(splitters) + 1)
    return np.asarray(points)[order], counts, pos


# ---------------------------------------------------------------------------
# the step before the path (snapshot -> coefficients) and
# the in-package caller that reuses a plan (tube refinement).
# ---------------------------------------------------------------------------


def mirror_extend(values: np.ndarray, a, b, mirror):
    """Append the index-reversed samples along mirrored axes; the box doubles
    there (gpe.py:81-101).  Returns (values, a, b_ext)."""
    b_ext = list(np.asarray(b, dtype=float))
    a = np.asarray(a, dtype=float)
    for d in range(3):
        if mirror[d]:
            values = np.concatenate([values, np.flip(values, axis=d)], axis=d)
            b_ext[d] = a[d] + 2.0 * (b_ext[d] - a[d])
    return values, a, np.asarray(b_ext)


def decompose(values: np.ndarray, a, b) -> np.ndarray:
    """Centred coefficients fftshift(fftn(v)) * prod(sqrt(w)/N) (fourier.py:183-188)."""
    n = np.array(values.shape)
    widths = np.asarray(b, dtype=float) - np.asarray(a, dtype=float)
    scale = float(np.prod(np.sqrt(widths) / n))
    return np.fft.fftshift(scipy.fft.fftn(values, workers=-1)) * scale


def tube_eval(values, a, b, mirror, thresholds, final_filter=None, sigma=2.0, m=6):
    """Adaptive low-density point extraction with one reused plan
    (tube.py:58-127).  Returns (points, density, level) sorted by lattice key."""
    thresholds = [float(t) for t in np.atleast_1d(thresholds)]
    levels = len(thresholds)
    ext, a_ext, b_ext = mirror_extend(values, a, b, mirror)
    coeffs = decompose(ext, a_ext, b_ext)
    shape = np.array(ext.shape)
    widths = b_ext - a_ext
    scale = 3 ** levels
    lattice = shape * scale
    rho_grid = (values.real ** 2 + values.imag ** 2).ravel()
    seeds = np.flatnonzero(rho_grid <= thresholds[0])
    empty = (np.empty((0, 3)), np.empty(0), np.empty(0, dtype=np.int64))
    if seeds.size == 0:
        return empty
    idx = (np.stack(np.unravel_index(seeds, values.shape), axis=1) * scale).astype(np.int64)
    rho = rho_grid[seeds]
    level = np.zeros(idx.shape[0], dtype=np.int64)
    grid, n, beta = oversampled_grid(coeffs, a_ext, b_ext, sigma, m)
    offs = np.stack(np.meshgrid([-1, 0, 1], [-1, 0, 1], [-1, 0, 1], indexing="ij")).reshape(3, 27).T
    for ell in range(1, levels + 1):
        keep = rho <= thresholds[ell - 1]
        if not keep.any():
            return empty
        parents, plevel = idx[keep], level[keep]
        step = 3 ** (levels - ell)
        idx = ((parents[:, None, :] + offs[None, :, :] * step).reshape(-1, 3)) % lattice
        level = np.full(idx.shape[0], ell, dtype=np.int64)
        level[13::27] = plevel
        coords = a_ext + idx * (widths / lattice)
        vals = gather_eval(grid, n, m, beta, coords, a_ext, b_ext)
        rho = vals.real ** 2 + vals.imag ** 2
    if final_filter is not None:
        keep = rho <= float(final_filter)
        idx, rho, level = idx[keep], rho[keep], level[keep]
    if idx.shape[0] == 0:
        return empty
    keys = (idx[:, 0] * lattice[1] + idx[:, 1]) * lattice[2] + idx[:, 2]
    order = np.argsort(keys, kind="stable")
    return a_ext + idx[order] * (widths / lattice), rho[order], level[order]
