"""Rectilinear evaluation on the device: the exact passes
(hand-written DMMA complex GEMM) and the separable 1D-NUFFT pass mode, vs
the CPU restatement of rectilinear.py:47-64 (oracle) and the NDFT."""

import numpy as np
import pytest

from conftest import random_spectral, rel_err
from oracle import nfft_oracle as O

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def vfb():
    import torch

    if not torch.cuda.is_available():
        pytest.skip("needs a GPU")
    import paper_1605_01244_b200 as pkg

    return pkg


@pytest.mark.parametrize("shape,M,m,tol", [
    ((16, 16, 16), (20, 17, 9), 6, 5e-12),
    ((32, 8, 64), (33, 40, 7), 6, 5e-12),
    ((8, 8, 8), (5, 300, 3), 7, 5e-13),
    ((16, 32, 16), (64, 64, 64), 4, 3e-8),  # m = 4: ~1e-9 per pass, three passes
    ((2, 4, 2), (3, 5, 4), 6, 5e-12),
    ((4, 4, 1024), (3, 4, 50), 6, 5e-12),   # n = 2048 on axis 3: scalar gather
    ((512, 2, 4), (40, 3, 5), 6, 5e-12),    # n = 1024 on axis 1: 8-line DMMA gather
])
def test_nufft_passes_match_exact(vfb, offset_box, shape, M, m, tol):
    spec = random_spectral(offset_box, shape, 1300 + sum(M))
    rng = np.random.default_rng(1310 + m)
    coords = [np.sort(rng.uniform(offset_box.a[d], offset_box.b[d], M[d])) for d in range(3)]
    coords[1][0] = offset_box.a[1]  # the left endpoint
    ref = O.rectilinear(spec.coeffs, offset_box.a, offset_box.b, coords)
    got = vfb.eval_rectilinear(spec, coords, mode="nufft", params=vfb.NufftParams(cutoff=m))
    l2, linf = rel_err(got, ref)
    assert l2 < tol and linf < tol, (l2, linf)
    exact = vfb.eval_rectilinear(spec, coords)
    l2, linf = rel_err(exact, ref)
    etol = 1e-13 if max(shape) <= 64 else 1e-12  # 1024-term axis sums: ~1e-13 rounding
    assert l2 < etol and linf < etol, (l2, linf)


def test_nufft_passes_config4_full(vfb):
    """Config 4 (128^3 -> 256^3 tanh-clustered grid) in NUFFT mode vs the
    exact device passes (themselves <= 1e-13 vs the oracle in
    test_gpu_parity.test_config4_rectilinear_full_size), device-resident."""
    import torch

    from paper_1605_01244_b200 import workloads

    w = workloads.WORKLOADS["c4"]
    spec = vfb.SpectralField(vfb.DomainBox(*w.box), torch.as_tensor(workloads.coefficients("c4"), device="cuda"))
    axes = workloads.rect_axes(256)
    exact = vfb.eval_rectilinear(spec, axes).cpu().numpy()
    fast = vfb.eval_rectilinear(spec, axes, mode="nufft").cpu().numpy()
    l2, linf = rel_err(fast, exact)
    assert l2 < 2e-12 and linf < 2e-12, (l2, linf)  # three passes of ~1e-13 each (gate 1e-10)
    # host coefficients and output: same bits as the device call
    host = vfb.eval_rectilinear(vfb.SpectralField(spec.domain, workloads.coefficients("c4")), axes, mode="nufft")
    np.testing.assert_array_equal(host, fast)


def test_nufft_passes_reject_unsupported_sizes(vfb, unit_box):
    spec = random_spectral(unit_box, (12, 16, 16), 1320)  # sigma N = 24: not a power of two
    coords = [np.linspace(0, 0.9, 5)] * 3
    with pytest.raises(ValueError, match="power of two"):
        vfb.eval_rectilinear(spec, coords, mode="nufft")
    with pytest.raises(ValueError, match="mode"):
        vfb.eval_rectilinear(spec, coords, mode="fast")
    got = vfb.eval_rectilinear(spec, coords)  # the exact mode covers it
    ref = O.rectilinear(spec.coeffs, unit_box.a, unit_box.b, coords)
    assert rel_err(got, ref)[1] < 1e-13


@pytest.mark.parametrize("M,K", [(1, 1), (7, 3), (65, 130), (200, 33)])
def test_exact_passes_ragged_gemm_shapes(vfb, offset_box, M, K):
    """Tile edges of the DMMA complex GEMM (64 x 64 x 16 tiles): mode counts
    and coordinate counts that are not tile multiples."""
    shape = (2 * K, 2 * ((K + 1) // 2 + 1), 2)
    spec = random_spectral(offset_box, shape, 1330 + M + K)
    rng = np.random.default_rng(1331 + M)
    coords = [rng.uniform(offset_box.a[d], offset_box.b[d], max(1, M - d)) for d in range(3)]
    ref = O.rectilinear(spec.coeffs, offset_box.a, offset_box.b, coords)
    got = vfb.eval_rectilinear(spec, coords)
    l2, linf = rel_err(got, ref)
    assert l2 < 1e-13 and linf < 1e-13, (l2, linf)


def test_nufft_passes_unsorted_duplicate_coordinates_and_out(vfb, offset_box):
    """The NUFFT passes take coordinate vectors in any order, with repeats and
    the left endpoint, host or device, and write into a caller's ``out``."""
    import torch

    spec = random_spectral(offset_box, (16, 8, 32), 1950)
    rng = np.random.default_rng(1951)
    coords = []
    for d, M in enumerate((11, 7, 13)):
        c = rng.uniform(offset_box.a[d], offset_box.b[d], M)
        c[2] = c[5]                      # a repeat
        c[0] = offset_box.a[d]           # the left endpoint
        coords.append(c)                 # unsorted
    ref = O.rectilinear(spec.coeffs, offset_box.a, offset_box.b, coords)
    host = vfb.eval_rectilinear(spec, coords, mode="nufft")
    assert rel_err(host, ref)[1] < 5e-12
    out = np.empty((11, 7, 13), dtype=np.complex128)
    assert vfb.eval_rectilinear(spec, coords, out=out, mode="nufft") is out
    np.testing.assert_array_equal(out, host)
    dspec = vfb.SpectralField(offset_box, torch.as_tensor(spec.coeffs, device="cuda"))
    dev = vfb.eval_rectilinear(dspec, coords, mode="nufft")
    np.testing.assert_array_equal(dev.cpu().numpy(), host)


@pytest.mark.parametrize("scalar", [False, True])
def test_nufft_passes_gather_variants(vfb, offset_box, scalar, monkeypatch):
    """The DMMA octet gather (sorted targets, 8 lines per CTA) and the scalar
    tap loop of the NUFFT passes agree with the exact passes, with clustered,
    sparse, unsorted and wrap-around coordinates."""
    if scalar:
        monkeypatch.setenv("VFN_RECT_SCALAR", "1")
    spec = random_spectral(offset_box, (32, 16, 64), 1960)
    rng = np.random.default_rng(1961)
    a, b = np.asarray(offset_box.a), np.asarray(offset_box.b)
    coords = [np.concatenate([rng.uniform(a[0], b[0], 20), a[0] + (b[0] - a[0]) * (1 - rng.uniform(0, 1e-3, 5))]),
              rng.uniform(a[1], b[1], 3),                                   # sparse: wide octet windows
              np.clip(rng.normal((a[2] + b[2]) / 2, 0.01, 70), a[2], np.nextafter(b[2], a[2]))]  # clustered
    exact = vfb.eval_rectilinear(spec, coords)
    fast = vfb.eval_rectilinear(spec, coords, mode="nufft")
    l2, linf = rel_err(fast, exact)
    assert l2 < 5e-12 and linf < 5e-12, (l2, linf)
