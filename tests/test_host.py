"""Host-side pieces of the drop-in API that need no GPU: parameter rules,
helper functions, boundary types, argument errors raised before any device
work (reference tests/test_nufft.py:80-129 and test_rectilinear.py:10-31)."""

import numpy as np
import pytest

import paper_1605_01244_b200 as vfb
from paper_1605_01244_b200.nufft import _kb_beta, _kb_transform, _kb_values, _oversampled_size


def test_params_rules():
    assert vfb.NufftParams.for_accuracy(1e-12).cutoff == 6
    assert vfb.NufftParams.for_accuracy(1e-3).cutoff == 2
    assert vfb.NufftParams.for_accuracy(1e-40).cutoff == 13
    assert vfb.NufftParams(cutoff=6).reached_eps() == pytest.approx(1e-13)
    with pytest.raises(ValueError):
        vfb.NufftParams(oversampling=0.5)
    with pytest.raises(ValueError):
        vfb.NufftParams(cutoff=0)
    with pytest.raises(ValueError):
        vfb.NufftParams(eps=1.0)


def test_kb_helpers():
    beta = _kb_beta(6, 2.0)
    assert beta == pytest.approx(30.501370212790203, rel=1e-15)
    vals = _kb_values(np.array([[0.0, 6.5, -6.5]]), 6, beta)
    assert vals[0, 0] == pytest.approx(1.0)
    assert vals[0, 1] == pytest.approx(1.0 / np.i0(beta), rel=1e-12)
    assert _kb_transform(np.array([0]), 32, 6, beta)[0] > 0
    assert _oversampled_size(16, 2.0) == 32
    assert _oversampled_size(10, 1.6) == 16
    with pytest.raises(ValueError, match="even"):
        _oversampled_size(10, 1.5)


def test_boundary_types(offset_box):
    assert offset_box.volume == pytest.approx(4.0 * 1.0 * 5.0)
    with pytest.raises(ValueError):
        vfb.DomainBox((0, 0, 0), (1, 1, 0))
    with pytest.raises(ValueError, match="even"):
        vfb.SpectralField(offset_box, np.zeros((3, 4, 4)))
    spec = vfb.SpectralField(offset_box, np.zeros((4, 6, 8)))
    assert spec.coeffs.dtype == np.complex128
    np.testing.assert_array_equal(spec.wavenumbers(1), np.arange(6) - 3)


def test_rescale_coeffs_known_answers(offset_box):
    coeffs = np.zeros((4, 6, 8), dtype=complex)
    coeffs[2, 3, 4] = 1.0
    coeffs[3, 3, 4] = 1.0
    fh = vfb.rescale_coeffs(vfb.SpectralField(offset_box, coeffs))
    assert fh[2, 3, 4] == pytest.approx(1.0 / np.sqrt(offset_box.volume), rel=1e-15)
    assert fh[3, 3, 4] == pytest.approx(-1.0 / np.sqrt(offset_box.volume), rel=1e-15)


def test_basis_matrix_checks(unit_box, offset_box):
    with pytest.raises(ValueError, match="right endpoint aliases the left"):
        vfb.basis_matrix(unit_box, 4, 1, np.array([0.5, 1.0]))
    with pytest.raises(ValueError, match="outside"):
        vfb.basis_matrix(unit_box, 4, 2, np.array([-0.01]))
    with pytest.raises(ValueError, match="axis"):
        vfb.basis_matrix(unit_box, 4, 3, np.array([0.5]))
    mat = vfb.basis_matrix(offset_box, 6, 0, np.array([-1.5, 0.0, 2.25]))
    np.testing.assert_allclose(np.abs(mat), 0.5, rtol=1e-14)


def test_rectilinear_argument_errors(unit_box):
    spec = vfb.SpectralField(unit_box, np.ones((4, 4, 4)))
    with pytest.raises(ValueError):
        vfb.eval_rectilinear(spec, [np.array([0.5]), np.array([0.5])])
    with pytest.raises(ValueError, match="outside"):
        vfb.eval_rectilinear(spec, [np.array([0.5]), np.array([1.5]), np.array([0.5])])


def test_points_shape_errors(unit_box):
    with pytest.raises(ValueError, match=r"\(M, 3\)"):
        vfb.map_to_torus(np.zeros((4, 2)), unit_box)


def test_tube_argument_errors():
    dom = vfb.DomainBox((0.0, 0.0, 0.0), (1.0, 1.0, 1.0))
    snap = vfb.Snapshot(dom, np.ones((8, 8, 8)), (False, False, False), 0.0)
    with pytest.raises(ValueError, match="thresholds"):
        vfb.tube_eval(snap, [])
    for bad in ([0.0], [0.2, -1.0]):
        with pytest.raises(ValueError, match="positive"):
            vfb.tube_eval(snap, bad)
    with pytest.raises(ValueError, match="inconsistent"):
        vfb.TubePointCloud(np.zeros((4, 3)), np.zeros(3), np.zeros(3, dtype=np.int64))
    assert vfb.computational_domain(dom, (True, False, True)).b == (2.0, 1.0, 2.0)
