"""Pin the CPU oracle (oracle/nfft_oracle.py) against golden vectors that
tests/golden/make_golden.py recorded from the real reference package."""

import numpy as np
import pytest

from conftest import golden, rel_err
from oracle import nfft_oracle as O


def test_torus_map_bit_exact():
    g = golden("torus_edges.npz")
    zeta = O.torus_map(g["points"], g["a"], g["b"])
    np.testing.assert_array_equal(zeta, g["zeta"])
    # the +1/2 edge (survey fact 5) is present in the fixture
    assert (g["zeta"] == 0.5).any()


def test_nearest_cells_bit_exact():
    g = golden("torus_edges.npz")
    _, l0 = O.nearest_cells(g["points"], g["a"], g["b"], g["n"])
    np.testing.assert_array_equal(l0, g["l0"])
    assert (g["l0"] == g["n"]).any()  # l0 == n edge


def test_kb_tables():
    g = golden("kb_tables.npz")
    for m, sigma, nmodes in ((6, 2.0, 32), (3, 2.0, 16), (13, 2.0, 24), (6, 1.6, 20)):
        key = f"m{m}_s{sigma}"
        beta = O.kb_beta(m, sigma)
        assert beta == float(g[key + "_beta"])
        n = O.grid_size(nmodes, sigma)
        assert n == int(g[key + "_n"])
        np.testing.assert_array_equal(O.kb_hat(O.centered_wavenumbers(nmodes), n, m, beta), g[key + "_hat"])
        np.testing.assert_array_equal(O.kb_window(g[key + "_v"], m, beta), g[key + "_win"])
    assert O.kb_beta(6, 2.0) == pytest.approx(30.501370212790203, rel=1e-15)


def test_grid_size_rules():
    assert O.grid_size(16, 2.0) == 32
    assert O.grid_size(10, 1.6) == 16
    with pytest.raises(ValueError, match="even"):
        O.grid_size(10, 1.5)
    with pytest.raises(ValueError):
        O.grid_size(16, 0.5)


def _cases():
    g = golden("nufft_cases.npz")
    for i in range(int(g["ncases"])):
        yield i, {k.split("_", 1)[1]: g[k] for k in g.files if k.startswith(f"case{i}_")}


@pytest.mark.parametrize("i", range(8))
def test_oversampled_grid_and_gather_match_reference(i):
    c = dict(_cases())[i]
    sigma, m = float(c["params"][0]), int(c["params"][1])
    grid, n, beta = O.oversampled_grid(c["coeffs"], c["a"], c["b"], sigma, m)
    if "grid" in c:
        np.testing.assert_array_equal(grid, c["grid"])
    out = O.gather_eval(grid, n, m, beta, c["points"], c["a"], c["b"])
    np.testing.assert_array_equal(out, c["nufft"])


@pytest.mark.parametrize("i", [0, 1, 5])
def test_ndft_matches_reference_direct(i):
    c = dict(_cases())[i]
    out = O.ndft(c["coeffs"], c["a"], c["b"], c["points"])
    l2, linf = rel_err(out, c["direct"])
    assert l2 < 1e-14 and linf < 1e-14


@pytest.mark.parametrize("i", [0, 1])
def test_scalar_series_matches_reference_direct(i):
    """The term-by-term scalar sum (the reference's own independent oracle,
    tests/oracles.py:19-33, restated) against the reference's eval_direct
    values on a few points of the golden cases."""
    c = dict(_cases())[i]
    pts = c["points"][:: max(1, len(c["points"]) // 6)][:6]
    ref = c["direct"][:: max(1, len(c["points"]) // 6)][:6]
    got = np.array([O.series_scalar(c["coeffs"], c["a"], c["b"], x) for x in pts])
    assert np.abs(got - ref).max() <= 1e-12 * np.abs(c["direct"]).max()


def test_config1_against_reference():
    from paper_1605_01244_b200 import workloads

    g = golden("config1.npz")
    coeffs = workloads.coefficients("c1")
    pts = workloads.points("c1")
    np.testing.assert_array_equal(
        np.array([coeffs.real.sum(), coeffs.imag.sum(), np.abs(coeffs).sum()]), g["coeffs_sum"]
    )
    np.testing.assert_array_equal(pts.sum(axis=0), g["points_sum"])
    a, b = workloads.UNIT_BOX
    out = O.nufft_eval(coeffs, a, b, pts)
    np.testing.assert_array_equal(out, g["nufft"])
    l2, linf = rel_err(out[:200], g["direct200"])
    assert l2 < 1e-12 and linf < 1e-12


def test_cluster_small_against_reference():
    g = golden("cluster_small.npz")
    from paper_1605_01244_b200 import workloads

    a, b = workloads.VORTEX_BOX
    out = O.nufft_eval(g["coeffs"], a, b, g["points"])
    np.testing.assert_array_equal(out, g["nufft"])
    np.testing.assert_array_equal(
        workloads.vortex_pair_spectrum((32, 32, 32), workloads.VORTEX_BOX), g["coeffs"]
    )


def test_rectilinear_against_reference():
    g = golden("rect_cases.npz")
    for i in range(int(g["ncases"])):
        a, b = g[f"case{i}_a"], g[f"case{i}_b"]
        coords = [g[f"case{i}_y{d}"] for d in range(3)]
        coeffs = g[f"case{i}_coeffs"]
        for d in range(3):
            np.testing.assert_array_equal(O.basis_matrix(a[d], b[d], coeffs.shape[d], coords[d]), g[f"case{i}_E{d}"])
        np.testing.assert_array_equal(O.rectilinear(coeffs, a, b, coords), g[f"case{i}_out"])


def test_bin_permutation_is_stable_sort_of_keys():
    g = golden("torus_edges.npz")
    keys = O.bin_keys(g["points"], g["a"], g["b"], g["n"])
    perm = O.bin_permutation(g["points"], g["a"], g["b"], g["n"])
    assert np.all(np.diff(keys[perm]) >= 0)
    # stability: equal keys keep input order
    same = keys[perm][1:] == keys[perm][:-1]
    assert np.all(perm[1:][same] > perm[:-1][same])


def test_domain_violation():
    a, b = (0.0, 0.0, 0.0), (1.0, 1.0, 1.0)
    pts = np.array([[0.5, 0.5, 0.5], [0.5, 1.0, 0.5], [np.nan, 0.1, 0.1]])
    assert O.domain_violation(pts, a, b) == 1
    assert O.domain_violation(pts[[0, 2]], a, b) == 1
    assert O.domain_violation(pts[:1], a, b) == -1


def test_tube_oracle_matches_reference():
    """The oracle's snapshot_spectral and tube_eval restatements reproduce the
    reference (tube.py:58-127, gpe.py:90-113) bit for bit."""
    g = golden("tube_case.npz")
    ext, a, b = O.mirror_extend(g["values"], g["a"], g["b"], g["mirror"])
    np.testing.assert_array_equal(O.decompose(ext, a, b), g["spectral"])
    for tag, thr, ff in (("two", [0.4, 0.3], None), ("one", [0.4], None), ("filt", [0.4, 0.3], 0.15)):
        p, rho, lev = O.tube_eval(g["values"], g["a"], g["b"], g["mirror"], thr, ff)
        np.testing.assert_array_equal(p, g[f"{tag}_points"])
        np.testing.assert_array_equal(rho, g[f"{tag}_density"])
        np.testing.assert_array_equal(lev, g[f"{tag}_level"])
    levels, counts = np.unique(g["two_level"], return_counts=True)
    assert counts.tolist() == [16, 992, 26208]  # reference test_tube.py:85-89
