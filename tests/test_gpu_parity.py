"""GPU parity: the CUDA path (through the C ABI) against the reference's golden
vectors and the CPU oracle, on the same seeded inputs.

Tolerances: integer/index work (torus map, nearest cell, bin key,
permutation) is bit-exact; floating point must match the reference within
1e-10 relative l2 / l-inf (north star), and in practice lands near 1e-14,
which is what most asserts below pin.
"""

import warnings

import numpy as np
import pytest

from conftest import golden, random_spectral, rel_err
from oracle import nfft_oracle as O

pytestmark = pytest.mark.gpu

TOL = 1e-10  # north-star gate (relative l2 and l-inf vs the reference)


@pytest.fixture(scope="module")
def vfb():
    import torch

    assert torch.cuda.is_available(), "GPU tests need a CUDA device"
    import paper_1605_01244_b200 as pkg

    return pkg


def cases():
    g = golden("nufft_cases.npz")
    out = []
    for i in range(int(g["ncases"])):
        out.append({k.split("_", 1)[1]: g[k] for k in g.files if k.startswith(f"case{i}_")})
    return out


CASES = cases()


def make_plan(vfb, c):
    sigma, m = float(c["params"][0]), int(c["params"][1])
    spec = vfb.SpectralField(vfb.DomainBox(tuple(c["a"]), tuple(c["b"])), c["coeffs"])
    with warnings.catch_warnings():
        warnings.simplefilter("ignore")
        return spec, vfb.NufftPlan(spec, vfb.NufftParams(oversampling=sigma, cutoff=m, eps=0.999))


# ---------------------------------------------------------------- K1 (bit-exact)


def test_map_to_torus_bit_exact(vfb):
    g = golden("torus_edges.npz")
    box = vfb.DomainBox(tuple(g["a"]), tuple(g["b"]))
    zeta = vfb.map_to_torus(g["points"], box)
    np.testing.assert_array_equal(zeta, g["zeta"])


@pytest.mark.parametrize("a,w", [((1.0e6, -3.0e5, 12.5), (2.0, 0.5, 3.0)),
                                 ((-7.25, 1.0e-3, 4.0e9), (1.0e-2, 3.0e-4, 1.0e3))])
def test_far_offset_and_tiny_boxes(vfb, a, w):
    """Boxes far from the origin or much smaller than 1: the torus map stays
    bit-exact vs the oracle (numpy's arithmetic; (x - a) / (a - b) loses the
    low bits the same way), bin keys and permutation bit-exact, values vs the
    oracle's gather on every path (binned tensor-core, warp per point)."""
    a = np.array(a)
    b = a + np.array(w)
    box = vfb.DomainBox(tuple(a), tuple(b))
    rng = np.random.default_rng(800)
    pts = a + rng.uniform(0.0, 1.0, (60000, 3)) * np.array(w)
    pts = np.minimum(pts, np.nextafter(b, a))
    pts[:4] = [a, np.nextafter(b, a), a + np.array(w) / 2, a + np.array(w) / 4]
    np.testing.assert_array_equal(vfb.map_to_torus(pts, box), O.torus_map(pts, a, b))
    spec = random_spectral(box, (12, 10, 14), 801)
    plan = vfb.NufftPlan(spec)
    keys, perm = plan.bin(pts)
    bx, tl = plan.geometry(len(pts))
    ref_keys = O.bin_keys(pts, a, b, plan._n, bx, tl, plan.key_shift())
    np.testing.assert_array_equal(keys.astype(np.int64), ref_keys)
    np.testing.assert_array_equal(perm, np.argsort(ref_keys, kind="stable"))
    grid, n, beta = O.oversampled_grid(spec.coeffs, tuple(a), tuple(b), 2.0, 6)
    sub = rng.choice(len(pts), 3000, replace=False)
    ref = O.gather_eval(grid, n, 6, beta, pts[sub], tuple(a), tuple(b))
    for variant in (0, 3):
        plan.set_gather(variant)
        l2, linf = rel_err(plan.evaluate(pts)[sub], ref)
        assert l2 < 1e-13 and linf < 1e-13, (variant, l2, linf)


def test_bin_sort_bit_exact_vs_cpu_stable_sort(vfb, offset_box):
    g = golden("torus_edges.npz")
    spec = random_spectral(vfb.DomainBox(tuple(g["a"]), tuple(g["b"])), (16, 16, 16), 7)
    plan = vfb.NufftPlan(spec)
    rng = np.random.default_rng(11)
    pts = np.vstack([g["points"], rng.uniform(g["a"], g["b"], (20000, 3))])
    keys, perm = plan.bin(pts)
    box, tile = plan.geometry(len(pts))
    ref_keys = O.bin_keys(pts, g["a"], g["b"], plan._n, box, tile, plan.key_shift())
    np.testing.assert_array_equal(keys.astype(np.int64), ref_keys)
    np.testing.assert_array_equal(perm, np.argsort(ref_keys, kind="stable"))


def test_bin_sort_bit_exact_clustered(vfb):
    g = golden("cluster_small.npz")
    from paper_1605_01244_b200 import workloads

    box = vfb.DomainBox(*workloads.VORTEX_BOX)
    plan = vfb.NufftPlan(vfb.SpectralField(box, g["coeffs"]))
    keys, perm = plan.bin(g["points"])
    bx, tl = plan.geometry(len(g["points"]))
    ref = O.bin_keys(g["points"], box.a, box.b, plan._n, bx, tl, plan.key_shift())
    np.testing.assert_array_equal(keys.astype(np.int64), ref)
    np.testing.assert_array_equal(perm, np.argsort(ref, kind="stable"))


# ---------------------------------------------------------------- K2 + K3


@pytest.mark.parametrize("i", [i for i, c in enumerate(CASES) if "grid" in c])
def test_plan_grid_matches_reference(vfb, i):
    c = CASES[i]
    _, plan = make_plan(vfb, c)
    l2, linf = rel_err(plan._grid, c["grid"])
    assert l2 < 1e-13 and linf < 1e-13, (l2, linf)


# ---------------------------------------------------------------- K4 end to end


@pytest.mark.parametrize("i", range(len(CASES)))
def test_evaluate_matches_reference(vfb, i):
    c = CASES[i]
    spec, plan = make_plan(vfb, c)
    out = plan.evaluate(c["points"])
    l2, linf = rel_err(out, c["nufft"])
    m = int(c["params"][1])
    tol = 1e-13 if m >= 3 else 1e-11
    assert l2 < tol and linf < tol, (l2, linf)
    # the reference's own accuracy budget vs the exact sum (test_nufft.py:136-146)
    if m >= 6 and float(c["params"][0]) == 2.0:
        mass = np.abs(vfb.rescale_coeffs(spec)).sum()
        assert np.abs(out - c["direct"]).max() <= 1e-12 * mass


@pytest.mark.parametrize("variant", [1, 2, 3])
def test_gather_variants_agree(vfb, variant):
    c = CASES[0]
    _, plan = make_plan(vfb, c)
    try:
        plan.set_gather(variant)
        out = plan.evaluate(c["points"])
    except ValueError as e:
        pytest.skip(str(e))
    l2, linf = rel_err(out, c["nufft"])
    assert l2 < 1e-13 and linf < 1e-13


def test_config1_full(vfb):
    from paper_1605_01244_b200 import workloads

    g = golden("config1.npz")
    spec = vfb.SpectralField(vfb.DomainBox(*workloads.UNIT_BOX), workloads.coefficients("c1"))
    out = vfb.NufftPlan(spec).evaluate(workloads.points("c1"))
    l2, linf = rel_err(out, g["nufft"])
    assert l2 < 1e-13 and linf < 1e-13, (l2, linf)
    l2, linf = rel_err(out[:200], g["direct200"])
    assert l2 < 1e-12 and linf < 1e-12


def test_cluster_seam(vfb):
    from paper_1605_01244_b200 import workloads

    g = golden("cluster_small.npz")
    spec = vfb.SpectralField(vfb.DomainBox(*workloads.VORTEX_BOX), g["coeffs"])
    out = vfb.NufftPlan(spec).evaluate(g["points"])
    l2, linf = rel_err(out, g["nufft"])
    assert l2 < 1e-13 and linf < 1e-13, (l2, linf)
    l2, linf = rel_err(out[:100], g["direct"])
    assert l2 < 1e-11 and linf < 1e-11


def test_edge_points(vfb):
    """zeta = +1/2 and l0 == n rows (survey fact 5) evaluate like the oracle."""
    g = golden("torus_edges.npz")
    box = vfb.DomainBox(tuple(g["a"]), tuple(g["b"]))
    spec = random_spectral(box, (16, 16, 16), 9)
    out = vfb.NufftPlan(spec).evaluate(g["points"])
    ref = O.nufft_eval(spec.coeffs, g["a"], g["b"], g["points"])
    l2, linf = rel_err(out, ref)
    assert l2 < 1e-13 and linf < 1e-13


# ---------------------------------------------------------------- determinism / API


def test_plan_reuse_is_bitwise_stable(vfb, offset_box):
    spec = random_spectral(offset_box, (12, 12, 12), 81)
    rng = np.random.default_rng(82)
    pts_a = rng.uniform(offset_box.a, offset_box.b, (40, 3))
    pts_b = rng.uniform(offset_box.a, offset_box.b, (25, 3))
    plan = vfb.NufftPlan(spec)
    first = plan.evaluate(pts_a)
    plan.evaluate(pts_b)
    np.testing.assert_array_equal(first, plan.evaluate(pts_a))
    np.testing.assert_array_equal(first, vfb.eval_nufft(spec, pts_a))


def test_batch_composition_invariance(vfb, offset_box):
    """A point's value does not depend on which other points share the call,
    on either gather (binned tensor-core: set_gather(2); warp per point: 3);
    the automatic choice by M switches between them, whose values agree to
    rounding."""
    spec = random_spectral(offset_box, (16, 16, 16), 90)
    rng = np.random.default_rng(91)
    pts = rng.uniform(offset_box.a, offset_box.b, (50000, 3))
    plan = vfb.NufftPlan(spec)
    plan.set_box(2)  # the automatic box width depends on M (density)
    sel = rng.permutation(len(pts))[:5000]
    fulls = []
    for variant in (2, 3):
        plan.set_gather(variant)
        full = plan.evaluate(pts)
        np.testing.assert_array_equal(full[:777], plan.evaluate(pts[:777]))
        np.testing.assert_array_equal(full[sel], plan.evaluate(pts[sel]))
        fulls.append(full)
    l2, linf = rel_err(fulls[1], fulls[0])
    assert l2 < 1e-14 and linf < 1e-14, (l2, linf)
    plan.set_gather(0)
    np.testing.assert_array_equal(plan.evaluate(pts), fulls[0])          # 50000 > WARP_MAX_M
    np.testing.assert_array_equal(plan.evaluate(pts[sel]), fulls[1][sel])  # 5000 <= WARP_MAX_M


@pytest.mark.parametrize("m", [2, 4, 5, 6, 7])
def test_gather_density_modes_are_bitwise_equal(vfb, offset_box, m, monkeypatch):
    """The tensor-core gather picks its CTA shape from the point density:
    16 warps, 12 warps, or half-units (even warps sum the real parts of a
    unit, odd warps the imaginary parts; vfn_gather_tc.cu SPLIT).  A value's
    bits must not depend on the mode (nufft.py:264-271 sums each point on its
    own), at both box widths and for sparse and dense sets."""
    spec = random_spectral(offset_box, (20, 16, 24), 93)
    rng = np.random.default_rng(94)
    with warnings.catch_warnings():
        warnings.simplefilter("ignore")
        plan = vfb.NufftPlan(spec, vfb.NufftParams(cutoff=m, eps=0.999))
    plan.set_graphs(False)  # the mode is read per launch; a replayed graph would keep the first one
    plan.set_gather(2)
    w = np.asarray(offset_box.b) - np.asarray(offset_box.a)
    sets = {
        "sparse": rng.uniform(offset_box.a, offset_box.b, (40000, 3)),
        "dense": np.asarray(offset_box.a) + w * (0.4 + 0.05 * rng.random((60000, 3))),
    }
    for name, pts in sets.items():
        for box in (1, 2):
            plan.set_box(box)
            outs = []
            for mode in ("16", "12", "s16"):
                monkeypatch.setenv("VFN_WARPS", mode)
                outs.append(plan.evaluate(pts))
            monkeypatch.delenv("VFN_WARPS")
            auto = plan.evaluate(pts)
            for o in outs[1:] + [auto]:
                np.testing.assert_array_equal(o, outs[0], err_msg=f"{name} box {box}")
    ref = vfb.eval_direct(spec, sets["sparse"][:200])
    l2, linf = rel_err(plan.evaluate(sets["sparse"])[:200], ref)
    assert linf < {2: 1e-3, 4: 1e-7, 5: 1e-9, 6: 1e-11, 7: 1e-12}[m], (l2, linf)


def test_torch_cuda_tensors_match_numpy(vfb, offset_box):
    import torch

    spec = random_spectral(offset_box, (16, 16, 16), 92)
    rng = np.random.default_rng(93)
    pts = rng.uniform(offset_box.a, offset_box.b, (5000, 3))
    host = vfb.NufftPlan(spec).evaluate(pts)
    dspec = vfb.SpectralField(offset_box, torch.as_tensor(spec.coeffs, device="cuda"))
    dev = vfb.NufftPlan(dspec).evaluate(torch.as_tensor(pts, device="cuda"))
    assert dev.is_cuda and dev.dtype == torch.complex128
    np.testing.assert_array_equal(dev.cpu().numpy(), host)


def test_empty_and_outside(vfb, unit_box):
    spec = random_spectral(unit_box, (8, 8, 8), 83)
    plan = vfb.NufftPlan(spec)
    out = plan.evaluate(np.empty((0, 3)))
    assert out.shape == (0,) and out.dtype == np.complex128
    with pytest.raises(ValueError, match=r"point \[1.0, 0.5, 0.5\] \(row 0\) lies outside"):
        plan.evaluate(np.array([[1.0, 0.5, 0.5]]))
    with pytest.raises(ValueError, match=r"\(row 2\)"):
        plan.evaluate(np.array([[0.1, 0.1, 0.1], [0.2, 0.2, 0.2], [np.nan, 0.5, 0.5], [2.0, 0, 0]]))
    with pytest.raises(ValueError, match="outside"):
        vfb.eval_direct(spec, np.array([[0.5, 0.5, 1.5]]))
    # the plan stays usable after an error
    assert plan.evaluate(np.array([[0.5, 0.5, 0.5]])).shape == (1,)


def test_warnings_match_reference(vfb, unit_box):
    spec = random_spectral(unit_box, (8, 8, 8), 57)
    with pytest.warns(vfb.AccuracyWarning, match="degraded"):
        vfb.NufftPlan(spec, vfb.NufftParams(cutoff=1))
    with pytest.warns(vfb.AccuracyWarning, match="short of"):
        vfb.NufftPlan(spec, vfb.NufftParams(cutoff=3, eps=1e-12))


def test_error_decreases_with_cutoff(vfb, offset_box):
    spec = random_spectral(offset_box, (16, 16, 16), 70)
    rng = np.random.default_rng(2070)
    pts = rng.uniform(offset_box.a, offset_box.b, (100, 3))
    ref = vfb.eval_direct(spec, pts)
    errs = []
    for m in (2, 3, 4, 6, 8):
        out = vfb.NufftPlan(spec, vfb.NufftParams(cutoff=m, eps=0.999)).evaluate(pts)
        errs.append(np.abs(out - ref).max())
    for lo, hi in zip(errs[1:], errs[:-1]):
        assert lo <= hi * 1.1


# ---------------------------------------------------------------- K6 / K5


@pytest.mark.parametrize("i", [0, 1, 5])
def test_direct_matches_reference(vfb, i):
    c = CASES[i]
    spec = vfb.SpectralField(vfb.DomainBox(tuple(c["a"]), tuple(c["b"])), c["coeffs"])
    out = vfb.eval_direct(spec, c["points"])
    l2, linf = rel_err(out, c["direct"])
    assert l2 < 1e-13 and linf < 1e-13


def test_direct_matches_scalar_series(vfb, offset_box):
    """The device NDFT (K6) against a term-by-term scalar sum in another
    summation order (oracle.series_scalar, after the reference's
    tests/oracles.py:19-33), as the reference's test_nufft.py:60-67 pins
    eval_direct."""
    spec = random_spectral(offset_box, (12, 10, 14), 2200)
    rng = np.random.default_rng(2201)
    pts = rng.uniform(offset_box.a, offset_box.b, (40, 3))
    out = vfb.eval_direct(spec, pts)
    scale = np.abs(out).max()
    for i in range(0, 40, 6):
        ref = O.series_scalar(spec.coeffs, offset_box.a, offset_box.b, pts[i])
        assert abs(out[i] - ref) <= 1e-12 * scale


def test_rectilinear_matches_reference(vfb):
    g = golden("rect_cases.npz")
    for i in range(int(g["ncases"])):
        box = vfb.DomainBox(tuple(g[f"case{i}_a"]), tuple(g[f"case{i}_b"]))
        spec = vfb.SpectralField(box, g[f"case{i}_coeffs"])
        out = vfb.eval_rectilinear(spec, [g[f"case{i}_y{d}"] for d in range(3)])
        ref = g[f"case{i}_out"]
        assert out.shape == ref.shape
        l2, linf = rel_err(out, ref)
        assert l2 < 1e-13 and linf < 1e-13, (i, l2, linf)


def test_rectilinear_out_argument_and_slabs(vfb):
    """eval_rectilinear(..., out=): device outputs are bitwise the device
    result; host outputs (pass 3 in slabs with overlapped downloads, also
    with fewer output rows than slabs) are bitwise identical for pageable and
    pinned memory and agree with the device result to rounding (cuBLAS may
    pick another kernel for a slab's GEMM shape)."""
    import torch

    g = golden("rect_cases.npz")
    for i in range(int(g["ncases"])):
        box = vfb.DomainBox(tuple(g[f"case{i}_a"]), tuple(g[f"case{i}_b"]))
        coeffs = g[f"case{i}_coeffs"]
        ys = [g[f"case{i}_y{d}"] for d in range(3)]
        for y0 in (ys[0], ys[0][:3]):
            axes = [y0, ys[1], ys[2]]
            shape = (len(y0), len(ys[1]), len(ys[2]))
            dev = vfb.eval_rectilinear(vfb.SpectralField(box, torch.as_tensor(coeffs, device="cuda")), axes)
            o = torch.empty(shape, dtype=torch.complex128, device="cuda")
            vfb.eval_rectilinear(vfb.SpectralField(box, torch.as_tensor(coeffs, device="cuda")), axes, out=o)
            assert torch.equal(o, dev)
            plain = vfb.eval_rectilinear(vfb.SpectralField(box, coeffs), axes)
            pinned = torch.empty(shape, dtype=torch.complex128, pin_memory=True).numpy()
            vfb.eval_rectilinear(vfb.SpectralField(box, coeffs), axes, out=pinned)
            ref = dev.cpu().numpy()
            assert np.array_equal(plain, pinned)
            l2, linf = rel_err(plain, ref)
            assert l2 < 1e-14 and linf < 1e-14, (i, l2, linf)
    with pytest.raises(ValueError):
        vfb.eval_rectilinear(vfb.SpectralField(box, coeffs), ys, out=np.empty((1, 1, 1), complex))


def test_rectilinear_axis_permutation_and_single_point(vfb, offset_box):
    """Properties the reference tests for the rectilinear path
    (test_rectilinear.py): permuting the axes of the coefficients, the box and
    the coordinate lists permutes the output (rtol 1e-12); a 1x1x1 grid
    equals the exact sum at that point (rel 1e-13)."""
    rng = np.random.default_rng(600)
    spec = random_spectral(offset_box, (6, 8, 10), 601)
    a, b = np.array(offset_box.a), np.array(offset_box.b)
    ys = [np.sort(rng.uniform(a[d], b[d], n)) for d, n in enumerate((5, 7, 9))]
    out = vfb.eval_rectilinear(spec, ys)
    perm = (2, 0, 1)
    pbox = vfb.DomainBox(tuple(a[list(perm)]), tuple(b[list(perm)]))
    pspec = vfb.SpectralField(pbox, np.ascontiguousarray(spec.coeffs.transpose(perm)))
    pout = vfb.eval_rectilinear(pspec, [ys[d] for d in perm])
    np.testing.assert_allclose(pout, out.transpose(perm), rtol=1e-12, atol=1e-12 * np.abs(out).max())
    x = np.array([[ys[0][2], ys[1][3], ys[2][4]]])
    one = vfb.eval_rectilinear(spec, [x[:, 0], x[:, 1], x[:, 2]])[0, 0, 0]
    direct = O.ndft(spec.coeffs, offset_box.a, offset_box.b, x)[0]
    assert abs(one - direct) <= 1e-13 * abs(direct)
    assert abs(vfb.eval_direct(spec, x)[0] - direct) <= 1e-13 * abs(direct)


def test_rectilinear_slabs_per_rank(vfb, offset_box):
    """parallel.eval_rectilinear_sharded: the axis-1 slabs of 1, 2, 3 and 5
    ranks (evaluated here one after another on this GPU) concatenate to
    the unsharded grid within 1e-14 (last-pass GEMM shapes differ)."""
    from paper_1605_01244_b200.parallel import eval_rectilinear_sharded

    rng = np.random.default_rng(700)
    spec = random_spectral(offset_box, (12, 10, 8), 701)
    a, b = np.array(offset_box.a), np.array(offset_box.b)
    coords = [np.sort(rng.uniform(a[d], b[d], n)) for d, n in enumerate((37, 20, 16))]
    full = vfb.eval_rectilinear(spec, coords)
    for world in (1, 2, 3, 5):
        slabs = [eval_rectilinear_sharded(spec, coords, r, world) for r in range(world)]
        got = np.concatenate(slabs, axis=0)
        l2, linf = rel_err(got, full)
        assert got.shape == full.shape and l2 < 1e-14 and linf < 1e-14, (world, l2, linf)


def test_rectilinear_unsorted_duplicate_and_edge_coordinates(vfb, offset_box):
    """Coordinate vectors need not be sorted (rectilinear.py:47-64): shuffled
    and repeated values and the left edge a (never b) on every axis, vs the
    oracle; a repeated coordinate gives bitwise equal slices."""
    rng = np.random.default_rng(990)
    spec = random_spectral(offset_box, (10, 12, 8), 991)
    a, b = np.array(offset_box.a), np.array(offset_box.b)
    ys = []
    for d, n in enumerate((9, 7, 11)):
        y = rng.uniform(a[d], b[d], n)
        y[1] = y[4]  # duplicate
        y[2] = a[d]  # left edge
        y[3] = np.nextafter(b[d], a[d])
        ys.append(y)
    out = vfb.eval_rectilinear(spec, ys)
    ref = O.rectilinear(spec.coeffs, offset_box.a, offset_box.b, ys)
    l2, linf = rel_err(out, ref)
    assert l2 < 1e-13 and linf < 1e-13, (l2, linf)
    assert np.array_equal(out[1], out[4]) and np.array_equal(out[:, 1], out[:, 4])
    with pytest.raises(ValueError, match="right endpoint aliases the left"):
        vfb.eval_rectilinear(spec, [np.append(ys[0], b[0]), ys[1], ys[2]])


def test_decompose_and_synthesize_regular(vfb, offset_box):
    """decompose / synthesize_regular (fourier.py:183-196) on the device vs
    numpy's restatement (fftshift(fftn(v)) * s and ifftn(ifftshift(c)) / s,
    s = prod sqrt(w) / N), the round trip, torch CUDA tensors in and out,
    and synthesize_regular vs the NUFFT at the regular grid points."""
    import torch

    rng = np.random.default_rng(995)
    shape = (12, 20, 16)
    vals = rng.standard_normal(shape) + 1j * rng.standard_normal(shape)
    s = float(np.prod(np.sqrt(offset_box.widths) / np.array(shape)))
    spec = vfb.decompose(vfb.PhysicalField(offset_box, vals))
    ref = np.fft.fftshift(np.fft.fftn(vals)) * s
    l2, linf = rel_err(spec.coeffs, ref)
    assert l2 < 1e-14 and linf < 1e-14, (l2, linf)
    back = vfb.synthesize_regular(spec).values
    l2, linf = rel_err(back, vals)
    assert l2 < 1e-14 and linf < 1e-14, (l2, linf)
    ref_back = np.fft.ifftn(np.fft.ifftshift(ref)) / s
    l2, linf = rel_err(back, ref_back)
    assert l2 < 1e-14 and linf < 1e-14, (l2, linf)
    dspec = vfb.decompose(vfb.PhysicalField(offset_box, torch.as_tensor(vals, device="cuda")))
    assert dspec.coeffs.is_cuda and np.array_equal(dspec.coeffs.cpu().numpy(), spec.coeffs)
    dback = vfb.synthesize_regular(dspec).values
    assert dback.is_cuda and np.array_equal(dback.cpu().numpy(), back)
    grid = np.stack(np.meshgrid(*vfb.regular_grid(offset_box, shape), indexing="ij"), -1).reshape(-1, 3)
    at_grid = vfb.NufftPlan(spec).evaluate(grid).reshape(shape)
    assert np.abs(at_grid - back).max() <= 1e-11 * np.abs(back).max()  # NUFFT truncation (white spectrum)
    with pytest.raises(ValueError, match="even"):
        vfb.PhysicalField(offset_box, np.zeros((3, 4, 4), complex))


def test_rectilinear_regular_grid_matches_fft(vfb, offset_box):
    spec = random_spectral(offset_box, (12, 12, 12), 43)
    axes = vfb.regular_grid(offset_box, spec.coeffs.shape)
    out = vfb.eval_rectilinear(spec, axes)
    # inverse DFT on the regular grid (fourier.py:191-196)
    n = np.array(spec.coeffs.shape)
    scale = float(np.prod(np.sqrt(offset_box.widths) / n))
    ref = np.fft.ifftn(np.fft.ifftshift(spec.coeffs)) / scale
    assert np.abs(out - ref).max() <= 1e-12 * np.abs(ref).max()


def test_acceptance_geometry_grid_and_points(vfb):
    """The reference's acceptance criteria 1-3 restated (test_acceptance.py:27-85):
    a 64^3 spectrum (real and imaginary parts N(0, 1/2), seed 2024) on the
    box [-20, 60)^3.  The rectilinear path on the regular grid and the NUFFT
    at every grid point must match the inverse FFT to 1e-11 absolute.  1000
    random points must match the exact sum to 1e-11."""
    box = vfb.DomainBox((-20.0,) * 3, (60.0,) * 3)
    rng = np.random.default_rng(2024)
    shape = (64, 64, 64)
    coeffs = (rng.standard_normal(shape) + 1j * rng.standard_normal(shape)) / np.sqrt(2.0)
    spec = vfb.SpectralField(box, coeffs)
    axes = vfb.regular_grid(box, shape)
    scale = float(np.prod(np.sqrt(box.widths) / np.array(shape)))
    ref = np.fft.ifftn(np.fft.ifftshift(coeffs)) / scale
    rect = vfb.eval_rectilinear(spec, axes)
    assert np.abs(rect - ref).max() <= 1e-11
    grid_pts = np.stack(np.meshgrid(*axes, indexing="ij"), axis=-1).reshape(-1, 3)
    plan = vfb.NufftPlan(spec)
    at_grid = plan.evaluate(grid_pts).reshape(shape)
    assert np.abs(at_grid - ref).max() <= 1e-11
    pts = rng.uniform(-20.0, 60.0, (1000, 3))
    direct = O.ndft(coeffs, box.a, box.b, pts)
    assert np.abs(plan.evaluate(pts) - direct).max() <= 1e-11
    assert np.abs(vfb.eval_direct(spec, pts) - direct).max() <= 1e-11


# ---------------------------------------------------------------- full-size properties


def test_config5_full_size(vfb):
    """BASELINE config 5 at full size on one GPU: N = 256^3 (decay 4096),
    2^28 uniform points generated on the device.  A 6000-point subset is
    checked against the oracle's gather on the same grid, and 2^20 of the
    points re-evaluated alone on the binned gather with the full call's box
    width are bitwise the full call's values."""
    import torch

    from paper_1605_01244_b200 import workloads

    w = workloads.WORKLOADS["c5"]
    coeffs = workloads.coefficients("c5")
    a, b = w.box
    plan = vfb.NufftPlan(vfb.SpectralField(vfb.DomainBox(a, b), torch.as_tensor(coeffs, device="cuda")))
    gen = torch.Generator(device="cuda")
    gen.manual_seed(2005)
    pts = torch.rand((w.npoints, 3), dtype=torch.float64, device="cuda", generator=gen) - 0.5
    out = plan.evaluate(pts)
    sub = torch.as_tensor(np.random.default_rng(5).choice(w.npoints, 6000, replace=False), device="cuda")
    psub = pts[sub].cpu().numpy()
    ref = O.nufft_eval(coeffs, a, b, psub)
    l2, linf = rel_err(out[sub].cpu().numpy(), ref)
    assert l2 < 1e-13 and linf < 1e-13, (l2, linf)
    box = plan.geometry(w.npoints)[0][0]
    part = pts[: 1 << 20]
    plan.set_gather(2)
    plan.set_box(box)
    assert torch.equal(plan.evaluate(part), out[: 1 << 20])
    del pts, out, part
    torch.cuda.empty_cache()


def test_config2_full_size(vfb):
    """BASELINE config 2 (64^3 modes, 1e6 points): a 20k-point subset against
    the oracle, the whole batch for determinism and batch invariance."""
    from paper_1605_01244_b200 import workloads

    coeffs = workloads.coefficients("c2")
    pts = workloads.points("c2")
    a, b = workloads.UNIT_BOX
    spec = vfb.SpectralField(vfb.DomainBox(a, b), coeffs)
    plan = vfb.NufftPlan(spec)
    out = plan.evaluate(pts)
    sub = np.random.default_rng(0).choice(len(pts), 20000, replace=False)
    ref = O.nufft_eval(coeffs, a, b, pts[sub])
    l2, linf = rel_err(out[sub], ref)
    assert l2 < TOL and linf < TOL
    assert l2 < 1e-13 and linf < 1e-13, (l2, linf)
    # 20000 points take the warp-per-point gather: rounding-level agreement;
    # on the binned gather with the full call's box width: bitwise
    l2, linf = rel_err(plan.evaluate(pts[sub]), out[sub])
    assert l2 < 1e-14 and linf < 1e-14, (l2, linf)
    plan.set_gather(2)
    plan.set_box(plan.geometry(len(pts))[0][0])
    np.testing.assert_array_equal(out[sub], plan.evaluate(pts[sub]))


def test_config3_clustered_full_size(vfb):
    """BASELINE config 3 (vortex-pair spectrum on [-8,8)^3, 1e7 points in a
    0.05-std cloud straddling the periodic seam): 20k-point subset vs oracle,
    and the automatic box choice must not change any value's bits compared
    with a fixed box on the same call geometry."""
    from paper_1605_01244_b200 import workloads

    coeffs = workloads.coefficients("c3")
    pts = workloads.points("c3")
    a, b = workloads.VORTEX_BOX
    plan = vfb.NufftPlan(vfb.SpectralField(vfb.DomainBox(a, b), coeffs))
    out = plan.evaluate(pts)
    sub = np.random.default_rng(1).choice(len(pts), 20000, replace=False)
    ref = O.nufft_eval(coeffs, a, b, pts[sub])
    l2, linf = rel_err(out[sub], ref)
    assert l2 < 1e-13 and linf < 1e-13, (l2, linf)
    box, _ = plan.geometry(len(pts))
    plan.set_box(box[0])
    np.testing.assert_array_equal(plan.evaluate(pts), out)


def test_config4_rectilinear_full_size(vfb):
    """BASELINE config 4: 128^3 coefficients on the 256^3 tanh-clustered grid,
    every value against the oracle (reference algorithm)."""
    from paper_1605_01244_b200 import workloads

    coeffs = workloads.coefficients("c4")
    axes = workloads.rect_axes(256)
    a, b = workloads.UNIT_BOX
    out = vfb.eval_rectilinear(vfb.SpectralField(vfb.DomainBox(a, b), coeffs), axes)
    ref = O.rectilinear(coeffs, a, b, axes)
    l2, linf = rel_err(out, ref)
    assert l2 < 1e-13 and linf < 1e-13, (l2, linf)


def test_box_widths_agree(vfb, offset_box):
    """Both gather box widths give the reference's values (to rounding)."""
    spec = random_spectral(offset_box, (16, 16, 16), 95)
    pts = np.random.default_rng(96).uniform(offset_box.a, offset_box.b, (40000, 3))
    plan = vfb.NufftPlan(spec)
    ref = O.nufft_eval(spec.coeffs, offset_box.a, offset_box.b, pts)
    for bxy in (1, 2):
        plan.set_box(bxy)
        out = plan.evaluate(pts)
        assert plan.geometry(len(pts))[0][0] == bxy
        l2, linf = rel_err(out, ref)
        assert l2 < 1e-13 and linf < 1e-13, (bxy, l2, linf)


# ---------------------------------------------------------------- SURVEY 8f next rows


def _tube_snap(vfb):
    g = golden("tube_case.npz")
    dom = vfb.DomainBox(tuple(g["a"]), tuple(g["b"]))
    return g, vfb.Snapshot(dom, g["values"], tuple(bool(x) for x in g["mirror"]), 0.0)


def test_snapshot_spectral_matches_reference(vfb):
    g, snap = _tube_snap(vfb)
    spec = vfb.snapshot_spectral(snap)
    assert spec.domain.b == (30.0, 30.0, 30.0)
    l2, linf = rel_err(spec.coeffs, g["spectral"])
    assert l2 < 1e-14 and linf < 1e-13, (l2, linf)


@pytest.mark.parametrize("tag,thr,ff", [("two", [0.4, 0.3], None), ("one", [0.4], None),
                                        ("filt", [0.4, 0.3], 0.15)])
def test_tube_eval_matches_reference(vfb, tag, thr, ff):
    """Same point set, levels and lattice order as the reference (bit-exact),
    densities to rounding (reference test_tube.py:85-115)."""
    g, snap = _tube_snap(vfb)
    cloud = vfb.tube_eval(snap, thr, final_filter=ff)
    np.testing.assert_array_equal(cloud.points, g[f"{tag}_points"])
    np.testing.assert_array_equal(cloud.level, g[f"{tag}_level"])
    np.testing.assert_allclose(cloud.density, g[f"{tag}_density"], rtol=0, atol=1e-13)
    if tag == "two":
        assert np.unique(cloud.level, return_counts=True)[1].tolist() == [16, 992, 26208]


def test_tube_empty_outcomes(vfb):
    import warnings as w

    dom = vfb.DomainBox((0.0, 0.0, 0.0), (1.0, 1.0, 1.0))
    snap = vfb.Snapshot(dom, np.ones((8, 8, 8)), (False, False, False), 0.0)
    with pytest.warns(RuntimeWarning, match="empty cloud"):
        cloud = vfb.tube_eval(snap, [0.5])
    assert len(cloud) == 0 and cloud.points.shape == (0, 3)
    with w.catch_warnings():
        w.simplefilter("error")
        assert len(vfb.tube_eval(snap, [1.5, 0.5])) == 0


def test_pipelined_host_path(vfb, unit_box):
    """Host buffers with M >= 2^23 take the chunked H2D/evaluate/D2H pipeline:
    same bits as the device-resident path for a fixed box width, and the first
    bad row is reported with its global index."""
    import torch

    spec = random_spectral(unit_box, (32, 32, 32), 97)
    rng = np.random.default_rng(98)
    M = (1 << 23) + 12345
    pts = rng.uniform(0.0, 1.0, (M, 3))
    plan = vfb.NufftPlan(spec)
    plan.set_box(2)
    host = plan.evaluate(pts)
    dev = plan.evaluate(torch.as_tensor(pts, device="cuda")).cpu().numpy()
    np.testing.assert_array_equal(host, dev)
    sub = rng.choice(M, 3000, replace=False)
    ref = O.nufft_eval(spec.coeffs, unit_box.a, unit_box.b, pts[sub])
    l2, linf = rel_err(host[sub], ref)
    assert l2 < 1e-13 and linf < 1e-13
    bad = pts.copy()
    bad[M - 7] = (0.5, 1.5, 0.5)  # in the second chunk
    bad[M - 3] = (np.nan, 0.5, 0.5)
    with pytest.raises(ValueError, match=rf"\(row {M - 7}\)"):
        plan.evaluate(bad)


@pytest.mark.parametrize("shape,sigma", [((18, 22, 26), 2.0), ((20, 30, 10), 1.6)])
def test_ragged_grids_many_points(vfb, offset_box, shape, sigma):
    """Oversampled sizes that are not multiples of the 4x4x8 tile (36x44x52,
    32x48x16 at sigma 1.6) with enough points for many work items per CTA,
    at both box widths, against the oracle."""
    spec = random_spectral(offset_box, shape, 99)
    rng = np.random.default_rng(100)
    pts = rng.uniform(offset_box.a, offset_box.b, (300000, 3))
    plan = vfb.NufftPlan(spec, vfb.NufftParams(oversampling=sigma))
    sub = rng.choice(len(pts), 4000, replace=False)
    grid, n, beta = O.oversampled_grid(spec.coeffs, offset_box.a, offset_box.b, sigma, 6)
    ref = O.gather_eval(grid, n, 6, beta, pts[sub], offset_box.a, offset_box.b)
    for bxy in (1, 2):
        plan.set_box(bxy)
        out = plan.evaluate(pts)
        l2, linf = rel_err(out[sub], ref)
        assert l2 < 1e-13 and linf < 1e-13, (bxy, l2, linf)


@pytest.mark.parametrize("m", [2, 3, 4, 5, 7, 8])
def test_tensor_core_gather_other_cutoffs(vfb, offset_box, m):
    """The tensor-core gather at m = 2, 3, 4, 5, 7, 8 (tiles 4x4x(20-2m), 4x2x6 at m = 7,
    2x2x4 at m = 8): uniform
    points plus a dense cluster (boxes with many units, every k-chunk count),
    at both box widths, against the oracle's gather on the same grid and
    against the thread-per-point gather."""
    shape = (18, 22, 26)
    spec = random_spectral(offset_box, shape, 110 + m)
    rng = np.random.default_rng(120 + m)
    a, b = np.array(offset_box.a), np.array(offset_box.b)
    uni = rng.uniform(a, b, (150000, 3))
    clu = np.clip(rng.normal((a + b) / 2, 0.01 * (b - a), (50000, 3)), a, np.nextafter(b, a))
    pts = np.vstack([uni, clu])
    plan = vfb.NufftPlan(spec, vfb.NufftParams(cutoff=m, eps=0.999))
    box, tile = plan.geometry(len(pts))
    assert tile == ((2, 2, 4) if m == 8 else (4, 2 if m == 7 else 4, 20 - 2 * m))
    sub = np.concatenate([rng.choice(150000, 2500, replace=False), 150000 + rng.choice(50000, 1500, replace=False)])
    grid, n, beta = O.oversampled_grid(spec.coeffs, offset_box.a, offset_box.b, 2.0, m)
    ref = O.gather_eval(grid, n, m, beta, pts[sub], offset_box.a, offset_box.b)
    outs = []
    for bxy in (1, 2):
        plan.set_box(bxy)
        out = plan.evaluate(pts)
        l2, linf = rel_err(out[sub], ref)
        assert l2 < 1e-13 and linf < 1e-13, (m, bxy, l2, linf)
        outs.append(out)
    plan.set_box(0)
    plan.set_gather(1)  # thread per point
    simple = plan.evaluate(pts)
    for out in outs:
        l2, linf = rel_err(out, simple)
        assert l2 < 1e-13 and linf < 1e-13


def test_shared_plan_from_several_threads(vfb, offset_box):
    """The reference allows one plan to be evaluated from several threads on
    disjoint point subsets (ctypes releases the GIL): host
    and CUDA-tensor inputs from 6 threads give the serial values bitwise."""
    import threading

    import torch

    spec = random_spectral(offset_box, (16, 20, 24), 400)
    rng = np.random.default_rng(401)
    pts = rng.uniform(offset_box.a, offset_box.b, (600000, 3))
    plan = vfb.NufftPlan(spec)
    parts = np.array_split(np.arange(len(pts)), 12)
    serial = [plan.evaluate(pts[ix]) for ix in parts]
    got = [None] * len(parts)
    errors = []

    def work(k):
        try:
            for j in range(k, len(parts), 6):
                if j % 2:
                    with torch.cuda.stream(torch.cuda.Stream()):
                        got[j] = plan.evaluate(torch.as_tensor(pts[parts[j]], device="cuda")).cpu().numpy()
                else:
                    got[j] = plan.evaluate(pts[parts[j]])
        except Exception as e:  # pragma: no cover - reported below
            errors.append(e)

    threads = [threading.Thread(target=work, args=(k,)) for k in range(6)]
    for th in threads:
        th.start()
    for th in threads:
        th.join()
    assert not errors, errors
    for a, b in zip(got, serial):
        assert np.array_equal(a, b)


@pytest.mark.parametrize("m", [1, 2, 4, 6, 9, 13])
def test_warp_gather_small_evaluates(vfb, offset_box, m):
    """The unbinned warp-per-point gather (automatic up to WARP_MAX_M points):
    vs the oracle at every cutoff family (W = 3 .. 27 lanes per row), M = 1,
    the threshold itself, outside / NaN rows reported with the reference's
    text, device and host inputs bitwise equal."""
    import torch

    spec = random_spectral(offset_box, (10, 14, 12), 500 + m)
    rng = np.random.default_rng(510 + m)
    a, b = np.array(offset_box.a), np.array(offset_box.b)
    plan = vfb.NufftPlan(spec, vfb.NufftParams(cutoff=m, eps=0.999))
    grid, n, beta = O.oversampled_grid(spec.coeffs, offset_box.a, offset_box.b, 2.0, m)
    for M in (1, 777, vfb.nufft.WARP_MAX_M):
        pts = rng.uniform(a, b, (M, 3))
        out = plan.evaluate(pts)
        assert plan.launch_count(M) == 2
        sub = np.arange(M) if M < 2000 else rng.choice(M, 2000, replace=False)
        ref = O.gather_eval(grid, n, m, beta, pts[sub], offset_box.a, offset_box.b)
        l2, linf = rel_err(out[sub], ref)
        # relative to max|ref| of the sample (one value at M = 1); the widest
        # windows deconvolve by the largest 1/phihat, so their grids carry
        # a few ulps more FFT rounding
        tol = (1e-13 if m <= 11 else 3e-13) if m >= 3 else 1e-11
        assert l2 < tol and linf < tol, (m, M, l2, linf)
        dev = plan.evaluate(torch.as_tensor(pts, device="cuda"))
        np.testing.assert_array_equal(dev.cpu().numpy(), out)
    pts = rng.uniform(a, b, (500, 3))
    pts[[123, 400], 1] = [b[1] + 0.5, np.nan]
    with pytest.raises(ValueError, match=r"\(row 123\) lies outside"):
        plan.evaluate(pts)
    pts[123, 1] = a[1]
    with pytest.raises(ValueError, match=r"\(row 400\) lies outside"):
        plan.evaluate(pts)
    pts[400, 1] = a[1]
    plan.evaluate(pts)  # the bad-row word was reset: a clean call passes


def test_rectilinear_and_direct_from_several_threads(vfb, offset_box):
    """Rectilinear and direct evaluations (both cuBLAS) running concurrently
    from different threads on one device give the serial values bitwise."""
    import threading

    rng = np.random.default_rng(900)
    spec = random_spectral(offset_box, (16, 12, 10), 901)
    a, b = np.array(offset_box.a), np.array(offset_box.b)
    axes = [np.sort(rng.uniform(a[d], b[d], n)) for d, n in enumerate((64, 48, 40))]
    pts = rng.uniform(a, b, (3000, 3))
    rect_ref = vfb.eval_rectilinear(spec, axes)
    direct_ref = vfb.eval_direct(spec, pts)
    errors = []

    def work(k):
        try:
            for _ in range(6):
                if k % 2:
                    assert np.array_equal(vfb.eval_rectilinear(spec, axes), rect_ref)
                else:
                    assert np.array_equal(vfb.eval_direct(spec, pts), direct_ref)
        except Exception as e:  # pragma: no cover - reported below
            errors.append(e)

    threads = [threading.Thread(target=work, args=(k,)) for k in range(4)]
    for th in threads:
        th.start()
    for th in threads:
        th.join()
    assert not errors, errors


def test_plans_release_device_memory(vfb, offset_box):
    """Creating, using and dropping plans repeatedly returns the device memory
    (grid, evaluate scratch, graphs); only process-wide caches (cuFFT plans,
    the window fit) may stay."""
    import gc

    import torch

    rng = np.random.default_rng(950)
    pts = rng.uniform(offset_box.a, offset_box.b, (200000, 3))
    spec = random_spectral(offset_box, (24, 20, 16), 951)

    def cycle():
        plan = vfb.NufftPlan(spec)
        plan.evaluate(pts)
        plan.evaluate(pts[:5000])
        plan.evaluate(torch.as_tensor(pts, device="cuda"))
        del plan
        gc.collect()

    cycle()  # warm the process-wide caches
    torch.cuda.synchronize()
    free0 = torch.cuda.mem_get_info()[0]
    for _ in range(12):
        cycle()
    torch.cuda.synchronize()
    free1 = torch.cuda.mem_get_info()[0]
    assert free0 - free1 < 64 << 20, (free0 - free1) / 2**20


@pytest.mark.parametrize("m", [6, 7, 8])
def test_pipelined_host_path_per_cutoff(vfb, offset_box, m):
    """The pipelined host path at m = 6 (four chunks) and m = 7, 8 (one
    chunk): pinned output, pinned and pageable inputs, bitwise the
    device-resident values."""
    import torch

    spec = random_spectral(offset_box, (16, 16, 16), 990 + m)
    rng = np.random.default_rng(991 + m)
    a, b = np.array(offset_box.a), np.array(offset_box.b)
    M = (1 << 23) + 77
    pts = rng.uniform(a, b, (M, 3))
    plan = vfb.NufftPlan(spec, vfb.NufftParams(2.0, m))
    ref = plan.evaluate(torch.as_tensor(pts, device="cuda")).cpu().numpy()
    pin_p = torch.empty((M, 3), dtype=torch.float64, pin_memory=True)
    pin_p.copy_(torch.as_tensor(pts))
    out = torch.empty(M, dtype=torch.complex128, pin_memory=True).numpy()
    for src in (pts, pin_p.numpy()):
        out[:] = np.nan
        plan.evaluate(src, out=out)
        assert np.array_equal(out, ref), src is pts
    sub = rng.choice(M, 2000, replace=False)
    l2, linf = rel_err(ref[sub], O.nufft_eval(spec.coeffs, offset_box.a, offset_box.b, pts[sub], m=m))
    assert l2 < 1e-12 and linf < 1e-12


@pytest.mark.parametrize("M", [300000, (1 << 23) + 5])
def test_pageable_and_pinned_host_buffers(vfb, offset_box, M):
    """Every mix of pageable (plain numpy, staged through pinned pieces) and
    pinned host buffers, on the simple and the pipelined host path, gives the
    device-resident values bitwise; an outside row is still reported."""
    import torch

    spec = random_spectral(offset_box, (16, 16, 16), 980)
    rng = np.random.default_rng(981)
    a, b = np.array(offset_box.a), np.array(offset_box.b)
    pts = rng.uniform(a, b, (M, 3))
    plan = vfb.NufftPlan(spec)
    plan.set_box(2)
    ref = plan.evaluate(torch.as_tensor(pts, device="cuda")).cpu().numpy()
    pin_p = torch.empty((M, 3), dtype=torch.float64, pin_memory=True)
    pin_p.copy_(torch.as_tensor(pts))
    for src in (pts, pin_p.numpy()):
        for pinned_out in (False, True):
            out = (torch.empty(M, dtype=torch.complex128, pin_memory=True).numpy() if pinned_out
                   else np.empty(M, dtype=np.complex128))
            plan.evaluate(src, out=out)
            assert np.array_equal(out, ref), (src is pts, pinned_out)
    bad = pts.copy()
    bad[M - 3] = np.nan
    with pytest.raises(ValueError, match=rf"\(row {M - 3}\)"):
        plan.evaluate(bad)


def test_cuda_graph_replay_matches_eager(vfb, offset_box):
    """Repeated small evaluates replay one CUDA graph (second call captures):
    values bitwise equal to the eager launches, new point values in the same
    buffers are picked up, out-of-domain rows still raise, M changes recapture."""
    import torch

    spec = random_spectral(offset_box, (16, 16, 16), 130)
    rng = np.random.default_rng(131)
    a, b = np.array(offset_box.a), np.array(offset_box.b)
    batches = [rng.uniform(a, b, (5000, 3)) for _ in range(3)]
    graphed = vfb.NufftPlan(spec)
    eager = vfb.NufftPlan(spec)
    eager.set_graphs(False)
    for plan in (graphed, eager):
        plan.set_gather(2)  # the binned path (graphs); small M would take the warp path
    for i in range(7):
        p = batches[i % 3]
        np.testing.assert_array_equal(graphed.evaluate(p), eager.evaluate(p))
    bad = batches[0].copy()
    bad[4321] = b + 1.0
    with pytest.raises(ValueError, match=r"\(row 4321\)"):
        graphed.evaluate(bad)
    np.testing.assert_array_equal(graphed.evaluate(batches[1]), eager.evaluate(batches[1]))
    # device-resident points and output, as bench.py drives it
    dpts = torch.as_tensor(batches[2], device="cuda")
    out = torch.empty(5000, dtype=torch.complex128, device="cuda")
    ref = eager.evaluate(batches[2])
    for _ in range(4):
        graphed.evaluate(dpts, out=out)
        np.testing.assert_array_equal(out.cpu().numpy(), ref)
    dpts.copy_(torch.as_tensor(batches[0], device="cuda"))
    graphed.evaluate(dpts, out=out)
    np.testing.assert_array_equal(out.cpu().numpy(), eager.evaluate(batches[0]))
    for M in (17, 3000, 17):
        np.testing.assert_array_equal(graphed.evaluate(batches[0][:M]), eager.evaluate(batches[0][:M]))
    # a larger call in between grows (reallocates) the plan's scratch: the
    # graph captured before must not be replayed on the freed buffers
    big = rng.uniform(a, b, (200000, 3))
    for p in (batches[1], batches[1], big, batches[1], batches[1]):
        np.testing.assert_array_equal(graphed.evaluate(p), eager.evaluate(p))


def test_batched_evaluate_beyond_batch_limit(vfb, offset_box, monkeypatch):
    """Calls larger than one sort batch (2^30 points; lowered here through
    VFN_MAX_BATCH) run as consecutive batches with one geometry: bitwise the
    single-batch values, outside rows reported with their global index, for
    device, host and pipelined-host inputs."""
    import torch

    spec = random_spectral(offset_box, (16, 16, 16), 140)
    rng = np.random.default_rng(141)
    a, b = np.array(offset_box.a), np.array(offset_box.b)
    pts = rng.uniform(a, b, (100000, 3))
    plan = vfb.NufftPlan(spec)
    plan.set_box(2)
    ref = plan.evaluate(pts)
    monkeypatch.setenv("VFN_MAX_BATCH", "30000")
    np.testing.assert_array_equal(plan.evaluate(pts), ref)
    dev = plan.evaluate(torch.as_tensor(pts, device="cuda"))
    np.testing.assert_array_equal(dev.cpu().numpy(), ref)
    bad = pts.copy()
    bad[71234] = np.nan
    with pytest.raises(ValueError, match=r"\(row 71234\)"):
        plan.evaluate(bad)
    big = rng.uniform(a, b, (1 << 23, 3))
    monkeypatch.delenv("VFN_MAX_BATCH")
    ref_big = plan.evaluate(big)
    monkeypatch.setenv("VFN_MAX_BATCH", str(1 << 21))
    np.testing.assert_array_equal(plan.evaluate(big), ref_big)


@pytest.mark.parametrize("shape", [(2, 2, 64), (64, 2, 2), (2, 4, 2), (2, 2, 2), (4, 30, 2)])
@pytest.mark.parametrize("m", [2, 6, 7])
def test_tiny_and_anisotropic_grids(vfb, offset_box, shape, m):
    """Mode counts of 2 along some axes (oversampled grids of 4 cells, far
    smaller than one tile plus its halo) on every gather variant, vs the oracle."""
    spec = random_spectral(offset_box, shape, 150 + m)
    rng = np.random.default_rng(151 + m)
    pts = rng.uniform(offset_box.a, offset_box.b, (3000, 3))
    plan = vfb.NufftPlan(spec, vfb.NufftParams(cutoff=m, eps=0.999))
    grid, n, beta = O.oversampled_grid(spec.coeffs, offset_box.a, offset_box.b, 2.0, m)
    ref = O.gather_eval(grid, n, m, beta, pts, offset_box.a, offset_box.b)
    for variant in (0, 1, 3):
        plan.set_gather(variant)
        l2, linf = rel_err(plan.evaluate(pts), ref)
        assert l2 < 1e-12 and linf < 1e-12, (shape, m, variant, l2, linf)


def test_c_abi_from_plain_c(tmp_path):
    """The boundary works without Python: examples/c_api_demo.c links
    libvfnfft.so directly, evaluates against vfn_direct_eval and checks the
    outside-point status (exit code 0 on success)."""
    import subprocess

    from conftest import REPO

    exe = tmp_path / "c_api_demo"
    lib = f"{REPO}/paper_1605_01244_b200"
    cc = subprocess.run(["gcc", "-O2", "-I", f"{REPO}/include", f"{REPO}/examples/c_api_demo.c",
                         "-L", lib, "-lvfnfft", f"-Wl,-rpath,{lib}", "-lm", "-o", str(exe)],
                        capture_output=True, text=True)
    assert cc.returncode == 0, cc.stderr
    run = subprocess.run([str(exe)], capture_output=True, text=True, timeout=120)
    assert run.returncode == 0, run.stdout + run.stderr
    assert "first bad row 17" in run.stdout


@pytest.mark.timeout(600)
def test_bench_under_torchrun_two_ranks(vfb):
    """bench.py's N > 1 path (torchrun, one JSON line from rank 0, max over
    ranks, strong scaling by key-range sharding: sample-sort splitters,
    all-to-all of points and values) with two ranks sharing this GPU over
    gloo (VFN_DIST_BACKEND=gloo; NCCL refuses two ranks on one device); the
    sharded values equal one unsharded evaluate bitwise."""
    import json
    import os
    import subprocess
    import sys

    from conftest import REPO

    env = dict(os.environ, VFN_DIST_BACKEND="gloo")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2",
           "--master-addr", "127.0.0.1", "--master-port", "29573", os.path.join(REPO, "bench.py"),
           "--gpus", "2", "--workload", "c2", "--steps", "3", "--warmup", "3"]
    res = subprocess.run(cmd, capture_output=True, text=True, timeout=540, cwd=REPO, env=env)
    assert res.returncode == 0, res.stderr[-2000:]
    lines = [ln for ln in res.stdout.splitlines() if ln.strip().startswith("{")]
    assert len(lines) == 1, res.stdout
    out = json.loads(lines[0])
    assert out["n_gpus"] == 2 and out["scaling"] == "strong" and out["config"]["points"] == 10 ** 6
    assert out["value"] > 0 and out["e2e"]["matches_device_result_bitwise"] is True
    sh = out["sharding"]
    assert sh["sharded_equals_unsharded_bitwise"] is True and sh["mode"] == "keyrange"
    assert 0.45e6 < sh["received_min"] <= sh["received_max"] < 0.55e6


@pytest.mark.parametrize("variant", [0, 1, 2, 3])
def test_first_bad_row_on_every_path(vfb, unit_box, variant):
    """Non-finite and out-of-domain rows deep inside a large call: every gather
    variant reports the FIRST bad row (reference nufft.py domain check), from
    host and device inputs, and the plan keeps working afterwards.  The
    CUDA-graph replay (variant 2 below 2^20 points) must report a row that was
    written into the captured input buffer in place."""
    import torch

    spec = random_spectral(unit_box, (16, 16, 16), 131)
    rng = np.random.default_rng(132)
    M = 100000
    pts = rng.uniform(0.0, 1.0, (M, 3))
    plan = vfb.NufftPlan(spec)
    plan.set_gather(variant)
    good = plan.evaluate(pts)
    bad = pts.copy()
    bad[77777] = (0.5, np.inf, 0.5)
    bad[88888] = (np.nan, 0.5, 0.5)
    bad[99999] = (-1e-300, 0.5, 0.5)
    for arr in (bad, torch.as_tensor(bad, device="cuda")):
        with pytest.raises(ValueError, match=r"\(row 77777\)"):
            plan.evaluate(arr)
    only_last = pts.copy()
    only_last[M - 1] = (0.5, 0.5, 1.0)
    with pytest.raises(ValueError, match=rf"\(row {M - 1}\)"):
        plan.evaluate(only_last)
    np.testing.assert_array_equal(plan.evaluate(pts), good)
    # same device buffer twice (graph capture + replay), then poisoned in place
    t = torch.as_tensor(pts, device="cuda")
    for _ in range(3):
        np.testing.assert_array_equal(plan.evaluate(t).cpu().numpy(), good)
    t[4242, 2] = float("nan")
    with pytest.raises(ValueError, match=r"\(row 4242\)"):
        plan.evaluate(t)
    t[4242, 2] = 0.25
    out = plan.evaluate(t).cpu().numpy()
    np.testing.assert_array_equal(np.delete(out, 4242), np.delete(good, 4242))


def test_evaluate_runs_on_the_callers_current_stream(vfb, unit_box):
    """Calls enqueue on torch's current stream (the stream handle passed through
    the C-ABI), so a caller's side stream orders them with its own work."""
    import torch

    from paper_1605_01244_b200 import nufft

    spec = random_spectral(unit_box, (16, 16, 16), 141)
    rng = np.random.default_rng(142)
    plan = vfb.NufftPlan(spec)
    for M in (3000, 60000):  # warp path and binned path
        pts = torch.as_tensor(rng.uniform(0.0, 1.0, (M, 3)), device="cuda")
        ref = plan.evaluate(pts).cpu().numpy()
        side = torch.cuda.Stream()
        with torch.cuda.stream(side):
            assert nufft._stream_of(plan.device).value == side.cuda_stream
            shifted = pts * 1.0  # produced on the side stream, consumed by the evaluate
            out = plan.evaluate(shifted)
            host = out.cpu().numpy()
        # the legacy default stream is handle 0 (c_void_p(0).value is None)
        assert (nufft._stream_of(plan.device).value or 0) == torch.cuda.current_stream().cuda_stream
        np.testing.assert_array_equal(host, ref)


def test_host_pipelined_call_takes_the_whole_calls_geometry(vfb):
    """A host-buffer call of >= 2^23 points runs in chunks; its bin geometry
    (box width) is chosen from the whole call's density sample, as the
    device-resident call chooses it, not from the first chunk — so the two
    give bitwise the same values even when the chunks' densities differ
    (first half uniform: box width 2 on its own; second half a tight cloud:
    the whole set takes width 1)."""
    import torch

    box = vfb.DomainBox((-0.5, -0.5, -0.5), (0.5, 0.5, 0.5))
    spec = random_spectral(box, (128, 128, 128), 1400)
    plan = vfb.NufftPlan(spec)
    rng = np.random.default_rng(1401)
    M = (1 << 23) + 5
    pts = rng.uniform(-0.5, 0.5, (M, 3))
    pts[M // 2:] = np.clip(rng.normal(0.1, 0.002, (M - M // 2, 3)), -0.5, 0.4999)
    dev = plan.evaluate(torch.as_tensor(pts, device="cuda")).cpu().numpy()
    assert plan.geometry(M)[0][0] == 1  # the whole set is dense enough for 1 x 1 boxes
    host = plan.evaluate(pts)
    np.testing.assert_array_equal(host, dev)


def test_hand_written_radix_sort_matches_stable_argsort(tmp_path):
    """The hand-written LSD radix sort (VFN_SORT=radix, csrc/vfn_sort.cu)
    gives the stable permutation of the bin keys and the same evaluate bits
    as the default sort (run in a subprocess: the choice is made once per
    process)."""
    import subprocess
    import sys

    from conftest import REPO

    code = r'''
import numpy as np, sys
sys.path.insert(0, %r)
import paper_1605_01244_b200 as vfb
from oracle import nfft_oracle as O
rng = np.random.default_rng(1600)
box = vfb.DomainBox((-1.5, 0.25, 2.0), (2.5, 1.25, 7.0))
coeffs = rng.standard_normal((32, 24, 16)) + 1j * rng.standard_normal((32, 24, 16))
plan = vfb.NufftPlan(vfb.SpectralField(box, coeffs))
for M in (70000, 1 << 20, (1 << 21) + 37):
    pts = rng.uniform(box.a, box.b, (M, 3))
    pts[: M // 3] = pts[0]
    keys, perm = plan.bin(pts)
    b, t = plan.geometry(M)
    ref = O.bin_keys(pts, box.a, box.b, plan._n, b, t, plan.key_shift())
    assert np.array_equal(keys.astype(np.int64), ref)
    assert np.array_equal(perm, np.argsort(ref, kind="stable"))
    np.save(%r + "/vals_%%d.npy" %% M, plan.evaluate(pts))
print("ok")
''' % (REPO, str(tmp_path))
    import os

    for env in ({"VFN_SORT": "radix"}, {}):
        res = subprocess.run([sys.executable, "-c", code], capture_output=True, text=True, timeout=600,
                             env=dict(os.environ, **env), cwd=REPO)
        assert res.returncode == 0 and "ok" in res.stdout, res.stderr[-2000:]
        if env:
            radix = {M: np.load(tmp_path / f"vals_{M}.npy") for M in (70000, 1 << 20, (1 << 21) + 37)}
    for M, v in radix.items():
        np.testing.assert_array_equal(v, np.load(tmp_path / f"vals_{M}.npy"))


def test_large_grid_bin_keys_and_units(vfb):
    """A 512^3 oversampled grid at m = 8 (1 x 1 x 4 boxes in 2 x 2 x 4 tiles:
    2^25 boxes, bin keys up to 2^26): the unit builder's multiply-shift division must stay
    exact past 2^25 (its 72-bit product), so the tensor-core gather matches
    the thread-per-point gather on the same grid."""
    import torch

    rng = np.random.default_rng(1900)
    N = 256
    coeffs = torch.complex(torch.randn((N, N, N), dtype=torch.float64, device="cuda"),
                           torch.randn((N, N, N), dtype=torch.float64, device="cuda"))
    box = vfb.DomainBox((-0.5, -0.5, -0.5), (0.5, 0.5, 0.5))
    plan = vfb.NufftPlan(vfb.SpectralField(box, coeffs), vfb.NufftParams(cutoff=8, eps=1e-16))
    pts = torch.as_tensor(rng.uniform(-0.5, 0.5, (1 << 20, 3)), device="cuda")
    plan.set_box(1)
    fast = plan.evaluate(pts)
    box_, tile = plan.geometry(1 << 20)
    assert tile == (2, 2, 4) and box_[0] == 1
    sub = pts[: 1 << 15]
    plan.set_gather(1)
    ref = plan.evaluate(sub)
    l2, linf = rel_err(fast[: 1 << 15].cpu().numpy(), ref.cpu().numpy())
    assert l2 < 1e-13 and linf < 1e-13, (l2, linf)
