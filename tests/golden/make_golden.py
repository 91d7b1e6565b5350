"""Generate the golden vectors under tests/golden/ from the REAL reference.

Run in the development container (where /root/reference exists):

    PYTHONDONTWRITEBYTECODE=1 python tests/golden/make_golden.py

It imports the unmodified reference package `vortexfourier` from
/root/reference/pkg/src and records its outputs on seeded inputs.  The
fixtures are small (~2 MB total) and are committed; the GPU box never reads
/root/reference.  Inputs are stored alongside outputs so the tests do not
depend on numpy RNG stability.
"""

from __future__ import annotations

import os
import sys
import warnings

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
REPO = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, "/root/reference/pkg/src")
sys.path.insert(0, REPO)

import vortexfourier as vf  # noqa: E402
from vortexfourier.nufft import _kb_beta, _kb_transform, _kb_values  # noqa: E402

from paper_1605_01244_b200 import workloads  # noqa: E402

OFFSET_BOX = vf.DomainBox((-1.5, 0.25, 2.0), (2.5, 1.25, 7.0))
UNIT_BOX = vf.DomainBox((0.0, 0.0, 0.0), (1.0, 1.0, 1.0))


def spectral(box, shape, seed):
    # the reference fixture convention (tests/conftest.py:24-27)
    rng = np.random.default_rng(seed)
    return vf.SpectralField(box, rng.standard_normal(shape) + 1j * rng.standard_normal(shape))


def box_arrays(box):
    return np.array(box.a), np.array(box.b)


def save(name, **arrays):
    path = os.path.join(HERE, name)
    np.savez_compressed(path, **arrays)
    print(f"wrote {name}: {os.path.getsize(path)} bytes")


def nufft_cases():
    """NUFFT vs the reference at several shapes/seeds/cutoffs/oversamplings."""
    cases = [
        # (box, shape, seed, sigma, m, npts)
        (OFFSET_BOX, (16, 16, 16), 60, 2.0, 6, 300),
        (OFFSET_BOX, (8, 24, 12), 61, 2.0, 6, 300),
        (OFFSET_BOX, (16, 16, 16), 70, 2.0, 2, 100),
        (OFFSET_BOX, (16, 16, 16), 71, 2.0, 3, 100),
        (OFFSET_BOX, (16, 16, 16), 72, 2.0, 8, 100),
        (OFFSET_BOX, (10, 20, 10), 73, 1.6, 6, 200),
        (UNIT_BOX, (12, 12, 12), 81, 2.0, 13, 60),
        (UNIT_BOX, (8, 8, 8), 82, 2.0, 1, 60),
        # cutoffs the tensor-core gather covers besides m = 6 (eps 1e-8, 1e-10,
        # a sigma = 1.5 m = 3 plan) and one past it (m = 7, general path)
        (OFFSET_BOX, (16, 16, 16), 74, 2.0, 4, 300),
        (OFFSET_BOX, (12, 20, 16), 75, 2.0, 5, 300),
        (UNIT_BOX, (20, 16, 12), 76, 1.5, 3, 400),
        (OFFSET_BOX, (8, 24, 12), 77, 2.0, 7, 200),
    ]
    out = {}
    for i, (box, shape, seed, sigma, m, npts) in enumerate(cases):
        spec = spectral(box, shape, seed)
        rng = np.random.default_rng(seed + 1000)
        pts = rng.uniform(box.a, box.b, (npts, 3))
        params = vf.NufftParams(oversampling=sigma, cutoff=m, eps=0.999)
        with warnings.catch_warnings():
            warnings.simplefilter("ignore")
            plan = vf.NufftPlan(spec, params)
        a, b = box_arrays(box)
        out[f"case{i}_a"] = a
        out[f"case{i}_b"] = b
        out[f"case{i}_coeffs"] = spec.coeffs
        out[f"case{i}_params"] = np.array([sigma, m], dtype=float)
        out[f"case{i}_points"] = pts
        out[f"case{i}_nufft"] = plan.evaluate(pts)
        out[f"case{i}_direct"] = vf.eval_direct(spec, pts)
        if np.prod(plan._n) <= 20000:
            out[f"case{i}_grid"] = plan._grid
    out["ncases"] = np.array(len(cases))
    save("nufft_cases.npz", **out)


def torus_edges():
    """map_to_torus and the gather's nearest-cell arithmetic at edge points:
    x = a + tiny (zeta can come out as +1/2), u just below an integer + 1/2,
    x = midpoint / quarter points, and random points on the offset box."""
    a, b = box_arrays(OFFSET_BOX)
    rng = np.random.default_rng(5)
    rows = [a, (a + b) / 2, a + (b - a) / 4, a + 1e-300, np.nextafter(a, b), np.nextafter(b, a)]
    # points whose torus coordinate sits exactly at / next to cell edges for n = 32
    n = np.array([32, 32, 32])
    for frac in (0.5, 0.5 / 32, 1.5 / 32, 31.5 / 32, 0.25, 0.75):
        x = a + (b - a) * frac
        rows += [x, np.nextafter(x, b), np.nextafter(x, a)]
    pts = np.vstack(rows + [rng.uniform(a, b, (400, 3))])
    zeta = vf.map_to_torus(pts, OFFSET_BOX)
    z = np.where(zeta < 0, zeta + 1.0, zeta)  # nufft.py:249
    u = z * n
    l0 = np.floor(u + 0.5).astype(np.int64)  # nufft.py:256-257
    # x just above the midpoint gives zeta = -tiny, z = 1 - tiny and l0 == n
    assert (l0 == n).any()
    save("torus_edges.npz", a=a, b=b, points=pts, zeta=zeta, n=n, l0=l0)


def kb_tables():
    out = {}
    for m, sigma, nmodes in ((6, 2.0, 32), (3, 2.0, 16), (13, 2.0, 24), (6, 1.6, 20)):
        beta = _kb_beta(m, sigma)
        n = int(round(sigma * nmodes))
        k = np.arange(nmodes) - nmodes // 2
        v = np.linspace(-(m + 0.5), m + 0.5, 101)
        key = f"m{m}_s{sigma}"
        out[key + "_beta"] = np.array(beta)
        out[key + "_hat"] = _kb_transform(k, n, m, beta)
        out[key + "_n"] = np.array(n)
        out[key + "_v"] = v
        out[key + "_win"] = _kb_values(v[None, :], m, beta)[0]
    save("kb_tables.npz", **out)


def config1():
    """BASELINE config 1 (N=32^3, M=1e4) through the reference: all 1e4 NUFFT
    values and a 200-point direct-NDFT subset."""
    coeffs = workloads.coefficients("c1")
    pts = workloads.points("c1")
    box = vf.DomainBox(*workloads.UNIT_BOX)
    spec = vf.SpectralField(box, coeffs)
    plan = vf.NufftPlan(spec)
    ref = plan.evaluate(pts)
    direct = vf.eval_direct(spec, pts[:200])
    save(
        "config1.npz",
        coeffs_sum=np.array([coeffs.real.sum(), coeffs.imag.sum(), np.abs(coeffs).sum()]),
        points_sum=pts.sum(axis=0),
        nufft=ref,
        direct200=direct,
    )


def cluster_small():
    """A reduced config-3 (32^3 vortex-pair spectrum on [-8,8)^3, 1500 points
    in a 0.05-std cloud around the origin) — exercises the periodic seam."""
    box = vf.DomainBox(*workloads.VORTEX_BOX)
    coeffs = workloads.vortex_pair_spectrum((32, 32, 32), workloads.VORTEX_BOX)
    pts = np.random.default_rng(2003).normal(0.0, 0.05, (1500, 3))
    spec = vf.SpectralField(box, coeffs)
    plan = vf.NufftPlan(spec)
    save(
        "cluster_small.npz",
        coeffs=coeffs,
        points=pts,
        nufft=plan.evaluate(pts),
        direct=vf.eval_direct(spec, pts[:100]),
    )


def rectilinear_cases():
    out = {}
    cases = [
        (OFFSET_BOX, (6, 4, 6), 41, (3, 2, 3)),
        (OFFSET_BOX, (16, 16, 16), 43, (20, 24, 28)),
        (UNIT_BOX, (8, 12, 10), 45, (1, 7, 33)),
    ]
    for i, (box, shape, seed, msz) in enumerate(cases):
        spec = spectral(box, shape, seed)
        rng = np.random.default_rng(seed + 1)
        coords = [rng.uniform(box.a[d], box.b[d], msz[d]) for d in range(3)]
        a, b = box_arrays(box)
        out[f"case{i}_a"] = a
        out[f"case{i}_b"] = b
        out[f"case{i}_coeffs"] = spec.coeffs
        for d in range(3):
            out[f"case{i}_y{d}"] = coords[d]
            out[f"case{i}_E{d}"] = vf.basis_matrix(box, shape[d], d, coords[d])
        out[f"case{i}_out"] = vf.eval_rectilinear(spec, coords)
    out["ncases"] = np.array(len(cases))
    save("rect_cases.npz", **out)




def tube_case():
    """tube_eval on the reference's single-vortex snapshot (tests/test_tube.py
    fixture): thresholds (0.4, 0.3), plus (0.4,) and a final filter."""
    from vortexfourier.gpe import Snapshot, snapshot_spectral
    from vortexfourier.tube import tube_eval

    dom = vf.DomainBox((-10.0, -10.0, -10.0), (10.0, 10.0, 10.0))
    spec = vf.VortexSpec(position=(0.0, 0.0, 0.0), direction=(0.0, 0.0, 1.0))
    init = vf.initial_field(dom, (16, 16, 16), [spec])
    snap = Snapshot(dom, init.values, (True, True, True), 0.0)
    out = {"values": snap.values, "a": np.array(dom.a), "b": np.array(dom.b),
           "mirror": np.array(snap.mirror), "spectral": snapshot_spectral(snap).coeffs}
    for tag, thr, ff in (("two", [0.4, 0.3], None), ("one", [0.4], None), ("filt", [0.4, 0.3], 0.15)):
        cloud = tube_eval(snap, thr, final_filter=ff)
        out[f"{tag}_points"] = cloud.points
        out[f"{tag}_density"] = cloud.density
        out[f"{tag}_level"] = cloud.level
    save("tube_case.npz", **out)


if __name__ == "__main__":
    nufft_cases()
    torus_edges()
    kb_tables()
    config1()
    cluster_small()
    rectilinear_cases()
    tube_case()
