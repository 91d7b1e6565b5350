"""File formats and the file-to-file commands on the B200:
snapshot -> HBM, CSV points -> HBM, density / VTK packing on the device,
device payloads streamed to files, and the eval-points / eval-grid / tube
commands end to end against the reference's own outputs recorded in
tests/golden/io/ (tests/golden/make_io_golden.py)."""

import os

import numpy as np
import pytest

from conftest import GOLDEN
from oracle import formats_oracle as O

pytestmark = pytest.mark.gpu

IO = os.path.join(GOLDEN, "io")
TOL = 1e-10  # the north-star accuracy gate, relative to max |ref|


def gold(name):
    return os.path.join(IO, name)


def raw(name):
    with open(gold(name), "rb") as fh:
        return fh.read()


@pytest.fixture(scope="module")
def torch():
    import torch

    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    return torch


@pytest.fixture(scope="module")
def F():
    from paper_1605_01244_b200 import formats

    return formats


def test_snapshot_to_device_and_back(F, torch, tmp_path):
    for name in ("snap_small.sfs", "snap_vortex.sfs"):
        host = F.read_snapshot(gold(name))
        dev = F.read_snapshot(gold(name), device=0)
        assert dev.values.is_cuda and dev.values.dtype == torch.complex128
        assert np.array_equal(dev.values.cpu().numpy().view(np.uint64), host.values.view(np.uint64))
        F.write_snapshot(tmp_path / name, dev)
        assert (tmp_path / name).read_bytes() == raw(name)


def test_large_snapshot_streams_through_pinned_chunks(F, torch, tmp_path):
    """> 2 staging chunks (16 MB each) in both directions."""
    from paper_1605_01244_b200 import DomainBox, Snapshot

    g = torch.Generator(device="cuda").manual_seed(3)
    v = torch.randn((64, 96, 80), dtype=torch.complex128, device="cuda", generator=g)  # 78.6 MB
    s = Snapshot(DomainBox((0.0, 0.0, 0.0), (1.0, 2.0, 3.0)), v, (True, False, False), 2.5)
    F.write_snapshot(tmp_path / "big.sfs", s)
    a, b, hv, m, t = O.unpack_snapshot((tmp_path / "big.sfs").read_bytes())
    assert np.array_equal(hv, v.cpu().numpy()) and m == (True, False, False) and t == 2.5
    back = F.read_snapshot(tmp_path / "big.sfs", device=0)
    assert torch.equal(back.values, v)


def test_points_to_device(F, torch):
    for name in ("eval_in.csv", "tube_out.csv"):
        host = F.read_points(gold(name))
        dev = F.read_points(gold(name), device=0)
        assert dev.is_cuda and np.array_equal(dev.cpu().numpy(), host)
    assert F.read_points(gold("pts_empty.csv"), device=0).shape == (0, 3)


def test_density_matches_numpy_bitwise(F, torch):
    g = torch.Generator(device="cuda").manual_seed(1)
    v = torch.randn(1 << 20, dtype=torch.complex128, device="cuda", generator=g) * 1e3
    rho = F.density(v)
    h = v.cpu().numpy()
    assert np.array_equal(rho.cpu().numpy().view(np.uint64), (h.real**2 + h.imag**2).view(np.uint64))


@pytest.mark.parametrize("tag", ["equi", "clus"])
def test_device_field_and_vtk_bytes(F, torch, tmp_path, tag):
    text = raw(f"grid_{tag}.hdr").decode()
    meta = dict(line.split("#")[0].strip().split(" = ", 1) for line in text.splitlines())
    coords = [np.array([float(x) for x in meta[f"coords_{d}"].split()]) for d in (1, 2, 3)]
    shape = tuple(len(c) for c in coords)
    psi = np.frombuffer(raw(f"grid_{tag}.psi.f64"), "<c16").reshape(shape)
    rho = np.frombuffer(raw(f"grid_{tag}.rho.f64"), "<f8").reshape(shape)
    dpsi = torch.as_tensor(psi.copy(), device="cuda")
    drho = F.density(dpsi)
    assert np.array_equal(drho.cpu().numpy(), rho)
    paths = F.write_field(tmp_path / f"grid_{tag}", coords, dpsi, drho, time=float(meta["time"]))
    for p in paths:
        assert p.read_bytes() == raw(p.name), p.name
    F.write_vtk_rectilinear(tmp_path / "x.vtk", coords, {"density": drho})
    assert (tmp_path / "x.vtk").read_bytes() == raw(f"grid_{tag}.vtk")


def test_device_vtk_large_transpose(F, torch, tmp_path):
    coords = F.equispaced_axes((37, 21, 50), (0.0, 1.0, -1.0, 1.0, 0.0, 5.0))
    g = torch.Generator(device="cuda").manual_seed(2)
    sc = torch.randn((37, 21, 50), dtype=torch.float64, device="cuda", generator=g)
    F.write_vtk_rectilinear(tmp_path / "d.vtk", coords, {"s": sc, "t": sc * 3})
    h = sc.cpu().numpy()
    assert (tmp_path / "d.vtk").read_bytes() == O.vtk_bytes(coords, {"s": h, "t": h * 3})


# ------------------------------------------------------------ commands


def _cols(path):
    return O.parse_points_csv(open(path, newline="").read())


def _check_eval_csv(path, ref_name):
    got, ref = _cols(path), _cols(gold(ref_name))
    assert list(got) == ["x1", "x2", "x3", "re", "im", "rho"]
    for k in ("x1", "x2", "x3"):
        assert np.array_equal(got[k], ref[k])
    zg = got["re"] + 1j * got["im"]
    zr = ref["re"] + 1j * ref["im"]
    assert np.abs(zg - zr).max() <= TOL * np.abs(zr).max()
    # rho written is numpy's re**2 + im**2 of the written values
    assert np.array_equal(got["rho"], got["re"] ** 2 + got["im"] ** 2)


def test_eval_points_command(tmp_path, torch):
    from paper_1605_01244_b200 import pipeline

    n = pipeline.eval_points(gold("snap_vortex.sfs"), gold("eval_in.csv"), tmp_path / "o.csv")
    assert n == 64
    _check_eval_csv(tmp_path / "o.csv", "eval_default.csv")


def test_eval_points_accuracy_flag(tmp_path, torch):
    """--accuracy 1e-6 -> cutoff 3 (nufft.py:67-73): the general gather path."""
    from paper_1605_01244_b200 import pipeline

    pipeline.eval_points(gold("snap_vortex.sfs"), gold("eval_in.csv"), tmp_path / "o.csv", accuracy=1e-6)
    _check_eval_csv(tmp_path / "o.csv", "eval_acc6.csv")


def test_eval_points_empty_and_missing_column(tmp_path, torch):
    from paper_1605_01244_b200 import pipeline

    assert pipeline.eval_points(gold("snap_vortex.sfs"), gold("pts_empty.csv"), tmp_path / "o.csv") == 0
    cols = _cols(tmp_path / "o.csv")
    assert list(cols) == ["x1", "x2", "x3", "re", "im", "rho"] and all(v.size == 0 for v in cols.values())
    (tmp_path / "in.csv").write_text("x1,x2\n1.0,2.0\n")
    with pytest.raises(ValueError, match="lacks column"):
        pipeline.eval_points(gold("snap_vortex.sfs"), tmp_path / "in.csv", tmp_path / "o2.csv")


@pytest.mark.parametrize("tag,grid", [
    ("equi", ["equispaced", "6", "5", "4", "-9", "9", "-9", "9", "-8", "8"]),
    ("clus", ["clustered", "9", "7", "5", "-9", "9", "-9", "9", "-8", "8", "0.5"]),
])
def test_eval_grid_command(F, tmp_path, torch, tag, grid):
    from paper_1605_01244_b200 import pipeline

    written = pipeline.eval_grid(gold("snap_vortex.sfs"), grid, tmp_path / f"grid_{tag}", vtk=True)
    assert [p.name for p in written] == [f"grid_{tag}.hdr", f"grid_{tag}.psi.f64", f"grid_{tag}.rho.f64",
                                         f"grid_{tag}.vtk"]
    assert written[0].read_bytes() == raw(f"grid_{tag}.hdr")  # coordinates and time identical
    coords, values, dens, meta = F.read_field(tmp_path / f"grid_{tag}")
    _, rvalues, _, _ = F.read_field(os.path.join(IO, f"grid_{tag}"))
    assert np.abs(values - rvalues).max() <= TOL * np.abs(rvalues).max()
    assert np.array_equal(dens, values.real**2 + values.imag**2)
    assert (tmp_path / f"grid_{tag}.vtk").read_bytes() == O.vtk_bytes(coords, {"density": dens})


def test_tube_command(tmp_path, torch):
    from paper_1605_01244_b200 import pipeline

    n = pipeline.tube(gold("snap_vortex.sfs"), [0.3, 0.2], tmp_path / "c.csv", final_filter=0.02)
    got, ref = _cols(tmp_path / "c.csv"), _cols(gold("tube_out.csv"))
    assert n == ref["x1"].size and list(got) == ["x1", "x2", "x3", "rho", "level"]
    for k in ("x1", "x2", "x3", "level"):
        assert np.array_equal(got[k], ref[k]), k
    assert np.abs(got["rho"] - ref["rho"]).max() <= TOL * np.abs(ref["rho"]).max()
