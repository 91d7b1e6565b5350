"""File formats on the CPU: the native readers / writers of
libvfnfft.so against the reference-written fixtures in tests/golden/io/
(made by tests/golden/make_io_golden.py) and against the plain-Python
restatement in oracle/formats_oracle.py.  Mirrors the reference's
tests/test_io.py cases (round trips, bad magic / version / truncation /
short payload, empty and ragged CSVs, VTK layout, field files)."""

import os
import struct

import numpy as np
import pytest

from conftest import GOLDEN
from oracle import formats_oracle as O

IO = os.path.join(GOLDEN, "io")


def gold(name):
    return os.path.join(IO, name)


def raw(name):
    with open(gold(name), "rb") as fh:
        return fh.read()


@pytest.fixture(scope="module")
def F():
    from paper_1605_01244_b200 import formats

    return formats


# ------------------------------------------------------------ oracle pinning


def test_oracle_reproduces_every_fixture():
    for name in ("snap_small.sfs", "snap_vortex.sfs"):
        a, b, v, m, t = O.unpack_snapshot(raw(name))
        assert O.pack_snapshot(a, b, v, m, t) == raw(name)
    for name in ("pts_small.csv", "pts_special.csv", "pts_empty.csv", "eval_in.csv", "eval_default.csv",
                 "tube_out.csv"):
        cols = O.parse_points_csv(raw(name).decode())
        pts = np.stack([cols.pop("x1"), cols.pop("x2"), cols.pop("x3")], axis=1)
        if name == "pts_small.csv":
            cols["level"] = cols["level"].astype(np.int64)
        if name == "pts_special.csv":
            cols["i"] = cols["i"].astype(np.int64)
        assert O.points_csv_bytes(pts, cols) == raw(name), name
    for tag in ("equi", "clus"):
        text = raw(f"grid_{tag}.hdr").decode()
        meta = dict(line.split("#")[0].strip().split(" = ", 1) for line in text.splitlines())
        coords = [np.array([float(x) for x in meta[f"coords_{d}"].split()]) for d in (1, 2, 3)]
        shape = tuple(len(c) for c in coords)
        assert O.field_header(shape, coords, f"grid_{tag}.psi.f64", f"grid_{tag}.rho.f64",
                              float(meta["time"])) == text
        rho = np.frombuffer(raw(f"grid_{tag}.rho.f64"), "<f8").reshape(shape)
        assert O.vtk_bytes(coords, {"density": rho}) == raw(f"grid_{tag}.vtk")


# ------------------------------------------------------------ snapshots


def test_snapshot_read_matches_reference_bytes(F):
    for name in ("snap_small.sfs", "snap_vortex.sfs"):
        s = F.read_snapshot(gold(name))
        a, b, v, m, t = O.unpack_snapshot(raw(name))
        assert s.domain.a == a and s.domain.b == b and s.mirror == m and s.time == t
        assert s.values.dtype == np.complex128
        assert np.array_equal(s.values.view(np.uint64), v.view(np.uint64))


def test_snapshot_write_is_byte_identical(F, tmp_path):
    for name in ("snap_small.sfs", "snap_vortex.sfs"):
        s = F.read_snapshot(gold(name))
        F.write_snapshot(tmp_path / name, s)
        assert (tmp_path / name).read_bytes() == raw(name)


def test_snapshot_round_trip_bit_exact(F, tmp_path):
    from paper_1605_01244_b200 import DomainBox, Snapshot

    rng = np.random.default_rng(5)
    v = rng.standard_normal((3, 5, 2)) + 1j * rng.standard_normal((3, 5, 2))
    v.flat[0] = complex(-0.0, np.inf)
    s = Snapshot(DomainBox((0.0, -1.0, 2.0), (1.0, 1.0, 3.5)), v, (False, True, False), 0.1 + 0.2)
    F.write_snapshot(tmp_path / "x.sfs", s)
    back = F.read_snapshot(tmp_path / "x.sfs")
    assert np.array_equal(back.values.view(np.uint64), v.view(np.uint64))
    assert back.time == 0.1 + 0.2 and back.mirror == (False, True, False)


def _corrupt(tmp_path, data):
    p = tmp_path / "state.sfs"
    p.write_bytes(data)
    return p


@pytest.mark.parametrize("mutate,match", [
    (lambda r: b"NOPE" + r[4:], r"not a snapshot file \(bad magic b'NOPE'\)"),
    (lambda r: r[:4] + (99).to_bytes(4, "little") + r[8:], "unsupported snapshot version 99"),
    (lambda r: b"SFS1\x01", "truncated snapshot header"),
    (lambda r: r[:-16], r"payload size 3056 does not match 6x4x8 complex values"),
    (lambda r: r + b"\0", r"payload size 3073 does not match 6x4x8 complex values"),
    (lambda r: b"S'\x00\xff" + r[4:], r"bad magic b\"S'\\x00\\xff\""),
])
def test_snapshot_rejects_like_the_reference(F, tmp_path, mutate, match):
    p = _corrupt(tmp_path, mutate(raw("snap_small.sfs")))
    with pytest.raises(ValueError, match=match):
        F.read_snapshot(p)
    # the same text as the oracle restatement
    with pytest.raises(ValueError, match=match):
        O.unpack_snapshot(p.read_bytes())


def test_snapshot_missing_file_is_oserror(F, tmp_path):
    with pytest.raises(OSError):
        F.read_snapshot(tmp_path / "absent.sfs")


# ------------------------------------------------------------ points CSV


@pytest.mark.parametrize("name", ["pts_small.csv", "pts_special.csv", "pts_empty.csv", "eval_in.csv",
                                  "eval_default.csv", "eval_acc6.csv", "tube_out.csv"])
def test_csv_read_matches_oracle(F, name):
    got = F.read_points_csv(gold(name))
    ref = O.parse_points_csv(raw(name).decode())
    assert list(got) == list(ref)
    for k in ref:
        assert got[k].dtype == np.float64
        assert np.array_equal(got[k].view(np.uint64), ref[k].view(np.uint64)), k


def test_csv_write_is_byte_identical(F, tmp_path):
    for name in ("pts_small.csv", "pts_special.csv", "pts_empty.csv", "eval_default.csv", "tube_out.csv"):
        cols = O.parse_points_csv(raw(name).decode())
        pts = np.stack([cols.pop("x1"), cols.pop("x2"), cols.pop("x3")], axis=1)
        if name == "pts_small.csv":
            cols["level"] = cols["level"].astype(np.int64)  # written from an int array
        if name == "pts_special.csv":
            cols["i"] = cols["i"].astype(np.int64)
        F.write_points_csv(tmp_path / name, pts, cols)
        assert (tmp_path / name).read_bytes() == raw(name), name


def test_csv_float_repr_fuzz(F, tmp_path):
    """Every bit pattern class: Python repr() is the oracle."""
    rng = np.random.default_rng(7)
    v = rng.integers(0, 2**64, 30000, dtype=np.uint64).view(np.float64)
    v = np.concatenate([v, rng.uniform(-1, 1, 30000) * 10.0 ** rng.integers(-25, 25, 30000),
                        np.round(rng.uniform(-1e6, 1e6, 3000) * 10.0 ** rng.integers(0, 6, 3000)) / 10.0 ** rng.integers(0, 6, 3000)])
    v = v[: v.size // 3 * 3].reshape(-1, 3)
    flags = rng.random(v.shape[0]) < 0.5
    F.write_points_csv(tmp_path / "f.csv", v, {"flag": flags, "k": np.arange(v.shape[0]) * -3})
    assert (tmp_path / "f.csv").read_bytes() == O.points_csv_bytes(v, {"flag": flags, "k": np.arange(v.shape[0]) * -3})
    F.write_points_csv(tmp_path / "g.csv", v, {"k": np.arange(v.shape[0]) * -3})
    back = F.read_points_csv(tmp_path / "g.csv")
    pts = np.stack([back["x1"], back["x2"], back["x3"]], axis=1)
    same = (pts.view(np.uint64) == v.view(np.uint64)) | (np.isnan(pts) & np.isnan(v))
    assert same.all()


def test_csv_strided_columns(F, tmp_path):
    rng = np.random.default_rng(3)
    vals = rng.standard_normal(50) + 1j * rng.standard_normal(50)
    pts = rng.standard_normal((50, 3))
    cols = {"re": vals.real, "im": vals.imag, "rho": vals.real**2 + vals.imag**2}
    F.write_points_csv(tmp_path / "s.csv", pts, cols)
    assert (tmp_path / "s.csv").read_bytes() == O.points_csv_bytes(pts, cols)


def test_csv_parse_like_python_float(F, tmp_path):
    text = ('x1, x2 ,"x3",q\n 1.5 ,+2,-inf,1_000.5\n\n"3e-400",1E5,  NaN,.5\r\n'
            '5.,Infinity,-0.0,1e400\r"7",\t8\t,9,10\n')
    (tmp_path / "t.csv").write_text(text, newline="")
    got = F.read_points_csv(tmp_path / "t.csv")
    ref = O.parse_points_csv(text)
    assert list(got) == list(ref) == ["x1", "x2", "x3", "q"]
    for k in ref:
        a, b = got[k], ref[k]
        assert ((a.view(np.uint64) == b.view(np.uint64)) | (np.isnan(a) & np.isnan(b))).all(), k


@pytest.mark.parametrize("text,exc,match", [
    ("", ValueError, "empty points file, expected a header row"),
    ("x1,x2,x3,density\n1.0,2.0,3.0\n", ValueError, "ragged"),
    ("x1,x2\n1,2,3\n", ValueError, "ragged"),
    ("x1\nabc\n", ValueError, "could not convert string to float: 'abc'"),
    ("x1\n1__0\n", ValueError, "could not convert string to float"),
    ("x1\nnan(1)\n", ValueError, "could not convert string to float"),
    ("x1,x2\n1,\n", ValueError, "could not convert string to float: ''"),
    ("x1\n0x10\n", ValueError, "could not convert string to float"),
])
def test_csv_rejects_like_the_reference(F, tmp_path, text, exc, match):
    (tmp_path / "e.csv").write_text(text, newline="")
    with pytest.raises(exc, match=match):
        F.read_points_csv(tmp_path / "e.csv")
    with pytest.raises(exc, match=match):
        O.parse_points_csv(text)


def test_csv_large_multithreaded_round_trip(F, tmp_path):
    """Big enough to split across host threads (chunk boundaries inside
    CRLF pairs, empty lines at chunk edges)."""
    rng = np.random.default_rng(9)
    pts = rng.uniform(-10, 10, (200000, 3))
    F.write_points_csv(tmp_path / "big.csv", pts, {"rho": pts[:, 0] ** 2})
    body = (tmp_path / "big.csv").read_bytes()
    assert body == O.points_csv_bytes(pts[:2000], {"rho": pts[:2000, 0] ** 2}) + \
        b"".join(O.points_csv_bytes(pts[2000:], {"rho": pts[2000:, 0] ** 2}).split(b"\r\n", 1)[1:])
    got = F.read_points(tmp_path / "big.csv")
    assert np.array_equal(got, pts)
    # blank lines anywhere are skipped (csv yields [] for them)
    (tmp_path / "gaps.csv").write_bytes(body.replace(b"\r\n", b"\r\n\r\n\n", 5000))
    assert np.array_equal(F.read_points(tmp_path / "gaps.csv"), pts)


def test_read_points_missing_column(F, tmp_path):
    (tmp_path / "p.csv").write_text("x1,x2\n1.0,2.0\n")
    with pytest.raises(ValueError, match="lacks column 'x3'"):
        F.read_points(tmp_path / "p.csv")


# ------------------------------------------------------------ fields / VTK


def _grid(tag):
    text = raw(f"grid_{tag}.hdr").decode()
    meta = dict(line.split("#")[0].strip().split(" = ", 1) for line in text.splitlines())
    coords = [np.array([float(x) for x in meta[f"coords_{d}"].split()]) for d in (1, 2, 3)]
    shape = tuple(len(c) for c in coords)
    psi = np.frombuffer(raw(f"grid_{tag}.psi.f64"), "<c16").reshape(shape)
    rho = np.frombuffer(raw(f"grid_{tag}.rho.f64"), "<f8").reshape(shape)
    return coords, psi, rho, float(meta["time"])


@pytest.mark.parametrize("tag", ["equi", "clus"])
def test_field_write_is_byte_identical(F, tmp_path, tag):
    coords, psi, rho, t = _grid(tag)
    paths = F.write_field(tmp_path / f"grid_{tag}", coords, psi, rho, time=t)
    assert [p.name for p in paths] == [f"grid_{tag}.hdr", f"grid_{tag}.psi.f64", f"grid_{tag}.rho.f64"]
    for p in paths:
        assert p.read_bytes() == raw(p.name), p.name
    rc, rv, rd, meta = F.read_field(tmp_path / f"grid_{tag}")
    assert all(np.array_equal(a, b) for a, b in zip(rc, coords))
    assert np.array_equal(rv, psi) and np.array_equal(rd, rho) and float(meta["time"]) == t


@pytest.mark.parametrize("tag", ["equi", "clus"])
def test_vtk_write_is_byte_identical(F, tmp_path, tag):
    coords, psi, rho, _ = _grid(tag)
    F.write_vtk_rectilinear(tmp_path / "x.vtk", coords, {"density": rho})
    assert (tmp_path / "x.vtk").read_bytes() == raw(f"grid_{tag}.vtk")


def test_vtk_two_scalars_and_title(F, tmp_path):
    coords = F.equispaced_axes((3, 4, 2), (0.0, 1.0, 0.0, 2.0, -1.0, 1.0))
    rng = np.random.default_rng(5)
    rho = rng.standard_normal((3, 4, 2))
    sc = {"density": rho, "phase": rho * 1e-40}
    F.write_vtk_rectilinear(tmp_path / "f.vtk", coords, sc, title="demo")
    assert (tmp_path / "f.vtk").read_bytes() == O.vtk_bytes(coords, sc, title="demo")
    with pytest.raises(ValueError, match="density"):
        F.write_vtk_rectilinear(tmp_path / "x.vtk", coords, {"density": np.zeros((3, 3))})


def test_field_shape_mismatch_and_unknown_format(F, tmp_path):
    coords = F.equispaced_axes((4, 4, 4), (0.0, 1.0) * 3)
    with pytest.raises(ValueError, match="does not match"):
        F.write_field(tmp_path / "out", coords, np.zeros((4, 4, 5), complex), np.zeros((4, 4, 5)))
    (tmp_path / "o.hdr").write_text("format = something-else\n")
    with pytest.raises(ValueError, match="unknown field format"):
        F.read_field(tmp_path / "o")


def test_axes_helpers(F):
    axes = F.equispaced_axes((5, 3, 2), (0.0, 1.0, -2.0, 2.0, 10.0, 20.0))
    assert [len(c) for c in axes] == [5, 3, 2] and axes[2][0] == 10.0 and axes[2][-1] == 20.0
    with pytest.raises(ValueError, match="direction 1"):
        F.equispaced_axes((4, 4, 4), (0.0, 1.0, 2.0, 2.0, 0.0, 1.0))
    c = F.clustered_axes((21, 11, 9), (-3.0, 5.0, 0.0, 1.0, -1.0, 1.0), 0.5)
    assert c[0][0] == -3.0 and c[0][-1] == 5.0 and np.all(np.diff(c[0]) > 0)
    with pytest.raises(ValueError, match="positive"):
        F.clustered_axes((8, 8, 8), (0.0, 1.0) * 3, 0.0)
    # identical to the coordinates recorded in the clustered fixture header
    coords, _, _, _ = _grid("clus")
    mine = F.clustered_axes((9, 7, 5), (-9.0, 9.0, -9.0, 9.0, -8.0, 8.0), 0.5)
    assert all(np.array_equal(a, b) for a, b in zip(mine, coords))


def test_parse_grid_specs(tmp_path):
    from paper_1605_01244_b200.pipeline import parse_grid

    (tmp_path / "axes.txt").write_text("-3 -1 0 1 3\n-2 0 2\n-1 1\n")
    c = parse_grid(["file", str(tmp_path / "axes.txt")])
    assert [len(x) for x in c] == [5, 3, 2]
    c = parse_grid(["equispaced", "6", "5", "4", "-3", "3", "-3", "3", "-2", "2"])
    assert [len(x) for x in c] == [6, 5, 4]
    with pytest.raises(ValueError, match="unknown grid kind"):
        parse_grid(["random", "4"])
    with pytest.raises(ValueError, match="three lines"):
        (tmp_path / "bad.txt").write_text("1 2\n3 4\n")
        parse_grid(["file", str(tmp_path / "bad.txt")])


def test_header_struct_layout():
    assert O.SFS1_HEADER.size == 79
    h = raw("snap_small.sfs")[:79]
    assert struct.unpack("<4sI", h[:8]) == (b"SFS1", 1)
