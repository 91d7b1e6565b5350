"""Generate the file-format fixtures under tests/golden/io/ with the REAL
reference writers (vortexfourier.snapshots / vortexfourier.fields) and the
bodies of its eval-points / eval-grid / tube commands (cli.py:90-142; the
cli module itself imports matplotlib, absent here, so the few lines of each
command body are repeated below with the reference's public functions).

    PYTHONDONTWRITEBYTECODE=1 python tests/golden/make_io_golden.py

Small files (~240 KB total), committed; the GPU box never reads
/root/reference.
"""

from __future__ import annotations

import os
import shutil
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
OUT = os.path.join(HERE, "io")
sys.path.insert(0, "/root/reference/pkg/src")

import vortexfourier as vf  # noqa: E402
from vortexfourier import fields  # noqa: E402
from vortexfourier.gpe import Snapshot, snapshot_spectral  # noqa: E402
from vortexfourier.nufft import NufftParams, NufftPlan  # noqa: E402
from vortexfourier.rectilinear import eval_rectilinear  # noqa: E402
from vortexfourier.snapshots import write_snapshot  # noqa: E402
from vortexfourier.tube import tube_eval  # noqa: E402


def p(name):
    return os.path.join(OUT, name)


def small_snapshot():
    # the reference's test_io.py:_random_snapshot shape/box/mirror/time
    rng = np.random.default_rng(0)
    values = rng.standard_normal((6, 4, 8)) + 1j * rng.standard_normal((6, 4, 8))
    dom = vf.DomainBox((-1.5, 0.25, 2.0), (2.5, 1.25, 7.0))
    write_snapshot(p("snap_small.sfs"), Snapshot(dom, values, (True, False, True), 3.25))


def vortex_snapshot():
    dom = vf.DomainBox((-10.0, -10.0, -10.0), (10.0, 10.0, 10.0))
    spec = vf.VortexSpec(position=(0.5, -0.25, 0.0), direction=(0.0, 0.6, 0.8))
    init = vf.initial_field(dom, (16, 12, 16), [spec])
    snap = Snapshot(dom, init.values, (True, False, True), 1.75)
    write_snapshot(p("snap_vortex.sfs"), snap)
    return snap


def csv_files():
    rng = np.random.default_rng(11)
    pts = rng.standard_normal((7, 3))
    rho = rng.random(7)
    level = np.array([0, 1, 2, 2, 1, 0, 2])
    fields.write_points_csv(p("pts_small.csv"), pts, {"density": rho, "level": level})
    fields.write_points_csv(p("pts_empty.csv"), np.empty((0, 3)), {"density": np.empty(0)})
    # awkward doubles: repr switches, signed zero, infinities, subnormals
    special = np.array([0.0, -0.0, np.inf, -np.inf, 1e16, 1e-5, 1e-4, 9999999999999998.0,
                        1234567890123456.0, 5e-324, 2.2250738585072014e-308, 1.7976931348623157e308,
                        0.1, 1 / 3, 9007199254740993.0, 1e22, -1e23, 123.0, 0.000123, 1e-310,
                        2.5e-5, 1.5, -2.75e100])
    bits = rng.integers(0, 2**63, 3 * 40, dtype=np.uint64).view(np.float64)
    bits = bits[np.isfinite(bits)]
    vals = np.concatenate([special, bits, rng.uniform(-1, 1, 60) * 10.0 ** rng.integers(-20, 20, 60)])
    vals = vals[: (vals.size // 3) * 3]
    pts = vals.reshape(-1, 3)
    fields.write_points_csv(p("pts_special.csv"), pts, {"nan": np.full(pts.shape[0], np.nan),
                                                         "i": np.arange(pts.shape[0]) - 7})


def eval_points(snap, tag, accuracy):
    rng = np.random.default_rng(2)
    pts = rng.uniform(-9.5, 9.5, size=(64, 3))
    fields.write_points_csv(p("eval_in.csv"), pts, {})
    # cmd_eval_points body (cli.py:108-125)
    spec = snapshot_spectral(snap)
    cols = fields.read_points_csv(p("eval_in.csv"))
    pts = np.stack([cols["x1"], cols["x2"], cols["x3"]], axis=1)
    params = None if accuracy is None else NufftParams.for_accuracy(accuracy)
    values = NufftPlan(spec, params).evaluate(pts)
    density = values.real**2 + values.imag**2
    fields.write_points_csv(p(f"eval_{tag}.csv"), pts, {"re": values.real, "im": values.imag, "rho": density})


def eval_grid(snap):
    # cmd_eval_grid body (cli.py:90-105), grids as test_cli.py uses them
    spec = snapshot_spectral(snap)
    for tag, coords in (
        ("equi", fields.equispaced_axes((6, 5, 4), (-9.0, 9.0, -9.0, 9.0, -8.0, 8.0))),
        ("clus", fields.clustered_axes((9, 7, 5), (-9.0, 9.0, -9.0, 9.0, -8.0, 8.0), 0.5)),
    ):
        values = eval_rectilinear(spec, coords)
        density = values.real**2 + values.imag**2
        fields.write_field(p(f"grid_{tag}"), coords, values, density, time=snap.time)
        fields.write_vtk_rectilinear(p(f"grid_{tag}.vtk"), coords, {"density": density})


def tube(snap):
    # cmd_tube body (cli.py:128-142)
    cloud = tube_eval(snap, [0.3, 0.2], final_filter=0.02)
    fields.write_points_csv(p("tube_out.csv"), cloud.points,
                            {"rho": cloud.density, "level": cloud.level.astype(float)})


if __name__ == "__main__":
    shutil.rmtree(OUT, ignore_errors=True)
    os.makedirs(OUT)
    small_snapshot()
    snap = vortex_snapshot()
    csv_files()
    eval_points(snap, "default", None)
    eval_points(snap, "acc6", 1e-6)
    eval_grid(snap)
    tube(snap)
    for f in sorted(os.listdir(OUT)):
        print(f, os.path.getsize(p(f)))
