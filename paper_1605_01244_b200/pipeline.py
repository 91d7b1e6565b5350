"""The reference's file-to-file evaluation commands (cli.py:64-142) with the
whole chain on the device: snapshot file -> HBM (pinned chunks) -> spectral
coefficients (vfn_decompose) -> plan -> evaluation -> density -> file, so
only the input file and the output bytes cross PCIe.

* ``eval_points``  <- ``cmd_eval_points`` (cli.py:108-125)
* ``eval_grid``    <- ``cmd_eval_grid``   (cli.py:90-105), without the figure
* ``tube``         <- ``cmd_tube``        (cli.py:128-142), without the figure
* ``parse_grid``   <- the grid argument of ``eval-grid`` (cli.py:64-87)

Each returns what the command prints about (the written paths / the point
count) instead of printing it; errors are the same ValueError / OSError the
CLI turns into ``error: ...`` lines.
"""

from __future__ import annotations

from pathlib import Path

import numpy as np

from . import formats
from .nufft import NufftParams, NufftPlan
from .rectilinear import eval_rectilinear
from .tube import snapshot_spectral, tube_eval

__all__ = ["eval_grid", "eval_points", "parse_grid", "tube"]


def _params(accuracy):
    # cli.py:28-31
    return None if accuracy is None else NufftParams.for_accuracy(accuracy)


def _device(device):
    if device is not None:
        return device
    import torch

    if not torch.cuda.is_available():
        raise RuntimeError("the evaluation pipeline needs a CUDA device")
    return torch.cuda.current_device()


_GRID_ARITY = {"equispaced": (9,), "clustered": (9, 10)}


def _axes_file(path) -> list[np.ndarray]:
    lines = [ln for ln in Path(path).read_text().strip().splitlines()]
    if len(lines) != 3:
        raise ValueError(f"grid file {path} must hold three lines of coordinates, one per axis")
    return [np.fromiter((float(t) for t in ln.split()), dtype=float) for ln in lines]


def parse_grid(tokens) -> list[np.ndarray]:
    """Grid spec tokens -> three coordinate vectors.  Accepted forms (the
    CLI's grid argument, cli.py:64-87): ``file PATH`` (three whitespace
    separated coordinate lines), ``equispaced M1 M2 M3 a1 b1 a2 b2 a3 b3`` and
    ``clustered M1 M2 M3 a1 b1 a2 b2 a3 b3 [strength]``."""
    kind, rest = tokens[0], list(tokens[1:])
    if kind == "file":
        if len(rest) != 1:
            raise ValueError("grid spec: file takes exactly one path")
        return _axes_file(rest[0])
    if kind not in _GRID_ARITY:
        raise ValueError(f"unknown grid kind {kind!r} (expected file, equispaced or clustered)")
    nums = [float(t) for t in rest]
    if len(nums) not in _GRID_ARITY[kind]:
        raise ValueError(f"grid spec: {kind} takes M1 M2 M3 a1 b1 a2 b2 a3 b3"
                         + (" [strength]" if kind == "clustered" else ""))
    counts, bounds = [int(v) for v in nums[:3]], nums[3:9]
    if kind == "equispaced":
        return formats.equispaced_axes(counts, bounds)
    return formats.clustered_axes(counts, bounds, nums[9] if len(nums) > 9 else 1.0)


def eval_grid(snapshot, grid, out, vtk: bool = False, device=None) -> list[Path]:
    """Snapshot on a rectilinear grid -> field files (+ VTK); ``grid`` is a
    token list for parse_grid or three coordinate vectors (cli.py:90-105)."""
    dev = _device(device)
    snap = formats.read_snapshot(snapshot, device=dev)
    spec = snapshot_spectral(snap)
    coords = parse_grid(grid) if isinstance(grid[0], str) else [np.asarray(c, dtype=float) for c in grid]
    values = eval_rectilinear(spec, coords)
    rho = formats.density(values)
    written = formats.write_field(out, coords, values, rho, time=snap.time)
    if vtk:
        vtk_path = Path(out).with_suffix(".vtk")
        formats.write_vtk_rectilinear(vtk_path, coords, {"density": rho})
        written.append(vtk_path)
    return written


def eval_points(snapshot, points, out, accuracy=None, device=None) -> int:
    """Snapshot at the points of a CSV -> CSV with re, im, rho columns
    (cli.py:108-125); returns the point count."""
    dev = _device(device)
    import torch

    snap = formats.read_snapshot(snapshot, device=dev)
    spec = snapshot_spectral(snap)
    pts = formats.read_points(points, device=dev)
    M = int(pts.shape[0])
    if M:
        values = NufftPlan(spec, _params(accuracy), device=pts.device.index).evaluate(pts)
    else:
        values = torch.empty(0, dtype=torch.complex128, device=pts.device)
    rho = formats.density(values)
    # one D2H of values + density; re / im are strided views of the values
    v = values.cpu().numpy()
    formats.write_points_csv(out, pts.cpu().numpy(), {"re": v.real, "im": v.imag, "rho": rho.cpu().numpy()})
    return M


def tube(snapshot, rhobar, out, final_filter=None, accuracy=None, device=None) -> int:
    """Low-density point cloud of a snapshot -> CSV with rho, level columns
    (cli.py:128-142); returns the point count."""
    dev = _device(device)
    snap = formats.read_snapshot(snapshot, device=dev)
    cloud = tube_eval(snap, rhobar, final_filter=final_filter, params=_params(accuracy))
    formats.write_points_csv(out, cloud.points, {"rho": cloud.density, "level": cloud.level.astype(float)})
    return len(cloud)
