"""CPU oracle for the file formats feeding the path — TEST INFRASTRUCTURE ONLY.

Plain-Python restatement (struct, csv, repr, numpy) of the reference's
on-disk formats, used by the tests as the checker of the native readers and
writers in csrc/vfn_io.cpp.  The product path never imports it.

Pinning: tests/golden/make_io_golden.py writes fixtures under
tests/golden/io/ with the real reference writers; tests/test_formats.py
checks that this restatement reproduces every fixture byte for byte and
reads every one back to the same values.

Paths are relative to /root/reference/pkg/src/vortexfourier/.
"""

from __future__ import annotations

import csv
import io
import struct

import numpy as np

__all__ = [
    "SFS1_HEADER",
    "pack_snapshot",
    "unpack_snapshot",
    "points_csv_bytes",
    "parse_points_csv",
    "field_header",
    "vtk_bytes",
]

# snapshots.py:29-31: "<4sI6d3I3Bd", 79 bytes
SFS1_HEADER = struct.Struct("<4sI6d3I3Bd")


def pack_snapshot(a, b, values, mirror, time) -> bytes:
    """snapshots.py:34-47"""
    n = values.shape
    head = SFS1_HEADER.pack(b"SFS1", 1, a[0], b[0], a[1], b[1], a[2], b[2], n[0], n[1], n[2],
                            *(1 if m else 0 for m in mirror), time)
    return head + np.ascontiguousarray(values, dtype="<c16").tobytes()


def unpack_snapshot(raw: bytes):
    """snapshots.py:50-72 -> (a, b, values, mirror, time); raises ValueError
    with the reference texts (path prefix omitted)."""
    if len(raw) < SFS1_HEADER.size:
        raise ValueError("truncated snapshot header")
    f = SFS1_HEADER.unpack_from(raw)
    if f[0] != b"SFS1":
        raise ValueError(f"not a snapshot file (bad magic {f[0]!r})")
    if f[1] != 1:
        raise ValueError(f"unsupported snapshot version {f[1]}")
    n = f[8:11]
    count = n[0] * n[1] * n[2]
    if len(raw) != SFS1_HEADER.size + 16 * count:
        raise ValueError(f"payload size {len(raw) - SFS1_HEADER.size} does not match "
                         f"{n[0]}x{n[1]}x{n[2]} complex values")
    values = np.frombuffer(raw, dtype="<c16", count=count, offset=SFS1_HEADER.size).reshape(n)
    return (f[2], f[4], f[6]), (f[3], f[5], f[7]), values.astype(np.complex128), \
        tuple(bool(v) for v in f[11:14]), f[14]


def points_csv_bytes(points, columns: dict) -> bytes:
    """fields.py:146-157: csv.writer rows of repr() values, CRLF."""
    points = np.asarray(points, dtype=float).reshape(-1, 3)
    buf = io.StringIO(newline="")
    w = csv.writer(buf)
    w.writerow(["x1", "x2", "x3"] + list(columns))
    for i in range(points.shape[0]):
        row = [repr(v.item()) for v in points[i]]
        for col in columns.values():
            row.append(repr(col[i].item() if hasattr(col[i], "item") else col[i]))
        w.writerow(row)
    return buf.getvalue().encode()


def parse_points_csv(text: str) -> dict:
    """fields.py:160-174"""
    reader = csv.reader(io.StringIO(text, newline=""))
    try:
        header = next(reader)
    except StopIteration:
        raise ValueError("empty points file, expected a header row")
    rows = [row for row in reader if row]
    data = np.array(rows, dtype=float) if rows else np.empty((0, len(header)))
    if data.ndim == 1:
        data = data[None, :]
    if data.size and data.shape[1] != len(header):
        raise ValueError("ragged CSV")
    return {name.strip(): data[:, i] for i, name in enumerate(header)}


def field_header(shape, coords, psi_name, rho_name, time=None) -> str:
    """fields.py:80-91"""
    lines = [
        "format = rectilinear-field-v1",
        f"size = {shape[0]} {shape[1]} {shape[2]}",
        "order = row-major third-index-fastest",
        f"payload_psi = {psi_name}  # complex, interleaved (re, im) f64, little-endian",
        f"payload_rho = {rho_name}  # f64, little-endian",
    ]
    if time is not None:
        lines.append(f"time = {time!r}")
    for d in range(3):
        lines.append(f"coords_{d + 1} = " + " ".join(repr(float(v)) for v in coords[d]))
    return "\n".join(lines) + "\n"


def vtk_bytes(coords, scalars: dict, title="field") -> bytes:
    """fields.py:119-143"""
    shape = tuple(len(c) for c in coords)
    out = [b"# vtk DataFile Version 3.0\n", title.encode() + b"\n", b"BINARY\n",
           b"DATASET RECTILINEAR_GRID\n", f"DIMENSIONS {shape[0]} {shape[1]} {shape[2]}\n".encode()]
    for name, c in zip("XYZ", coords):
        out.append(f"{name}_COORDINATES {len(c)} double\n".encode())
        out.append(np.ascontiguousarray(c, dtype=">f8").tobytes() + b"\n")
    out.append(f"POINT_DATA {shape[0] * shape[1] * shape[2]}\n".encode())
    for name, data in scalars.items():
        out.append(f"SCALARS {name} float 1\nLOOKUP_TABLE default\n".encode())
        out.append(np.ascontiguousarray(data.transpose(2, 1, 0), dtype=">f4").tobytes() + b"\n")
    return b"".join(out)
