"""Throughput of the file-format row on the GPU box: native
readers/writers (libvfnfft.so) vs the Python the reference executes for the
same files (csv.writer of repr() values / csv.reader + float array,
fields.py:146-174; numpy frombuffer of the SFS1 payload, snapshots.py:50-72),
and the eval-points command end to end.  Prints one JSON object.

    python tools/bench_io.py [--points 4194304] [--grid 256]
"""

import argparse
import csv
import io
import json
import os
import sys
import tempfile
import time

import numpy as np

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, REPO)

import torch  # noqa: E402

from paper_1605_01244_b200 import DomainBox, Snapshot, formats, pipeline  # noqa: E402


def py_csv_write(points, columns) -> str:
    # the loop of fields.py:146-157
    buf = io.StringIO(newline="")
    w = csv.writer(buf)
    w.writerow(["x1", "x2", "x3"] + list(columns))
    for i in range(points.shape[0]):
        w.writerow([repr(v.item()) for v in points[i]] + [repr(c[i].item()) for c in columns.values()])
    return buf.getvalue()


def py_csv_read(text: str):
    # fields.py:160-174
    reader = csv.reader(io.StringIO(text, newline=""))
    header = next(reader)
    data = np.array([row for row in reader if row], dtype=float)
    return {name.strip(): data[:, i] for i, name in enumerate(header)}


def timed(fn, reps=3):
    best = float("inf")
    out = None
    for _ in range(reps):
        torch.cuda.synchronize()
        t = time.perf_counter()
        out = fn()
        torch.cuda.synchronize()
        best = min(best, time.perf_counter() - t)
    return best, out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--points", type=int, default=1 << 22)
    ap.add_argument("--grid", type=int, default=256)
    ap.add_argument("--py-rows", type=int, default=200000, help="rows timed for the Python restatement")
    args = ap.parse_args()
    d = tempfile.mkdtemp(dir="/tmp")
    res = {"cpu_threads": os.cpu_count()}

    # snapshot file -> HBM
    n = args.grid
    g = torch.Generator(device="cuda").manual_seed(1)
    v = torch.randn((n, n, n // 2), dtype=torch.complex128, device="cuda", generator=g)
    snap = Snapshot(DomainBox((-1.0, -1.0, -1.0), (1.0, 1.0, 1.0)), v, (True, True, False), 1.0)
    path = os.path.join(d, "s.sfs")
    t_w, _ = timed(lambda: formats.write_snapshot(path, snap))
    t_r, back = timed(lambda: formats.read_snapshot(path, device=0))
    assert torch.equal(back.values, v)
    nbytes = v.numel() * 16
    raw = open(path, "rb").read()
    t_py, _ = timed(lambda: np.frombuffer(raw, dtype="<c16", offset=79).astype(np.complex128), reps=2)
    res["snapshot"] = {"bytes": nbytes, "write_GBps_from_hbm": nbytes / t_w / 1e9,
                       "read_GBps_to_hbm": nbytes / t_r / 1e9,
                       "python_unpack_GBps_host_only": nbytes / t_py / 1e9}

    # points CSV
    M = args.points
    rng = np.random.default_rng(2)
    pts = rng.uniform(-1, 1, (M, 3))
    vals = rng.standard_normal(M) + 1j * rng.standard_normal(M)
    cols = {"re": vals.real, "im": vals.imag, "rho": vals.real**2 + vals.imag**2}
    cpath = os.path.join(d, "p.csv")
    t_cw, _ = timed(lambda: formats.write_points_csv(cpath, pts, cols))
    size = os.path.getsize(cpath)
    t_cr, dev_pts = timed(lambda: formats.read_points(cpath, device=0))
    assert np.array_equal(dev_pts.cpu().numpy(), pts)
    k = min(args.py_rows, M)
    t_pw, text = timed(lambda: py_csv_write(pts[:k], {c: a[:k] for c, a in cols.items()}), reps=1)
    t_pr, _ = timed(lambda: py_csv_read(text), reps=1)
    res["points_csv"] = {"rows": M, "bytes": size, "native_write_rows_per_s": M / t_cw,
                         "native_read_to_hbm_rows_per_s": M / t_cr,
                         "python_write_rows_per_s": k / t_pw, "python_read_rows_per_s": k / t_pr,
                         "python_sample_rows": k}

    # eval-points command: snapshot + CSV in, CSV out (cli.py:108-125)
    small = Snapshot(DomainBox((-1.0, -1.0, -1.0), (1.0, 1.0, 1.0)),
                     torch.randn((64, 64, 32), dtype=torch.complex128, device="cuda", generator=g),
                     (False, False, True), 0.5)
    spath = os.path.join(d, "small.sfs")
    formats.write_snapshot(spath, small)
    formats.write_points_csv(cpath, pts * 0.999, {})
    opath = os.path.join(d, "o.csv")
    t_e, cnt = timed(lambda: pipeline.eval_points(spath, cpath, opath), reps=2)
    res["eval_points_command"] = {"points": cnt, "snapshot": [64, 64, 32], "seconds": t_e,
                                  "points_per_s": cnt / t_e}
    print(json.dumps(res))


if __name__ == "__main__":
    main()
