"""Per-call host overhead of a tiny device-resident evaluate, split into the
Python wrapper and the native vfn_plan_eval call (wall clock, M = 1).

    python tools/call_overhead.py
"""
import ctypes
import time

import numpy as np
import torch

import paper_1605_01244_b200 as vfb
from paper_1605_01244_b200 import _lib, nufft


def per_call(fn, n=3000):
    for _ in range(200):
        fn()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(n):
        fn()
    torch.cuda.synchronize()
    return (time.perf_counter() - t0) / n * 1e6


def main():
    rng = np.random.default_rng(1)
    box = vfb.DomainBox((0.0, 0.0, 0.0), (1.0, 1.0, 1.0))
    c = rng.standard_normal((32, 32, 32)) + 1j * rng.standard_normal((32, 32, 32))
    plan = vfb.NufftPlan(vfb.SpectralField(box, c))
    for M in (1, 1000, 10000):
        pts = torch.as_tensor(rng.uniform(0, 1, (M, 3)), device="cuda")
        out = torch.empty(M, dtype=torch.complex128, device="cuda")
        lib = _lib.load()
        h, pp, po = plan._handle, pts.data_ptr(), out.data_ptr()
        stream = nufft._stream_of(plan.device)
        bad = ctypes.c_int64(-1)
        rows = {
            "plan.evaluate(pts)": lambda: plan.evaluate(pts),
            "plan.evaluate(pts, out=out)": lambda: plan.evaluate(pts, out=out),
            "native vfn_plan_eval only": lambda: lib.vfn_plan_eval(h, pp, M, po, 1, ctypes.byref(bad), stream),
            "_points_arg": lambda: nufft._points_arg(pts),
            "torch.empty": lambda: torch.empty(M, dtype=torch.complex128, device="cuda"),
            "_stream_of": lambda: nufft._stream_of(plan.device),
            "torch.cuda.is_available": lambda: torch.cuda.is_available(),
            "current_stream(dev).cuda_stream": lambda: torch.cuda.current_stream(plan.device).cuda_stream,
            "_C._cuda_getCurrentRawStream": lambda: torch._C._cuda_getCurrentRawStream(plan.device),
            "_lib.load": lambda: _lib.load(),
        }
        x = torch.zeros(1, device="cuda")
        s = torch.cuda.current_stream()
        rows["floor: 1 torch launch + stream sync"] = lambda: (x.add_(1), s.synchronize())
        rows["floor: 2 torch launches + stream sync"] = lambda: (x.add_(1), x.add_(1), s.synchronize())
        for k, f in rows.items():
            print(f"M={M:6d} {k:40s} {per_call(f):8.2f} us")
        plan.evaluate(pts)
        g, tot = plan.last_timing()
        print(f"M={M:6d} device events: gather {g * 1e3:.2f} us, ev0->ev3 {tot * 1e3:.2f} us")


if __name__ == "__main__":
    main()
