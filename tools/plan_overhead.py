"""Per-call host overhead of small plans: one-shot eval_nufft (the reference's
acceptance criterion 3 shape: 64^3 coefficients, 1000 points), plan build
breakdown (vfn_plan_build_timing) and evaluate time.

    python tools/plan_overhead.py
"""
import json
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    import torch

    import paper_1605_01244_b200 as vfb

    torch.cuda.set_device(0)
    rng = np.random.default_rng(2024)
    dom = vfb.DomainBox((-20.0,) * 3, (60.0,) * 3)
    out = {}
    for shape in [(16, 16, 16), (64, 64, 64), (128, 128, 128)]:
        coeffs = (rng.standard_normal(shape) + 1j * rng.standard_normal(shape)) / np.sqrt(2)
        spec = vfb.SpectralField(dom, coeffs)
        pts = np.stack([rng.uniform(dom.a[d], dom.b[d], 1000) for d in range(3)], axis=1)
        vfb.eval_nufft(spec, pts)
        ts, bs, es, ds = [], [], [], []
        for _ in range(10):
            t0 = time.perf_counter()
            plan = vfb.NufftPlan(spec)
            t1 = time.perf_counter()
            plan.evaluate(pts)
            t2 = time.perf_counter()
            bs.append(plan.build_timing())
            del plan
            t3 = time.perf_counter()
            ts.append((t1 - t0) * 1e3)
            es.append((t2 - t1) * 1e3)
            ds.append((t3 - t2) * 1e3)
        t0 = time.perf_counter()
        for _ in range(10):
            vfb.eval_direct(spec, pts)
        direct = (time.perf_counter() - t0) * 100
        out[str(shape)] = {"plan_ms": float(np.median(ts)), "evaluate_1000_ms": float(np.median(es)),
                           "destroy_ms": float(np.median(ds)), "direct_1000_ms": direct,
                           "breakdown_ms": {k: float(np.median([b[k] for b in bs])) for k in bs[0]}}
    print(json.dumps(out, indent=1))


if __name__ == "__main__":
    main()
