"""Small end-to-end cases for compute-sanitizer (every kernel family once):
m=6 TMA/DMMA gather at both box widths, generic DMMA gather (m=3), thread-per-
point gather (m=13), rectilinear, direct NDFT, map/bin."""
import os
import sys
import warnings

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import paper_1605_01244_b200 as vfb

rng = np.random.default_rng(0)
box = vfb.DomainBox((-1.5, 0.25, 2.0), (2.5, 1.25, 7.0))
coeffs = rng.standard_normal((16, 24, 12)) + 1j * rng.standard_normal((16, 24, 12))
spec = vfb.SpectralField(box, coeffs)
pts = rng.uniform(box.a, box.b, (20000, 3))
for m in (6, 3, 13):
    with warnings.catch_warnings():
        warnings.simplefilter("ignore")
        plan = vfb.NufftPlan(spec, vfb.NufftParams(cutoff=m, eps=0.999))
    for bxy in ((1, 2) if m == 6 else (0,)):
        plan.set_box(bxy)
        out = plan.evaluate(pts)
        print("m", m, "box", bxy, "ok", np.isfinite(out).all())
    keys, perm = plan.bin(pts[:1000])
print("direct", np.isfinite(vfb.eval_direct(spec, pts[:50])).all())
print("rect", vfb.eval_rectilinear(spec, [np.linspace(-1.5, 2.4, 7), np.linspace(0.25, 1.2, 5), np.linspace(2, 6.9, 9)]).shape)
print("torus", vfb.map_to_torus(pts[:10], box).shape)
torch.cuda.synchronize()
