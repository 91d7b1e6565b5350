"""e2e (pinned host in/out) time of one c5 evaluate for several pipeline
schedules, device-resident step for reference.  Each argument is a chunk
size (VFN_PIPE_CHUNK) or a comma list of chunk fractions (VFN_PIPE_SPLIT).
Usage: python tools/e2e_chunks.py [134217728 | 0.2,0.6,0.2 ...]"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import paper_1605_01244_b200 as vfb
from paper_1605_01244_b200 import workloads

w = workloads.WORKLOADS["c5"]
dev = torch.device("cuda", 0)
spec = vfb.SpectralField(vfb.DomainBox(*w.box), torch.as_tensor(workloads.coefficients("c5")).to(dev))
plan = vfb.NufftPlan(spec)
g = torch.Generator(device=dev)
g.manual_seed(2005)
pts = torch.rand((w.npoints, 3), dtype=torch.float64, device=dev, generator=g) - 0.5
ph = torch.empty((w.npoints, 3), dtype=torch.float64, pin_memory=True)
ph.copy_(pts)
oh = torch.empty(w.npoints, dtype=torch.complex128, pin_memory=True)
pn, on = ph.numpy(), oh.numpy()
out = torch.empty(w.npoints, dtype=torch.complex128, device=dev)
for _ in range(2):
    plan.evaluate(pts, out=out)
torch.cuda.synchronize()
t = time.perf_counter()
for _ in range(3):
    plan.evaluate(pts, out=out)
torch.cuda.synchronize()
print("device", round((time.perf_counter() - t) / 3 * 1e3, 1), "ms", flush=True)
ref = None
for c in sys.argv[1:] or ["134217728", "67108864", "33554432"]:
    os.environ.pop("VFN_PIPE_CHUNK", None)
    os.environ.pop("VFN_PIPE_SPLIT", None)
    os.environ["VFN_PIPE_SPLIT" if "," in c else "VFN_PIPE_CHUNK"] = c
    plan.evaluate(pn, out=on)
    ts = []
    for _ in range(3):
        t = time.perf_counter()
        plan.evaluate(pn, out=on)
        ts.append((time.perf_counter() - t) * 1e3)
    if ref is None:
        ref = on.copy()
    print("schedule", c, "e2e", [round(x, 1) for x in ts], "bitwise", bool(np.array_equal(on, ref)), flush=True)
