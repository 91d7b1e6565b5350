"""e2e (pinned host in/out) time of one c5 evaluate for several pipeline
chunk sizes (VFN_PIPE_CHUNK), device-resident step for reference.
Usage: python tools/e2e_chunks.py [chunk ...]"""
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
for c in sys.argv[1:] or ["134217728", "67108864", "33554432"]:
    os.environ["VFN_PIPE_CHUNK"] = c
    plan.evaluate(pn, out=on)
    ts = []
    for _ in range(3):
        t = time.perf_counter()
        plan.evaluate(pn, out=on)
        ts.append((time.perf_counter() - t) * 1e3)
    print("chunk", c, "e2e", [round(x, 1) for x in ts], "gather/total ms", plan.last_timing(), flush=True)
