"""Small driver for ncu: build a plan for a workload and evaluate its points
a few times (device-resident).
Usage: python tools/profile_gather.py c2 [gather_variant] [reps] [cutoff]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import paper_1605_01244_b200 as vfb
from paper_1605_01244_b200 import workloads

name = sys.argv[1] if len(sys.argv) > 1 else "c2"
variant = int(sys.argv[2]) if len(sys.argv) > 2 else 0
reps = int(sys.argv[3]) if len(sys.argv) > 3 else 2
cutoff = int(sys.argv[4]) if len(sys.argv) > 4 else 6
w = workloads.WORKLOADS[name]
dev = torch.device("cuda", 0)
spec = vfb.SpectralField(vfb.DomainBox(*w.box), torch.as_tensor(workloads.coefficients(name)).to(dev))
plan = vfb.NufftPlan(spec, vfb.NufftParams(cutoff=cutoff, eps=0.999))
plan.set_gather(variant)
if name == "c5":
    g = torch.Generator(device=dev)
    g.manual_seed(2005)
    pts = torch.rand((w.npoints, 3), dtype=torch.float64, device=dev, generator=g) - 0.5
else:
    pts = torch.as_tensor(workloads.points(name)).to(dev)
out = torch.empty(pts.shape[0], dtype=torch.complex128, device=dev)
for _ in range(reps):
    plan.evaluate(pts, out=out)
torch.cuda.synchronize()
print("gather_ms", plan.last_timing())
