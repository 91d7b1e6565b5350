"""Per-call time of small evaluates on the unbinned warp-per-point gather
(variant 3) vs the binned tensor-core path (variant 2, CUDA-graph replay),
device-resident points, c1's plan (32^3 modes, 64^3 grid) and c2's (64^3
modes, 128^3 grid), optionally c3 / c5's: where the automatic switch
(VFN_WARP_MAX_M) belongs.  Usage: python tools/small_m_sweep.py [c1 c2 c3 c5]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import paper_1605_01244_b200 as vfb
from paper_1605_01244_b200 import workloads

dev = torch.device("cuda", 0)
SIZES = {"c1": (1000, 4000, 10000, 16384, 32768, 65536, 131072, 262144),
         "c2": (1000, 4000, 10000, 16384, 32768, 65536, 131072, 262144),
         "c3": (32768, 131072, 262144, 524288),
         "c5": (32768, 131072, 524288, 2097152)}
for name in sys.argv[1:] or ("c1", "c2"):
    w = workloads.WORKLOADS[name]
    spec = vfb.SpectralField(vfb.DomainBox(*w.box), torch.as_tensor(workloads.coefficients(name)).to(dev))
    plan = vfb.NufftPlan(spec)
    g = torch.Generator(device=dev)
    g.manual_seed(7)
    lo, hi = (torch.tensor(v, dtype=torch.float64, device=dev) for v in w.box)
    for M in SIZES[name]:
        pts = lo + (hi - lo) * torch.rand((M, 3), dtype=torch.float64, device=dev, generator=g)
        out = torch.empty(M, dtype=torch.complex128, device=dev)
        row = []
        for variant in (3, 2):
            plan.set_gather(variant)
            for _ in range(3):
                plan.evaluate(pts, out=out)
            torch.cuda.synchronize()
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record()
            for _ in range(20):
                plan.evaluate(pts, out=out)
            b.record()
            torch.cuda.synchronize()
            row.append(a.elapsed_time(b) / 20 * 1e3)
        print(f"{name} M={M}: warp {row[0]:.1f} us, binned {row[1]:.1f} us", flush=True)
