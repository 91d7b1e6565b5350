"""Steady-state timing of eval_direct (K6, exact NDFT) on the c2 / c3 coefficients."""
import sys, time
sys.path.insert(0, '/root/repo')
import numpy as np, torch
import paper_1605_01244_b200 as vfb
from paper_1605_01244_b200 import workloads
for name, M in (("c2", 10000), ("c3", 2000)):
    w = workloads.WORKLOADS[name]
    spec = vfb.SpectralField(vfb.DomainBox(*w.box), workloads.coefficients(name))
    pts = workloads.points(name)[:M]
    vfb.eval_direct(spec, pts)
    torch.cuda.synchronize(); t = time.perf_counter()
    for _ in range(3):
        out = vfb.eval_direct(spec, pts)
    torch.cuda.synchronize(); dt = (time.perf_counter() - t) / 3
    terms = M * np.prod(w.modes)
    print(name, M, 'points', round(dt*1e3, 1), 'ms', '%.3e terms/s' % (terms / dt), flush=True)
