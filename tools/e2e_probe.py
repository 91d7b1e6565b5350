"""Time the host-buffer (pinned) evaluate for a workload at several chunk sizes."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_1605_01244_b200 as vfb
from paper_1605_01244_b200 import workloads
name = sys.argv[1] if len(sys.argv) > 1 else "c5"
w = workloads.WORKLOADS[name]
dev = torch.device("cuda", 0)
plan = vfb.NufftPlan(vfb.SpectralField(vfb.DomainBox(*w.box), torch.as_tensor(workloads.coefficients(name)).to(dev)))
g = torch.Generator(device=dev); g.manual_seed(2005)
pts = torch.rand((w.npoints, 3), dtype=torch.float64, device=dev, generator=g) - 0.5
ph = torch.empty((w.npoints, 3), dtype=torch.float64, pin_memory=True); ph.copy_(pts)
oh = torch.empty(w.npoints, dtype=torch.complex128, pin_memory=True)
od = torch.empty(w.npoints, dtype=torch.complex128, device=dev)
plan.evaluate(pts, out=od); torch.cuda.synchronize()
t0 = time.perf_counter(); plan.evaluate(pts, out=od); torch.cuda.synchronize(); print("device", (time.perf_counter()-t0)*1e3, "ms")
t0 = time.perf_counter(); oh.copy_(od); torch.cuda.synchronize(); print("D2H only", (time.perf_counter()-t0)*1e3)
t0 = time.perf_counter(); pts.copy_(ph); torch.cuda.synchronize(); print("H2D only", (time.perf_counter()-t0)*1e3)
for ch in [w.npoints * 2, 1 << 27, 1 << 26, 1 << 25, 1 << 24]:
    os.environ["VFN_PIPE_CHUNK"] = str(ch)
    plan.evaluate(ph.numpy(), out=oh.numpy())
    t0 = time.perf_counter(); plan.evaluate(ph.numpy(), out=oh.numpy()); dt = time.perf_counter() - t0
    print("chunk", ch, "%.1f ms" % (dt * 1e3), "same" if np.array_equal(oh.numpy(), od.cpu().numpy()) else "DIFF")
