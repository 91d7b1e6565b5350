import sys, time, numpy as np, torch
sys.path.insert(0, '.')
import paper_1605_01244_b200 as vfb
from paper_1605_01244_b200 import workloads
torch.cuda.set_device(0)
w = workloads.WORKLOADS["c4"]
spec = vfb.SpectralField(vfb.DomainBox(*w.box), torch.as_tensor(workloads.coefficients("c4"), device="cuda"))
axes = workloads.rect_axes(256)
for _ in range(3): vfb.eval_rectilinear(spec, axes, mode="nufft")
torch.cuda.synchronize()
for mode in ("nufft",):
    ts = []
    for _ in range(10):
        t0 = time.perf_counter(); vfb.eval_rectilinear(spec, axes, mode=mode); torch.cuda.synchronize(); ts.append(time.perf_counter() - t0)
    print(mode, "wall ms", np.median(ts) * 1e3)
