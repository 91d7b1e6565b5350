"""PCIe and per-chunk evaluate costs behind the pipelined host path (c5):
H2D / D2H GB/s from pinned memory alone and concurrently, and the
device-resident evaluate time of the first f*M points for several f.
Usage: python tools/pcie_probe.py"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import paper_1605_01244_b200 as vfb
from paper_1605_01244_b200 import workloads


def timed(fn, reps=3):
    fn()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(reps):
        fn()
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) / reps


dev = torch.device("cuda", 0)
w = workloads.WORKLOADS["c5"]
M = w.npoints
hp = torch.empty((M, 3), dtype=torch.float64, pin_memory=True)
ho = torch.empty(M, dtype=torch.complex128, pin_memory=True)
dp = torch.empty((M, 3), dtype=torch.float64, device=dev)
do = torch.empty(M, dtype=torch.complex128, device=dev)
t_in = timed(lambda: dp.copy_(hp, non_blocking=True))
t_out = timed(lambda: ho.copy_(do, non_blocking=True))
s2 = torch.cuda.Stream()


def both():
    with torch.cuda.stream(s2):
        ho.copy_(do, non_blocking=True)
    dp.copy_(hp, non_blocking=True)
    torch.cuda.current_stream().wait_stream(s2)


t_both = timed(both)
print(f"H2D {hp.nbytes / t_in / 1e6:.1f} GB/s ({t_in:.1f} ms), D2H {ho.nbytes / t_out / 1e6:.1f} GB/s "
      f"({t_out:.1f} ms), both concurrently {t_both:.1f} ms", flush=True)
spec = vfb.SpectralField(vfb.DomainBox(*w.box), torch.as_tensor(workloads.coefficients("c5")).to(dev))
plan = vfb.NufftPlan(spec)
g = torch.Generator(device=dev)
g.manual_seed(2005)
dp.copy_(torch.rand((M, 3), dtype=torch.float64, device=dev, generator=g) - 0.5)
for f in (0.06, 0.12, 0.25, 0.38, 0.5, 1.0):
    n = int(f * M)
    t = timed(lambda: plan.evaluate(dp[:n], out=do[:n]))
    print(f"f={f}: evaluate {t:.1f} ms (gather {plan.last_timing()[0]:.1f} ms), {t / f:.1f} ms per full set",
          flush=True)
