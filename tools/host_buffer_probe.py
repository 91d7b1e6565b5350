"""Evaluate from pageable numpy arrays (what a reference user passes) vs
pinned host buffers vs device-resident points, c5's plan, several M.
Usage: python tools/host_buffer_probe.py"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import paper_1605_01244_b200 as vfb
from paper_1605_01244_b200 import workloads

dev = torch.device("cuda", 0)
w = workloads.WORKLOADS["c5"]
spec = vfb.SpectralField(vfb.DomainBox(*w.box), torch.as_tensor(workloads.coefficients("c5")).to(dev))
plan = vfb.NufftPlan(spec)
rng = np.random.default_rng(3)
for M in (1 << 20, 1 << 23, 1 << 26, 1 << 28):
    pts = rng.uniform(-0.5, 0.5, (M, 3))
    pin_p = torch.empty((M, 3), dtype=torch.float64, pin_memory=True)
    pin_p.copy_(torch.as_tensor(pts))
    pin_o = torch.empty(M, dtype=torch.complex128, pin_memory=True)
    dpts = torch.as_tensor(pts, device=dev)
    res = {}
    reuse = np.empty(M, dtype=np.complex128)
    reuse[:] = 0
    for name, call in (("pageable (fresh out)", lambda: plan.evaluate(pts)),
                       ("pageable (reused out)", lambda: plan.evaluate(pts, out=reuse)),
                       ("pinned in/out", lambda: plan.evaluate(pin_p.numpy(), out=pin_o.numpy())),
                       ("device", lambda: plan.evaluate(dpts))):
        call()
        torch.cuda.synchronize()
        t = time.perf_counter()
        for _ in range(3):
            call()
        torch.cuda.synchronize()
        res[name] = (time.perf_counter() - t) / 3 * 1e3
    print(f"M=2^{M.bit_length() - 1}: " + ", ".join(f"{k} {v:.1f} ms" for k, v in res.items()), flush=True)
