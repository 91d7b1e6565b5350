"""Drive small device-resident evaluates (M = 1 and 10^4) for an ncu launch
list: `ncu --metrics gpu__time_duration.sum -k regex:k_gather_warp ...`."""
import numpy as np
import torch

import paper_1605_01244_b200 as vfb

rng = np.random.default_rng(1)
box = vfb.DomainBox((0.0, 0.0, 0.0), (1.0, 1.0, 1.0))
c = rng.standard_normal((32, 32, 32)) + 1j * rng.standard_normal((32, 32, 32))
plan = vfb.NufftPlan(vfb.SpectralField(box, c))
for M in (1, 10000):
    pts = torch.as_tensor(rng.uniform(0, 1, (M, 3)), device="cuda")
    for _ in range(210):
        plan.evaluate(pts)
