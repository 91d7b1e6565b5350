import sys, numpy as np, torch
sys.path.insert(0, '.')
import paper_1605_01244_b200 as vfb
from paper_1605_01244_b200 import workloads
torch.cuda.set_device(0)
for N, M in [(64, 1 << 20), (128, 1 << 20), (256, 1 << 20), (256, 1 << 24)]:
    rng = np.random.default_rng(5)
    coeffs = rng.standard_normal((N,) * 3) + 1j * rng.standard_normal((N,) * 3)
    box = vfb.DomainBox((-0.5,) * 3, (0.5,) * 3)
    plan = vfb.NufftPlan(vfb.SpectralField(box, torch.as_tensor(coeffs, device='cuda')), vfb.NufftParams(2.0, 8, eps=1e-16))
    pts = torch.rand((M, 3), dtype=torch.float64, device='cuda', generator=torch.Generator('cuda').manual_seed(3)) - 0.5
    try:
        v = plan.evaluate(pts)
        torch.cuda.synchronize()
        print(N, M, 'ok', plan.geometry(M), flush=True)
    except Exception as e:
        print(N, M, 'FAIL', e, flush=True)
        break
