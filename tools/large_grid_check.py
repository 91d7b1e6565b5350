"""Largest-size check on one B200: N = 512^3 coefficients (oversampled grid
1024^3, 17 GB), 2^26 uniform points, values of a 256-point subset against
the device NDFT (exact sum), plus the same subset evaluated on its own
(bitwise equal: batch composition does not change a point's value).

    python tools/large_grid_check.py [--modes 512] [--points 67108864] > gpurun_out/large_grid.json
"""
from __future__ import annotations

import argparse
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--modes", type=int, default=512)
    ap.add_argument("--points", type=int, default=1 << 26)
    ap.add_argument("--check", type=int, default=256)
    a = ap.parse_args()
    import torch

    import paper_1605_01244_b200 as vfb

    dev = torch.device("cuda", 0)
    torch.cuda.set_device(dev)
    N = a.modes
    g = torch.Generator(device=dev)
    g.manual_seed(7)
    k = torch.arange(-N // 2, N // 2, device=dev, dtype=torch.float64)
    decay = torch.exp(-(k * k) / (16.0 * N))
    coeffs = torch.randn((N, N, N, 2), dtype=torch.float64, device=dev, generator=g)
    coeffs *= (decay[:, None, None] * decay[None, :, None] * decay[None, None, :])[..., None]
    coeffs = torch.view_as_complex(coeffs)
    box = vfb.DomainBox((-0.5, -0.5, -0.5), (0.5, 0.5, 0.5))
    spec = vfb.SpectralField(box, coeffs)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    plan = vfb.NufftPlan(spec)
    torch.cuda.synchronize()
    t_plan = time.perf_counter() - t0
    pts = torch.rand((a.points, 3), dtype=torch.float64, device=dev, generator=g) - 0.5
    out = plan.evaluate(pts)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    out = plan.evaluate(pts)
    torch.cuda.synchronize()
    t_eval = time.perf_counter() - t0
    gather_ms, total_ms = plan.last_timing()
    idx = torch.linspace(0, a.points - 1, a.check, device=dev, dtype=torch.float64).long()
    sub = pts[idx].contiguous()
    ref = vfb.eval_direct(spec, sub)
    got = out[idx]
    err = float((got - ref).abs().max() / ref.abs().max())
    alone = plan.evaluate(torch.cat([sub, pts[: 1 << 20]]).contiguous())[: a.check]
    print(json.dumps({
        "modes": [N, N, N], "grid": list(plan._n), "points": a.points,
        "plan_build_s": t_plan, "evaluate_s": t_eval, "gather_ms": gather_ms, "device_ms": total_ms,
        "points_per_s": a.points / t_eval,
        "rel_linf_vs_direct": err, "checked_points": a.check,
        "subset_in_other_batch_bitwise_equal": bool(torch.equal(alone, got)),
        "hbm_allocated_gb": torch.cuda.max_memory_allocated() / 1e9,
    }))


if __name__ == "__main__":
    main()
