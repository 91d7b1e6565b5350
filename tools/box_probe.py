"""Device time of one c5 evaluate (2^28 points, device-resident) per box
width at a given cutoff, and the box the automatic choice takes.

    python tools/box_probe.py --cutoff 8
"""
import argparse
import json
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--cutoff", type=int, default=8)
    ap.add_argument("--reps", type=int, default=3)
    args = ap.parse_args()
    import torch

    import paper_1605_01244_b200 as vfb
    from paper_1605_01244_b200 import workloads

    dev = torch.device("cuda", 0)
    torch.cuda.set_device(dev)
    w = workloads.WORKLOADS["c5"]
    spec = vfb.SpectralField(vfb.DomainBox(*w.box), torch.as_tensor(workloads.coefficients("c5")).to(dev))
    plan = vfb.NufftPlan(spec, vfb.NufftParams(2.0, args.cutoff, eps=1e-16))
    pts = workloads.device_points("c5", 0, w.npoints, dev)
    res = {"cutoff": args.cutoff}
    vals = {}
    for b in (0, 1, 2):
        plan.set_box(b)
        out = None
        ts = []
        for _ in range(args.reps + 1):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            out = plan.evaluate(pts)
            e1.record()
            torch.cuda.synchronize()
            ts.append((e0.elapsed_time(e1), plan.last_timing()[0]))
        vals[b] = out[:1 << 20].cpu().numpy()
        res[f"box{b or 'auto'}"] = {"evaluate_ms": float(np.median([t[0] for t in ts[1:]])),
                                   "gather_ms": float(np.median([t[1] for t in ts[1:]])),
                                   "geometry": str(plan.geometry(w.npoints))}
    res["box1_vs_box2_max_rel"] = float(np.abs(vals[1] - vals[2]).max() / np.abs(vals[1]).max())
    print(json.dumps(res, indent=1))


if __name__ == "__main__":
    main()
