"""Device cost of evaluating the first f * M rows of config 5 (what one chunk
of the pipelined host-buffer evaluate computes), per fraction f and box
width, against f times the whole call: how much the lower point density of a
chunk inflates its gather.

    python tools/chunk_cost_probe.py [--cutoff 6] > gpurun_out/chunk_cost.json
"""

from __future__ import annotations

import argparse
import json
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--cutoff", type=int, default=6)
    ap.add_argument("--reps", type=int, default=3)
    ap.add_argument("--fractions", default="0.06,0.1,0.15,0.22,0.28,0.44,0.5,1.0")
    args = ap.parse_args()
    import torch

    import paper_1605_01244_b200 as vfb
    from paper_1605_01244_b200 import workloads
    from paper_1605_01244_b200.parallel import density_sample_rows

    dev = torch.device("cuda", 0)
    torch.cuda.set_device(dev)
    w = workloads.WORKLOADS["c5"]
    spec = vfb.SpectralField(vfb.DomainBox(*w.box), torch.as_tensor(workloads.coefficients("c5")).to(dev))
    plan = vfb.NufftPlan(spec, vfb.NufftParams(2.0, args.cutoff))
    M = w.npoints
    pts = workloads.device_points("c5", 0, M, dev)
    stride, cnt = density_sample_rows(M, plan.DENSITY_SAMPLE)
    variant, box = plan.decide(M, pts[torch.arange(cnt, device=dev) * stride])

    def run(n):
        seg = pts[:n]
        tot, gat = [], []
        for _ in range(args.reps + 1):
            plan.evaluate(seg)
            torch.cuda.synchronize()
            g, t = plan.last_timing()
            tot.append(t)
            gat.append(g)
        return float(np.median(tot[1:])), float(np.median(gat[1:]))

    rows = []
    full = {}
    for b in (box, 3 - box):
        plan.pin(variant, b)
        full[b] = run(M)
        for f in [float(x) for x in args.fractions.split(",")]:
            n = int(f * M)
            t, g = run(n)
            rows.append({"box": b, "f": f, "points": n, "device_ms": t, "gather_ms": g,
                         "vs_share": t / (f * full[b][0]), "gather_vs_share": g / (f * full[b][1])})
    print(json.dumps({"cutoff": args.cutoff, "whole_call_box": box, "variant": variant,
                      "full_ms": {str(b): v for b, v in full.items()}, "chunks": rows}, indent=1))


if __name__ == "__main__":
    main()
