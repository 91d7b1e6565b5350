"""One-GPU proxy of config-5 strong scaling.

On one B200: the whole 2^28-point set is split into P key ranges exactly as
P ranks would split it (parallel.evaluate_sharded: sampled partition keys ->
splitters -> vfn_plan_partition), and each range is evaluated on its own as
the owning rank would (pinned to the unsharded call's decisions).  The same
is done with P input-order blocks (what each rank would gather without the
exchange).  Reports per-range evaluate and gather times against 1/P of the
unsharded call, checks that the ranges' values are bitwise the unsharded
values, and projects the P-GPU step = slowest range + partition + the two
all-to-alls at an assumed NVLink rate.

    python tools/shard_proxy.py [--ranks 8] [--reps 3] > profiles/r02/shard_proxy_c5.json
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
    ap.add_argument("--ranks", type=int, default=8)
    ap.add_argument("--reps", type=int, default=3)
    ap.add_argument("--workload", default="c5")
    ap.add_argument("--nvlink-gbs", type=float, default=700.0,
                    help="assumed per-GPU all-to-all rate (GB/s) for the projection")
    args = ap.parse_args()
    import torch

    import paper_1605_01244_b200 as vfb
    from paper_1605_01244_b200 import workloads
    from paper_1605_01244_b200.parallel import density_sample_rows, shard_range, splitters_from_samples

    dev = torch.device("cuda", 0)
    torch.cuda.set_device(dev)
    w = workloads.WORKLOADS[args.workload]
    spec = vfb.SpectralField(vfb.DomainBox(*w.box), torch.as_tensor(workloads.coefficients(args.workload)).to(dev))
    plan = vfb.NufftPlan(spec, vfb.NufftParams(2.0, 6))
    M, P = w.npoints, args.ranks
    pts = workloads.device_points(args.workload, 0, M, dev)

    def timed(fn, reps):
        ts, gs = [], []
        for _ in range(reps):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            r = fn()
            e1.record()
            torch.cuda.synchronize()
            ts.append(e0.elapsed_time(e1))
            gs.append(plan.last_timing()[0])
        return r, float(np.median(ts)), float(np.median(gs))

    full, full_ms, full_g = timed(lambda: plan.evaluate(pts), args.reps)
    full = full.clone()
    stride, cnt = density_sample_rows(M, plan.DENSITY_SAMPLE)
    sample = pts[torch.arange(cnt, device=dev) * stride]
    variant, box = plan.decide(M, sample)
    plan.pin(variant, box)
    # key ranges: splitters from the same per-rank samples evaluate_sharded draws
    kstride = max(1, M // ((1 << 18) * P))
    keys = torch.cat([plan.part_keys(pts[slice(*shard_range(M, P, r))], kstride, shard_range(M, P, r)[0])
                      for r in range(P)])
    split = splitters_from_samples(keys, P)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    send, counts, pos = plan.partition(pts, split, 0)
    e1.record()
    torch.cuda.synchronize()
    part_ms = e0.elapsed_time(e1)  # one partition of all M (a rank partitions M / P)
    offs = np.concatenate([[0], np.cumsum(counts)])
    ranges, blocks = [], []
    ok = True
    for r in range(P):
        seg = send[offs[r]:offs[r + 1]]
        vals, ms, g = timed(lambda: plan.evaluate(seg), args.reps)
        ranges.append({"points": int(counts[r]), "evaluate_ms": ms, "gather_ms": g})
        back = full[torch.nonzero((pos >= offs[r]) & (pos < offs[r + 1])).flatten()]
        ok &= bool(torch.equal(vals, back))
        lo, hi = shard_range(M, P, r)
        blk = pts[lo:hi]
        vb, ms_b, g_b = timed(lambda: plan.evaluate(blk), args.reps)
        ok &= bool(torch.equal(vb, full[lo:hi]))
        blocks.append({"points": hi - lo, "evaluate_ms": ms_b, "gather_ms": g_b})
    slow_k = max(x["evaluate_ms"] for x in ranges)
    slow_b = max(x["evaluate_ms"] for x in blocks)
    a2a_bytes = (M // P) * (P - 1) / P * (24 + 16)  # points out + values back per rank
    a2a_ms = a2a_bytes / (args.nvlink_gbs * 1e9) * 1e3
    proj = slow_k + part_ms / P + a2a_ms
    res = {
        "workload": args.workload, "points": M, "ranks": P, "box": box, "variant": variant,
        "unsharded": {"evaluate_ms": full_ms, "gather_ms": full_g},
        "ideal_share_ms": full_ms / P, "ideal_gather_share_ms": full_g / P,
        "key_ranges": ranges, "input_order_blocks": blocks,
        "slowest_key_range_gather_vs_share": max(x["gather_ms"] for x in ranges) / (full_g / P),
        "slowest_block_gather_vs_share": max(x["gather_ms"] for x in blocks) / (full_g / P),
        "partition_all_points_ms": part_ms,
        "projected": {
            "all_to_all_ms_assumed": a2a_ms, "nvlink_gbs_assumed": args.nvlink_gbs,
            "keyrange_step_ms": proj, "keyrange_efficiency": (full_ms / P) / proj,
            "block_step_ms": slow_b, "block_efficiency": (full_ms / P) / slow_b,
        },
        "values_bitwise_equal_unsharded": ok,
    }
    print(json.dumps(res, indent=1))


if __name__ == "__main__":
    main()
