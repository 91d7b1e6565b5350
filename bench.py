#!/usr/bin/env python
"""3D NFFT trafo throughput (points/s, fp64 complex) on B200, with its FP64
roofline fraction and the reference CPU path timed beside it.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--workload c5]
    python bench.py --impl reference ...      # CPU reference arm (oracle port)

A "step" is one `NufftPlan.evaluate` over the workload's points (all ranks
together), i.e. validate + map + bin-sort + gather on a built plan — the
reference's own plan/evaluate split (nufft.py:190-196).  The plan (deconvolve,
pad, 3D FFT) is built once per rank and reported separately.

* ``value``   — points/s with points and results resident in HBM;
* ``e2e``     — the same through the public API with pinned HOST buffers, H2D of
                the points and D2H of the results inside the timed region;
* ``roofline``— the gather kernel's algorithmic FP64 rate (2[(2m+1)^3+(2m+1)^2
                +(2m+1)] real FMA = 9516 flop per point at m=6) over its CUDA-event time, against the
                DFMA peak measured on this device by vfn_bench_fp64_peak;
* ``cpu_baseline`` — the oracle port of the reference (oracle/nfft_oracle.py,
                numpy, fork-sharded over all host cores) on a bounded sample.

Multi-GPU (torchrun): rank 0 builds the coefficients and NCCL-broadcasts them
(the path's one exchange); every rank builds its own replicated plan and
evaluates its share of ONE workload-sized point set (strong scaling, the
BASELINE config-5 definition); ``--scaling weak`` gives every rank its own
full workload-sized block instead.  At N=1 both are the same run.
"""

from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import threading
import time

import numpy as np

REPO = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, REPO)

from paper_1605_01244_b200 import workloads  # noqa: E402

METRIC = "3D NFFT trafo points/sec (fp64 complex)"
SIGMA, CUTOFF = 2.0, 6


def flop_per_point(m: int) -> int:
    """Algorithmic work of the gather per point: (2m+1)^3 + (2m+1)^2 + (2m+1)
    complex-by-real multiply-adds (nufft.py:269-271), 2 real FMA = 4 flop each."""
    w = 2 * m + 1
    return 4 * (w ** 3 + w ** 2 + w)


def parse():
    p = argparse.ArgumentParser()
    p.add_argument("--gpus", type=int, default=1)
    p.add_argument("--steps", type=int, default=5)
    p.add_argument("--warmup", type=int, default=3)
    p.add_argument("--impl", choices=["ours", "reference"], default="ours")
    p.add_argument("--workload", choices=["c1", "c2", "c3", "c4", "c5", "tube"], default="c5")
    p.add_argument("--cpu-seconds", type=float, default=12.0)
    p.add_argument("--no-cpu-baseline", action="store_true")
    p.add_argument("--gather", type=int, default=0, help="0 auto, 1 simple, 2 box/DMMA")
    p.add_argument("--scaling", choices=["weak", "strong"], default="strong",
                   help="strong (default, BASELINE config 5): one point set split across the ranks; "
                        "weak: every rank evaluates its own full workload-sized point set")
    p.add_argument("--shard-mode", choices=["keyrange", "block"], default="keyrange",
                   help="strong scaling over N>1 ranks: keyrange (sample sort + all-to-all, default) or "
                        "block (each rank gathers its own input-order block)")
    p.add_argument("--values", choices=["p2p", "nccl"], default="p2p",
                   help="sharded evaluate: values stored by the gather into their owners' buffers over NVLink "
                        "(p2p, default) or returned by an NCCL all-to-all")
    p.add_argument("--cutoff", type=int, default=6,
                   help="window half-width m (BASELINE's metric is quoted at the default 6)")
    return p.parse_args()


def workload_config(name: str, n_gpus: int, scaling: str = "weak") -> dict:
    w = workloads.WORKLOADS[name]
    per_gpu = w.npoints if scaling == "weak" else -(-w.npoints // n_gpus)
    return {
        "workload": f"{name}: N={w.modes[0]}^3 complex128 coefficients, M={w.npoints} "
        f"{'Gaussian-cloud' if w.kind == 'cluster' else 'uniform'} points on "
        f"{list(w.box[0])}..{list(w.box[1])}, sigma={SIGMA}, m={CUTOFF}",
        "modes": list(w.modes),
        "points": w.npoints * (n_gpus if scaling == "weak" else 1),
        "points_per_gpu": per_gpu,
        "sigma": SIGMA,
        "m": CUTOFF,
        "parallelism": (f"{n_gpus} GPU(s), each evaluating its own {w.npoints}-point block (weak scaling); "
                        if scaling == "weak" else f"{w.npoints} points split over {n_gpus} GPU(s); ")
        + "coefficients NCCL-broadcast from rank 0, oversampled grid replicated",
        "l2_flush": "none needed: per-step inputs (points) exceed the 126 MB L2"
        if w.npoints * 24 > 2 * 126e6
        else "inputs smaller than L2 (warm-L2 number)",
    }


# ---------------------------------------------------------------- CPU side


_G = {}


def _cpu_worker(args):
    lo, hi, deadline = args
    from oracle import nfft_oracle as O

    g = _G
    pts = g["pts"][lo:hi]
    outs = []
    done = 0
    chunk = 2048
    while done < len(pts) and time.perf_counter() < deadline:
        part = pts[done : done + chunk]
        outs.append(O.gather_eval(g["grid"], g["n"], CUTOFF, g["beta"], part, g["a"], g["b"]))
        done += len(part)
    return lo, done, (np.concatenate(outs) if outs else np.empty(0, np.complex128))


def cpu_port_run(name: str, coeffs: np.ndarray, seconds: float, sample_cap: int = 8_000_000):
    """The reference algorithm (oracle port) fork-sharded over every host core
    (SURVEY 8d mode B): plan once, then each worker gathers a contiguous slice
    of a sample of the workload's points until `seconds` run out."""
    import multiprocessing as mp

    from oracle import nfft_oracle as O

    w = workloads.WORKLOADS[name]
    a, b = w.box
    cores = len(os.sched_getaffinity(0))
    t0 = time.perf_counter()
    grid, n, beta = O.oversampled_grid(coeffs, a, b, SIGMA, CUTOFF)
    plan_s = time.perf_counter() - t0
    budget = int(min(sample_cap, max(cores * 3e4 * seconds, 20000)))
    pts = cpu_sample_points(name, budget)
    _G.update(grid=grid, n=n, beta=beta, a=a, b=b, pts=pts)
    bounds = np.linspace(0, len(pts), cores + 1).astype(int)
    ctx = mp.get_context("fork")
    t1 = time.perf_counter()
    deadline = t1 + seconds
    with ctx.Pool(cores) as pool:
        res = pool.map(_cpu_worker, [(bounds[i], bounds[i + 1], deadline) for i in range(cores)])
    elapsed = time.perf_counter() - t1
    count = sum(r[1] for r in res)
    idx = np.concatenate([np.arange(r[0], r[0] + r[1]) for r in res])
    vals = np.concatenate([r[2] for r in res])
    _G.clear()
    return {
        "value": count / elapsed,
        "points": count,
        "seconds": elapsed,
        "cores": cores,
        "plan_s": plan_s,
        "sample_points": pts[idx],
        "sample_values": vals,
    }


def cpu_sample_points(name: str, count: int) -> np.ndarray:
    w = workloads.WORKLOADS[name]
    if w.kind == "cluster":
        return workloads.points(name, count)
    rng = np.random.default_rng(4000 + int(name[1:]))
    return rng.uniform(-0.5, 0.5, (count, 3))


def cpu_model() -> str:
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


# ---------------------------------------------------------------- clocks


class ClockSampler:
    FIELDS = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap,power.draw")

    def __init__(self, index: int):
        self.lines = []
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(index), f"--query-gpu={self.FIELDS}",
                 "--format=csv,noheader,nounits", "-lms", "100"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.thread = threading.Thread(target=self._read, daemon=True)
            self.thread.start()
            # nvidia-smi's start-up (NVML init) stalls CUDA calls of this
            # process: wait for its first sample before the timed region
            t0 = time.perf_counter()
            while not self.lines and time.perf_counter() - t0 < 3.0:
                time.sleep(0.01)
        except OSError:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def stop(self) -> dict:
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        time.sleep(0.25)
        self.proc.terminate()
        self.proc.wait()
        sm, mx, reasons, power = [], [], set(), []
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for line in self.lines:
            parts = [p.strip() for p in line.split(",")]
            if len(parts) < 7:
                continue
            try:
                sm.append(float(parts[0]))
                mx.append(float(parts[1]))
                power.append(float(parts[6]))
            except ValueError:
                continue
            for nm, v in zip(names, parts[2:6]):
                if v.lower().startswith("active"):
                    reasons.add(nm)
        return {
            "sm_mhz": float(np.median(sm)) if sm else None,
            "sm_max_mhz": max(mx) if mx else None,
            "reasons": sorted(reasons),
            "samples": len(sm),
            "power_w_max": max(power) if power else None,
        }


# ---------------------------------------------------------------- GPU side


def dist_setup(args):
    import torch
    import torch.distributed as dist

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world > 1:
        # VFN_DIST_BACKEND=gloo + fewer GPUs than ranks: plumbing check of the
        # torchrun path on a 1-GPU box (ranks share a device; timings meaningless)
        backend = os.environ.get("VFN_DIST_BACKEND", "nccl")
        local = local % max(1, torch.cuda.device_count()) if backend != "nccl" else local
        torch.cuda.set_device(local)
        if backend == "nccl":
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        else:
            dist.init_process_group(backend)
    else:
        torch.cuda.set_device(0)
    return world, rank, local


def run_ours(args):
    import torch
    import torch.distributed as dist

    import paper_1605_01244_b200 as vfb
    from paper_1605_01244_b200 import _lib
    from paper_1605_01244_b200.parallel import broadcast_coefficients, shard_range

    name = args.workload
    w = workloads.WORKLOADS[name]
    world, rank, local = dist_setup(args)
    dev = torch.device("cuda", local)

    def barrier():
        if world > 1:
            dist.barrier()

    def max_over_ranks(x: float) -> float:
        if world == 1:
            return x
        t = torch.tensor([x], dtype=torch.float64, device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    # CPU baseline first (rank 0, N=1 only), before this process touches CUDA
    coeffs_host = workloads.coefficients(name) if rank == 0 else None
    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        cpu = cpu_port_run(name, coeffs_host, args.cpu_seconds)

    # coefficients: rank 0 -> all ranks over NCCL (the one exchange per plan)
    if rank == 0:
        coeffs_dev = torch.as_tensor(coeffs_host).to(dev)
    else:
        coeffs_dev = torch.empty(w.modes, dtype=torch.complex128, device=dev)
    coeffs_dev = broadcast_coefficients(coeffs_dev, src=0, group=None if world > 1 else False)
    spec = vfb.SpectralField(vfb.DomainBox(*w.box), coeffs_dev)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    plan = vfb.NufftPlan(spec, vfb.NufftParams(SIGMA, CUTOFF))
    torch.cuda.synchronize()
    plan_first_ms = max_over_ranks((time.perf_counter() - t0) * 1e3)
    # steady state: a second plan for the same field (cuFFT plan cached, the
    # first plan's grid recycled through the device pool)
    del plan
    t0 = time.perf_counter()
    plan = vfb.NufftPlan(spec, vfb.NufftParams(SIGMA, CUTOFF))
    torch.cuda.synchronize()
    plan_ms = max_over_ranks((time.perf_counter() - t0) * 1e3)
    plan_breakdown = plan.build_timing()
    if args.gather:
        plan.set_gather(args.gather)

    # this rank's block of points, resident in HBM: a 1/world block of ONE
    # point set (strong; the same global set at every world size) or a whole
    # workload-sized set per rank (weak)
    from paper_1605_01244_b200.parallel import ShardStats, evaluate_sharded

    lo, hi = shard_range(w.npoints, world, rank) if args.scaling == "strong" else (0, w.npoints)
    M = hi - lo
    if args.scaling == "strong" or world == 1:
        pts = workloads.device_points(name, lo, hi, dev)
    elif name == "c5":
        gen = torch.Generator(device=dev)
        gen.manual_seed(2005 + 7919 * rank)
        pts = torch.rand((M, 3), dtype=torch.float64, device=dev, generator=gen) - 0.5
    else:
        pts = torch.as_tensor(workloads.points(name)[lo:hi]).to(dev)
    out = torch.empty(M, dtype=torch.complex128, device=dev)
    stream = torch.cuda.current_stream(dev)
    # strong scaling over several ranks: key-range sharding (sample sort +
    # NCCL all-to-all of points and values, parallel.evaluate_sharded)
    sharded = world > 1 and args.scaling == "strong"
    stats = ShardStats() if sharded else None

    def step(p, o):
        if sharded:
            return evaluate_sharded(plan, p, out=o, stats=stats, mode=args.shard_mode, values=args.values)
        return plan.evaluate(p, out=o)

    # ---- device-resident timing
    for _ in range(args.warmup):
        step(pts, out)
    torch.cuda.synchronize()
    clocks = ClockSampler(dev.index if dev.index is not None else 0)
    barrier()
    torch.cuda.synchronize()
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    gather_ms = []
    e0.record(stream)
    for _ in range(args.steps):
        step(pts, out)
        gather_ms.append(plan.last_timing()[0])
    e1.record(stream)
    torch.cuda.synchronize()
    barrier()
    clk = clocks.stop()
    step_ms = max_over_ranks(e0.elapsed_time(e1) / args.steps)
    M_gather = stats.received if sharded else M  # points of this rank's gather launch
    if M_gather < (1 << 20) and M_gather > plan_warp_max() and not sharded:
        # graph-replayed evaluates report the whole graph's time; the
        # roofline needs the gather kernel alone: a few eager evaluates
        plan.set_graphs(False)
        gather_ms = []
        for _ in range(3):
            plan.evaluate(pts, out=out)
            gather_ms.append(plan.last_timing()[0])
        plan.set_graphs(True)
    g_mean = float(np.mean(gather_ms))
    g_ms = max_over_ranks(g_mean)
    shard_info = None
    if sharded:
        shard_info = {
            "mode": args.shard_mode,
            "exchange": "p2p: the partition kernel stores each point into its destination's IPC-shared receive "
                        "buffer and the gather's epilogue stores each value into its owner's output buffer, both "
                        "over NVLink (no all-to-all on the data path)" if args.values == "p2p"
                        else "nccl: all_to_all_single of the points and of the values, then a reorder",
            "partition_count_ms": max_over_ranks(stats.partition_ms),
            "points_exchange_ms": max_over_ranks(stats.exchange_in_ms),
            "evaluate_ms": max_over_ranks(stats.evaluate_ms),
            "values_return_ms": max_over_ranks(stats.exchange_out_ms),
            "output_copy_ms": max_over_ranks(stats.restore_ms),
            "decide_ms": max_over_ranks(stats.decide_ms),
            "received_max": int(max_over_ranks(float(stats.received))),
            "received_min": int(-max_over_ranks(-float(stats.received))),
            "note": "last timed step, CUDA events on each rank, max over ranks",
        }

    # ---- end to end through the public API: pinned host in, pinned host out
    # (pageable if the host cannot pin 40 B per point for every rank)
    try:
        pts_host = torch.empty((M, 3), dtype=torch.float64, pin_memory=True)
        out_host = torch.empty(M, dtype=torch.complex128, pin_memory=True)
        pinned = True
    except RuntimeError:
        pts_host = torch.empty((M, 3), dtype=torch.float64)
        out_host = torch.empty(M, dtype=torch.complex128)
        pinned = False
    pts_host.copy_(pts)
    pts_np, out_np = pts_host.numpy(), out_host.numpy()

    def e2e_step():
        if sharded:  # this rank's block: H2D, sharded evaluate, D2H
            pts.copy_(pts_host, non_blocking=True)
            r = evaluate_sharded(plan, pts, out=out, mode=args.shard_mode, values=args.values)
            out_host.copy_(r, non_blocking=True)
            torch.cuda.current_stream(dev).synchronize()
        else:
            plan.evaluate(pts_np, out=out_np)  # returns after the D2H has landed

    for _ in range(2):  # untimed: the first host-buffer calls size the plan's staging buffers
        e2e_step()
    torch.cuda.synchronize()
    barrier()
    e2e_ms = []
    for _ in range(max(2, min(args.steps, 5))):
        t0 = time.perf_counter()
        e2e_step()
        e2e_ms.append((time.perf_counter() - t0) * 1e3)
    e2e_step_ms = max_over_ranks(float(np.mean(e2e_ms)))
    dev_vals = out.cpu().numpy()
    same = bool(np.array_equal(out_np, dev_vals)) if not sharded else None
    sharded_equal = None
    if sharded:
        # bitwise against ONE unsharded evaluate of the whole set on this rank's plan
        plan.set_gather(0)
        plan.set_box(0)
        whole = workloads.device_points(name, 0, w.npoints, dev)
        ref = plan.evaluate(whole)[lo:hi].cpu().numpy()
        del whole
        sharded_equal = bool(np.array_equal(dev_vals, ref)) and bool(np.array_equal(out_np, ref))
        sharded_equal = bool(max_over_ranks(0.0 if sharded_equal else 1.0) == 0.0)
        same = sharded_equal

    # ---- roofline of the gather kernel (per rank, max-time rank)
    peak = None
    if rank == 0:
        import ctypes

        tf, mhz = ctypes.c_double(), ctypes.c_double()
        _lib.check(_lib.load().vfn_bench_fp64_peak(dev.index or 0, 0.5, ctypes.byref(tf), ctypes.byref(mhz)))
        peak = tf.value

    total_points = w.npoints * (world if args.scaling == "weak" else 1)
    value = total_points / (step_ms * 1e-3)
    fl = float(flop_per_point(CUTOFF))
    # the slowest rank's gather rate (its own launch's points and time); a
    # collective, so every rank computes it before rank 0 reports
    achieved = -max_over_ranks(-(fl * M_gather / (g_mean * 1e-3) / 1e12)) if world > 1 else \
        fl * M_gather / (g_ms * 1e-3) / 1e12
    if rank != 0:
        return
    result = {
        "metric": METRIC,
        "value": value,
        "unit": "points/s",
        "n_gpus": world,
        "steps": args.steps,
        "warmup": args.warmup,
        "ms_per_step": step_ms,
        "higher_is_better": True,
        "scaling": args.scaling,
        "vs_baseline": None,
        "dtype": "f64",
        "data": "synthetic, seeded (SURVEY 8d recipe); no dataset exists for this benchmark",
        "config": workload_config(name, world, args.scaling),
        "e2e": {
            "value": total_points / (e2e_step_ms * 1e-3),
            "unit": "points/s",
            "h2d_bytes_per_step": int(total_points * 24),
            "d2h_bytes_per_step": int(total_points * 16),
            "ms_per_step": e2e_step_ms,
            "steps_ms": [round(x, 3) for x in e2e_ms],  # this rank's timed host-buffer evaluates (the mean is reported)
            "matches_device_result_bitwise": same,
            "pinned_host_buffers": pinned,
        },
        "roofline": {
            "bound": "tensor",
            "pipe": "FP64: DMMA (mma.sync m8n8k4 f64) and DFMA share one datapath; peak = measured DFMA rate",
            "kernel": "gather (K4)",
            "achieved": achieved,
            "peak": peak,
            "unit": "TFLOP/s",
            "frac": achieved / peak if peak else None,
            "traffic": None,
            "algorithmic": f"{int(fl)} flop/point = 2*((2m+1)^3+(2m+1)^2+(2m+1)) real FMA at m={CUTOFF}; "
            f"{M_gather} points per launch",
            "peak_source": "measured DFMA peak on this device (vfn_bench_fp64_peak, 0.5 s); "
            "MEASURED_PEAKS.json has no FP64 figure",
            "gather_ms": g_ms,
            "gather_share_of_step": g_ms / step_ms,
        },
        "plan_build_ms": plan_ms,
        "plan_build": {"first_ms": plan_first_ms, "steady_ms": plan_ms,
                       "steady_breakdown_ms": plan_breakdown},
        "gpu_launches": None,
        "clocks": clk,
    }
    tr = profiled_traffic(name)
    ng = 1
    for v in plan._n:
        ng *= v
    result["roofline"]["algorithmic_bytes"] = 40 * M_gather + 16 * ng  # points in/out + grid once
    if shard_info is not None:
        shard_info["sharded_equals_unsharded_bitwise"] = sharded_equal
        result["sharding"] = shard_info
    if tr is not None and world == 1 and CUTOFF == 6:  # the committed capture is m = 6
        result["roofline"]["traffic"] = tr[0]
        result["roofline"]["traffic_source"] = tr[1]
    result["gpu_launches"] = (launches_per_step(plan, M_gather) + (5 if sharded else 0)) * args.steps
    if cpu is not None:
        sp = cpu["sample_points"]
        gpu_vals = plan.evaluate(sp)
        ref = cpu["sample_values"]
        err_l2 = float(np.linalg.norm(gpu_vals - ref) / np.linalg.norm(ref))
        err_inf = float(np.abs(gpu_vals - ref).max() / np.abs(ref).max())
        result["cpu_baseline"] = {
            "value": cpu["value"],
            "unit": "points/s",
            "cores": cpu["cores"],
            "kind": "port",
            "sample": f"{cpu['points']} points of the {name} distribution in {cpu['seconds']:.1f} s, "
            f"oracle/nfft_oracle.py (numpy restatement of nufft.py:244-272) fork-sharded over "
            f"{cpu['cores']} cores after a {cpu['plan_s']:.2f} s plan build; CPU {cpu_model()}",
        }
        result["parity_vs_cpu"] = {"points": int(len(ref)), "rel_l2": err_l2, "rel_linf": err_inf}
    print(json.dumps(result), flush=True)


def profiled_traffic(name: str):
    """dram__bytes_read.sum + dram__bytes_write.sum of the gather kernel from the
    committed ncu --set full capture for this workload (profiles/), or None."""
    t = None
    for rnd in ("r02", "r01"):  # the newest capture of the current kernel first
        try:
            t = json.load(open(os.path.join(REPO, "profiles", rnd, "traffic.json")))[name]
            break
        except (OSError, KeyError, ValueError):
            continue
    if t is None:
        return None
    return t["dram_bytes_read"] + t["dram_bytes_write"], t["source"]


def run_rect(args):
    """Config 4: rectilinear 128^3 -> 256^3 tanh-clustered tensor grid through
    eval_rectilinear (three exact separable passes).  Points = grid points."""
    import torch

    import paper_1605_01244_b200 as vfb

    world, rank, local = dist_setup(args)
    if rank != 0:
        return
    dev = torch.device("cuda", local)
    w = workloads.WORKLOADS["c4"]
    coeffs = workloads.coefficients("c4")
    axes = workloads.rect_axes(256)
    box = vfb.DomainBox(*w.box)
    cpu = None
    if not args.no_cpu_baseline:
        from oracle import nfft_oracle as O

        t0 = time.perf_counter()
        ref = O.rectilinear(coeffs, box.a, box.b, axes)
        cpu = {"seconds": time.perf_counter() - t0, "ref": ref}
    spec_d = vfb.SpectralField(box, torch.as_tensor(coeffs).to(dev))
    for _ in range(args.warmup):
        out = vfb.eval_rectilinear(spec_d, axes)
    torch.cuda.synchronize()
    stream = torch.cuda.current_stream(dev)
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    clocks = ClockSampler(local)
    e0.record(stream)
    for _ in range(args.steps):
        out = vfb.eval_rectilinear(spec_d, axes)
    e1.record(stream)
    torch.cuda.synchronize()
    clk = clocks.stop()
    step_ms = e0.elapsed_time(e1) / args.steps
    npts = 256 ** 3
    # e2e through the public API: pinned host coefficients in, pinned host
    # values out (the download overlaps the last pass slab by slab), warmed
    # up like the device loop
    c_pin = torch.empty(coeffs.shape, dtype=torch.complex128, pin_memory=True)
    c_pin.copy_(torch.as_tensor(coeffs))
    o_pin = torch.empty((256, 256, 256), dtype=torch.complex128, pin_memory=True)
    spec_h = vfb.SpectralField(box, c_pin.numpy())
    host = o_pin.numpy()
    vfb.eval_rectilinear(spec_h, axes, out=host)
    e2e_runs = []
    for _ in range(max(2, min(args.steps, 5))):
        t0 = time.perf_counter()
        vfb.eval_rectilinear(spec_h, axes, out=host)
        e2e_runs.append((time.perf_counter() - t0) * 1e3)
    e2e_ms = float(np.mean(e2e_runs))
    N, Mx = 128, 256
    cmacs = N * N * N * Mx + N * N * Mx * Mx + N * Mx * Mx * Mx  # the three passes
    achieved = 8.0 * cmacs / (step_ms * 1e-3) / 1e12
    import ctypes

    from paper_1605_01244_b200 import _lib

    tf, mhz = ctypes.c_double(), ctypes.c_double()
    _lib.check(_lib.load().vfn_bench_fp64_peak(local, 0.5, ctypes.byref(tf), ctypes.byref(mhz)))
    result = {
        "metric": "3D rectilinear-grid evaluation points/sec (fp64 complex)",
        "value": npts / (step_ms * 1e-3),
        "unit": "points/s",
        "n_gpus": 1,
        "steps": args.steps,
        "warmup": args.warmup,
        "ms_per_step": step_ms,
        "higher_is_better": True,
        "scaling": "strong",
        "vs_baseline": None,
        "dtype": "f64",
        "data": "synthetic, seeded (SURVEY 8d recipe)",
        "config": {"workload": "c4: N=128^3 coefficients -> 256^3 tanh-clustered rectilinear grid",
                   "modes": [128, 128, 128], "points": npts},
        "e2e": {"value": npts / (e2e_ms * 1e-3), "unit": "points/s",
                "h2d_bytes_per_step": int(coeffs.nbytes + 3 * 256 * 8), "d2h_bytes_per_step": int(npts * 16),
                "ms_per_step": e2e_ms,
                "matches_device_result_bitwise": bool(np.array_equal(host, out.cpu().numpy()))},
        "roofline": {"bound": "tensor", "pipe": "FP64: DMMA (mma.sync m8n8k4 f64), peak = measured DFMA rate",
                     "kernel": "3 separable passes, hand-written DMMA complex GEMM (vfn_zgemm.cu)", "achieved": achieved,
                     "peak": tf.value, "unit": "TFLOP/s", "frac": achieved / tf.value, "traffic": None,
                     "algorithmic": f"{cmacs} complex MACs = 8 flop each"},
        "gpu_launches": (3 + 2 + 8) * args.steps,  # k_basis per axis, passes 1-2, pass 3 (8 slabs for host output)
        "clocks": clk,
    }
    # the separable 1D-NUFFT pass mode: HBM-bound, one fused
    # kernel per pass; algorithmic bytes = each pass's input + output once
    for _ in range(2):
        fast = vfb.eval_rectilinear(spec_d, axes, mode="nufft")
    torch.cuda.synchronize()
    e0.record(stream)
    for _ in range(args.steps):
        fast = vfb.eval_rectilinear(spec_d, axes, mode="nufft")
    e1.record(stream)
    torch.cuda.synchronize()
    nufft_ms = e0.elapsed_time(e1) / args.steps
    pass_bytes = 16 * (N ** 3 + 2 * N * N * Mx + 2 * N * Mx * Mx + Mx ** 3)
    hbm = measured_hbm_gbs()
    fast_np = fast.cpu().numpy()
    exact_np = out.cpu().numpy()
    result["nufft_mode"] = {
        "value": npts / (nufft_ms * 1e-3), "unit": "points/s", "ms_per_step": nufft_ms,
        "params": "sigma 2, m 6 per pass",
        "rel_l2_vs_exact": float(np.linalg.norm(fast_np - exact_np) / np.linalg.norm(exact_np)),
        "rel_linf_vs_exact": float(np.abs(fast_np - exact_np).max() / np.abs(exact_np).max()),
        "roofline": {"bound": "hbm", "achieved": pass_bytes / (nufft_ms * 1e-3) / 1e9, "peak": hbm,
                     "unit": "GB/s", "frac": pass_bytes / (nufft_ms * 1e-3) / 1e9 / hbm if hbm else None,
                     "traffic": None, "algorithmic": f"{pass_bytes} B: each pass's input and output once",
                     "peak_source": "MEASURED_PEAKS.json hbm_gbs"},
    }
    if cpu is not None:
        ref = cpu["ref"]
        result["nufft_mode"]["rel_linf_vs_cpu"] = float(np.abs(fast_np - ref).max() / np.abs(ref).max())
        result["cpu_baseline"] = {"value": npts / cpu["seconds"], "unit": "points/s",
                                  "cores": len(os.sched_getaffinity(0)), "kind": "port",
                                  "sample": "full c4 through oracle.rectilinear (numpy/BLAS restatement of rectilinear.py:47-64)"}
        result["parity_vs_cpu"] = {
            "points": npts,
            "rel_l2": float(np.linalg.norm(host - ref) / np.linalg.norm(ref)),
            "rel_linf": float(np.abs(host - ref).max() / np.abs(ref).max()),
        }
    print(json.dumps(result), flush=True)


def run_tube(args):
    """tube_eval (tube.py:58-127) on a synthetic two-vortex
    snapshot (64^3 samples on [-8,8)^3, mirrored on all axes -> 128^3
    computational box), thresholds (0.2, 0.05) as the reference's
    acceptance criterion 7.  One step = one whole call: decompose, plan,
    seeds, two refinement passes, compaction and sort, cloud to host."""
    import torch

    import paper_1605_01244_b200 as vfb

    world, rank, local = dist_setup(args)
    if rank != 0:
        return
    dev = torch.device("cuda", local)
    shape = (64, 64, 64)
    box = workloads.VORTEX_BOX
    values = workloads.vortex_pair_field(shape, box)
    mirror = (True, True, True)
    thr = [0.2, 0.05]
    snap = vfb.Snapshot(vfb.DomainBox(*box), values, mirror, 0.0)
    dsnap = vfb.Snapshot(vfb.DomainBox(*box), torch.as_tensor(values, device=dev), mirror, 0.0)
    for _ in range(args.warmup):
        cloud = vfb.tube_eval(dsnap, thr)
    torch.cuda.synchronize()
    clocks = ClockSampler(local)
    t0 = time.perf_counter()
    for _ in range(args.steps):
        cloud = vfb.tube_eval(dsnap, thr)
    torch.cuda.synchronize()
    step_ms = (time.perf_counter() - t0) * 1e3 / args.steps
    clk = clocks.stop()
    host_cloud = vfb.tube_eval(snap, thr)  # untimed: first host-input call (pinned staging set-up)
    e2e_runs = []
    for _ in range(max(2, min(args.steps, 5))):
        t0 = time.perf_counter()
        host_cloud = vfb.tube_eval(snap, thr)
        e2e_runs.append((time.perf_counter() - t0) * 1e3)
    e2e_ms = float(np.mean(e2e_runs))
    result = {
        "metric": "tube_eval wall time (snapshot -> refined low-density cloud)",
        "value": step_ms,
        "unit": "ms",
        "n_gpus": 1,
        "steps": args.steps,
        "warmup": args.warmup,
        "ms_per_step": step_ms,
        "higher_is_better": False,
        "scaling": "strong",
        "vs_baseline": None,
        "dtype": "f64",
        "data": "synthetic two-vortex snapshot (workloads.vortex_pair_field)",
        "config": {"workload": "tube: 64^3 samples on [-8,8)^3, mirror (T,T,T), thresholds (0.2, 0.05), sigma 2, m 6",
                   "cloud_points": len(cloud)},
        "e2e": {"value": e2e_ms, "unit": "ms", "h2d_bytes_per_step": int(values.nbytes),
                "d2h_bytes_per_step": int(len(host_cloud) * (24 + 8 + 8))},
        "roofline": None,
        "gpu_launches": None,
        "clocks": clk,
    }
    if not args.no_cpu_baseline:
        from oracle import nfft_oracle as O

        t0 = time.perf_counter()
        rp, rd, rl = O.tube_eval(values, np.array(box[0]), np.array(box[1]), mirror, thr)
        cpu_s = time.perf_counter() - t0
        result["cpu_baseline"] = {"value": cpu_s * 1e3, "unit": "ms", "cores": len(os.sched_getaffinity(0)),
                                  "kind": "port",
                                  "sample": "one full call of oracle.tube_eval (numpy restatement of tube.py:58-127)"}
        same = rp.shape == host_cloud.points.shape and np.array_equal(rp, host_cloud.points) and \
            np.array_equal(rl, host_cloud.level)
        result["parity_vs_cpu"] = {"points": int(len(rp)), "points_and_levels_identical": bool(same),
                                   "density_rel_linf": float(np.abs(rd - host_cloud.density).max() / np.abs(rd).max())
                                   if same and len(rd) else None}
    print(json.dumps(result), flush=True)


def measured_hbm_gbs():
    """HBM copy bandwidth of this pool's B200s (MEASURED_PEAKS.json), else the
    profiling recipe's fallback."""
    try:
        return float(json.load(open(os.path.join(REPO, "MEASURED_PEAKS.json")))["hbm_gbs"])
    except (OSError, KeyError, ValueError):
        return 6527.5


def plan_warp_max() -> int:
    from paper_1605_01244_b200 import nufft

    return nufft.WARP_MAX_M


def launches_per_step(plan, M: int) -> int:
    """Kernels of ours launched by one evaluate: map+key, the CUB onesweep
    radix sort (1 histogram + one pass per 8 key bits), box offsets and the
    gather (DESIGN.md lists them)."""
    return plan.launch_count(M)


def run_reference(args):
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    name = args.workload
    if name == "tube":
        from oracle import nfft_oracle as O

        box = workloads.VORTEX_BOX
        values = workloads.vortex_pair_field((64, 64, 64), box)
        times = []
        for i in range(args.warmup + args.steps):
            t0 = time.perf_counter()
            O.tube_eval(values, np.array(box[0]), np.array(box[1]), (True, True, True), [0.2, 0.05])
            if i >= args.warmup:
                times.append(time.perf_counter() - t0)
        ms = float(np.mean(times)) * 1e3
        print(json.dumps({
            "metric": "tube_eval wall time (snapshot -> refined low-density cloud)", "value": ms, "unit": "ms",
            "n_gpus": world, "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms,
            "higher_is_better": False, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic two-vortex snapshot (workloads.vortex_pair_field)",
            "config": {"workload": "tube: 64^3 samples on [-8,8)^3, mirror (T,T,T), thresholds (0.2, 0.05), sigma 2, m 6"},
            "impl": "reference",
            "cpu_baseline": {"value": ms, "unit": "ms", "cores": len(os.sched_getaffinity(0)), "kind": "port",
                             "sample": "one full call of oracle.tube_eval per step (numpy restatement of tube.py:58-127)"},
            "e2e": {"value": ms, "unit": "ms", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        }), flush=True)
        return
    coeffs = workloads.coefficients(name)
    if name == "c4":
        from oracle import nfft_oracle as O

        w = workloads.WORKLOADS["c4"]
        axes = workloads.rect_axes(256)
        times = []
        for i in range(args.warmup + args.steps):
            t0 = time.perf_counter()
            O.rectilinear(coeffs, w.box[0], w.box[1], axes)
            if i >= args.warmup:
                times.append(time.perf_counter() - t0)
        value = 256 ** 3 / float(np.mean(times))
        cores = len(os.sched_getaffinity(0))
        print(json.dumps({
            "metric": "3D rectilinear-grid evaluation points/sec (fp64 complex)", "value": value,
            "unit": "points/s", "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": float(np.mean(times)) * 1e3, "higher_is_better": True, "scaling": "strong",
            "vs_baseline": None, "dtype": "f64", "data": "synthetic, seeded (SURVEY 8d recipe)",
            "config": {"workload": "c4: N=128^3 coefficients -> 256^3 tanh-clustered rectilinear grid",
                       "modes": [128, 128, 128], "points": 256 ** 3},
            "impl": "reference",
            "cpu_baseline": {"value": value, "unit": "points/s", "cores": cores, "kind": "port",
                             "sample": "full c4 per step, oracle.rectilinear (numpy + OpenBLAS threads)"},
            "e2e": {"value": value, "unit": "points/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        }), flush=True)
        return
    runs = []
    per_step = max(3.0, args.cpu_seconds / 4)
    for i in range(args.warmup + args.steps):
        r = cpu_port_run(name, coeffs, per_step)
        if i >= args.warmup:
            runs.append(r)
    value = float(np.mean([r["value"] for r in runs]))
    cores = runs[0]["cores"]
    sample = (f"each step: the {name} plan (oracle port, numpy/scipy) then its gather fork-sharded over "
              f"{cores} cores for {per_step:.0f} s (~{int(np.mean([r['points'] for r in runs]))} points); "
              f"CPU {cpu_model()}")
    out = {
        "metric": METRIC,
        "value": value,
        "unit": "points/s",
        "n_gpus": world,
        "steps": args.steps,
        "warmup": args.warmup,
        "ms_per_step": float(np.mean([r["seconds"] for r in runs]) * 1e3),
        "higher_is_better": True,
        "scaling": args.scaling,
        "vs_baseline": None,
        "dtype": "f64",
        "data": "synthetic, seeded (SURVEY 8d recipe)",
        "config": workload_config(name, world, args.scaling),
        "impl": "reference",
        "cpu_baseline": {"value": value, "unit": "points/s", "cores": cores, "kind": "port", "sample": sample},
        "e2e": {"value": value, "unit": "points/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(out), flush=True)


def main():
    global CUTOFF
    args = parse()
    CUTOFF = args.cutoff
    if args.impl == "reference":
        run_reference(args)
    elif args.workload == "c4":
        run_rect(args)
    elif args.workload == "tube":
        run_tube(args)
    else:
        run_ours(args)
    if int(os.environ.get("WORLD_SIZE", "1")) > 1 and args.impl == "ours":
        import torch.distributed as dist

        dist.destroy_process_group()


if __name__ == "__main__":
    main()
