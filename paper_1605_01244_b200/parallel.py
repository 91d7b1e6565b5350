"""Multi-GPU plumbing for the trafo: one process per GPU,
torch.distributed for the control plane.

* The coefficients (N1 N2 N3 complex128) are broadcast once per plan from
  rank 0 over NCCL (NVLink/NVSwitch on an 8xB200 box) — the path's only
  exchange step.  Every rank then builds its own replicated plan.
* Points are partitioned into contiguous 1/P blocks in input order
  (`shard_range`); each rank evaluates its block with no data-path
  collective.  Results are bitwise independent of P because a point's value
  depends only on the (identical) replicated grid and the point itself.
* `gather_results` optionally assembles the full output on one rank.
"""

from __future__ import annotations


def shard_range(total: int, world: int, rank: int) -> tuple[int, int]:
    """Contiguous block [lo, hi) of `total` items owned by `rank` (sizes differ by <= 1)."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError("bad world/rank")
    base, extra = divmod(int(total), int(world))
    lo = rank * base + min(rank, extra)
    return lo, lo + base + (1 if rank < extra else 0)


def broadcast_coefficients(coeffs, src: int = 0, group=None):
    """Broadcast a coefficient tensor from `src` to every rank (in place).
    `group=False` means single process: return the tensor unchanged."""
    if group is False:
        return coeffs
    import torch.distributed as dist

    if not dist.is_initialized() or dist.get_world_size(group) == 1:
        return coeffs
    dist.broadcast(coeffs, src=src, group=group)
    return coeffs


def gather_results(local, total: int, dst: int = 0, group=None):
    """Concatenate every rank's shard result (1-D tensors of complex128 or
    any dtype, contiguous shards in rank order) on `dst`; other ranks get None."""
    import torch
    import torch.distributed as dist

    world = dist.get_world_size(group)
    rank = dist.get_rank(group)
    sizes = [shard_range(total, world, r) for r in range(world)]
    width = max(hi - lo for lo, hi in sizes)
    real = torch.view_as_real(local) if local.is_complex() else local
    pad = torch.zeros((width,) + tuple(real.shape[1:]), dtype=real.dtype, device=real.device)
    pad[: real.shape[0]] = real
    bufs = [torch.empty_like(pad) for _ in range(world)] if rank == dst else None
    dist.gather(pad, bufs, dst=dst, group=group)
    if rank != dst:
        return None
    parts = [b[: hi - lo] for b, (lo, hi) in zip(bufs, sizes)]
    full = torch.cat(parts)
    return torch.view_as_complex(full) if local.is_complex() else full


def evaluate_sharded(plan, points, rank: int, world: int, out=None):
    """Evaluate this rank's contiguous block of `points` (global array) with `plan`."""
    lo, hi = shard_range(points.shape[0], world, rank)
    return plan.evaluate(points[lo:hi], out=out)


def eval_rectilinear_sharded(spec, coords, rank: int, world: int, evaluator=None):
    """This rank's slab of a rectilinear evaluation: the
    (replicated, broadcast) coefficients are contracted for the rank's
    contiguous block of axis-1 coordinates only, so each rank produces
    output rows [lo, hi) of the (M1, M2, M3) grid and no collective is
    needed beyond the coefficient broadcast; `gather_results` on the
    flattened slabs (or writing them in place) assembles the grid.  Values
    agree with the unsharded call to rounding (the last pass's GEMM shape
    changes with the slab).  `evaluator` defaults to `eval_rectilinear`."""
    if evaluator is None:
        from .rectilinear import eval_rectilinear as evaluator
    lo, hi = shard_range(len(coords[0]), world, rank)
    return evaluator(spec, [coords[0][lo:hi], coords[1], coords[2]])
