"""Multi-GPU trafo: one process per GPU, torch.distributed (NCCL
over NVLink/NVSwitch) for the collectives, the device steps in libvfnfft.

Plan build.  The coefficients (N1 N2 N3 complex128) are broadcast once from
rank 0 (`broadcast_coefficients`); every rank builds the same replicated
oversampled grid.

Evaluate (`evaluate_sharded`).  Every rank holds a block of ONE point set in
input order and gets the values of its own block back, in order.  The
reference allows evaluating disjoint point subsets on a shared immutable
plan; how the subsets are formed is this layer's choice:

* ``mode="keyrange"`` (default): a distributed sample sort by the partition
  key (tile of the nearest oversampled cell, then global row;
  include/vfnfft.h vfn_plan_partition).  Splitters come from an all-gather
  of key samples, the points move to the rank owning their key range with
  one all-to-all, each rank evaluates a spatially compact range of whole
  tiles at full point density, and the values come back with a second
  all-to-all and are put back in input order on the device — or, by
  default, the gathers store every value straight into its owner's
  IPC-shared output buffer over NVLink (the return exchange fused into the
  gather's epilogue, `vfn_plan_eval_to_peers`).  Input-order
  blocks would instead leave every rank with a sparse sample of the whole
  box: each grid tile staged for 1/P of its points (profiles/r01/
  pcie_chunks.md: a 1/8 block costs 2.3x its share of the gather).
* ``mode="block"``: each rank evaluates its own block (no exchange).

Determinism.  Before evaluating, the ranks pin the gather decisions the
unsharded call would take (`vfn_plan_decide`: warp-per-point vs binned
from the global M, the box width from the density sample rows
j * (M // 16384) of the whole set, assembled from the ranks' blocks).  A
point's value then depends only on the point, the replicated grid and those
pinned settings, so results are bitwise independent of the rank count P
and of the mode, and equal to one `NufftPlan.evaluate` of the whole set.

`gather_results` assembles per-rank outputs on one rank when wanted.
"""

from __future__ import annotations

from dataclasses import dataclass, field


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


# ---------------------------------------------------------------- collectives


class _Comm:
    """The few collectives the sharded evaluate needs, over a process group
    (or a single process).  NCCL takes CUDA tensors directly; other backends
    (gloo: CPU tests, ranks sharing one GPU) go through host copies."""

    def __init__(self, group=None):
        import torch.distributed as dist

        self.dist = dist if dist.is_available() and dist.is_initialized() else None
        self.group = group
        self.world = self.dist.get_world_size(group) if self.dist else 1
        self.rank = self.dist.get_rank(group) if self.dist else 0
        self.nccl = bool(self.dist) and self.dist.get_backend(group) == "nccl"

    def _io(self, t):
        return t if self.nccl or not t.is_cuda else t.cpu()

    def all_gather_ints(self, values: list[int]) -> list[list[int]]:
        import torch

        if self.world == 1:
            return [list(values)]
        dev = torch.device("cuda", torch.cuda.current_device()) if self.nccl else torch.device("cpu")
        mine = torch.tensor(values, dtype=torch.int64, device=dev)
        parts = [torch.empty_like(mine) for _ in range(self.world)]
        self.dist.all_gather(parts, mine, group=self.group)
        return [p.tolist() for p in parts]

    def all_gather_rows(self, t, counts: list[int]):
        """Concatenate every rank's (counts[r], ...) tensor in rank order."""
        import torch

        if self.world == 1:
            return t
        width = max(max(counts), 1)
        src = self._io(t)
        pad = torch.zeros((width,) + tuple(src.shape[1:]), dtype=src.dtype, device=src.device)
        pad[: src.shape[0]] = src
        parts = [torch.empty_like(pad) for _ in range(self.world)]
        self.dist.all_gather(parts, pad, group=self.group)
        out = torch.cat([p[:c] for p, c in zip(parts, counts)])
        return out.to(t.device)

    def barrier(self):
        if self.world > 1:
            self.dist.barrier(group=self.group)

    def all_reduce_min(self, v: int) -> int:
        import torch

        if self.world == 1:
            return v
        dev = torch.device("cuda", torch.cuda.current_device()) if self.nccl else torch.device("cpu")
        x = torch.tensor([v], dtype=torch.int64, device=dev)
        self.dist.all_reduce(x, op=self.dist.ReduceOp.MIN, group=self.group)
        return int(x.item())

    def all_reduce_sum(self, t):
        if self.world == 1:
            return t
        x = self._io(t).clone()
        self.dist.all_reduce(x, group=self.group)
        return x.to(t.device)

    def all_to_all(self, send, send_counts: list[int], recv_counts: list[int]):
        """Rows of `send` (destination-major, send_counts[d] rows for rank d)
        to their ranks; returns the received rows, source-major."""
        import torch

        if self.world == 1:
            return send
        src = self._io(send)
        recv = torch.empty((sum(recv_counts),) + tuple(src.shape[1:]), dtype=src.dtype, device=src.device)
        self.dist.all_to_all_single(recv, src, output_split_sizes=list(recv_counts),
                                    input_split_sizes=list(send_counts), group=self.group)
        return recv.to(send.device)


# ---------------------------------------------------------------- sharded evaluate


@dataclass
class ShardStats:
    """Where a sharded evaluate's time went on this rank (ms, CUDA events on
    the current stream; host-side syncs of the exchange included)."""

    decide_ms: float = 0.0
    partition_ms: float = 0.0
    exchange_in_ms: float = 0.0
    evaluate_ms: float = 0.0
    exchange_out_ms: float = 0.0
    restore_ms: float = 0.0
    sent: list = field(default_factory=list)
    received: int = 0

    @property
    def exchange_ms(self) -> float:
        return self.exchange_in_ms + self.exchange_out_ms


def density_sample_rows(total: int, sample: int) -> tuple[int, int]:
    """(stride, count) of the density sample rows j * stride, j < count."""
    return max(1, total // sample), sample


def splitters_from_samples(keys, world: int):
    """world - 1 ascending splitters at the count quantiles of the sorted
    key sample (int64 tensor): rank r owns keys in [s[r-1], s[r])."""
    import torch

    ks, _ = torch.sort(keys)
    n = int(ks.shape[0])
    if world <= 1 or n == 0:
        return ks[:0]
    idx = torch.tensor([(r * n) // world for r in range(1, world)], dtype=torch.int64, device=ks.device)
    return ks[idx].contiguous()


def _gather_values(values, pos):
    if values.is_cuda:
        from .nufft import gather_values

        return gather_values(values, pos)
    return values[pos.long()]  # host tensors: the CPU plumbing tests only


class _PeerBuffers:
    """Per rank, two slots of IPC-shared device buffers (allocated by the
    library with cudaMalloc, exported as CUDA IPC handles and mapped by every
    other rank; ranks in the same process — tests/simcomm.py threads — use
    each other's pointers directly):

    * ``out`` — the values of this rank's own block; every rank's gather
      stores into it over NVLink (vfn_plan_eval_to_peers);
    * ``in``  — the points (24 B) and their rows in their owners' blocks
      (4 B) that the other ranks' partition kernels scatter into it over
      NVLink (vfn_plan_partition_scatter_peers).

    The slots alternate between calls on a slot number the ranks agree on:
    a rank still reading call k's buffers is never written by a call k + 1
    kernel (that uses the other slot), and call k + 2 cannot start before
    every rank has passed call k + 1's collectives."""

    KINDS = ("out", "in")

    def __init__(self, device: int):
        self.device = device
        self.cap = {"out": 0, "in": 0}
        self.local = {"out": [None, None], "in": [None, None]}  # (address, handle bytes) per slot
        self.opened = {}  # (rank, handle) -> mapped address
        self.calls = 0

    def _alloc(self, kind: str, cap: int, elem: int):
        import ctypes

        from . import _lib

        lib = _lib.load()
        for k in range(2):
            if self.local[kind][k] is not None:
                lib.vfn_ipc_free(self.device, self.local[kind][k][0])
            ptr = ctypes.c_void_p()
            h = (ctypes.c_ubyte * 64)()
            _lib.check(lib.vfn_ipc_alloc(self.device, elem * cap, ctypes.byref(ptr), h))
            self.local[kind][k] = (ptr.value, bytes(h))
        self.cap[kind] = cap

    def prepare(self, comm, m_out: int, m_in: int = 0):
        """Collective: this rank's slots hold m_out values and m_in received
        points; returns (slot, {kind: local address}, {kind: addresses by rank})."""
        import ctypes
        import os

        import numpy as np

        from . import _lib

        good = 1
        try:
            for kind, m, elem in (("out", m_out, 16), ("in", m_in, 28)):
                if m > self.cap[kind] or self.local[kind][0] is None:
                    self._alloc(kind, max(m + m // 4, 1024), elem)
        except Exception:  # allocation failed: still join the collective below
            good = 0
        mine = [os.getpid(), self.calls, self.cap["in"] if good else 0, good]
        for kind in self.KINDS:
            for k in range(2):
                entry = self.local[kind][k] if good else None
                mine.append(entry[0] if entry else 0)
                mine.extend(int(x) for x in np.frombuffer(entry[1], dtype=np.int64)) if entry else mine.extend([0] * 8)
        allv = comm.all_gather_ints(mine)
        if min(row[3] for row in allv) == 0:
            raise RuntimeError("a rank could not allocate its peer buffers")
        pid = os.getpid()
        # one slot for the whole call, agreed by all ranks (their call counts
        # may differ: a plan can join later calls of another rank set)
        c = max(row[1] for row in allv)
        slot = c & 1
        self.calls = c + 1
        addrs = {kind: [0] * comm.world for kind in self.KINDS}
        caps_in = [row[2] for row in allv]
        for r, row in enumerate(allv):
            for ki, kind in enumerate(self.KINDS):
                base = 4 + 9 * (2 * ki + slot)
                ptr = row[base]
                handle = np.asarray(row[base + 1: base + 9], dtype=np.int64).tobytes()
                if r == comm.rank or row[0] == pid:
                    addrs[kind][r] = ptr
                    continue
                key = (r, handle)
                if key not in self.opened:
                    out = ctypes.c_void_p()
                    _lib.check(_lib.load().vfn_ipc_open(self.device, (ctypes.c_ubyte * 64)(*handle),
                                                        ctypes.byref(out)))
                    self.opened[key] = out.value
                addrs[kind][r] = self.opened[key]
        local = {kind: self.local[kind][slot][0] for kind in self.KINDS}
        self.caps_in = caps_in
        return slot, local, addrs

    def close(self):
        from . import _lib

        if _lib._lib is None:
            return
        lib = _lib._lib
        for addr in self.opened.values():
            lib.vfn_ipc_close(self.device, addr)
        self.opened.clear()
        for kind in self.KINDS:
            for k in range(2):
                if self.local[kind][k] is not None:
                    lib.vfn_ipc_free(self.device, self.local[kind][k][0])
                    self.local[kind][k] = None


class _Timer:
    def __init__(self, enabled: bool):
        import torch

        self.on = enabled and torch.cuda.is_available() and torch.cuda.is_initialized()
        self.marks = []
        if self.on:
            self.torch = torch

    def mark(self):
        if self.on:
            e = self.torch.cuda.Event(enable_timing=True)
            e.record()
            self.marks.append(e)

    def spans(self, n: int) -> list[float]:
        if not self.on or len(self.marks) < 2:
            return [0.0] * n
        self.torch.cuda.current_stream().synchronize()
        return [a.elapsed_time(b) for a, b in zip(self.marks, self.marks[1:])]


def evaluate_sharded(plan, points, group=None, mode: str = "keyrange", out=None, stats: ShardStats | None = None,
                     samples_per_rank: int = 1 << 18, comm=None, values: str = "p2p"):
    """Values of this rank's block of one point set, in input order (see the
    module docstring).  ``points``: this rank's (m, 3) block (a CUDA tensor
    on the plan's device); the blocks of ranks 0..P-1 concatenated in rank
    order are the whole set.  Every rank of ``group`` must call this.
    ``comm`` replaces the torch.distributed group with an object offering
    `_Comm`'s methods (tests run P ranks as threads of one process).
    ``values``: how points and values move — "p2p" (default): the partition
    kernel stores every point into its destination's IPC-shared receive
    buffer and the gather's epilogue stores every value into its owner's
    output buffer, both over NVLink (the two all-to-alls fused into the
    kernels around them); "nccl": all-to-alls of points and values and a
    local reorder."""
    import torch

    if mode not in ("keyrange", "block"):
        raise ValueError("mode must be 'keyrange' or 'block'")
    if values not in ("p2p", "nccl"):
        raise ValueError("values must be 'p2p' or 'nccl'")
    comm = comm if comm is not None else _Comm(group)
    if points.dim() != 2 or points.shape[1] != 3:
        raise ValueError(f"points must be an (M, 3) array, got shape {tuple(points.shape)}")
    points = points.to(torch.float64).contiguous()
    m = int(points.shape[0])
    timer = _Timer(stats is not None)
    timer.mark()
    sizes = [c[0] for c in comm.all_gather_ints([m])]
    total = sum(sizes)
    row0 = sum(sizes[: comm.rank])

    # the unsharded call's decisions, from the global M and global sample rows
    sample = None
    if total >= (1 << 20):
        stride, cnt = density_sample_rows(total, plan.DENSITY_SAMPLE)
        j0 = -(-row0 // stride)
        j1 = min(cnt, -(-(row0 + m) // stride))
        local = points[torch.arange(max(j0, 0), max(j1, j0), device=points.device) * stride - row0] \
            if j1 > j0 else points[:0]
        counts = [c[0] for c in comm.all_gather_ints([int(local.shape[0])])]
        sample = comm.all_gather_rows(local, counts)
    prev = (plan._gather, getattr(plan, "_box", 0))
    variant, box = plan.decide(total, sample)
    plan.pin(variant, box)
    timer.mark()
    try:
        if mode == "block" or comm.world == 1 or variant == 3:
            # the warp-per-point gather is point-local: no exchange needed
            res = plan.evaluate(points, out=out)
            timer.mark()
            if stats is not None:
                sp = timer.spans(2)
                stats.decide_ms, stats.evaluate_ms = sp[0], sp[1]
                stats.sent, stats.received = [m], m
            return res
        # splitters from an all-gather of key samples (same stride on every
        # rank, so each rank's share of the sample follows its block size)
        kstride = max(1, total // (samples_per_rank * comm.world))
        keys = plan.part_keys(points, kstride, row0)
        kcounts = [c[0] for c in comm.all_gather_ints([int(keys.shape[0])])]
        split = splitters_from_samples(comm.all_gather_rows(keys, kcounts), comm.world)
        p2p = (values == "p2p" and points.is_cuda and hasattr(plan, "partition_scatter_peers")
               and not getattr(plan, "_p2p_failed", False))
        if p2p:
            send_counts, bad = plan.partition_count(points, split, row0)
        else:
            send, send_counts, pos, bad = plan.partition(points, split, row0, raise_outside=False)
        # an outside point anywhere fails every rank with the global first row
        first = comm.all_reduce_min(row0 + bad if bad >= 0 else total)
        if first < total:
            mine = torch.zeros(3, dtype=torch.float64, device=points.device)
            if row0 <= first < row0 + m:
                mine = points[first - row0].clone()
            bad_pt = comm.all_reduce_sum(mine).cpu().tolist()
            raise ValueError(f"point {bad_pt} (row {first}) lies outside the domain "
                             f"{list(plan.domain.a)} .. {list(plan.domain.b)}")
        timer.mark()
        cmat = comm.all_gather_ints(send_counts)  # cmat[source][destination]
        recv_counts = [c[comm.rank] for c in cmat]
        if p2p:
            # the points go straight into the destinations' receive buffers and
            # the values straight into their owners' output buffers, both over
            # NVLink (IPC-mapped); no all-to-all on the data path
            r_in = sum(recv_counts)
            po = getattr(plan, "_peer_buffers", None)
            if po is None:
                po = plan._peer_buffers = _PeerBuffers(plan.device)
            try:
                slot, local, addrs = po.prepare(comm, m, r_in)
                ok = 1
            except Exception:  # e.g. no peer access between two GPUs: every rank falls back
                ok = 0
            if comm.all_reduce_min(ok) == 0:
                plan._p2p_failed = True
                return evaluate_sharded(plan, points, group, mode, out, stats, samples_per_rank, comm, "nccl")
            dst_off = [sum(cmat[s_][d] for s_ in range(comm.rank)) for d in range(comm.world)]
            rows_of = [addrs["in"][d] + 24 * po.caps_in[d] for d in range(comm.world)]
            plan.partition_scatter_peers(points, dst_off, addrs["in"], rows_of)
            comm.barrier()  # every rank's points are in my receive buffer
            timer.mark()
            seg = [0]
            for c in recv_counts:
                seg.append(seg[-1] + c)
            plan.evaluate_to_peers(local["in"], local["in"] + 24 * po.cap["in"], seg, addrs["out"], M=r_in)
            timer.mark()
            comm.barrier()  # every rank's values for my block are in my output buffer
            timer.mark()
            if out is None:
                out = torch.empty(m, dtype=torch.complex128, device=points.device)
            from . import _lib
            from .nufft import _stream_of

            _lib.check(_lib.load().vfn_copy_device(plan.device, out.data_ptr(), local["out"], 16 * m,
                                                   _stream_of(plan.device)))
            res = out
        else:
            recv = comm.all_to_all(send, send_counts, recv_counts)
            timer.mark()
            vals = plan.evaluate(recv)
            timer.mark()
            back = comm.all_to_all(torch.view_as_real(vals), recv_counts, send_counts)
            timer.mark()
            res = _gather_values(torch.view_as_complex(back.contiguous()), pos)
            if out is not None:
                out.copy_(res)
                res = out
        timer.mark()
        if stats is not None:
            sp = timer.spans(6)
            (stats.decide_ms, stats.partition_ms, stats.exchange_in_ms, stats.evaluate_ms,
             stats.exchange_out_ms, stats.restore_ms) = sp[:6]
            stats.sent, stats.received = list(send_counts), int(sum(recv_counts))
        return res
    finally:
        plan.set_gather(prev[0])
        plan.set_box(prev[1])


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
