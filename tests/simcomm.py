"""P ranks as threads of one process: the collectives of
paper_1605_01244_b200.parallel._Comm over shared slots and a barrier, so the
sharded evaluate can be exercised for P = 1..8 on one GPU (each thread has
its own plan, as each rank would).  Test infrastructure only."""

from __future__ import annotations

import threading


class ThreadGroup:
    def __init__(self, world: int):
        self.world = world
        self.barrier = threading.Barrier(world)
        self.slots = [None] * world

    def comm(self, rank: int) -> "ThreadComm":
        return ThreadComm(self, rank)


class ThreadComm:
    def __init__(self, g: ThreadGroup, rank: int):
        self.g, self.rank, self.world = g, rank, g.world

    def _exchange(self, value):
        self.g.slots[self.rank] = value
        self.g.barrier.wait()
        vals = list(self.g.slots)
        self.g.barrier.wait()
        return vals

    def barrier(self):
        self.g.barrier.wait()

    def all_gather_ints(self, values):
        return [list(v) for v in self._exchange(list(values))]

    def all_gather_rows(self, t, counts):
        import torch

        parts = self._exchange(t.clone())
        return torch.cat([p.to(t.device) for p in parts])

    def all_reduce_min(self, v):
        return min(self._exchange(int(v)))

    def all_reduce_sum(self, t):
        parts = self._exchange(t.clone())
        acc = parts[0].clone()
        for p in parts[1:]:
            acc += p.to(acc.device)
        return acc

    def all_to_all(self, send, send_counts, recv_counts):
        import torch

        offs = [0]
        for c in send_counts:
            offs.append(offs[-1] + c)
        pieces = self._exchange([send[offs[d]:offs[d + 1]].clone() for d in range(self.world)])
        return torch.cat([pieces[src][self.rank].to(send.device) for src in range(self.world)])


def run_ranks(world: int, fn):
    """fn(rank, comm) in `world` threads; returns the per-rank results
    (re-raises the first exception)."""
    g = ThreadGroup(world)
    res = [None] * world
    errs = []

    def body(r):
        try:
            res[r] = fn(r, g.comm(r))
        except BaseException as e:  # noqa: BLE001
            errs.append(e)
            g.barrier.abort()

    ts = [threading.Thread(target=body, args=(r,)) for r in range(world)]
    for t in ts:
        t.start()
    for t in ts:
        t.join()
    if errs:
        raise errs[0]
    return res
