"""Multi-process host logic of the sharded trafo on CPU (gloo, world 2):
coefficient broadcast, contiguous point shards, result assembly, and
P-invariance of the assembled output.  The per-rank evaluator here is the
CPU oracle standing in for the GPU plan (the device path is covered by the
-m gpu tests); what is under test is the plumbing in parallel.py."""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_1605_01244_b200.parallel import broadcast_coefficients, gather_results, shard_range


def test_shard_range_partitions():
    for total in (0, 1, 7, 1000, 2 ** 28):
        for world in (1, 2, 3, 4, 8):
            spans = [shard_range(total, world, r) for r in range(world)]
            assert spans[0][0] == 0 and spans[-1][1] == total
            assert all(spans[i][1] == spans[i + 1][0] for i in range(world - 1))
            sizes = [hi - lo for lo, hi in spans]
            assert max(sizes) - min(sizes) <= 1
    with pytest.raises(ValueError):
        shard_range(10, 2, 2)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from oracle import nfft_oracle as O

    a, b = (-1.5, 0.25, 2.0), (2.5, 1.25, 7.0)
    if rank == 0:
        rng = np.random.default_rng(3)
        coeffs = torch.as_tensor(rng.standard_normal((8, 8, 8)) + 1j * rng.standard_normal((8, 8, 8)))
    else:
        coeffs = torch.zeros((8, 8, 8), dtype=torch.complex128)
    coeffs = broadcast_coefficients(coeffs, src=0)
    pts = np.random.default_rng(4).uniform(a, b, (1001, 3))
    lo, hi = shard_range(len(pts), world, rank)
    local = torch.as_tensor(O.nufft_eval(coeffs.numpy(), a, b, pts[lo:hi]))
    full = gather_results(local, len(pts), dst=0)
    if rank == 0:
        q.put((coeffs.numpy(), full.numpy()))
    dist.barrier()
    dist.destroy_process_group()


def test_two_rank_broadcast_shard_gather():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    coeffs, full = q.get(timeout=120)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    from oracle import nfft_oracle as O

    a, b = (-1.5, 0.25, 2.0), (2.5, 1.25, 7.0)
    pts = np.random.default_rng(4).uniform(a, b, (1001, 3))
    rng = np.random.default_rng(3)
    ref_coeffs = rng.standard_normal((8, 8, 8)) + 1j * rng.standard_normal((8, 8, 8))
    np.testing.assert_array_equal(coeffs, ref_coeffs)
    # sharded == single-process, bitwise
    np.testing.assert_array_equal(full, O.nufft_eval(ref_coeffs, a, b, pts))


def _rect_worker(rank, world, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from oracle import nfft_oracle as O
    from paper_1605_01244_b200.parallel import eval_rectilinear_sharded

    a, b = (-1.5, 0.25, 2.0), (2.5, 1.25, 7.0)
    coeffs = torch.zeros((6, 8, 10), dtype=torch.complex128)
    if rank == 0:
        rng = np.random.default_rng(5)
        coeffs = torch.as_tensor(rng.standard_normal((6, 8, 10)) + 1j * rng.standard_normal((6, 8, 10)))
    coeffs = broadcast_coefficients(coeffs, src=0)
    rng = np.random.default_rng(6)
    coords = [np.sort(rng.uniform(a[d], b[d], n)) for d, n in enumerate((7, 5, 9))]

    class Spec:  # oracle stand-in for the GPU evaluator (plumbing under test)
        pass

    spec = Spec()
    spec.coeffs = coeffs.numpy()
    slab = eval_rectilinear_sharded(spec, coords, rank, world,
                                    evaluator=lambda s, c: O.rectilinear(s.coeffs, a, b, c))
    parts = [None] * world
    dist.all_gather_object(parts, slab)
    if rank == 0:
        q.put((np.concatenate(parts, axis=0), O.rectilinear(spec.coeffs, a, b, coords)))
    dist.barrier()
    dist.destroy_process_group()


def test_two_rank_rectilinear_slabs():
    """Axis-1 slabs of a rectilinear evaluation on 2 gloo ranks concatenate
    to the unsharded grid (oracle evaluator)."""
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_rect_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    got, ref = q.get(timeout=120)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert got.shape == ref.shape
    np.testing.assert_allclose(got, ref, rtol=1e-13, atol=1e-13 * np.abs(ref).max())


class _OraclePlan:
    """CPU stand-in for NufftPlan in the key-range plumbing test: the
    partition keys, stable split and values come from the oracle (the device
    steps are covered by tests/test_gpu_shard.py)."""

    DENSITY_SAMPLE = 16384

    def __init__(self, coeffs, a, b):
        from oracle import nfft_oracle as O

        self.O, self.coeffs, self.a, self.b = O, coeffs, a, b
        self._n = tuple(2 * s for s in coeffs.shape)
        self.tile = (4, 4, 8)
        self._gather, self._box = 0, 0
        self.evaluated = []

        class D:
            pass

        self.domain = D()
        self.domain.a, self.domain.b = a, b

    def decide(self, M, sample=None):
        return (3 if M <= 32768 else 4), 2

    def pin(self, v, b):
        self._gather, self._box = v, b

    def set_gather(self, v):
        self._gather = v

    def set_box(self, b):
        self._box = b

    def part_keys(self, pts, stride=1, row0=0):
        k = self.O.partition_keys(pts.numpy(), self.a, self.b, self._n, self.tile, row0)
        return torch.as_tensor(k[::stride].copy())

    def partition(self, pts, split, row0=0, raise_outside=True):
        bad = self.O.domain_violation(pts.numpy(), self.a, self.b)
        send, counts, pos = self.O.partition(pts.numpy(), self.a, self.b, self._n, self.tile,
                                             split.numpy(), row0)
        return torch.as_tensor(send), counts.tolist(), torch.as_tensor(pos.astype(np.int32)), bad

    def evaluate(self, pts, out=None):
        self.evaluated.append(int(pts.shape[0]))
        return torch.as_tensor(self.O.nufft_eval(self.coeffs, self.a, self.b, pts.numpy()))


def _keyrange_worker(rank, world, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_1605_01244_b200.parallel import ShardStats, evaluate_sharded

    a, b = (-1.5, 0.25, 2.0), (2.5, 1.25, 7.0)
    coeffs = np.random.default_rng(7).standard_normal((8, 8, 8)) + 0j
    pts = np.random.default_rng(8).uniform(a, b, (40000, 3))
    lo, hi = shard_range(len(pts), world, rank)
    plan = _OraclePlan(coeffs, a, b)
    st = ShardStats()
    got = evaluate_sharded(plan, torch.as_tensor(pts[lo:hi]), stats=st, samples_per_rank=512)
    bad = pts.copy()
    bad[30001, 1] = 9.0
    blo, bhi = shard_range(len(bad), world, rank)
    try:
        evaluate_sharded(plan, torch.as_tensor(bad[blo:bhi]))
        msg = None
    except ValueError as e:
        msg = str(e)
    q.put((rank, got.numpy(), plan.evaluated, st.sent, msg))
    dist.barrier()
    dist.destroy_process_group()


def test_two_rank_keyrange_exchange():
    """The key-range sharded evaluate on 2 gloo ranks: sample-sort splitters,
    all-to-all of points and values, values back in input order equal the
    unsharded oracle bitwise; every rank evaluates only its key range; an
    outside point fails both ranks with the global row."""
    from oracle import nfft_oracle as O

    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_keyrange_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = sorted([q.get(timeout=180) for _ in range(2)], key=lambda x: x[0])
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    a, b = (-1.5, 0.25, 2.0), (2.5, 1.25, 7.0)
    coeffs = np.random.default_rng(7).standard_normal((8, 8, 8)) + 0j
    pts = np.random.default_rng(8).uniform(a, b, (40000, 3))
    ref = O.nufft_eval(coeffs, a, b, pts)
    np.testing.assert_array_equal(np.concatenate([r[1] for r in res]), ref)
    # each rank evaluated one key range (x-slab of tiles), about half the points
    for r in res:
        assert abs(r[2][0] - 20000) < 2000, r[2]
        assert sum(r[3]) == 20000
    # rank 0 sent most of its points' second half elsewhere: a real exchange
    assert res[0][3][1] > 5000 and res[1][3][0] > 5000
    for r in res:
        assert r[4] is not None and "(row 30001) lies outside" in r[4]
