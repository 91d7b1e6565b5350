"""Key-range sharding of one point set over P ranks (
paper_1605_01244_b200/parallel.py): the device partition vs the CPU
restatement, and the sharded evaluate's bitwise P-invariance in the DEFAULT
mode (no set_box / set_gather by the caller).  P ranks run as threads of
this process (tests/simcomm.py), each with its own plan, as each GPU has its
replicated plan; the torchrun test in test_gpu_parity.py runs the
torch.distributed path."""

import numpy as np
import pytest

from conftest import random_spectral
from oracle import nfft_oracle as O
from simcomm import run_ranks

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def vfb():
    import torch

    if not torch.cuda.is_available():
        pytest.skip("needs a GPU")
    import paper_1605_01244_b200 as pkg

    return pkg


def tile_of_plan(plan):
    box, tile = plan.geometry(1 << 22)  # the tensor-core tile (independent of the box width)
    return tile


@pytest.mark.parametrize("nparts", [1, 2, 3, 8, 37])
def test_partition_matches_cpu_restatement(vfb, offset_box, nparts):
    import torch

    spec = random_spectral(offset_box, (24, 20, 16), 1200 + nparts)
    plan = vfb.NufftPlan(spec)
    rng = np.random.default_rng(1210 + nparts)
    pts = rng.uniform(offset_box.a, offset_box.b, (50000, 3))
    pts[:300] = pts[0]  # a dense run inside one tile: ties split by row
    row0 = 123456
    dpts = torch.as_tensor(pts, device="cuda")
    keys = plan.part_keys(dpts, 1, row0).cpu().numpy()
    tile = tile_of_plan(plan)
    ref_keys = O.partition_keys(pts, offset_box.a, offset_box.b, plan._n, tile, row0)
    np.testing.assert_array_equal(keys, ref_keys)
    np.testing.assert_array_equal(plan.part_keys(dpts, 7, row0).cpu().numpy(), ref_keys[::7])
    split = np.sort(rng.choice(ref_keys, nparts - 1, replace=False)) if nparts > 1 else np.empty(0, np.int64)
    split[: min(2, len(split))] = ref_keys[150]  # equal splitters: an empty destination
    split = np.sort(split)
    send, counts, pos = plan.partition(dpts, torch.as_tensor(split, device="cuda"), row0)
    rsend, rcounts, rpos = O.partition(pts, offset_box.a, offset_box.b, plan._n, tile, split, row0)
    assert counts == rcounts.tolist()
    np.testing.assert_array_equal(pos.cpu().numpy(), rpos)
    np.testing.assert_array_equal(send.cpu().numpy(), rsend)
    vals = torch.as_tensor(rng.standard_normal(len(pts)) + 1j * rng.standard_normal(len(pts)), device="cuda")
    back = vfb.nufft.gather_values(vals, pos).cpu().numpy()
    np.testing.assert_array_equal(back, vals.cpu().numpy()[rpos])


def test_partition_reports_outside_rows(vfb, unit_box):
    import torch

    plan = vfb.NufftPlan(random_spectral(unit_box, (8, 8, 8), 1220))
    pts = np.random.default_rng(1221).uniform(0, 1, (9000, 3))
    pts[[4097, 8000], 2] = [1.0, np.nan]
    split = torch.tensor([1 << 40], dtype=torch.int64, device="cuda")
    with pytest.raises(ValueError, match=r"\(row 4097\) lies outside"):
        plan.partition(torch.as_tensor(pts, device="cuda"), split)


def _sets(vfb):
    from paper_1605_01244_b200 import workloads

    rng = np.random.default_rng(1230)
    uni = rng.uniform(-0.5, 0.5, (1 << 22, 3))
    cloud = np.clip(rng.normal(0.0, 0.02, (1 << 22, 3)), -0.5, 0.4999)
    return {"uniform": uni, "cloud": cloud}


@pytest.mark.parametrize("kind", ["uniform", "cloud"])
def test_sharded_default_mode_is_bitwise_P_invariant(vfb, kind):
    """2^22 points as P = 1, 2, 4, 8 input-order blocks, default plan
    settings: the key-range sharded evaluate (and the block mode) equals one
    unsharded evaluate bitwise."""
    import torch

    from paper_1605_01244_b200.parallel import ShardStats, evaluate_sharded, shard_range

    box = vfb.DomainBox((-0.5, -0.5, -0.5), (0.5, 0.5, 0.5))
    spec = random_spectral(box, (64, 64, 64), 1240)
    pts = _sets(vfb)[kind]
    dpts = torch.as_tensor(pts, device="cuda")
    ref = vfb.NufftPlan(spec).evaluate(dpts).cpu().numpy()
    plans = [vfb.NufftPlan(spec) for _ in range(8)]
    for P in (1, 2, 4, 8):
        for mode in ("keyrange", "block"):
            def rank(r, comm):
                lo, hi = shard_range(len(pts), P, r)
                st = ShardStats()
                v = evaluate_sharded(plans[r], dpts[lo:hi], mode=mode, comm=comm, stats=st)
                torch.cuda.synchronize()
                return v.cpu().numpy(), st

            res = run_ranks(P, rank)
            got = np.concatenate([v for v, _ in res])
            np.testing.assert_array_equal(got, ref, err_msg=f"{kind} P={P} {mode}")
            if mode == "keyrange" and P > 1 and kind == "uniform":
                recv = [st.received for _, st in res]
                assert max(recv) <= 1.05 * len(pts) / P, recv  # balanced key ranges
    for p in plans:  # the caller's settings are restored
        assert p._gather == 0 and p._box == 0


@pytest.mark.parametrize("M", [20000, 100000])
def test_sharded_small_sets(vfb, offset_box, M):
    """Below the warp-path threshold (point-local gather, no exchange) and a
    binned set below the density-sampling size."""
    import torch

    from paper_1605_01244_b200.parallel import evaluate_sharded, shard_range

    spec = random_spectral(offset_box, (20, 24, 16), 1250)
    pts = np.random.default_rng(1251).uniform(offset_box.a, offset_box.b, (M, 3))
    dpts = torch.as_tensor(pts, device="cuda")
    ref = vfb.NufftPlan(spec).evaluate(dpts).cpu().numpy()
    plans = [vfb.NufftPlan(spec) for _ in range(4)]
    for P in (2, 3, 4):
        res = run_ranks(P, lambda r, comm: evaluate_sharded(
            plans[r], dpts[slice(*shard_range(M, P, r))], comm=comm).cpu().numpy())
        np.testing.assert_array_equal(np.concatenate(res), ref)


def test_sharded_outside_point_fails_every_rank(vfb, unit_box):
    import torch

    from paper_1605_01244_b200.parallel import evaluate_sharded, shard_range

    spec = random_spectral(unit_box, (16, 16, 16), 1260)
    pts = np.random.default_rng(1261).uniform(0, 1, (200000, 3))
    pts[150001, 0] = 1.5
    dpts = torch.as_tensor(pts, device="cuda")
    plans = [vfb.NufftPlan(spec) for _ in range(3)]

    def rank(r, comm):
        with pytest.raises(ValueError, match=r"\(row 150001\) lies outside"):
            evaluate_sharded(plans[r], dpts[slice(*shard_range(len(pts), 3, r))], comm=comm)
        return True

    assert all(run_ranks(3, rank))


@pytest.mark.parametrize("draw", range(8))
def test_sharded_fuzz(vfb, draw):
    """Random rank counts, sizes (warp path, binned without and with the
    density sample), boxes, grids and point distributions (uniform, clouds
    straddling the periodic seam, mixtures, a single repeated point): the
    key-range sharded evaluate equals the unsharded call bitwise."""
    import torch

    from paper_1605_01244_b200.parallel import evaluate_sharded, shard_range

    rng = np.random.default_rng(1500 + draw)
    a = rng.uniform(-3, 3, 3)
    w = rng.uniform(0.5, 4, 3)
    box = vfb.DomainBox(tuple(a), tuple(a + w))
    shape = tuple(int(2 * rng.integers(4, 33)) for _ in range(3))
    spec = random_spectral(box, shape, 1510 + draw)
    M = int(rng.choice([20000, 300000, 1 << 20, 2500000]))
    kind = draw % 4
    if kind == 0:
        u = rng.uniform(0, 1, (M, 3))
    elif kind == 1:  # a cloud over the seam at 0 / 1
        u = np.mod(rng.normal(0.0, 0.01, (M, 3)), 1.0)
    elif kind == 2:  # mixture
        u = np.concatenate([rng.uniform(0, 1, (M // 2, 3)),
                            np.mod(rng.normal(rng.uniform(0, 1, 3), 0.003, (M - M // 2, 3)), 1.0)])
        u = u[rng.permutation(M)]
    else:  # one point repeated, plus a few others
        u = np.repeat(rng.uniform(0, 1, (1, 3)), M, axis=0)
        u[:: 97] = rng.uniform(0, 1, (len(u[:: 97]), 3))
    pts = np.asarray(box.a) + np.minimum(u, np.nextafter(1.0, 0.0)) * (np.asarray(box.b) - np.asarray(box.a))
    pts = np.minimum(pts, np.nextafter(np.asarray(box.b), -np.inf))
    dpts = torch.as_tensor(pts, device="cuda")
    ref = vfb.NufftPlan(spec).evaluate(dpts).cpu().numpy()
    P = int(rng.choice([2, 3, 5, 8]))
    plans = [vfb.NufftPlan(spec) for _ in range(P)]
    res = run_ranks(P, lambda r, comm: evaluate_sharded(
        plans[r], dpts[slice(*shard_range(M, P, r))], comm=comm).cpu().numpy())
    np.testing.assert_array_equal(np.concatenate(res), ref, err_msg=f"draw {draw}: P={P} M={M} kind={kind}")


@pytest.mark.parametrize("values", ["p2p", "nccl"])
def test_value_return_modes(vfb, offset_box, values):
    """Both ways values get back to their owners — stored straight into the
    owners' buffers by the gather (p2p, the default) or an all-to-all and a
    reorder (nccl) — give the unsharded values bitwise, also with a
    caller-provided ``out`` and on repeated calls (alternating buffers)."""
    import torch

    from paper_1605_01244_b200.parallel import evaluate_sharded, shard_range

    spec = random_spectral(offset_box, (20, 24, 16), 1700)
    pts = np.random.default_rng(1701).uniform(offset_box.a, offset_box.b, (400000, 3))
    dpts = torch.as_tensor(pts, device="cuda")
    ref = vfb.NufftPlan(spec).evaluate(dpts).cpu().numpy()
    plans = [vfb.NufftPlan(spec) for _ in range(3)]

    def rank(r, comm):
        lo, hi = shard_range(len(pts), 3, r)
        outs = []
        for rep in range(3):
            o = torch.empty(hi - lo, dtype=torch.complex128, device="cuda") if rep == 1 else None
            v = evaluate_sharded(plans[r], dpts[lo:hi], comm=comm, values=values, out=o)
            outs.append(v.cpu().numpy())
        return outs

    res = run_ranks(3, rank)
    for rep in range(3):
        np.testing.assert_array_equal(np.concatenate([x[rep] for x in res]), ref)


def _ipc_worker(rank, world, port, q):
    import os

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    import numpy as np
    import torch
    import torch.distributed as dist

    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import paper_1605_01244_b200 as vfb
    from paper_1605_01244_b200.parallel import ShardStats, evaluate_sharded, shard_range

    try:
        box = vfb.DomainBox((-0.5, -0.5, -0.5), (0.5, 0.5, 0.5))
        rng = np.random.default_rng(1710)
        coeffs = rng.standard_normal((32, 32, 32)) + 1j * rng.standard_normal((32, 32, 32))
        spec = vfb.SpectralField(box, coeffs)
        pts = np.random.default_rng(1711).uniform(-0.5, 0.5, (1 << 20, 3))
        dpts = torch.as_tensor(pts, device="cuda")
        plan = vfb.NufftPlan(spec)
        ref = plan.evaluate(dpts).cpu().numpy()
        lo, hi = shard_range(len(pts), world, rank)
        ok = True
        for _ in range(3):
            st = ShardStats()
            got = evaluate_sharded(plan, dpts[lo:hi], stats=st).cpu().numpy()
            ok &= bool(np.array_equal(got, ref[lo:hi]))
        q.put((rank, ok, st.received, None))
    except Exception:  # noqa: BLE001
        import traceback

        q.put((rank, False, 0, traceback.format_exc()))
    dist.barrier()
    dist.destroy_process_group()


def test_two_processes_store_values_over_ipc():
    """Two processes (gloo control plane, both on this GPU): each evaluates a
    key range and the gather stores the values into the OTHER process's
    IPC-mapped output buffer (cudaIpcOpenMemHandle), as ranks on separate
    GPUs do over NVLink; every rank gets its block's unsharded values
    bitwise, on repeated calls."""
    import socket

    import torch.multiprocessing as mp

    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_ipc_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = sorted([q.get(timeout=300) for _ in range(2)])
    for p in procs:
        p.join(timeout=120)
    for rank, ok, received, err in res:
        assert err is None, err
        assert ok, f"rank {rank}: sharded values differ"
        assert 0.4 * (1 << 20) < received < 0.6 * (1 << 20)


def test_peer_buffer_failure_falls_back_on_every_rank(vfb, offset_box):
    """If one rank cannot allocate its IPC buffers, every rank takes the NCCL
    exchange for that call and later ones (no rank left waiting in a
    collective), with the same values."""
    import torch

    from paper_1605_01244_b200.parallel import _PeerBuffers, evaluate_sharded, shard_range

    spec = random_spectral(offset_box, (16, 16, 16), 1800)
    pts = np.random.default_rng(1801).uniform(offset_box.a, offset_box.b, (300000, 3))
    dpts = torch.as_tensor(pts, device="cuda")
    ref = vfb.NufftPlan(spec).evaluate(dpts).cpu().numpy()
    plans = [vfb.NufftPlan(spec) for _ in range(3)]

    def broken_alloc(self, kind, cap, elem):
        raise RuntimeError("simulated allocation failure")

    pb = _PeerBuffers(plans[1].device)
    pb._alloc = broken_alloc.__get__(pb)
    plans[1]._peer_buffers = pb

    def rank(r, comm):
        lo, hi = shard_range(len(pts), 3, r)
        return [evaluate_sharded(plans[r], dpts[lo:hi], comm=comm).cpu().numpy() for _ in range(2)]

    res = run_ranks(3, rank)
    for k in range(2):
        np.testing.assert_array_equal(np.concatenate([x[k] for x in res]), ref)
    assert all(getattr(p, "_p2p_failed", False) for p in plans)
