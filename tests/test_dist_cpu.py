"""Multi-process (gloo, world_size 2, CPU) checks of the sharded algorithm:
every rank derives the same shard plan from the same inputs, the plan
partitions points and edges exactly, and the sharded decomposition the
device path uses -- camera-sized sums allreduced, point blocks local --
reproduces the full (single-process) gradient and Hessian-vector product of
the reference restatement."""
import os
import socket

import numpy as np
import pytest
import torch.distributed as dist
import torch.multiprocessing as mp

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def worker(rank, world, port, outq):
    import sys

    sys.path.insert(0, ROOT)
    import torch

    from oracle import restatement as R
    from paper_2509_26581_b200 import bal

    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank, world_size=world)
    try:
        p = bal.synthetic_bal(24, 900, 5400, seed=3)
        tiles, pts, edges, owner = bal.shard_plan(p, world)
        plan = torch.tensor(np.concatenate([tiles.ravel(), pts.ravel(), edges.astype(np.uint32)]).astype(np.int64))
        plans = [torch.zeros_like(plan) for _ in range(world)]
        dist.all_gather(plans, plan)
        same_plan = all(bool(torch.equal(plans[0], x)) for x in plans)
        own = torch.tensor(owner.astype(np.int64))
        owners = [torch.zeros_like(own) for _ in range(world)]
        dist.all_gather(owners, own)
        same_owner = all(bool(torch.equal(owners[0], x)) for x in owners)

        # full restatement (what a single device computes)
        gf = R.build_graph(p, "fp64")
        R.activate(gf, 0)
        lf = R.LinearSystem(gf)
        lf.linearize()
        v = np.random.default_rng(0).standard_normal(gf.N)
        lam = 0.3
        full_hvp = lf.hvp(v, lam)
        # this rank's shard: only edges of its points are active
        mine = owner[p.point_index] == rank
        gr = R.build_graph(p, "fp64", levels=np.where(mine, 0, 1))
        R.activate(gr, 0)
        lr = R.LinearSystem(gr)
        lr.linearize()
        ncam = 9 * p.num_cameras
        bc = torch.tensor(lr.b[:ncam].copy())
        dist.all_reduce(bc)  # camera gradient: allreduce over shards
        lr.D = lf.D  # D comes from the allreduced diagonal on device
        part = lr.hvp(v, 0.0)
        cam = torch.tensor(part[:ncam].copy())
        dist.all_reduce(cam)
        cam_hvp = cam.numpy() + lam * v[:ncam]
        pcols = ncam + 3 * np.nonzero(owner == rank)[0]
        pcols = (pcols[:, None] + np.arange(3)).ravel()
        ok_b = np.allclose(bc.numpy(), lf.b[:ncam], rtol=1e-11, atol=1e-9 * np.abs(lf.b).max())
        ok_bp = np.allclose(lr.b[pcols], lf.b[pcols], rtol=1e-12, atol=0)
        ok_h = np.allclose(cam_hvp, full_hvp[:ncam], rtol=1e-11, atol=1e-11 * np.abs(full_hvp).max())
        ok_hp = np.allclose(part[pcols] + lam * v[pcols], full_hvp[pcols], rtol=1e-12, atol=1e-14)
        cover = int(edges.sum()) == p.num_observations and sorted(set(owner.tolist())) == list(range(world))
        outq.put((rank, same_plan, same_owner, bool(ok_b), bool(ok_bp), bool(ok_h), bool(ok_hp), cover))
    finally:
        dist.destroy_process_group()


def test_sharded_decomposition_gloo_world2():
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = free_port()
    procs = [ctx.Process(target=worker, args=(r, world, port, q)) for r in range(world)]
    for pr in procs:
        pr.start()
    res = [q.get(timeout=240) for _ in range(world)]
    for pr in procs:
        pr.join(60)
    for r in res:
        assert all(r[1:]), r


def test_shard_plan_partitions():
    import sys

    sys.path.insert(0, ROOT)
    from paper_2509_26581_b200 import bal

    p = bal.synthetic_bal(49, 7776, 31843, seed=42)
    for world in (1, 2, 3, 8):
        tiles, pts, edges, owner = bal.shard_plan(p, world)
        assert tiles[0, 0] == 0 and pts[0, 0] == 0 and pts[-1, 1] == p.num_points
        assert np.all(tiles[1:, 0] == tiles[:-1, 1]) and np.all(pts[1:, 0] == pts[:-1, 1])
        assert int(edges.sum()) == p.num_observations
        assert np.bincount(owner, minlength=world).sum() == p.num_points
        if world > 1:  # balanced by edge count
            assert edges.max() <= 1.2 * edges.mean() + 600


# ---------------------------------------------------------------------------
# The product's shared-memory reducer (kind 2) between real processes: sums
# in rank order (every rank gets identical bits), max, multi-slot messages,
# broadcast. The same collectives carry the sharded GPU solve in
# tests/test_gpu_sharded.py::test_shm_processes_match_single_gpu.
def shm_worker(rank, world, key, n, outq):
    import sys

    sys.path.insert(0, ROOT)
    from paper_2509_26581_b200 import _abi

    L = _abi.lib()
    rng = np.random.default_rng(100 + rank)
    data = rng.standard_normal(n)
    mx = data.copy()
    bc = np.full(5000, float(rank))
    rc1 = L.gb_shm_allreduce_selftest(world, rank, key, data.ctypes.data, n, 0, bc.ctypes.data, bc.size)
    rc2 = L.gb_shm_allreduce_selftest(world, rank, key + 1, mx.ctypes.data, n, 1, None, 0)
    outq.put((rank, rc1, rc2, data, mx, bc))


@pytest.mark.parametrize("world,n", [(3, 1000), (2, 1_500_000)])
def test_shm_reducer_processes(world, n):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    key = 0x5EED0000 + world * 7 + os.getpid() % 1000 * 16
    procs = [ctx.Process(target=shm_worker, args=(r, world, key, n, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = sorted((q.get(timeout=300) for _ in range(world)), key=lambda t: t[0])
    for p in procs:
        p.join(60)
        assert p.exitcode == 0
    ins = [np.random.default_rng(100 + r).standard_normal(n) for r in range(world)]
    want = ins[0].copy()
    for x in ins[1:]:
        want = want + x  # rank order
    want_max = np.maximum.reduce(ins)
    for rank, rc1, rc2, data, mx, bc in res:
        assert rc1 == 0 and rc2 == 0
        assert np.array_equal(data.view(np.uint64), want.view(np.uint64))
        assert np.array_equal(mx, want_max)
        assert np.all(bc == world - 1)
